"""Developer: run one small fast-path call in this process (GPU); prints ok / the error.
   FBP_DBG=<mask> python tools/dev_bisect.py <N> <bp|rec>   (needs a -DFBP_DEV_MASK=1 build)"""
import json, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2007_06289_b200 as pkg
import phantoms as P
N = int(sys.argv[1]); mode = sys.argv[2]
c = json.load(open(os.path.join(ROOT, "coeffs", f"iir_q3_n{N}_dc0.json")))
plan = pkg.Plan(N, c["b"], c["a"], max_batch=1)
L = P.integer_linogram(N, 1, seed=3).cuda()
try:
    out = plan.backproject(L, scale=1.0) if mode == "bp" else plan.reconstruct(L)
    torch.cuda.synchronize()
    print("DBG", os.environ.get("FBP_DBG"), N, mode, "ok", float(out.abs().max()))
except Exception as e:
    print("DBG", os.environ.get("FBP_DBG"), N, mode, "ERR", str(e).splitlines()[0])
