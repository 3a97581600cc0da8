"""Small fast-path workload for compute-sanitizer runs (GPU):
   compute-sanitizer --tool <memcheck|racecheck|synccheck> python tools/sanitize_case.py N B
Runs fbp_reconstruct (fused sweep + pair kernels), fbp_fht_backproject and
fbp_fht_forward once each at size N with B slices."""
import json, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2007_06289_b200 as pkg
import phantoms as P
N, B = int(sys.argv[1]), int(sys.argv[2])
c = json.load(open(os.path.join(ROOT, "coeffs", f"iir_q3_n{N}_dc0.json")))
plan = pkg.Plan(N, c["b"], c["a"], max_batch=B)
S = P.random_linogram(N, B, seed=1, scale=10.0).cuda()
img = plan.reconstruct(S)
bp = plan.backproject(S, scale=1.0 / N)
fw = plan.forward(img)
torch.cuda.synchronize()
print("sanitize case", N, B, plan.path(), "ok", float(img.abs().max()), float(bp.abs().max()), float(fw.abs().max()))
