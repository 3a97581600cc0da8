"""Developer: KS/KB kernel times (CUDA events inside libfbp) under the FBP_DBG skip
mask of a -DFBP_DEV_MASK=1 build (results invalid when the mask is set).
   FBP_DBG=<mask> python tools/dev_timing2.py [N] [B]"""
import json, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2007_06289_b200 as pkg
import phantoms as P
N = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
B = int(sys.argv[2]) if len(sys.argv) > 2 else 16
c = json.load(open(os.path.join(ROOT, "coeffs", f"iir_q3_n{N}_dc0.json")))
plan = pkg.Plan(N, c["b"], c["a"], max_batch=B)
S = torch.empty((B, 4, N, 2 * N), device="cuda")
for i in range(B):
    S[i] = P.make_slice(3, i, device="cuda", N=N)
img = torch.empty((B, N, N), device="cuda")
for _ in range(3):
    plan.reconstruct(S, out=img)
torch.cuda.synchronize()
plan.profile(True)
K = 10
for _ in range(K):
    plan.reconstruct(S, out=img)
torch.cuda.synchronize()
kt = plan.kernel_times()
plan.profile(False)
print("DBG", os.environ.get("FBP_DBG", "0"), " ".join(f"{k}={v[0] / K:.4f}ms" for k, v in kt.items() if v[1]))
