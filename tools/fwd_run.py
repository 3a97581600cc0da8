"""Developer: run the forward FHT (fbp_fht_forward) K times on B slices of N (ncu driver).
    python tools/fwd_run.py [N] [B] [K]"""
import os, sys, json
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2007_06289_b200 as pkg
N = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
B = int(sys.argv[2]) if len(sys.argv) > 2 else 16
K = int(sys.argv[3]) if len(sys.argv) > 3 else 3
c = json.load(open(os.path.join(ROOT, "coeffs", f"iir_q3_n{N}_dc0.json")))
plan = pkg.Plan(N, c["b"], c["a"], max_batch=B)
img = torch.randn((B, N, N), device="cuda")
out = torch.empty((B, 4, N, 2 * N), device="cuda")
for _ in range(K):
    plan.forward(img, out=out)
torch.cuda.synchronize()
plan.profile(True)
for _ in range(K):
    plan.forward(img, out=out)
torch.cuda.synchronize()
print({k: v[0] / K for k, v in plan.kernel_times().items() if v[1]})
