#!/usr/bin/env python
"""Developer timing (GPU): per-kernel times of fbp_reconstruct and fbp_fht_backproject
at N=2048 on one batch (CUDA events inside libfbp).  Not a test."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2007_06289_b200 as pkg  # noqa: E402
import phantoms as P  # noqa: E402

N = int(os.environ.get("N", "2048"))
B = int(os.environ.get("B", "16"))
c = json.load(open(os.path.join(ROOT, "coeffs", f"iir_q3_n{N}_dc0.json")))
plan = pkg.Plan(N, c["b"], c["a"], max_batch=B)
S = torch.empty((B, 4, N, 2 * N), device="cuda", dtype=torch.float32)
for i in range(B):
    S[i] = P.make_slice(3 if N == 2048 else 2, i, device="cuda", N=N)
img = torch.empty((B, N, N), device="cuda")
for name, fn in (("reconstruct", lambda: plan.reconstruct(S, out=img)),
                 ("backproject", lambda: plan.backproject(S, scale=1.0 / N, out=img))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    plan.profile(True)
    for _ in range(5):
        fn()
    kt = plan.kernel_times()
    plan.profile(False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(name, {k: round(v[0] / 5, 4) for k, v in kt.items()}, "ms per call of", B, "slices;",
          "wall %.4f ms" % (e0.elapsed_time(e1) / 10), flush=True)
