#!/usr/bin/env python
"""Developer timing (GPU): fbp_iir_filter (K1) throughput at N=2048, 16 slices, vs the
HBM roofline on its 64 N^2 algorithmic bytes per slice (read S, write F).  Not a test."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2007_06289_b200 as pkg  # noqa: E402
import phantoms as P  # noqa: E402

N, B = int(os.environ.get("N", "2048")), int(os.environ.get("B", "16"))
c = json.load(open(os.path.join(ROOT, "coeffs", f"iir_q3_n{N}_dc0.json")))
plan = pkg.Plan(N, c["b"], c["a"], max_batch=B)
S = torch.empty((B, 4, N, 2 * N), device="cuda")
for i in range(B):
    S[i] = P.make_slice(3 if N == 2048 else 2, i, device="cuda", N=N)
F = torch.empty_like(S)
for _ in range(3):
    plan.iir_filter(S, out=F)
torch.cuda.synchronize()
plan.profile(True)
K = 10
for _ in range(K):
    plan.iir_filter(S, out=F)
kt = plan.kernel_times()
plan.profile(False)
ms = kt["iir"][0] / K
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6454.6) \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6454.6
gbs = 64.0 * N * N * B / (ms / 1e3) / 1e9
print(f"iir_filter N={N} B={B}: {ms:.3f} ms/call, {B / (ms / 1e3):.0f} slices/s, {gbs:.0f} GB/s "
      f"({gbs / peak:.3f} of {peak} GB/s)")
