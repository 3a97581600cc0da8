#!/usr/bin/env python
"""Developer workload for profiling the forward FHT (ncu -k regex:k_fwd): N=2048, 4 slices,
three fbp_fht_forward calls.  Not a test."""
import json, os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2007_06289_b200 as pkg
N, B = 2048, 4
c = json.load(open("coeffs/iir_q3_n2048_dc0.json"))
plan = pkg.Plan(N, c["b"], c["a"], max_batch=B)
img = torch.rand((B, N, N), device="cuda")
out = torch.empty((B, 4, N, 2 * N), device="cuda")
for _ in range(3):
    plan.forward(img, out=out)
torch.cuda.synchronize()
