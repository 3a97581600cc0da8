#!/usr/bin/env python
"""Developer check (GPU): fast-path parity vs the oracle on a few cases, with
timings.  Not a test; prints one line per case."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2007_06289_b200 as pkg  # noqa: E402
import phantoms as P  # noqa: E402
from oracle import fbp_oracle as O  # noqa: E402


def coeffs(N, v="dc0"):
    c = json.load(open(os.path.join(ROOT, "coeffs", f"iir_q3_n{N}_{v}.json")))
    return c["b"], c["a"]


def rel(g, r):
    return float(np.max(np.abs(g.astype(np.float64) - r)) / max(np.max(np.abs(r)), 1e-300))


for N in [int(a) for a in (sys.argv[1:] or ["512", "1024", "2048"])]:
    for v in ("dc0", "spec"):
        b, a = coeffs(N, v)
        plan = pkg.Plan(N, b, a, max_batch=2)
        print("N", N, v, plan.path(), plan.info(), flush=True)
        L = P.integer_linogram(N, 1, seed=3)
        out = plan.backproject(L.cuda(), scale=1.0).cpu().numpy()[0]
        ref = O.combine(O.fht_backproject(L[0].double().numpy()), 1.0)
        print("  int BP exact:", np.array_equal(out.astype(np.float64), ref),
              "maxdiff", float(np.max(np.abs(out - ref))), flush=True)
        cfg = {512: 2, 1024: 4, 2048: 3}[N]
        S = P.make_slice(cfg, 0)
        t0 = time.time()
        img = plan.reconstruct(S[None].cuda()).cpu().numpy()[0]
        ref = O.reconstruct(S.double().numpy(), b, a)
        print("  recon rel err %.3e (oracle %.1fs)" % (rel(img, ref), time.time() - t0), flush=True)
