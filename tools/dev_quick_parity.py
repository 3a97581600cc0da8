#!/usr/bin/env python
"""Developer check (GPU, seconds): the fast path (KS + KB) against the general path
(K1/K2/K3, untouched by fast-path edits) on the same inputs — integer back
projections bit-equal, reconstructions within 1e-5 of the slice peak — at the bench
launch sizes.  The general path is the exact schedule pinned against the oracle by
tests/test_gpu_parity.py; this is an iteration aid, not a test.

    python tools/dev_quick_parity.py [512 1024 2048 4096]
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2007_06289_b200 as pkg  # noqa: E402
import phantoms as P  # noqa: E402

ok = True
for N in [int(a) for a in (sys.argv[1:] or ["512", "1024", "2048", "4096"])]:
    B = {512: 16, 1024: 16, 2048: 16, 4096: 8}.get(N, 4)
    for v in ("dc0", "spec"):
        c = json.load(open(os.path.join(ROOT, "coeffs", f"iir_q3_n{N}_{v}.json")))
        fast = pkg.Plan(N, c["b"], c["a"], max_batch=B)
        gen = pkg.Plan(N, list(c["b"]) + [0.0], c["a"], max_batch=B)   # M = 4: general path
        assert fast.path()["fast"] and not gen.path()["fast"]
        L = P.integer_linogram(N, B, seed=N).cuda()
        a = fast.backproject(L, scale=1.0)
        b = gen.backproject(L, scale=1.0)
        ex = bool(torch.equal(a, b))
        S = P.random_linogram(N, B, seed=N + 1).cuda()
        r1 = fast.reconstruct(S)
        r2 = gen.reconstruct(S)
        torch.cuda.synchronize()
        err = float(((r1 - r2).abs().amax(dim=(1, 2)) / r2.abs().amax(dim=(1, 2))).max())
        good = ex and err < 1e-5
        ok &= good
        print(f"N={N} B={B} {v}: int BP bit-equal {ex}, recon max rel diff {err:.2e} {'OK' if good else 'FAIL'}",
              flush=True)
        if v == "dc0":
            # forward FHT (NEXT-1) by the exact adjoint identity <fwd(img), P> = <img, BP(P)>
            # on small integers, BP from the general path
            img = P.integer_image(N, 2, seed=N + 2, lo=-15, hi=15).cuda()
            Li = P.integer_linogram(N, 2, seed=N + 3, lo=-15, hi=15).cuda()
            fw = fast.forward(img).double()
            bp = gen.backproject(Li, scale=1.0).double()
            lhs = float((fw * Li.double()).sum())
            rhs = float((img.double() * bp).sum())
            adj = lhs == rhs
            ok &= adj
            print(f"N={N} forward adjoint identity exact {adj} ({lhs:.0f} vs {rhs:.0f})", flush=True)
        fast.close()
        gen.close()
print("ALL OK" if ok else "FAILURES")
sys.exit(0 if ok else 1)
