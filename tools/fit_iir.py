#!/usr/bin/env python
"""Offline IIR coefficient fit (§3, §5).

The paper fits the causal recursive filter so that its impulse response matches
the causal half h+ of the discrete ramp kernel (Eq.7, Eq.10) in mean square, by
"the Simplex method".  It prints no coefficient values, so they
are produced here once and FROZEN in ``coeffs/*.json`` (reading R13):

  * objective  sum_{n=0}^{K} (h_iir(n) - h+(n))^2,  K = N; the
    JSON records it as ``sse`` and as the mean square error ``mse`` = sse/(K+1)
  * Nelder-Mead, 8 seeded restarts, initial simplex scale 0.1, xatol/fatol 1e-10,
    <= 20000 evaluations, stability penalty 1e6 * max(0, max|pole| - 1 + 1e-6)
    
  * two variants: ``spec`` (plain MSE) and ``dc0`` (same objective
    with the hard constraint sum(b) = 0, i.e. zero DC gain, reading R14).

Standalone CPU tool: uses scipy only; imports neither ``oracle`` nor the product.
Usage:  python tools/fit_iir.py --n 64 512 1024 2048 4096 --order 3
        python tools/fit_iir.py --sweep 1 2 3 4 5 --k 512     (NEXT-3 order sweep,
            M = Q = q, both variants -> coeffs/sweep/iir_q<q>_<variant>.json)
"""
from __future__ import annotations

import argparse
import json
import math
import os

import numpy as np
from scipy import optimize, signal


def half_ramp(K: int) -> np.ndarray:
    n = np.arange(K + 1)
    h = np.where(n % 2 == 1, -1.0 / (np.maximum(n, 1) * math.pi) ** 2, 0.0)
    h[0] = 0.125
    return h


def unpack(p, M, Q, dc0):
    if dc0:
        b = np.concatenate([p[: M - 1], [-np.sum(p[: M - 1])]])
        a = p[M - 1: M - 1 + Q]
    else:
        b = p[:M]
        a = p[M: M + Q]
    return b, a


def fit(K: int, M: int, Q: int, dc0: bool, restarts: int = 8, seed: int = 0, target=None):
    """Nelder-Mead fit of b (M taps), a (Q taps) so that the causal impulse response
    matches `target` (default: the causal half h+ of the ramp kernel, Eq.10) in
    least squares over lags 0..K."""
    target = half_ramp(K) if target is None else np.asarray(target, dtype=np.float64)[: K + 1]
    imp = np.zeros(K + 1)
    imp[0] = 1.0

    def obj(p):
        b, a = unpack(p, M, Q, dc0)
        roots = np.roots(np.concatenate([[1.0], a])) if Q else np.zeros(0)
        excess = max(0.0, (np.max(np.abs(roots)) if len(roots) else 0.0) - (1.0 - 1e-6))
        if excess > 0:
            return 1e6 * excess + 1.0
        h = signal.lfilter(b, np.concatenate([[1.0], a]), imp)
        return float(np.sum((h - target) ** 2))

    rng = np.random.default_rng(seed)
    npar = (M - 1 if dc0 else M) + Q
    best = None
    for r in range(restarts):
        x0 = rng.normal(0.0, 0.3, npar)
        # start from a stable single pole near 0.5
        if Q:
            x0[(M - 1 if dc0 else M)] = -0.5 + 0.1 * rng.normal()
        sim = np.vstack([x0] + [x0 + 0.1 * np.eye(npar)[i] for i in range(npar)])
        res = optimize.minimize(obj, x0, method="Nelder-Mead",
                                options=dict(initial_simplex=sim, xatol=1e-10, fatol=1e-14,
                                             maxfev=20000, maxiter=20000))
        if best is None or res.fun < best[0]:
            best = (res.fun, res.x, r, res.nfev)
    b, a = unpack(best[1], M, Q, dc0)
    poles = np.roots(np.concatenate([[1.0], a])) if Q else np.zeros(0)
    return dict(M=M, Q=Q, b=[float(v) for v in b], a=[float(v) for v in a],
                sse=float(best[0]), mse=float(best[0]) / (K + 1), max_pole=float(np.max(np.abs(poles))) if Q else 0.0,
                dc_gain=float(2.0 * np.sum(b) / (1.0 + np.sum(a))), K=K,
                restart=int(best[2]), nfev=int(best[3]), seed=seed,
                variant="dc0" if dc0 else "spec")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="+", default=[64, 512, 1024, 2048, 4096])
    ap.add_argument("--order", type=int, default=3)
    ap.add_argument("--sweep", type=int, nargs="*", default=None, help="orders q of the NEXT-3 sweep")
    ap.add_argument("--k", type=int, default=512, help="fit range K of the sweep")
    ap.add_argument("--out", default=os.path.join(os.path.dirname(__file__), "..", "coeffs"))
    args = ap.parse_args()
    os.makedirs(args.out, exist_ok=True)
    if args.sweep:
        out = os.path.join(args.out, "sweep")
        os.makedirs(out, exist_ok=True)
        for q in args.sweep:
            for dc0 in (False, True):
                r = fit(args.k, q, q, dc0)
                path = os.path.join(out, f"iir_q{q}_{r['variant']}.json")
                with open(path, "w") as fh:
                    json.dump(r, fh, indent=1)
                print(path, "mse", r["mse"], "max|p|", r["max_pole"], "dc", r["dc_gain"])
        return
    for N in args.n:
        for dc0 in (False, True):
            r = fit(N, args.order, args.order, dc0)
            path = os.path.join(args.out, f"iir_q{args.order}_n{N}_{r['variant']}.json")
            with open(path, "w") as fh:
                json.dump(r, fh, indent=1)
            print(path, r["mse"], r["max_pole"], r["dc_gain"])


if __name__ == "__main__":
    main()
