"""NEXT-3: the offline IIR coefficient fit and its order sweep
(-m "not gpu").

PAPER.md:151-153 (§3): the causal recursive filter's coefficients minimise the mean
square error between the impulse responses of the FIR ramp filter (Eq.8, causal half
h+ of Eq.10) and the IIR filter (Eq.9), by a simplex search.
tools/fit_iir.py implements that fit (reading R13); coeffs/sweep/ holds the q = 1..5
sweep (Fig. 2a analogue) it writes.  The end-to-end quality checks go through the
fp64 oracle (test infrastructure) on a seeded phantom.
"""
import json
import math
import os
import sys

import numpy as np
import pytest
from scipy import signal

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import fit_iir  # noqa: E402

SWEEP = os.path.join(ROOT, "coeffs", "sweep")


def sweep(q, v):
    return json.load(open(os.path.join(SWEEP, f"iir_q{q}_{v}.json")))


def test_planted_filter_recovered():
    """A target that IS the impulse response of a stable (M, Q) = (2, 2) filter is
    matched to rounding by the simplex fit (SPEC.md fit_iir example)."""
    b, a = [0.3, -0.12], [-0.7, 0.2]
    K = 64
    imp = np.zeros(K + 1)
    imp[0] = 1.0
    h = signal.lfilter(b, [1.0] + a, imp)
    r = fit_iir.fit(K, 2, 2, dc0=False, target=h, restarts=8)
    assert r["sse"] < 1e-20
    assert np.allclose(r["b"], b, atol=1e-9) and np.allclose(r["a"], a, atol=1e-9)


def test_half_ramp_is_eq10():
    """Target of the fit: h+(0) = h(0)/2 = 1/8, h+(n) = h(n) = -1/(n pi)^2 for odd n,
    0 for even n > 0 (Eq.7, Eq.10)."""
    h = fit_iir.half_ramp(9)
    assert h[0] == 0.125
    for n in range(1, 10):
        assert h[n] == (-1.0 / (n * math.pi) ** 2 if n % 2 else 0.0)


@pytest.mark.parametrize("v", ["spec", "dc0"])
def test_sweep_mse_non_increasing_in_order(v):
    """More taps never fit worse (the q-tap optimum is feasible for q+1 with zero
    taps; the simplex restarts find it): MSE(q) non-increasing for q = 1..5."""
    mse = [sweep(q, v)["mse"] for q in range(1, 6)]
    for q in range(1, 5):
        assert mse[q] <= mse[q - 1] * (1 + 1e-9), (v, q, mse)
    assert mse[4] < 1e-3 * mse[0]


@pytest.mark.parametrize("q", [1, 2, 3, 4, 5])
def test_sweep_files_consistent(q):
    """Each frozen file reproduces its recorded fit error, is stable and,
    for dc0, has zero DC gain exactly (sum b = 0, reading R14)."""
    for v in ("spec", "dc0"):
        c = sweep(q, v)
        assert c["M"] == q and c["Q"] == q and len(c["b"]) == q and len(c["a"]) == q
        K = c["K"]
        imp = np.zeros(K + 1)
        imp[0] = 1.0
        h = signal.lfilter(c["b"], [1.0] + c["a"], imp)
        sse = float(np.sum((h - fit_iir.half_ramp(K)) ** 2))
        assert sse == pytest.approx(c["sse"], rel=1e-9, abs=1e-18)
        assert np.max(np.abs(np.roots([1.0] + c["a"]))) < 1.0
        if v == "dc0":
            assert abs(sum(c["b"])) < 1e-15


def _phantom(N, seed, axes):
    import phantoms
    E = phantoms.draw_ellipses(N, 10, axes, seed)
    return phantoms.image_of_ellipses(E, N)


def _fit(rec, ref):
    scale = float(np.sum(rec * ref) / np.sum(ref * ref))
    rel = float(np.sqrt(np.mean((rec - ref) ** 2)) / np.sqrt(np.mean(ref ** 2)))
    return scale, rel


def test_order_sweep_quality_n64():
    """Fig. 2a analogue at N = 64 through the oracle (dyadic line sums of a seeded
    10-ellipse phantom, semi-axes N/16..N/4, densities in [-0.5, 1]): the FIR reference
    (L0 = 2N) reproduces the phantom (scale 1); q = 1 is useless (plain MSE: DC leak,
    scale ~6.5; zero DC: the one-pole fit degenerates to b = 0); the zero-DC fits
    approach the FIR result as q grows (rel-RMSE vs FIR 0.50 / 0.046 / 0.011 at
    q = 2 / 3 / 5) and beat the plain-MSE fits at q = 3 (0.47).  Quality, not parity:
    profiles/r02_next3_order_sweep.md has N up to 2048."""
    from oracle import fbp_oracle as O
    N = 64
    ph = _phantom(N, 11, (N / 16, N / 4))
    S = O.fht_forward(ph)
    fir = O.combine(O.fht_backproject(O.fir_filter(S, O.ramp_kernel(2 * N))), 1.0 / N)
    s_fir, r_fir = _fit(fir, ph)
    assert abs(s_fir - 1.0) < 0.02 and r_fir < 0.15
    res = {}
    for q in (1, 2, 3, 5):
        for v in ("spec", "dc0"):
            c = sweep(q, v)
            res[(q, v)] = _fit(O.reconstruct(S, c["b"], c["a"]), fir)
    assert res[(1, "spec")][0] > 3.0                     # DC leak of the plain-MSE fit
    assert res[(1, "dc0")][1] > 0.99                     # degenerate one-pole zero-DC fit
    assert res[(5, "dc0")][1] < res[(3, "dc0")][1] < res[(2, "dc0")][1]
    assert res[(3, "dc0")][1] < 0.5 * res[(3, "spec")][1]
    assert abs(res[(5, "dc0")][0] - 1.0) < 0.02 and res[(5, "dc0")][1] < 0.03
