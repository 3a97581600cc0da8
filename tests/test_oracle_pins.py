"""Pins of the CPU oracle against things other than itself (-m "not gpu").

Each test names the passage / mathematical fact it checks.  A plausible mistake
in the oracle (dropped term, wrong sign or index, transposed operand, wrong
mirror, wrong weight) fails at least one of them.
"""
import json
import math
import os

import numpy as np
import pytest
from scipy import integrate, signal

from oracle import fbp_oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")))
COEFF_DIR = os.path.join(os.path.dirname(os.path.dirname(__file__)), "coeffs")


def load_coeffs(N=512, variant="dc0"):
    c = json.load(open(os.path.join(COEFF_DIR, f"iir_q3_n{N}_{variant}.json")))
    return np.array(c["b"]), np.array(c["a"]), c


# ----------------------------------------------------------------- ramp kernel
def test_ramp_kernel_spec_examples():
    assert np.array_equal(O.ramp_kernel(0), np.array(GOLD["ramp_kernel_L0_0"]["taps"]))
    g = GOLD["ramp_kernel_L0_2"]
    assert np.allclose(O.ramp_kernel(2), g["taps"], atol=g["tol"])


def test_ramp_kernel_equals_eq6_integral():
    """Eq.6: h(n) = 2 int_0^{1/2} |w| e^{2 pi i w n} dw, by quadrature."""
    h = O.ramp_kernel(9)
    for n in range(-9, 10):
        val, _ = integrate.quad(lambda w: 2.0 * w * math.cos(2 * math.pi * w * n), 0.0, 0.5,
                                epsabs=1e-14, epsrel=1e-14, limit=200)
        assert abs(val - h[n + 9]) < 1e-12, n


def test_ramp_kernel_equals_eq6_sinc_form():
    """Eq.6 right-hand side: sinc(pi n)/2 - sinc^2(pi n/2)/4 (numpy's normalised sinc)."""
    n = np.arange(-50, 51)
    rhs = np.sinc(n) / 2.0 - np.sinc(n / 2.0) ** 2 / 4.0
    assert np.allclose(O.ramp_kernel(50), rhs, atol=1e-15)


def test_ramp_kernel_dc_sum_closed_form():
    """sum_n h(n) -> 0 (sum over odd k of 1/k^2 = pi^2/8); finite L0 leaves the tail."""
    for L0 in (1, 7, 64, 1001):
        s = O.ramp_kernel(L0).sum()
        tail = 2.0 * sum(1.0 / (k * math.pi) ** 2 for k in range(L0 + 1 if L0 % 2 == 0 else L0 + 2, 200001, 2))
        # remaining tail beyond 200001 < 2/(pi^2 * 200001) ~ 1e-6 / 1
        assert abs(s - tail) < 2.0 / (math.pi ** 2 * 200000), L0


def test_causal_target_split():
    g = GOLD["causal_target_L0_2"]
    assert np.allclose(O.causal_target(2), g["taps"], atol=g["tol"])
    for L0 in (0, 5, 16):
        hp = O.causal_target(L0)
        h = O.ramp_kernel(L0)
        full = np.concatenate([hp[::-1], [0.0] * 0])  # h-(n) = h+(-n)
        rec = np.zeros(2 * L0 + 1)
        rec[L0:] += hp
        rec[: L0 + 1] += hp[::-1]
        assert np.allclose(rec, h, atol=0), L0   # Eq.10/11 split exactness
        assert len(full) == L0 + 1


# ----------------------------------------------------------------------- IIR
def test_iir_spec_examples():
    g = GOLD["iir_geometric"]
    r = O.iir_impulse_response(g["b"], g["a"], len(g["response"]) - 1)
    assert np.array_equal(r, np.array(g["response"]))
    g = GOLD["iir_pure_gain"]
    r = O.iir_impulse_response(g["b"], g["a"], len(g["response"]) - 1)
    assert np.array_equal(r, np.array(g["response"]))
    # closed form 0.5^n over a long horizon
    r = O.iir_impulse_response([1.0], [-0.5], 60)
    assert np.array_equal(r, 0.5 ** np.arange(61))


def test_iir_impulse_response_partial_fractions():
    """Closed form from the roots of A(z): h(n) = sum_i r_i p_i^n (+ direct terms)."""
    b, a, _ = load_coeffs(512, "spec")
    n = np.arange(200)
    r, p, k = signal.residuez(b, np.concatenate([[1.0], a]))
    h = np.real(sum(ri * pi ** n for ri, pi in zip(r, p)))
    for j, kj in enumerate(k):
        h[j] += np.real(kj)
    assert np.allclose(O.iir_impulse_response(b, a, 199), h, atol=1e-12)


@pytest.mark.parametrize("variant", ["spec", "dc0"])
def test_iir_matches_lfilter(variant):
    """Library routine: scipy.signal.lfilter forward, and on the reversed row."""
    b, a, _ = load_coeffs(512, variant)
    rng = np.random.default_rng(3)
    x = rng.normal(size=(5, 300))
    A = np.concatenate([[1.0], a])
    yc = signal.lfilter(b, A, x, axis=-1)
    ya = signal.lfilter(b, A, x[:, ::-1], axis=-1)[:, ::-1]
    assert np.allclose(O.iir_causal(x, b, a), yc, atol=1e-12)
    assert np.allclose(O.iir_anticausal(x, b, a), ya, atol=1e-12)
    assert np.allclose(O.iir_symmetric(x, b, a), yc + ya, atol=1e-12)


@pytest.mark.parametrize("variant", ["spec", "dc0"])
def test_iir_symmetric_equals_own_impulse_convolution(variant):
    """North-star check 1: symmetric IIR == direct convolution with its
    own two-sided impulse response g(m) = h(|m|), g(0) = 2 h(0) (Eq.10-12)."""
    b, a, _ = load_coeffs(512, variant)
    L = 256
    h = O.iir_impulse_response(b, a, L)
    g = np.concatenate([h[:0:-1], [2 * h[0]], h[1:]])       # lags -L..L
    rng = np.random.default_rng(4)
    x = rng.normal(size=(3, L))
    ref = np.stack([np.convolve(row, g)[L: L + L] for row in x])
    assert np.allclose(O.iir_symmetric(x, b, a), ref, atol=1e-9)


def test_iir_symmetric_impulse_is_symmetric():
    b, a, _ = load_coeffs(512, "spec")
    x = np.zeros((1, 201))
    x[0, 100] = 1.0
    y = O.iir_symmetric(x, b, a)[0]
    assert np.allclose(y[100 + np.arange(1, 100)], y[100 - np.arange(1, 100)], atol=1e-15)
    assert abs(y[100] - 2 * b[0]) < 1e-15


@pytest.mark.parametrize("variant", ["spec", "dc0"])
def test_iir_fit_error_matches_frozen_file(variant):
    """The frozen coefficients reproduce their recorded fit error against h+ (Eq.10)."""
    b, a, c = load_coeffs(2048, variant)
    K = c["K"]
    e = O.iir_impulse_response(b, a, K) - O.causal_target(K)
    assert abs(np.mean(e ** 2) - c["mse"]) <= 1e-6 * c["mse"]
    assert np.all(np.abs(O.iir_poles(a)) < 1.0)
    # the ramp approximation is good to the fit error: per-lag RMS ~ sqrt(mse)
    assert math.sqrt(c["mse"]) < 1e-4


def test_fir_filter_against_numpy_convolve():
    taps = O.ramp_kernel(20)
    rng = np.random.default_rng(5)
    x = rng.normal(size=(2, 100))
    ref = np.stack([np.convolve(r, taps)[20:120] for r in x])
    assert np.allclose(O.fir_filter(x, taps), ref, atol=1e-13)


# ------------------------------------------------------------- dyadic patterns
def test_dyadic_table_N8_golden():
    rows = GOLD["dyadic_offsets_N8"]["rows"]
    ref = np.array([[int(c) for c in r] for r in rows])
    assert np.array_equal(O.dyadic_offsets(8), ref)


@pytest.mark.parametrize("N", [1, 2, 4, 8, 16, 32, 64, 128])
def test_dyadic_properties(N):
    d = O.dyadic_offsets(N)
    assert np.array_equal(d, O.dyadic_offsets_closed_form(N))
    for y in range(N):
        assert np.array_equal(d[:, y], O.dyadic_offsets_column(N, y))
    assert np.array_equal(d, d.T)                       # d_t(y) = d_y(t)  (R5)
    assert np.all(d[:, 0] == 0)
    assert np.array_equal(d[:, N - 1], np.arange(N))     # pattern ends at shift t
    if N > 1:
        steps = np.diff(d, axis=1)
        assert np.all((steps == 0) | (steps == 1))       # one pixel per row, connected
        y = np.arange(N)
        dev = np.abs(d - np.arange(N)[:, None] * y[None, :] / (N - 1))
        assert dev.max() <= 0.5 + math.log2(N) / 4       # approximates a straight line


# ---------------------------------------------------------- forward projection
def test_forward_2x2_spec_example():
    g = GOLD["fht_2x2"]
    S = O.forward_project(np.array(g["image"], dtype=float))
    assert list(S[0, 0, 2:4]) == g["Lv_plus_t0_cols_2_3"]
    assert S[0, 1, 2] == g["Lv_plus_t1_col_2"]
    g2 = GOLD["fht_2x2_all_families"]
    assert np.array_equal(S, np.array(g2["S"], dtype=float))


@pytest.mark.parametrize("N", [2, 8, 32])
def test_forward_sample_matches_forward_project(N):
    """forward_sample (one sample, closed-form d_t) == forward_project (recursive
    pattern table, pinned below by brute force / SPEC identities) at every sample."""
    rng = np.random.default_rng(100 + N)
    img = rng.integers(-50, 50, size=(N, N)).astype(float)
    S = O.forward_project(img)
    for f in range(4):
        for t in range(N):
            for s in range(2 * N):
                assert O.forward_sample(img, f, t, s) == S[f, t, s]


@pytest.mark.parametrize("N", [2, 4, 8, 16])
def test_forward_brute_force_and_fht_forward_bit_exact(N):
    """FHT == brute-force dyadic sums on random integer images, exactly;
    SPEC.md:44/475: every (family, t) row sums to the image total; t=0
    rows of the v families are column sums."""
    rng = np.random.default_rng(N)
    for _ in range(3):
        img = rng.integers(-50, 50, size=(N, N)).astype(float)
        S = O.forward_project(img)
        assert np.array_equal(S, O.fht_forward(img))
        assert np.all(S.sum(axis=2) == img.sum())
        assert np.array_equal(S[0, 0, N:], img.sum(axis=0))
        assert np.array_equal(S[1, 0, N:], img.sum(axis=0)[::-1])
        # support of row t is [N - t, 2N)   (R2)
        for t in range(N):
            assert np.all(S[:, t, : N - t] == 0)


# ------------------------------------------------------------- back projection
def test_backprojection_2x2_golden():
    g = GOLD["fht_2x2_all_families"]
    S = np.array(g["S"], dtype=float)
    out = O.combine(O.fht_backproject(S), 1.0)
    assert np.array_equal(out, np.array(g["unweighted_backprojection"], dtype=float))
    assert np.array_equal(O.combine(O.backproject_direct(S), 1.0), out)


def test_backprojection_impulse_peak():
    g = GOLD["impulse_N4"]
    img = np.zeros((4, 4))
    img[g["y"], g["x"]] = 1.0
    out = O.combine(O.fht_backproject(O.forward_project(img)), 1.0)
    assert out[g["y"], g["x"]] == g["peak"] == out.max()
    assert np.argmax(out) == g["y"] * 4 + g["x"]


@pytest.mark.parametrize("N", [2, 4, 8, 16])
def test_backprojection_is_exact_adjoint(N):
    """<R f, P> = <f, B P> exactly on integers: pins the back projection (incl. the
    family un-mirror/un-transpose of Eq.20-22) to the pinned forward projection."""
    rng = np.random.default_rng(100 + N)
    img = rng.integers(-20, 20, size=(N, N)).astype(float)
    P = rng.integers(-20, 20, size=(4, N, 2 * N)).astype(float)
    lhs = float(np.sum(O.forward_project(img) * P))
    rhs = float(np.sum(img * O.combine(O.backproject_direct(P), 1.0)))
    assert lhs == rhs
    rhs2 = float(np.sum(img * O.combine(O.fht_backproject(P), 1.0)))
    assert lhs == rhs2


@pytest.mark.parametrize("N", [2, 4, 8, 16, 32, 64])
def test_fht_backprojection_bit_exact_vs_direct_integers(N):
    """North-star check 2: FHT == brute-force sums along every dyadic pattern, bit-exact."""
    rng = np.random.default_rng(200 + N)
    P = rng.integers(-511, 512, size=(4, N, 2 * N)).astype(float)
    assert np.array_equal(O.fht_backproject(P), O.backproject_direct(P))
    d = O.dyadic_offsets(N)
    for _ in range(10):
        f, y, x = rng.integers(0, 4), rng.integers(0, N), rng.integers(0, N)
        assert O.backproject_pixel(P, f, y, x, d) == O.fht_backproject(P)[f, y, x]


def test_fht_backprojection_float_vs_direct_N256():
    """North-star check 3: direct Theta(N^3) BP == FHT BP to float64 rounding."""
    N = 256
    rng = np.random.default_rng(7)
    P = rng.normal(size=(4, N, 2 * N))
    A = O.fht_backproject(P)
    B = O.backproject_direct(P)
    assert np.max(np.abs(A - B)) <= 1e-12 * np.max(np.abs(B))


def test_zero_in_zero_out():
    b, a, _ = load_coeffs(64, "spec")
    assert np.all(O.reconstruct(np.zeros((4, 8, 16)), b, a) == 0)


# ------------------------------------------------- end-to-end convention pins
def _raster_ellipses(N, ell):
    """Point-sampled (pixel centres) ellipse phantom, test-local."""
    yy, xx = np.mgrid[0:N, 0:N] + 0.5
    img = np.zeros((N, N))
    for cx, cy, a, b, phi, rho in ell:
        u = (xx - cx) * math.cos(phi) + (yy - cy) * math.sin(phi)
        v = -(xx - cx) * math.sin(phi) + (yy - cy) * math.cos(phi)
        img += rho * ((u / a) ** 2 + (v / b) ** 2 <= 1.0)
    return img


def _phantom(N, seed):
    rng = np.random.default_rng(seed)
    ell = []
    for _ in range(10):
        r = 0.8 * N / 2 * math.sqrt(rng.uniform())
        th = rng.uniform(0, 2 * math.pi)
        ell.append((N / 2 + r * math.cos(th), N / 2 + r * math.sin(th),
                    rng.uniform(N / 16, N / 4), rng.uniform(N / 16, N / 4),
                    rng.uniform(0, math.pi), rng.uniform(0.2, 1.0)))
    return _raster_ellipses(N, ell)


def _fit(rec, ph):
    scale = float(np.sum(rec * ph) / np.sum(ph * ph))
    rel = float(np.sqrt(np.mean((rec - ph) ** 2)) / np.sqrt(np.mean(ph ** 2)))
    return scale, rel


@pytest.mark.parametrize("N", [32, 64])
def test_fir_fbp_recovers_phantom_scale(N):
    """Weight w = 1/N (R7) and the family geometry (R4): FIR-ramp-filtered (Eq.8,
    L0 = 2N) FHT back projection of the dyadic projection of a phantom reproduces
    it with best-fit scale 1 (a wrong weight, mirror or transpose gives 0.4-0.6 or 2)."""
    ph = _phantom(N, 11)
    S = O.fht_forward(ph)
    F = O.fir_filter(S, O.ramp_kernel(2 * N))
    rec = O.combine(O.fht_backproject(F), 1.0 / N)
    scale, rel = _fit(rec, ph)
    assert abs(scale - 1.0) < 0.03, scale
    assert rel < 0.12, rel


def test_iir_fbp_dc0_recovers_phantom():
    """Quality sanity (not parity): the fitted M=Q=3 zero-DC recursive pair (Eq.12-13)
    gives a recognisable reconstruction at N=64 (scale 0.84, rel-RMSE 0.24 measured).
    The 3-pole fit cannot follow the 1/n^2 tail of Eq.7, so quality falls with N
    (DESIGN.md §3 R14); coefficients are an input, parity does not depend on them."""
    N = 64
    b, a, _ = load_coeffs(N, "dc0")
    ph = _phantom(N, 12)
    S = O.fht_forward(ph)
    rec = O.reconstruct(S, b, a)
    scale, rel = _fit(rec, ph)
    assert abs(scale - 1.0) < 0.25, scale
    assert rel < 0.35, rel


# ------------------------------------------------- NEXT-2: (r,theta) -> (s,t)
def _family_line_np(f, A, k, N):
    """P0, D of the phantom generator's line model (input-side code, not the oracle)."""
    import torch
    from phantoms.generator import _family_line
    (px, py), (dx, dy) = _family_line(f, torch.tensor(float(A), dtype=torch.float64),
                                      torch.tensor(float(k), dtype=torch.float64), N)
    return (float(px), float(py)), (float(dx), float(dy))


def test_linogram_line_rtheta_geometry():
    """Every point of the R2 line (phantom generator's model) satisfies (p - c).n = r;
    theta ranges are the paper's four classes: f1 = L_v- [0, pi/4],
    f3 = L_h- [pi/4, pi/2], f2 = L_h+ [pi/2, 3pi/4], f0 = L_v+ [3pi/4, pi) (t = 0: 0)."""
    import math
    N = 16
    rng = np.random.default_rng(5)
    rngs = {1: (0, math.pi / 4), 3: (math.pi / 4, math.pi / 2), 2: (math.pi / 2, 3 * math.pi / 4),
            0: (3 * math.pi / 4, math.pi)}
    for _ in range(200):
        f, t, s = int(rng.integers(4)), int(rng.integers(N)), int(rng.integers(2 * N))
        r, th, L = O.linogram_line_rtheta(f, t, s, N)
        k = t / (N - 1)
        P0, D = _family_line_np(f, s - N + 0.5 - 0.5 * k, k, N)
        assert abs(L - math.hypot(*D)) < 1e-12 and 0.0 <= th < math.pi
        for tau in (0.0, 3.7, float(N)):
            px, py = P0[0] + tau * D[0], P0[1] + tau * D[1]
            assert abs((px - N / 2) * math.cos(th) + (py - N / 2) * math.sin(th) - r) < 1e-9
        lo, hi = rngs[f]
        if not (f == 0 and t == 0):
            assert lo - 1e-12 <= th <= hi + 1e-12, (f, t, th)
    assert O.linogram_line_rtheta(0, 0, 5, N)[1] == 0.0          # vertical line, normal along x


def test_sinogram_sample_wrap_and_bins():
    """Linear interpolation in both indices; the row after P-1 is row 0 at -r; bins
    outside the detector read 0 (R23)."""
    import math
    P_, R_ = 8, 9
    p = np.zeros((P_, R_))
    p[0, 2] = 1.0                                  # r = (2 - 4) * 1 = -2 at theta = 0
    # theta half-way between rows 7 and 8 == row 0 at -r: r = +2 reads p[0][2] with weight 1/2
    th = (P_ - 0.5) * math.pi / P_
    assert abs(O.sinogram_sample(p, th, 2.0, 1.0) - 0.5) < 1e-12
    assert abs(O.sinogram_sample(p, 0.0, -1.5, 1.0) - 0.5) < 1e-12   # half-way between bins 2, 3
    assert O.sinogram_sample(p, 0.0, 100.0, 1.0) == 0.0


def test_resample_zero_and_linear():
    N = 8
    rng = np.random.default_rng(2)
    p1, p2 = rng.normal(size=(16, 15)), rng.normal(size=(16, 15))
    assert not O.resample_sinogram(np.zeros((16, 15)), N).any()
    lhs = O.resample_sinogram(2.0 * p1 - 3.0 * p2, N)
    rhs = 2.0 * O.resample_sinogram(p1, N) - 3.0 * O.resample_sinogram(p2, N)
    assert np.allclose(lhs, rhs, atol=1e-12)


def _blob_case(N, n_angles, dr, seed=0):
    """Gaussian blobs: analytic sinogram p = A sqrt(2 pi) s exp(-q^2 / 2 s^2) and the
    analytic linogram along the phantom generator's lines, A sqrt(2 pi) s exp(-d^2/2s^2)/|D|
    (blobs far inside the square)."""
    import math
    rng = np.random.default_rng(seed)
    blobs = [(N / 2 + rng.uniform(-0.25, 0.25) * N, N / 2 + rng.uniform(-0.25, 0.25) * N,
              rng.uniform(0.5, 1.5), rng.uniform(N / 16, N / 8)) for _ in range(4)]
    nb = int(math.ceil(N * math.sqrt(2) / dr)) + 4
    th = np.arange(n_angles) * math.pi / n_angles
    r = (np.arange(nb) - 0.5 * (nb - 1)) * dr
    sino = np.zeros((n_angles, nb))
    for ex, ey, A, sg in blobs:
        q = r[None, :] - ((ex - N / 2) * np.cos(th)[:, None] + (ey - N / 2) * np.sin(th)[:, None])
        sino += A * math.sqrt(2 * math.pi) * sg * np.exp(-q * q / (2 * sg * sg))
    ref = np.zeros((4, N, 2 * N))
    for f in range(4):
        for t in range(N):
            k = t / (N - 1)
            for s in range(2 * N):
                P0, D = _family_line_np(f, s - N + 0.5 - 0.5 * k, k, N)
                L = math.hypot(*D)
                for ex, ey, A, sg in blobs:
                    d = ((ex - P0[0]) * D[1] - (ey - P0[1]) * D[0]) / L
                    ref[f, t, s] += A * math.sqrt(2 * math.pi) * sg * math.exp(-d * d / (2 * sg * sg)) / L
    return sino, ref


def test_resample_smooth_blobs_second_order():
    """PAPER.md:178 linear interpolation + Eq.15 stretch: on smooth blobs the error
    vs the analytic linogram is O(h^2) (x4 per halving of the sampling), which only
    an exact (r, theta) geometry and the right k_t direction give."""
    errs = []
    for n_angles, dr in ((64, 1.0), (128, 0.5)):
        sino, ref = _blob_case(32, n_angles, dr)
        S = O.resample_sinogram(sino, 32, dr)
        errs.append(np.abs(S - ref).max() / np.abs(ref).max())
    assert errs[1] < 6e-3 and errs[0] / errs[1] > 3.0, errs


def test_resample_ellipses_close_to_analytic_linogram():
    """Sharp ellipses (inside the square): relative RMS error ~1 % at N = 64 (edges are
    not smooth), below the 2 % SPEC-style interpolation tolerance."""
    import phantoms as P
    N = 64
    E = P.draw_ellipses(N, 6, (N / 16, N / 5), seed=N)
    E.cx = N / 2 + 0.5 * (E.cx - N / 2)
    E.cy = N / 2 + 0.5 * (E.cy - N / 2)
    ref = P.linogram_of_ellipses(E, N).numpy()
    sino = P.sinogram_of_ellipses(E, N, 4 * N, int(math.ceil(N * math.sqrt(2) / 0.5)) + 4, 0.5).numpy()
    S = O.resample_sinogram(sino, N, 0.5)
    assert math.sqrt(((S - ref) ** 2).mean()) / math.sqrt((ref ** 2).mean()) < 0.02


# ------------------------------------------- NEXT-4: conventional (r, theta) FBP
def test_backproject_rtheta_single_angle_smears():
    """Eq.5 with one nonzero angle: the back projection of a row
    that is linear in the bin index is constant along the line direction and equals
    pi/P times the row at r = x.n (linear interpolation is exact on a linear row).
    theta = 0 (normal +x): constant down columns; theta = pi/2 (normal +y): constant
    along rows.  Pins the angle origin, the centre (N/2, N/2) and the pi/P weight."""
    N, P, R = 16, 8, 40
    c = np.arange(N) + 0.5 - N / 2.0
    q = np.zeros((P, R))
    q[0] = np.arange(R) * 2.0 + 1.0              # value 2j + 1 at bin j
    img = O.backproject_rtheta(q, N)
    expect_x = math.pi / P * (2.0 * (c + 0.5 * (R - 1)) + 1.0)
    assert np.allclose(img, np.broadcast_to(expect_x[None, :], (N, N)), atol=1e-12)
    q = np.zeros((P, R))
    q[P // 2] = np.arange(R) * 2.0 + 1.0
    img = O.backproject_rtheta(q, N, dr=0.5)     # bin j at r = (j - (R-1)/2) / 2
    expect_y = math.pi / P * (2.0 * (2.0 * c + 0.5 * (R - 1)) + 1.0)
    assert np.allclose(img, np.broadcast_to(expect_y[:, None], (N, N)), atol=1e-12)


def test_backproject_rtheta_constant_and_outside():
    """A constant sinogram back-projects to pi * constant (sum of P weights pi/P);
    bins outside the detector read 0 (a detector narrower than the image leaves
    the corners' far angles empty)."""
    N, P = 32, 24
    R = int(math.ceil(N * math.sqrt(2))) + 4
    img = O.backproject_rtheta(np.full((P, R), 3.0), N)
    assert np.allclose(img, 3.0 * math.pi, atol=1e-12)
    img = O.backproject_rtheta(np.full((P, 9), 1.0), N)   # |r| <= 4 only
    assert abs(img[N // 2, N // 2] - math.pi) < 1e-12
    assert img[0, 0] < 0.5 * math.pi


def test_ramp_filter_rtheta_zero_dc_and_spacing():
    """Eq.7 taps sum to zero over the full band (sum_odd 1/n^2 = pi^2/8), so a long
    constant row filters to ~0 in its interior; halving dr scales the kernel by
    1/dr (h_dr(m) = h(m)/dr^2, times dr)."""
    R = 401
    q = O.ramp_filter_rtheta(np.ones((1, R)), dr=1.0, L0=4000)[0]
    assert abs(q[R // 2]) < 2e-3            # tail beyond the row end: sum_{|m|>200} ~ 1/(pi^2 200)
    x = np.random.default_rng(5).standard_normal((2, 64))
    assert np.allclose(O.ramp_filter_rtheta(x, dr=0.5), 2.0 * O.ramp_filter_rtheta(x, dr=1.0),
                       atol=1e-13)


def _disc_sinogram(P, R, dr, rho, x0=0.0, y0=0.0):
    """Closed-form chord lengths of a unit-density disc of radius rho centred at
    (x0, y0) relative to the image centre: p(r, theta) = 2 sqrt(rho^2 - (r - x0 cos
    - y0 sin)^2) (textbook; independent of the oracle)."""
    th = np.arange(P) * math.pi / P
    r = (np.arange(R) - 0.5 * (R - 1)) * dr
    d = r[None, :] - (x0 * np.cos(th) + y0 * np.sin(th))[:, None]
    return 2.0 * np.sqrt(np.clip(rho * rho - d * d, 0.0, None))


@pytest.mark.parametrize("dr", [1.0, 0.5])
def test_fbp_rtheta_recovers_disc(dr):
    """FBP (Eq.3 + Eq.5) inverts the Radon transform: an off-centre unit disc is
    recovered with density 1 inside and 0 outside (pins the |omega| kernel scale,
    the 1/dr spacing, the pi/P half-turn weight and the centre/orientation: a
    flipped theta or axis would move the disc)."""
    N, P = 64, 128
    R = int(math.ceil(N * math.sqrt(2) / dr)) + 8
    x0, y0, rho = 9.0, -12.0, 10.0
    img = O.fbp_rtheta(_disc_sinogram(P, R, dr, rho, x0, y0), N, dr)
    c = np.arange(N) + 0.5 - N / 2.0
    X, Y = np.meshgrid(c, c)
    d = np.hypot(X - x0, Y - y0)
    inside, outside = img[d < 0.8 * rho], img[(d > 1.3 * rho) & (np.hypot(X, Y) < N / 2 - 2)]
    assert abs(inside.mean() - 1.0) < 0.01 and np.max(np.abs(inside - 1.0)) < 0.05
    assert abs(outside.mean()) < 0.01 and np.max(np.abs(outside)) < 0.1   # edge streaks
    # the mirrored disc position must NOT match (orientation pin)
    dm = np.hypot(X - x0, Y + y0)
    assert img[(dm < 0.5 * rho) & (d > 1.3 * rho)].mean() < 0.05


def test_fbp_rtheta_recovers_ellipse_phantom():
    """End to end on the phantom generator's analytic (r, theta) sinogram (textbook
    ellipse projection, R23 geometry): best-fit scale 1 and a small RMSE
    against the pixel-centre phantom (edges dominate the residual)."""
    import phantoms
    N, P = 64, 128
    R = int(math.ceil(N * math.sqrt(2))) + 8
    E = phantoms.draw_ellipses(N, 10, (6.0, 20.0), seed=41)
    p = phantoms.sinogram_of_ellipses(E, N, P, R).numpy()
    img = O.fbp_rtheta(p, N)
    ref = phantoms.image_of_ellipses(E, N)
    scale = float(np.sum(img * ref) / np.sum(ref * ref))
    assert abs(scale - 1.0) < 0.03
    assert np.sqrt(np.mean((img - ref) ** 2)) / np.sqrt(np.mean(ref ** 2)) < 0.2
