"""CPU float64 ORACLE for the fast-FBP hot path of arXiv 2007.06289.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import, call or
execute anything under ``oracle/``.  The product path (``paper_2007_06289_b200``)
never imports this module and shares no code, table or constant with it.

Plain, slow, obviously-correct NumPy float64.  Every function follows the passage
of ``PAPER.md`` it cites (``PAPER.md:<line>`` = line in the paper's LaTeX, plus
section / equation).  Where the paper is silent or garbled the reading taken is
the one listed in DESIGN.md §3 ("Readings"), referenced here as R<k>.

Notation:
  * N = 2**n, image ``img[y][x]`` (row y, column x).
  * linogram / sinogram ``S[f][t][s]``: family f in {0: L_v+, 1: L_v-, 2: L_h+,
    3: L_h-} (SPEC.md:41 order), shift t in [0, N), intercept s in [0, 2N)
    with s = x0 + N (R2).
  * family views  G_0 = img[y][x], G_1 = img[y][N-1-x], G_2 = img[x][y],
    G_3 = img[N-1-x][y]  (Eq.16 transpose + mirror for the shift sign, R4).

Pinned by ``tests/test_oracle_pins.py`` (closed forms, SPEC worked examples,
library routines, brute force, exact adjoint identities; the NEXT-2 resampling
against the phantom generator's own line model and analytic linograms).  Parity status per
function is listed in DESIGN.md §4; nothing here is "parity unpinned" except the
numeric values of the paper's own (unprinted) IIR coefficients, which are an
input, not a computation.
"""
from __future__ import annotations

import math

import numpy as np

__all__ = [
    "ramp_kernel", "causal_target", "iir_impulse_response", "iir_causal",
    "iir_anticausal", "iir_symmetric", "fir_filter", "dyadic_offsets",
    "dyadic_offsets_closed_form", "dyadic_offsets_column", "family_views", "forward_project",
    "backproject_direct", "backproject_pixel", "fht_backproject", "combine",
    "reconstruct", "iir_poles", "fht_forward",
    "ramp_filter_rtheta", "backproject_rtheta", "fbp_rtheta",
]


# --------------------------------------------------------------------------
# §3  Fast recursive filtering
# --------------------------------------------------------------------------

def ramp_kernel(L0: int) -> np.ndarray:
    """Band-limited discrete ramp kernel h(n), n = -L0..L0.

    PAPER.md:97-101 (§3, Eq.7): h(0) = 1/4, h(n) = 0 for even n != 0,
    h(n) = -1/(n*pi)^2 for odd n.  Returns the 2*L0+1 taps (Eq.8, L = 2L0+1).
    """
    n = np.arange(-L0, L0 + 1)
    h = np.zeros(2 * L0 + 1, dtype=np.float64)
    for i, k in enumerate(n):
        if k == 0:
            h[i] = 0.25
        elif k % 2 == 0:
            h[i] = 0.0
        else:
            h[i] = -1.0 / (k * math.pi) ** 2
    return h


def causal_target(L0: int) -> np.ndarray:
    """Causal half h+(n), n = 0..L0 of the ramp kernel.

    PAPER.md:119-133 (§3, Eq.10): h+(0) = h(0)/2, h+(n) = h(n) for n > 0.
    """
    h = ramp_kernel(L0)
    hp = h[L0:].copy()
    hp[0] = h[L0] / 2.0
    return hp


def iir_impulse_response(b, a, n_max: int) -> np.ndarray:
    """Run the difference equation Eq.9 on a unit impulse, zero initial state.

    PAPER.md:112-117 (§3, Eq.9):
        p~(n) = sum_{k=0}^{M-1} b_k p(n-k) - sum_{k=1}^{Q} a_k p~(n-k).
    ``b`` = (b_0..b_{M-1}), ``a`` = (a_1..a_Q).  Returns outputs n = 0..n_max.
    """
    x = np.zeros(n_max + 1)
    x[0] = 1.0
    return iir_causal(x[None, :], b, a)[0]


def iir_causal(x: np.ndarray, b, a) -> np.ndarray:
    """Causal pass p~+ of Eq.13 (upper signs) along the last axis.

    PAPER.md:145-149 (§3, Eq.13):
        p~+(n) = sum_k b_k p(n-k) - sum_k a_k p~+(n-k),   n = 0 .. len-1,
    with per-direction feedback (R10) and zero initial state / zero extension
    (R11).  Vectorised over leading axes, loop over n.
    """
    x = np.asarray(x, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    a = np.asarray(a, dtype=np.float64)
    L = x.shape[-1]
    y = np.zeros_like(x)
    for n in range(L):
        acc = np.zeros(x.shape[:-1])
        for k in range(len(b)):
            if n - k >= 0:
                acc = acc + b[k] * x[..., n - k]
        for k in range(1, len(a) + 1):
            if n - k >= 0:
                acc = acc - a[k - 1] * y[..., n - k]
        y[..., n] = acc
    return y


def iir_anticausal(x: np.ndarray, b, a) -> np.ndarray:
    """Anticausal pass p~- of Eq.13 (lower signs) along the last axis.

    PAPER.md:145-149 (§3, Eq.13):
        p~-(n) = sum_k b_k p(n+k) - sum_k a_k p~-(n+k),   n = len-1 .. 0,
    with a^- = a^+, b^- = b^+ (PAPER.md:153), per-direction feedback (R10),
    zero state / zero extension beyond the row end (R11).
    """
    x = np.asarray(x, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    a = np.asarray(a, dtype=np.float64)
    L = x.shape[-1]
    y = np.zeros_like(x)
    for n in range(L - 1, -1, -1):
        acc = np.zeros(x.shape[:-1])
        for k in range(len(b)):
            if n + k < L:
                acc = acc + b[k] * x[..., n + k]
        for k in range(1, len(a) + 1):
            if n + k < L:
                acc = acc - a[k - 1] * y[..., n + k]
        y[..., n] = acc
    return y


def iir_symmetric(x: np.ndarray, b, a) -> np.ndarray:
    """Symmetric recursive ramp filter: p~ = p~+ + p~- (Eq.12).

    Both passes include the lag-0 term b_0 p(n) (Eq.10 h+-(0) = h(0)/2, R12).
    """
    return iir_causal(x, b, a) + iir_anticausal(x, b, a)


def iir_poles(a) -> np.ndarray:
    """Roots of the feedback polynomial z^Q + a_1 z^{Q-1} + ... + a_Q (Eq.9, R15).

    The filter is stable iff every root has |z| < 1.
    """
    a = np.asarray(a, dtype=np.float64)
    if len(a) == 0:
        return np.zeros(0)
    return np.roots(np.concatenate([[1.0], a]))


def fir_filter(x: np.ndarray, taps: np.ndarray) -> np.ndarray:
    """Direct FIR convolution of Eq.8 along the last axis, zero padded.

    PAPER.md:103-107 (§3, Eq.8): p~(n) = sum_{k=-L0}^{L0} p(n-k) h(k); output
    length = input length.  ``taps`` are h(-L0..L0).
    """
    x = np.asarray(x, dtype=np.float64)
    L0 = (len(taps) - 1) // 2
    L = x.shape[-1]
    y = np.zeros_like(x)
    for k in range(-L0, L0 + 1):
        hk = taps[k + L0]
        if hk == 0.0:
            continue
        # y[n] += h(k) x[n-k]
        if k >= 0:
            if k < L:
                y[..., k:] += hk * x[..., : L - k]
        else:
            if -k < L:
                y[..., : L + k] += hk * x[..., -k:]
    return y


# --------------------------------------------------------------------------
# §4.4  Dyadic patterns (Brady; Ershov et al.)
# --------------------------------------------------------------------------

def dyadic_offsets(N: int) -> np.ndarray:
    """Dyadic line pattern table d[t][y] (shift t, row y), by the recursion.

    PAPER.md:242 (§4.4): partial sums over segments of length 2^i computed
    recursively over "dyadic patterns".  Reading R3 (standard recursion):
        D_1(0) = [0];
        D_2h(t) = D_h(floor(t/2))  ++  (D_h(floor(t/2)) + ceil(t/2)).
    """
    if N < 1 or (N & (N - 1)) != 0:
        raise ValueError("N must be a power of two")
    D = {0: [0]}          # height 1
    h = 1
    while h < N:
        newD = {}
        for t in range(2 * h):
            lo = D[t // 2]
            newD[t] = lo + [v + (t + 1) // 2 for v in lo]
        D = newD
        h *= 2
    return np.array([D[t] for t in range(N)], dtype=np.int64)


def dyadic_offsets_closed_form(N: int) -> np.ndarray:
    """Closed form d_t(y) = sum_k bit_{n-1-k}(y) * ceil(floor(t/2^k)/2) (R3)."""
    n = N.bit_length() - 1
    d = np.zeros((N, N), dtype=np.int64)
    for t in range(N):
        for y in range(N):
            v = 0
            for k in range(n):
                if (y >> (n - 1 - k)) & 1:
                    v += ((t >> k) + 1) // 2
            d[t, y] = v
    return d


# --------------------------------------------------------------------------
# §4.3  Forward / back projection in (s,t), the four line families
# --------------------------------------------------------------------------

def family_views(img: np.ndarray) -> list:
    """The four family views of Eq.16 (transpose) plus the shift-sign mirror.

    PAPER.md:166-170 (§4.1) four line classes; PAPER.md:194-198 (Eq.16)
    R_h = R_v applied to the transposed image.  Reading R4:
      G_0 = img[y][x] (L_v+), G_1 = img[y][N-1-x] (L_v-),
      G_2 = img[x][y] (L_h+), G_3 = img[N-1-x][y] (L_h-).
    """
    img = np.asarray(img)
    return [img, img[:, ::-1], img.T, img[::-1, :].T]


def forward_project(img: np.ndarray) -> np.ndarray:
    """Forward dyadic projection (Eq.17 discretised), direct sums.  S[f][t][s].

    PAPER.md:199-202 (Eq.17): P_v(s,t) = int f(s + t y / N, y) dy; discretised
    along dyadic patterns (§4.4):
        S[f][t][s] = sum_{y=0}^{N-1} G_f[y][s - N + d_t(y)],
    terms whose column falls outside [0, N) dropped (R1, R2).
    """
    img = np.asarray(img, dtype=np.float64)
    N = img.shape[0]
    d = dyadic_offsets(N)
    S = np.zeros((4, N, 2 * N), dtype=img.dtype)
    for f, G in enumerate(family_views(img)):
        for t in range(N):
            for s in range(2 * N):
                acc = 0.0
                for y in range(N):
                    x = s - N + d[t, y]
                    if 0 <= x < N:
                        acc += G[y, x]
                S[f, t, s] = acc
    return S


def forward_sample(img: np.ndarray, f: int, t: int, s: int) -> float:
    """One linogram sample of the forward projection, direct definition (Eq.17).

    PAPER.md:199-202 (Eq.17) discretised along dyadic patterns (R1-R3), family
    view G_f of Eq.16 (R4): S[f][t][s] = sum_{y<N} G_f[y][s - N + d_t(y)], terms
    outside [0, N) dropped, summed in order y = 0..N-1; d_t(y) by the closed form
    of R3 for all y at once.  Same definition as ``forward_project`` (pinned against
    it in tests/test_oracle_pins.py), one sample at a time for full-size checks.
    """
    G = family_views(np.asarray(img, dtype=np.float64))[f]
    N = G.shape[0]
    n = N.bit_length() - 1
    y = np.arange(N, dtype=np.int64)
    d = np.zeros(N, dtype=np.int64)
    for k in range(n):
        d += ((y >> (n - 1 - k)) & 1) * (((t >> k) + 1) // 2)
    x = s - N + d
    ok = (x >= 0) & (x < N)
    acc = 0.0
    for yy in y[ok]:
        acc += float(G[yy, x[yy]])
    return acc


def dyadic_offsets_column(N: int, y: int) -> np.ndarray:
    """d_t(y) for all t at one row y, by the closed form of R3 (vectorised over t)."""
    n = N.bit_length() - 1
    t = np.arange(N, dtype=np.int64)
    v = np.zeros(N, dtype=np.int64)
    for k in range(n):
        if (y >> (n - 1 - k)) & 1:
            v += ((t >> k) + 1) // 2
    return v


def backproject_pixel(F: np.ndarray, f: int, y: int, x: int, d=None) -> float:
    """One pixel of the family-f back projection, direct definition (O5).

    PAPER.md:204-212 (Eq.18-19) read as the exact adjoint of ``forward_project``
    (R4, R5): B_f[y][x] = sum_{t=0}^{N-1} F[f][t][x + N - d_t(y)], summed in
    order t = 0..N-1.  ``d`` is an optional full table d[t][y].
    """
    N = F.shape[1]
    col = dyadic_offsets_column(N, y) if d is None else np.asarray(d)[:, y]
    acc = 0.0
    for t in range(N):
        acc += float(F[f, t, x + N - col[t]])
    return acc


def backproject_direct(F: np.ndarray) -> np.ndarray:
    """Direct Theta(N^3) back projection of all four families (O5).  B[f][y][x].

    PAPER.md:73-80 (§2, Eq.5 discretised: Theta(N^3))
    (Eq.18-20) as the adjoint of Eq.17 (R4).
    """
    F = np.asarray(F, dtype=np.float64)
    N = F.shape[1]
    d = dyadic_offsets(N)
    B = np.zeros((4, N, N))
    xs = np.arange(N)
    for f in range(4):
        for y in range(N):
            acc = np.zeros(N)
            for t in range(N):
                acc += F[f, t, xs + N - d[t, y]]
            B[f, y] = acc
    return B


def fht_backproject(F: np.ndarray) -> np.ndarray:
    """Back projection by the Fast Hough Transform, all four families.  B[f][y][x].

    PAPER.md:240-245 (§4.4): Brady's recursion, partial sums over segments of
    length 2^i, i = 1..log2 N (R3), additions only.  PAPER.md:251-260 (§4.5,
    Eq.19-21): back projection = forward projection with the sign of one
    parameter changed, i.e. the FHT run in the negative shift direction over
    the linogram viewed as rows t x columns s.  Level recursion (h -> 2h):
        R_2h[b][y'][u] = R_h[2b][floor(y'/2)][u] + R_h[2b+1][floor(y'/2)][u - ceil(y'/2)]
    with R_1[t][0][u] = F[t][u] and zero outside [0, 2N).  After log2 N levels
    R_N[0][y][u] = sum_t F[t][u - d_y(t)] = B[y][u - N] (d_y(t) = d_t(y), R5).
    """
    F = np.asarray(F, dtype=np.float64)
    N = F.shape[1]
    W = 2 * N
    B = np.zeros((4, N, N))
    for f in range(4):
        R = F[f].reshape(N, 1, W).copy()       # [blocks][shifts][u]
        h = 1
        while h < N:
            nb = R.shape[0] // 2
            newR = np.zeros((nb, 2 * h, W))
            for bb in range(nb):
                A = R[2 * bb]
                Bk = R[2 * bb + 1]
                for yp in range(2 * h):
                    lo = yp // 2
                    sh = (yp + 1) // 2
                    shifted = np.zeros(W)
                    shifted[sh:] = Bk[lo, : W - sh]
                    newR[bb, yp] = A[lo] + shifted
            R = newR
            h *= 2
        B[f] = R[0][:, N:]
    return B


def fht_forward(img: np.ndarray) -> np.ndarray:
    """Forward FHT (Eq.17 via §4.4 recursion, positive direction).  S[f][t][s].

    Same level recursion as ``fht_backproject`` with u + ceil(y'/2), applied to
    each family view G_f placed at columns [N, 2N) ... read along s = x0 + N
    (R2): S[f][t][s] = sum_y G_f[y][s - N + d_t(y)].
    """
    img = np.asarray(img, dtype=np.float64)
    N = img.shape[0]
    W = 2 * N
    S = np.zeros((4, N, W))
    for f, G in enumerate(family_views(img)):
        # row y of the "image" is placed so that column s reads G[y][s - N]
        R = np.zeros((N, 1, W))
        R[:, 0, N:] = G
        h = 1
        while h < N:
            nb = R.shape[0] // 2
            newR = np.zeros((nb, 2 * h, W))
            for bb in range(nb):
                A = R[2 * bb]
                Bk = R[2 * bb + 1]
                for tp in range(2 * h):
                    lo = tp // 2
                    sh = (tp + 1) // 2
                    shifted = np.zeros(W)
                    shifted[: W - sh] = Bk[lo, sh:]
                    newR[bb, tp] = A[lo] + shifted
            R = newR
            h *= 2
        S[f] = R[0]
    return S


# --------------------------------------------------------------------------
# §4.2  (r, theta) -> (s, t) transition (NEXT-2)
# --------------------------------------------------------------------------

def linogram_line_rtheta(f: int, t: int, s: int, N: int):
    """(r, theta, |D|) of linogram sample (f, t, s): Eq.14 for the line model of R2.

    PAPER.md:172-178 (Eq.14) relates (s, t) to (r, theta); here the exact line of
    reading R2 is used: view line X'(tau) = A + k tau, Y' = tau, A = s - N + 0.5 -
    0.5 k, k = t/(N-1), mapped to image coordinates per family (R4):
      f=0: P0 = (A, 0), D = (k, 1)        f=1: P0 = (N - A, 0), D = (-k, 1)
      f=2: P0 = (0, A), D = (1, k)        f=3: P0 = (0, N - A), D = (1, -k).
    Unit normal n = (D_y, -D_x)/|D|, flipped so that theta = atan2(n_y, n_x) lies
    in [0, pi) (R23); r = (P0 - c).n, c = (N/2, N/2).
    """
    k = t / (N - 1)
    A = s - N + 0.5 - 0.5 * k
    P0, D = {0: ((A, 0.0), (k, 1.0)), 1: ((N - A, 0.0), (-k, 1.0)),
             2: ((0.0, A), (1.0, k)), 3: ((0.0, N - A), (1.0, -k))}[f]
    L = math.hypot(D[0], D[1])
    nx, ny = D[1] / L, -D[0] / L
    th = math.atan2(ny, nx)
    if th < 0.0 or th >= math.pi:
        nx, ny = -nx, -ny
        th = math.atan2(ny, nx)
    r = (P0[0] - N / 2.0) * nx + (P0[1] - N / 2.0) * ny
    return r, th, L


def sinogram_sample(p: np.ndarray, theta: float, r: float, dr: float) -> float:
    """Linear interpolation of a scanner sinogram p[k][j] at (theta, r) (R23).

    PAPER.md:178 ("transition ... using linear interpolation"): linear in the
    angle index u = theta/(pi/P) between rows k0 = floor(u) and k0 + 1, linear in
    the bin index w = r/dr + (R-1)/2 within a row, bins outside [0, R) read 0; the
    row after k = P-1 is row 0 at -r (p(r, theta + pi) = p(-r, theta)).
    """
    P, R = p.shape

    def row(k, rr):
        w = rr / dr + 0.5 * (R - 1)
        j0 = math.floor(w)
        b = w - j0
        v = 0.0
        if 0 <= j0 < R:
            v += (1.0 - b) * p[k, j0]
        if 0 <= j0 + 1 < R:
            v += b * p[k, j0 + 1]
        return v

    u = theta / (math.pi / P)
    k0 = min(int(math.floor(u)), P - 1)
    a = u - k0
    v0 = row(k0, r)
    v1 = row(k0 + 1, r) if k0 + 1 < P else row(0, -r)
    return (1.0 - a) * v0 + a * v1


def resample_sinogram(p: np.ndarray, N: int, dr: float = 1.0) -> np.ndarray:
    """Sinogram -> linogram (NEXT-2), S[f][t][s].  PAPER.md:172-188 (Eq.14-15).

    Each linogram sample is the sinogram linearly interpolated at the (r, theta) of
    its line (Eq.14 for the R2 line model) divided by the stretch factor of Eq.15,
    k_t = |D| = sqrt(1 + (t/(N-1))^2) for that line model (R23): the linogram
    integrates along the row coordinate (dY', Eq.17), the scanner along arc length.
    """
    p = np.asarray(p, dtype=np.float64)
    S = np.zeros((4, N, 2 * N))
    for f in range(4):
        for t in range(N):
            for s in range(2 * N):
                r, th, L = linogram_line_rtheta(f, t, s, N)
                S[f, t, s] = sinogram_sample(p, th, r, dr) / L
    return S


# --------------------------------------------------------------------------
# §2  Conventional (r, theta) FBP — the NEXT-4 comparison baseline
# --------------------------------------------------------------------------

def ramp_filter_rtheta(p: np.ndarray, dr: float = 1.0, L0: int | None = None) -> np.ndarray:
    """Ramp-filter every projection row of a scanner sinogram p[k][j] (Eq.3, Eq.8).

    PAPER.md:63-66 (Eq.3) with the band-limited kernel of Eq.7
    sampled at bin spacing dr (R24): q(r_j) = dr * sum_m h_dr(m) p(r_{j-m}),
    h_dr(m) = h(m) / dr^2.  L0 defaults to R (the kernel covers the whole row).
    """
    p = np.asarray(p, dtype=np.float64)
    R = p.shape[-1]
    taps = ramp_kernel(R if L0 is None else L0) / (dr * dr)
    return dr * fir_filter(p, taps)


def backproject_rtheta(q: np.ndarray, N: int, dr: float = 1.0) -> np.ndarray:
    """Direct back projection in (r, theta), Theta(N^2 P) (Eq.5, R24).

    PAPER.md:72-77 (Eq.5): f(x, y) = integral over theta of q_theta(x cos theta +
    y sin theta); discretised on the P angles theta_k = k pi / P in [0, pi) with
    weight pi / P: p(r, theta + pi) = p(-r, theta) folds Eq.5's [0, 2 pi) onto
    [0, pi), and the inversion with the |omega| kernel of Eq.4 integrates one
    half-turn (Eq.5's missing 1/2, reading R24); q linear in r (bins outside the detector read 0).
    Pixel (y, x) sits at (x + 0.5, y + 0.5), r measured from the centre (N/2, N/2)
    (the geometry of R23).  Returns img[y][x].
    """
    q = np.asarray(q, dtype=np.float64)
    P, R = q.shape
    c = np.arange(N) + 0.5 - N / 2.0
    X, Y = np.meshgrid(c, c)            # X[y][x] = x + 0.5 - N/2, Y[y][x] = y + 0.5 - N/2
    img = np.zeros((N, N))
    for k in range(P):
        th = k * math.pi / P
        w = (X * math.cos(th) + Y * math.sin(th)) / dr + 0.5 * (R - 1)
        j0 = np.floor(w).astype(np.int64)
        a = w - j0
        row = np.concatenate([[0.0], q[k], [0.0]])       # index j + 1; 0 outside [0, R)
        i0 = np.clip(j0 + 1, 0, R + 1)
        i1 = np.clip(j0 + 2, 0, R + 1)
        img += (1.0 - a) * row[i0] + a * row[i1]
    return img * (math.pi / P)


def fbp_rtheta(p: np.ndarray, N: int, dr: float = 1.0) -> np.ndarray:
    """Conventional FBP on a scanner sinogram: Eq.3 filtering, then Eq.5 direct
    back projection ("the sequential application of two
    operations"); the Theta(N^3) "Radon" back projection of Fig. 2b
    (PAPER.md:238, 273), the NEXT-4 comparison baseline."""
    return backproject_rtheta(ramp_filter_rtheta(p, dr), N, dr)


def combine(B: np.ndarray, w: float) -> np.ndarray:
    """Sum of the four family images (Eq.22), weight w (R7).

    Un-mirror / un-transpose each family (Eq.16, Eq.20-21 read as R4):
        out[y][x] = w * ((B_0[y][x] + B_1[y][N-1-x]) + (B_2[x][y] + B_3[x][N-1-y])).
    """
    B = np.asarray(B, dtype=np.float64)
    v = B[0] + B[1][:, ::-1]
    h = B[2].T + B[3][:, ::-1].T
    return w * (v + h)


def reconstruct(S: np.ndarray, b, a) -> np.ndarray:
    """Full hot path on one slice: IIR ramp filter (Eq.12-13) then FHT back
    projection (Eq.19-22) with w = 1/N (R7).  S: [4][N][2N] -> img [N][N]."""
    S = np.asarray(S, dtype=np.float64)
    N = S.shape[1]
    F = iir_symmetric(S, b, a)
    return combine(fht_backproject(F), 1.0 / N)
