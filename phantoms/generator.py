"""Ellipse phantoms -> analytic (s,t) line integrals -> noise.  See package doc.

Geometry (readings R1/R2/R18):
  * image domain [0,N]^2, pixel (x,y) centred at (x+0.5, y+0.5);
  * family views f = 0..3: view coordinates (X',Y') map to image coordinates
        f=0: (X, Y) = (X', Y')          f=1: (X, Y) = (N - X', Y')
        f=2: (X, Y) = (Y', X')          f=3: (X, Y) = (Y', N - X')
  * line (s, t) of a family: x0 = s - N, passing through view points
        (x0 + 0.5, 0.5) and (x0 + t + 0.5, N - 0.5),
    i.e. X'(Y') = x0 + 0.5 + t (Y' - 0.5)/(N - 1);
  * value = integral over Y' in [0, N] of f(X'(Y'), Y') dY', restricted to the
    image square (one unit of Y' per image row, like a row-sampled line sum).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

# BASELINE.json configs (index 1..5), DESIGN.md §5 table.
CONFIGS = {
    1: dict(N=64, slices=1, ellipses=10, axes=(2.0, 20.0), noise=None),
    2: dict(N=512, slices=1, ellipses=30, axes=(4.0, 160.0), noise=("gauss", 0.01)),
    3: dict(N=2048, slices=1, ellipses=50, axes=(16.0, 640.0), noise=None),
    4: dict(N=1024, slices=256, ellipses=40, axes=(8.0, 320.0), noise=("poisson", 1e5)),
    5: dict(N=4096, slices=64, ellipses=80, axes=(32.0, 1280.0), noise=("poisson", 1e4)),
}


@dataclass
class EllipseSet:
    cx: np.ndarray
    cy: np.ndarray
    a: np.ndarray
    b: np.ndarray
    phi: np.ndarray
    rho: np.ndarray


def draw_ellipses(N: int, n_ellipses: int, axes, seed: int) -> EllipseSet:
    """Random ellipses: centres area-uniform in the disc of radius 0.8*N/2 about the
    image centre, semi-axes U[axes], rotation U[0, pi), density U[-0.5, 1]."""
    rng = np.random.default_rng(seed)
    R = 0.8 * N / 2.0
    r = R * np.sqrt(rng.uniform(0.0, 1.0, n_ellipses))
    th = rng.uniform(0.0, 2.0 * math.pi, n_ellipses)
    cx = N / 2.0 + r * np.cos(th)
    cy = N / 2.0 + r * np.sin(th)
    a = rng.uniform(axes[0], axes[1], n_ellipses)
    b = rng.uniform(axes[0], axes[1], n_ellipses)
    phi = rng.uniform(0.0, math.pi, n_ellipses)
    rho = rng.uniform(-0.5, 1.0, n_ellipses)
    return EllipseSet(cx, cy, a, b, phi, rho)


def _family_line(f: int, A, k, N):
    """Image-space line P(tau) = P0 + tau * D for view line X' = A + k tau, Y' = tau."""
    if f == 0:
        return (A, torch.zeros_like(A)), (k, torch.ones_like(k))
    if f == 1:
        return (N - A, torch.zeros_like(A)), (-k, torch.ones_like(k))
    if f == 2:
        return (torch.zeros_like(A), A), (torch.ones_like(k), k)
    return (torch.zeros_like(A), N - A), (torch.ones_like(k), -k)


def linogram_of_ellipses(E: EllipseSet, N: int, device="cpu",
                         dtype=torch.float64) -> torch.Tensor:
    """Analytic line integrals S[f][t][s] of the ellipse phantom, float64."""
    dev = torch.device(device)
    t = torch.arange(N, device=dev, dtype=dtype).view(N, 1)
    s = torch.arange(2 * N, device=dev, dtype=dtype).view(1, 2 * N)
    k = (t / (N - 1)).expand(N, 2 * N)
    x0 = (s - N).expand(N, 2 * N)
    A = x0 + 0.5 - 0.5 * k                      # X'(tau) = A + k tau
    # domain: tau in [0, N] and 0 <= A + k tau <= N
    lo = torch.zeros_like(A)
    hi = torch.full_like(A, float(N))
    kpos = k > 0
    safe_k = torch.where(kpos, k, torch.ones_like(k))
    lo = torch.where(kpos, torch.maximum(lo, -A / safe_k), lo)
    hi = torch.where(kpos, torch.minimum(hi, (N - A) / safe_k), hi)
    inside0 = (A >= 0) & (A <= N)
    hi = torch.where(~kpos & ~inside0, lo, hi)
    S = torch.zeros((4, N, 2 * N), device=dev, dtype=dtype)
    for f in range(4):
        (px, py), (dx, dy) = _family_line(f, A, k, N)
        acc = torch.zeros((N, 2 * N), device=dev, dtype=dtype)
        for i in range(len(E.cx)):
            c, sn = math.cos(E.phi[i]), math.sin(E.phi[i])
            ia2, ib2 = 1.0 / E.a[i] ** 2, 1.0 / E.b[i] ** 2
            ex, ey = px - E.cx[i], py - E.cy[i]
            u0 = ex * c + ey * sn
            v0 = -ex * sn + ey * c
            du = dx * c + dy * sn
            dv = -dx * sn + dy * c
            al = du * du * ia2 + dv * dv * ib2
            be = u0 * du * ia2 + v0 * dv * ib2
            ga = u0 * u0 * ia2 + v0 * v0 * ib2 - 1.0
            disc = be * be - al * ga
            sq = torch.sqrt(torch.clamp(disc, min=0.0))
            t1 = (-be - sq) / al
            t2 = (-be + sq) / al
            a1 = torch.maximum(t1, lo)
            a2 = torch.minimum(t2, hi)
            seg = torch.clamp(a2 - a1, min=0.0)
            seg = torch.where(disc > 0, seg, torch.zeros_like(seg))
            acc = acc + E.rho[i] * seg
        S[f] = acc
    return S


def add_noise(S: torch.Tensor, noise, seed: int) -> torch.Tensor:
    """Noise models of BASELINE configs 2/4/5 (reading R19).

    ("gauss", frac): S + N(0, (frac * max S)^2) on every entry.
    ("poisson", I0): counts ~ Poisson(I0 exp(-(2/N) S)), clamped >= 1,
                     S' = -ln(counts / I0) on every entry.
    """
    if noise is None:
        return S
    g = torch.Generator(device=S.device)
    g.manual_seed(int(seed))
    kind, par = noise
    if kind == "gauss":
        sigma = par * float(S.max())
        return S + sigma * torch.randn(S.shape, generator=g, device=S.device, dtype=S.dtype)
    if kind == "poisson":
        N = S.shape[-2]
        lam = par * torch.exp(-(2.0 / N) * S)
        counts = torch.poisson(lam, generator=g)
        counts = torch.clamp(counts, min=1.0)
        return -torch.log(counts / par)
    raise ValueError(kind)


def make_slice(config: int, slice_index: int = 0, device="cpu", N: int | None = None) -> torch.Tensor:
    """One seeded synthetic linogram [4][N][2N] as float32 (the shared input bytes)."""
    cfg = CONFIGS[config]
    N = N or cfg["N"]
    axes = cfg["axes"]
    if N != cfg["N"]:   # scale the semi-axis range with N (R18)
        axes = (axes[0] * N / cfg["N"], axes[1] * N / cfg["N"])
    seed = 1000 * config + slice_index
    E = draw_ellipses(N, cfg["ellipses"], axes, seed)
    S = linogram_of_ellipses(E, N, device=device)
    S = add_noise(S, cfg["noise"], seed)
    return S.to(torch.float32)


def make_batch(config: int, n_slices: int, first: int = 0, device="cpu",
               N: int | None = None) -> torch.Tensor:
    """[n_slices][4][N][2N] float32, slice i seeded with 1000*config + first + i."""
    return torch.stack([make_slice(config, first + i, device=device, N=N)
                        for i in range(n_slices)])


def random_linogram(N: int, batch: int, seed: int, device="cpu",
                    scale: float = 1.0) -> torch.Tensor:
    """Uniform random [batch][4][N][2N] float32 in [-scale, scale) (parity stress)."""
    g = torch.Generator(device="cpu")
    g.manual_seed(int(seed))
    x = (torch.rand((batch, 4, N, 2 * N), generator=g, dtype=torch.float64) * 2 - 1) * scale
    return x.to(torch.float32).to(device)


def integer_linogram(N: int, batch: int, seed: int, lo: int = -511, hi: int = 511,
                     device="cpu") -> torch.Tensor:
    """Integer-valued [batch][4][N][2N] float32 in [lo, hi] (bit-exact FHT tests, R21)."""
    g = torch.Generator(device="cpu")
    g.manual_seed(int(seed))
    x = torch.randint(lo, hi + 1, (batch, 4, N, 2 * N), generator=g, dtype=torch.int64)
    return x.to(torch.float32).to(device)


def integer_image(N: int, batch: int, seed: int, lo: int = -511, hi: int = 511,
                  device="cpu") -> torch.Tensor:
    """Integer-valued [batch][N][N] float32 image in [lo, hi] (bit-exact forward FHT tests)."""
    g = torch.Generator(device="cpu")
    g.manual_seed(int(seed))
    x = torch.randint(lo, hi + 1, (batch, N, N), generator=g, dtype=torch.int64)
    return x.to(torch.float32).to(device)


def random_image(N: int, batch: int, seed: int, device="cpu") -> torch.Tensor:
    """Uniform random [batch][N][N] float32 image in [0, 1) (forward FHT stress)."""
    g = torch.Generator(device="cpu")
    g.manual_seed(int(seed))
    x = torch.rand((batch, N, N), generator=g, dtype=torch.float64)
    return x.to(torch.float32).to(device)


def image_of_ellipses(E: EllipseSet, N: int) -> np.ndarray:
    """The ellipse phantom sampled at pixel centres (x + 0.5, y + 0.5), img[y][x],
    float64 (reference image of the NEXT-3/NEXT-4 quality studies)."""
    yy, xx = np.mgrid[0:N, 0:N] + 0.5
    img = np.zeros((N, N))
    for cx, cy, a, b, phi, rho in zip(E.cx, E.cy, E.a, E.b, E.phi, E.rho):
        u = (xx - cx) * np.cos(phi) + (yy - cy) * np.sin(phi)
        v = -(xx - cx) * np.sin(phi) + (yy - cy) * np.cos(phi)
        img += rho * ((u / a) ** 2 + (v / b) ** 2 <= 1.0)
    return img


def sinogram_of_ellipses(E: EllipseSet, N: int, n_angles: int, n_bins: int, dr: float = 1.0,
                         dtype=torch.float64) -> torch.Tensor:
    """Scanner sinogram p[k][j] of the ellipse phantom (arc-length line integrals,
    whole line, no square restriction), float64.  Geometry (reading R23):
    theta_k = k*pi/n_angles is the angle of the line normal n = (cos, sin) in image
    coordinates (x = column, y = row), r_j = (j - (n_bins-1)/2) * dr is the signed
    distance of the line from the image centre (N/2, N/2).  Per ellipse (textbook
    projection of an ellipse): p = 2 rho a b sqrt(max(0, m^2 - q^2)) / m^2 with
    m^2 = a^2 cos^2(theta - phi) + b^2 sin^2(theta - phi), q = r - (e - c).n."""
    th = torch.arange(n_angles, dtype=dtype) * (math.pi / n_angles)
    r = (torch.arange(n_bins, dtype=dtype) - 0.5 * (n_bins - 1)) * dr
    c, sn = torch.cos(th).view(-1, 1), torch.sin(th).view(-1, 1)
    out = torch.zeros((n_angles, n_bins), dtype=dtype)
    for i in range(len(E.cx)):
        m2 = (E.a[i] * torch.cos(th - E.phi[i])) ** 2 + (E.b[i] * torch.sin(th - E.phi[i])) ** 2
        m2 = m2.view(-1, 1)
        q = r.view(1, -1) - ((E.cx[i] - N / 2.0) * c + (E.cy[i] - N / 2.0) * sn)
        out = out + 2.0 * E.rho[i] * E.a[i] * E.b[i] * torch.sqrt(torch.clamp(m2 - q * q, min=0.0)) / m2
    return out
