"""Seeded input generator checks (-m "not gpu")."""
import math

import numpy as np
import pytest
import torch

import phantoms as P
from oracle import fbp_oracle as O


def test_deterministic_and_shape():
    a = P.make_slice(1, 0)
    b = P.make_slice(1, 0)
    assert a.dtype == torch.float32 and a.shape == (4, 64, 128)
    assert torch.equal(a, b)
    assert not torch.equal(a, P.make_slice(1, 1))
    n2 = P.make_slice(2, 0, N=64)
    assert n2.shape == (4, 64, 128) and torch.isfinite(n2).all()
    p4 = P.make_slice(4, 3, N=32)
    assert torch.isfinite(p4).all() and float(p4.abs().max()) < 10


def test_row_mass_equals_phantom_mass():
    """Lines of one (family, t) row are 1 px apart along x' per unit of y': the row
    sum of the analytic line integrals is a unit-spacing quadrature of the phantom's
    mass (Radon invariant, §4.2): equal up to the sampling error of chord lengths."""
    N = 64
    E = P.draw_ellipses(N, 6, (2.0, 8.0), 5)   # small: entirely inside the square
    mass = float(np.sum(E.rho * math.pi * E.a * E.b))
    S = P.linogram_of_ellipses(E, N)
    rs = S.sum(dim=2)
    assert torch.allclose(rs, torch.full_like(rs, mass), rtol=0.06)
    assert abs(float(rs.mean()) - mass) < 0.005 * mass


def test_analytic_linogram_close_to_dyadic_sums_of_raster():
    """Analytic straight-line integrals vs the oracle's dyadic sums of the rasterised
    phantom: same geometry (R1/R2/R4), differing only by discretisation."""
    N = 32
    E = P.draw_ellipses(N, 5, (4.0, 10.0), 9)
    yy, xx = np.mgrid[0:N, 0:N] + 0.5
    img = np.zeros((N, N))
    for i in range(len(E.cx)):
        c, s = math.cos(E.phi[i]), math.sin(E.phi[i])
        u = (xx - E.cx[i]) * c + (yy - E.cy[i]) * s
        v = -(xx - E.cx[i]) * s + (yy - E.cy[i]) * c
        img += E.rho[i] * ((u / E.a[i]) ** 2 + (v / E.b[i]) ** 2 <= 1)
    Sd = O.forward_project(img)
    Sa = P.linogram_of_ellipses(E, N).numpy()
    rel = np.abs(Sa - Sd).mean() / np.abs(Sd).mean()
    assert rel < 0.12, rel
    # wrong family orientation would give O(1) differences
    assert np.abs(Sa[2] - Sd[3]).mean() / np.abs(Sd).mean() > 0.2


def test_integer_and_random_generators():
    x = P.integer_linogram(8, 2, 1)
    assert x.shape == (2, 4, 8, 16)
    assert torch.equal(x, torch.round(x)) and x.abs().max() <= 511
    r = P.random_linogram(8, 1, 2)
    assert r.abs().max() <= 1.0
