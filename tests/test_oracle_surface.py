"""Pins the CPU restatement of the minimal-surface oracle (oracle/surface.py)
with the reference's own cases (P/tests/test_oracles.cpp:65-125, 321-324)."""
import math

import numpy as np

from oracle import pyoracle as O
from oracle.surface import MinimalSurface, make_surface


def fd_order(e1, e2, h1, h2):   # test_oracles.cpp:14-16
    return math.log(e1 / e2) / math.log(h1 / h2)


def test_flat_and_planar_closed_forms():   # test_oracles.cpp:65-81
    ms = MinimalSurface(16, 0.0)
    zero = np.zeros(ms.n)
    assert abs(ms.value(zero) - 1.0) <= 1e-13   # unit area
    assert np.linalg.norm(ms.gradient(zero)) == 0.0
    a = 0.75
    tilt = MinimalSurface(16, 0.0)
    tilt.set_boundary(lambda x, y: a * x)
    plane = np.zeros(tilt.n)
    for j in range(1, 17):
        for i in range(1, 17):
            plane[tilt.index(i, j)] = a * tilt.h * i
    assert abs(tilt.value(plane) - math.sqrt(1 + a * a)) <= 1e-12 * math.sqrt(1 + a * a)
    assert np.linalg.norm(tilt.gradient(plane)) < 1e-12


def test_flat_hessian_is_five_point_laplacian():   # test_oracles.cpp:83-93
    ms = MinimalSurface(8, 0.0)
    h = ms.hessian(np.zeros(ms.n)).toarray()
    for j in range(1, 9):
        for i in range(1, 9):
            r = ms.index(i, j)
            assert abs(h[r, r] - 4.0) < 1e-12
            if i > 1:
                assert abs(h[r, ms.index(i - 1, j)] + 1.0) < 1e-12
            if i < 8:
                assert abs(h[r, ms.index(i + 1, j)] + 1.0) < 1e-12


def test_gradient_and_hessian_central_differences():   # test_oracles.cpp:95-112
    ms = MinimalSurface(10)
    m = 0.1 * O.gaussian(81, ms.n, 1)[:, 0]
    nu = O.gaussian(82, ms.n, 1)[:, 0]
    nu /= np.linalg.norm(nu)
    g_dot = ms.gradient(m) @ nu
    h1, h2 = 1e-2, 1e-3
    e1 = abs((ms.value(m + h1 * nu) - ms.value(m - h1 * nu)) / (2 * h1) - g_dot)
    e2 = abs((ms.value(m + h2 * nu) - ms.value(m - h2 * nu)) / (2 * h2) - g_dot)
    assert fd_order(e1, e2, h1, h2) >= 1.9
    hv = ms.hessian(m) @ nu
    d1 = (ms.gradient(m + h1 * nu) - ms.gradient(m - h1 * nu)) / (2 * h1) - hv
    d2 = (ms.gradient(m + h2 * nu) - ms.gradient(m - h2 * nu)) / (2 * h2) - hv
    assert fd_order(np.linalg.norm(d1), np.linalg.norm(d2), h1, h2) >= 1.9


def test_hessian_spd_at_the_rim_state():   # test_oracles.cpp:114-125
    ms = MinimalSurface(12)
    m = ms.newton_state(1)
    h = ms.hessian(m).toarray()
    assert np.allclose(h, h.T, rtol=0, atol=1e-14)
    assert np.linalg.eigvalsh(h).min() > 0.0


def test_registry_surface16():   # test_oracles.cpp:321-324
    ms, state, hs = make_surface("surface16")
    assert hs.shape == (256, 256) and ms.n == 256
    assert np.count_nonzero(state) == 0   # newton_steps defaults to 0: the flat start
