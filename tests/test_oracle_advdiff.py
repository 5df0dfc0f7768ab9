"""Pins the CPU restatement of the advection-diffusion oracle (oracle/advdiff.py)
with the reference's own cases (P/tests/test_oracles.cpp:259-310)."""
import numpy as np

from oracle import pyoracle as O
from oracle.advdiff import AdvDiff2D


def test_zero_symmetry_psd_adjoint_consistency():   # test_oracles.cpp:259-292
    ad = AdvDiff2D(grid=16, num_observations=40)
    assert np.linalg.norm(ad.misfit_hessvec(np.zeros(ad.n))) == 0.0
    x, y = O.gaussian(87, ad.n, 2).T
    a = x @ ad.misfit_hessvec(y)
    b = y @ ad.misfit_hessvec(x)
    assert abs(a - b) <= 1e-10 * abs(b)
    assert x @ ad.misfit_hessvec(x) >= 0.0
    nu = O.gaussian(88, ad.n, 1)[:, 0]
    w = np.zeros(ad.n)
    w[ad.obs] = 1.0
    assert np.isfinite(ad.solve_state(nu) @ w)
    pair1 = w @ ad.misfit_hessvec(nu)
    pair2 = nu @ ad.misfit_hessvec(w)
    assert abs(pair1 - pair2) <= 1e-12 * abs(pair2)
    hd = ad.misfit_hessvec(np.eye(ad.n))
    assert np.linalg.norm(hd - hd.T) / np.linalg.norm(hd) < 1e-10


def test_numerical_rank_grows_with_observations():   # test_oracles.cpp:294-310
    def rank_at(obs):
        ad = AdvDiff2D(grid=16, kappa=1e-3, num_observations=obs)
        ev = np.linalg.eigvalsh(ad.misfit_hessvec(np.eye(ad.n)))
        return int(np.count_nonzero(ev > 1e-4 * ev.max()))
    r10, r60 = rank_at(10), rank_at(60)
    assert r10 <= 10
    assert r60 > r10


def test_solve_counter_and_errors():   # advdiff2d.hpp:48-64
    ad = AdvDiff2D(grid=8, num_observations=10)
    ad.misfit_hessvec(np.ones((ad.n, 2)))
    assert ad.solves == 2
    import pytest
    with pytest.raises(ValueError):
        AdvDiff2D(grid=8, kappa=0.0)
    with pytest.raises(ValueError):
        AdvDiff2D(grid=8, num_observations=1000)
