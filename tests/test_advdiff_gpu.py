"""Device advection-diffusion misfit Hessian ("advdiff-<G>") against the CPU
restatement (oracle/advdiff.py: sparse LU solves, pinned by the reference's
test_oracles.cpp:259-310), plus the reference's operator and registry cases."""
import numpy as np
import pytest

from oracle import pyoracle as O
from oracle.advdiff import AdvDiff2D as OraAdvDiff
from paper_2003_10173_b200 import (AdvDiff2D, PeelConfig, build_block_tree, build_cluster_tree, make_oracle,
                                   peel_construct)

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("grid,kappa,obs", [(16, 1e-3, 40), (20, 1e-2, 60), (32, 1e-3, 100)])
def test_hessvec_matches_oracle(cuda, grid, kappa, obs):
    dev = AdvDiff2D(grid=grid, kappa=kappa, num_observations=obs)
    ora = OraAdvDiff(grid=grid, kappa=kappa, num_observations=obs)
    assert np.array_equal(dev.observation_nodes(), np.asarray(ora.obs))   # the same std::shuffle pick
    assert abs(dev.sigma() - ora.sigma) <= 1e-12 * ora.sigma
    for b in (1, 4, 9):
        x = O.gaussian(400 + b, grid * grid, b)
        assert rel(dev.misfit_hessvec(x), ora.misfit_hessvec(x)) < 1e-10, (grid, b)


def test_zero_symmetry_psd_and_counter(cuda):   # test_oracles.cpp:259-292
    ad = AdvDiff2D(grid=16, num_observations=40)
    assert np.linalg.norm(ad.misfit_hessvec(np.zeros(ad.n()))) == 0.0
    x, y = O.gaussian(87, ad.n(), 2).T
    a = x @ ad.misfit_hessvec(y)
    b = y @ ad.misfit_hessvec(x)
    assert abs(a - b) <= 1e-10 * abs(b)
    assert x @ ad.misfit_hessvec(x) >= 0.0
    hd = ad.misfit_hessvec(np.eye(ad.n()))
    assert rel(hd, hd.T) < 1e-10
    before = ad.solves()
    ad.misfit_hessvec(np.ones((ad.n(), 3)))
    assert ad.solves() - before == 2   # one forward and one adjoint solve per application
    with pytest.raises(ValueError):
        AdvDiff2D(grid=8, kappa=0.0)
    with pytest.raises(ValueError):
        AdvDiff2D(grid=8, num_observations=1000)
    none = AdvDiff2D(grid=8, num_observations=0)   # no observations: a zero misfit Hessian
    assert np.count_nonzero(none.misfit_hessvec(np.ones((64, 2)))) == 0


def test_numerical_rank_grows_with_observations(cuda):   # test_oracles.cpp:294-310
    def rank_at(obs):
        ad = AdvDiff2D(grid=16, kappa=1e-3, num_observations=obs)
        ev = np.linalg.eigvalsh(ad.misfit_hessvec(np.eye(ad.n())))
        return int(np.count_nonzero(ev > 1e-4 * ev.max()))
    r10, r60 = rank_at(10), rank_at(60)
    assert r10 <= 10 and r60 > r10


def test_registry_and_hara(cuda):   # test_oracles.cpp:333-336
    a = make_oracle("advdiff-16-k1e-2-obs50")
    assert a.op.dim() == 256
    assert a.advdiff.config["kappa"] == 1e-2
    assert a.advdiff.config["num_observations"] == 50
    assert a.leaf == 64
    o = make_oracle("advdiff-24", {"leaf": "16"})
    ct = build_cluster_tree(o.points, o.leaf)
    bt = build_block_tree(ct, ct, o.eta, o.mode)
    eps = 1e-6
    res = peel_construct(o.op, bt, PeelConfig(eps=eps))
    n = o.op.dim()
    h = o.advdiff.misfit_hessvec(np.eye(n))
    err = np.linalg.norm(res.matrix.matvec(np.eye(n)) - h, 2) / np.linalg.norm(h, 2)
    assert err <= 3 * eps, err
