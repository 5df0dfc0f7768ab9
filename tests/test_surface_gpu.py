"""Device minimal-surface Hessian ("surface<N>", cfg5's operator) against the CPU
restatement (oracle/surface.py, itself pinned by the reference's
test_oracles.cpp:65-125) and the reference's operator / registry cases."""
import numpy as np
import pytest

from oracle import pyoracle as O
from oracle.surface import MinimalSurface as OraSurface
from paper_2003_10173_b200 import (Admissibility, MinimalSurface, PeelConfig, build_block_tree, build_cluster_tree,
                                   make_oracle, peel_construct)

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("g,rim,steps", [(16, 0.5, 0), (12, 0.5, 1), (9, 0.0, 0), (20, 0.3, 2)])
def test_hessvec_matches_oracle(cuda, g, rim, steps):
    dev = MinimalSurface(g, rim, steps)
    ora = OraSurface(g, rim)
    state = ora.newton_state(steps)
    assert rel(dev.state(), state) < 1e-10 if steps else np.count_nonzero(dev.state()) == 0
    hs = ora.hessian(state)
    assert dev.nnz() == hs.nnz
    for b in (1, 3, 7):
        x = O.gaussian(300 + b, g * g, b)
        assert rel(dev.hessvec(x), hs @ x) < 1e-12, (g, steps, b)


def test_flat_hessian_is_five_point_laplacian(cuda):   # test_oracles.cpp:83-93
    dev = MinimalSurface(8, 0.0)
    h = dev.hessvec(np.eye(64))
    ora = OraSurface(8, 0.0)
    for j in range(1, 9):
        for i in range(1, 9):
            r = ora.index(i, j)
            assert abs(h[r, r] - 4.0) < 1e-12
            if i > 1:
                assert abs(h[r, ora.index(i - 1, j)] + 1.0) < 1e-12
            if i < 8:
                assert abs(h[r, ora.index(i + 1, j)] + 1.0) < 1e-12


def test_spd_at_rim_state_and_operator_adapter(cuda):   # test_oracles.cpp:114-125
    dev = MinimalSurface(12, 0.5, 1)
    h = dev.hessvec(np.eye(144))
    assert np.array_equal(h, h.T)
    assert np.linalg.eigvalsh(h).min() > 0.0
    x = O.gaussian(82, 144, 3)
    op = dev.hessian_operator()
    assert rel(op.apply(x), dev.hessvec(x)) == 0.0
    assert op.columns_applied() == 3


def test_registry_surface(cuda):   # test_oracles.cpp:321-324
    s = make_oracle("surface16")
    assert s.op.dim() == 256
    assert s.mode == Admissibility.strong
    assert s.leaf == 64
    assert s.points.shape == (256, 2)
    o = make_oracle("surface12", {"rim": "0.25", "newton_steps": "1", "leaf": "16"})
    assert o.leaf == 16 and o.surface.newton_steps == 1 and o.surface.rim == 0.25
    with pytest.raises(ValueError):
        MinimalSurface(3)


def test_peel_construct_surface_to_tolerance(cuda):
    # HARA of the surface Hessian on its own (strong) block tree: the sparse
    # operator is captured to the construction tolerance (3 eps)
    o = make_oracle("surface24", {"leaf": "32"})
    ct = build_cluster_tree(o.points, o.leaf)
    bt = build_block_tree(ct, ct, o.eta, o.mode)
    eps = 1e-6
    res = peel_construct(o.op, bt, PeelConfig(eps=eps))
    n = o.op.dim()
    a = o.surface.hessvec(np.eye(n))
    x = np.eye(n)
    hm = res.matrix.matvec(x)
    err = np.linalg.norm(hm - a, 2) / np.linalg.norm(a, 2)
    assert err <= 3 * eps, err
