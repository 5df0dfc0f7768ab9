"""Device 1D diffusion Hessian (cfg3's black-box operator) against the CPU
restatement (oracle/diffusion1d.hpp) and the reference's own operator tests
(test_oracles.cpp:126-238, 321-331)."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2003_10173_b200 import (Admissibility, Diffusion1D, PeelConfig, build_block_tree, build_cluster_tree,
                                   estimate_relative_error, make_oracle, peel_construct)

# the solve is a different (chunked) evaluation order of the reference's LU
# recurrences; A+ = M/dt + K/2 is ill-conditioned (kappa ~ 4 dt / (h^2 rho)), so
# parity is a relative tolerance, not bits
TOL = 1e-10


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def both(**kw):
    ref_keys = dict(n="n", steps="steps", final_time="T", t_p="tp", t_0="t0", source_amplitude="amp", alpha="alpha",
                    beta="beta", pad="pad", source_positions="sources", num_receivers="receivers")
    ora = O.Diff1D(**{ref_keys[k]: v for k, v in kw.items()})
    return Diffusion1D(**kw), ora


@pytest.mark.gpu
@pytest.mark.parametrize("kw", [dict(n=64, steps=96), dict(n=512, steps=64),
                                dict(n=1000, steps=40, pad=0.3, final_time=12.0, source_positions=[-0.3, 0.4],
                                     num_receivers=5),
                                dict(n=4099, steps=24, t_p=0.5)])
@pytest.mark.parametrize("b", [1, 5, 70])
def test_hessvec_matches_oracle(cuda, kw, b):
    d, ora = both(**kw)
    x = O.gaussian(7 + b, kw["n"], b)
    for tv in (True, False):
        y = d.hessvec_at_target(x, include_tv=tv)
        yo = ora.hessvec(x, include_tv=tv, threads=4)
        assert rel(y, yo) <= TOL, (tv, rel(y, yo))
    # column-wise too: every column is its own Hessian application
    yo = ora.hessvec(x, threads=4)
    y = d.hessvec_at_target(x)
    for j in range(b):
        assert rel(y[:, j], yo[:, j]) <= TOL


@pytest.mark.gpu
def test_state_field_matches_oracle(cuda):
    d, ora = both(n=300, steps=80)
    inf = ora.info()
    k = inf["npad"] - 1 + np.arange(300)
    for s in range(3):
        u = d.state_field(s)
        uo = ora.state(s)[k, :]
        assert rel(u, uo) <= 1e-11
        assert np.all(u[:, 0] == 0.0)


@pytest.mark.gpu
def test_silenced_source_leaves_only_tv(cuda):   # test_oracles.cpp:126-136
    d, ora = both(n=64, steps=64, t_0=1e9)
    assert np.all(d.state_field(0) == 0.0)
    x = O.gaussian(3, 64, 4)
    assert np.all(d.hessvec_at_target(x, include_tv=False) == 0.0)
    assert rel(d.hessvec_at_target(x), ora.hessvec(x)) <= 1e-14


@pytest.mark.gpu
def test_hessian_symmetric_psd_zero_maps_to_zero(cuda):   # test_oracles.cpp:205-225
    d = Diffusion1D(n=64, steps=96)
    op = d.hessian_operator(True)
    assert np.linalg.norm(op.apply(np.zeros((64, 1)))) == 0.0
    x, y = O.gaussian(85, 64, 1), O.gaussian(86, 64, 1)
    a = (x.T @ op.apply(y)).item()
    b = (y.T @ op.apply(x)).item()
    assert abs(a - b) <= 1e-10 * abs(b)
    assert (x.T @ op.apply(x)).item() >= 0.0
    hd = d.hessian_operator(False).apply(np.eye(64))   # dense_assemble of the misfit Hessian
    assert rel(hd, hd.T) < 1e-10
    ev = np.linalg.eigvalsh((hd + hd.T) / 2)
    assert ev.min() >= -1e-8 * ev.max()


@pytest.mark.gpu
def test_two_marches_per_source(cuda):   # test_oracles.cpp:227-238
    d = Diffusion1D(n=48, steps=48)
    assert d.pde_solves() == 3   # the cached state marches
    op = d.hessian_operator()
    op.apply(np.zeros((48, 2)))
    before = d.pde_solves()
    op.apply(O.gaussian(86, 48, 1))
    assert d.pde_solves() - before == 2 * 3
    assert op.columns_applied() == 3


@pytest.mark.gpu
def test_registry_names_and_overrides(cuda):   # test_oracles.cpp:321-331
    o = make_oracle("diff1d-64", {"steps": "32", "leaf": "16"})
    assert o.op.dim() == 64
    assert o.leaf == 16
    assert o.mode == Admissibility.weak
    assert o.diffusion.steps == 32
    with pytest.raises(ValueError):
        make_oracle("nonsense")


@pytest.mark.gpu
def test_rejects_bad_config(cuda):
    with pytest.raises(ValueError):
        Diffusion1D(n=4)
    with pytest.raises(ValueError):
        Diffusion1D(n=64, beta=0.0)
    d = Diffusion1D(n=64, steps=8)
    with pytest.raises(ValueError):
        d.hessvec_at_target(np.zeros((63, 1)))


@pytest.mark.gpu
def test_hara_compresses_the_device_hessian(cuda):
    """cfg3 at desk scale: peel_construct on the device operator reaches eps
    against the dense assembly (SPEC.md:707's 3 eps acceptance)."""
    o = make_oracle("diff1d-512", {"steps": "64"})
    bt = o.default_block_tree()
    eps = 1e-6
    res = peel_construct(o.op, bt, PeelConfig(eps=eps))
    hd = o.op.apply(np.eye(512))
    hd = (hd + hd.T) / 2
    assert np.linalg.norm(res.matrix.matvec(np.eye(512)) - hd, 2) <= 3 * eps * np.linalg.norm(hd, 2)
    assert estimate_relative_error(o.op, res.matrix) <= 3 * eps
    # the same construction on the CPU restatement's operator, densely: ranks agree within 2
    ora = O.Diff1D(n=512, steps=64)
    hdo = ora.hessvec(np.eye(512), threads=8)
    assert rel(o.op.apply(np.eye(512)), hdo) <= TOL
    tree = O.Tree(o.points, 32, 1.0, True)
    _, st = O.peel_dense(tree, (hdo + hdo.T) / 2, True, eps=eps)
    got = [lv.max_rank for lv in res.stats.levels]
    assert len(got) == len(st["level_max_rank"])
    assert all(abs(a - b) <= 2 for a, b in zip(got, st["level_max_rank"]))
