"""The CPU restatement of the diffusion Hessian (oracle/diffusion1d.hpp) pinned
by the reference's own operator tests (test_oracles.cpp:126-238); no GPU."""
import numpy as np
import pytest

from oracle import pyoracle as O


def test_oracle_geometry_matches_reference_formulas():   # diffusion1d.hpp:77-85
    d = O.Diff1D(n=262144, steps=1, T=30.0)
    inf = d.info()
    assert inf["npad"] == 65536 and inf["nstate"] == 393214   # SURVEY §8(d) cfg3 sizes
    assert inf["dt"] == 30.0
    assert inf["marches"] == 3


def test_oracle_silenced_source_zero_state():   # test_oracles.cpp:126-136
    d = O.Diff1D(n=64, steps=64, t0=1e9)
    assert np.all(d.state(0) == 0.0)
    x = O.gaussian(1, 64, 2)
    assert np.all(d.hessvec(x, include_tv=False) == 0.0)


def test_oracle_energy_decays_after_source():   # test_oracles.cpp:149-167
    d = O.Diff1D(n=96, steps=256, T=30.0)
    u = d.state(0)
    quiet = int((1.4 * 1.0 + 4 * 1.0) / d.info()["dt"]) + 1
    prev = float(np.sum(u[:, quiet] ** 2))
    assert prev > 0.0
    for j in range(quiet + 1, 257):
        e = float(np.sum(u[:, j] ** 2))
        assert e <= prev * (1 + 1e-12)
        prev = e


def test_oracle_hessian_symmetric_psd():   # test_oracles.cpp:205-225
    d = O.Diff1D(n=64, steps=96)
    assert np.linalg.norm(d.hessvec(np.zeros((64, 1)))) == 0.0
    x, y = O.gaussian(85, 64, 1), O.gaussian(86, 64, 1)
    a = (x.T @ d.hessvec(y)).item()
    b = (y.T @ d.hessvec(x)).item()
    assert a == pytest.approx(b, rel=1e-10)
    assert (x.T @ d.hessvec(x)).item() >= 0.0
    hd = d.hessvec(np.eye(64), include_tv=False, threads=4)
    assert np.linalg.norm(hd - hd.T) / np.linalg.norm(hd) < 1e-10
    ev = np.linalg.eigvalsh((hd + hd.T) / 2)
    assert ev.min() >= -1e-8 * ev.max()


def test_oracle_two_marches_per_source():   # test_oracles.cpp:227-238
    d = O.Diff1D(n=48, steps=48)
    d.hessvec(np.zeros((48, 2)))
    before = d.info()["marches"]
    d.hessvec(O.gaussian(86, 48, 1))
    assert d.info()["marches"] - before == 6


def test_oracle_threads_do_not_change_bits():
    d = O.Diff1D(n=200, steps=32)
    x = O.gaussian(5, 200, 7)
    assert np.array_equal(d.hessvec(x, threads=1), d.hessvec(x, threads=3))


def test_registry_rejects_unknown_names():   # registry.hpp:152-154 (host logic only)
    from paper_2003_10173_b200 import make_oracle
    with pytest.raises(ValueError):
        make_oracle("nonsense")
