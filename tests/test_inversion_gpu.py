"""Iterative inversion and low-rank updates on the B200, restated from the
reference's test_inversion.cpp and test_algebra.cpp (dense numpy expansions
and the oracle's to_dense are the checkers)."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2003_10173_b200 import (Admissibility, DenseOperator, H2Matrix, PeelConfig, ThresholdSchedule,
                                   build_block_tree, build_cluster_tree, desymmetrized, divergence_error,
                                   h_hyperpower, h_newton_schulz, h_unrolled, low_rank_update, make_operator,
                                   ns_sampler, peel_construct, pnorm_estimate, residual_norm, scaled_identity,
                                   scaled_identity_start, threshold_schedule, unrolled_sampler)


def n2(a):
    return np.linalg.norm(a, 2)


def tree1d(n, leaf):   # test_inversion.cpp:12-15
    pts = O.grid1d(n, 0, 1)
    ct = build_cluster_tree(pts, leaf)
    return build_block_tree(ct, ct, 1.0, Admissibility.weak), O.Tree(pts, leaf, 1.0, True)


def kernel_matrix(n):   # test_inversion.cpp:18-25
    i = np.arange(n)
    return np.exp(-np.abs(i[:, None] - i[None, :]) / (0.2 * n)) + 0.5 * np.eye(n)


def dense(m, ref):
    rr, cr = m.ranks()
    sym = m.symmetric
    return O.H2.from_packed(ref, sym, rr, None if sym else cr, m.download()).to_dense()


def compress_dense(a, bt, eps, seed=42):   # test_inversion.cpp:27-34
    return peel_construct(DenseOperator(a, True), bt, PeelConfig(eps=eps, seed=seed)).matrix


def test_threshold_schedule():   # test_inversion.cpp:38-46 (host logic, no GPU)
    assert threshold_schedule(0.5, 3, 1e-6, ThresholdSchedule()) == 1e-6
    dyn = ThresholdSchedule(dynamic=True)
    assert threshold_schedule(1.0, 0, 1e-6, dyn) == 1e-2
    assert threshold_schedule(1e-3, 5, 1e-6, dyn) == 1e-6
    assert abs(threshold_schedule(3e-2, 2, 1e-6, dyn) - 9e-5) < 1e-18


@pytest.mark.gpu
def test_unrolled_sampler_scalar_recurrence(cuda):   # test_inversion.cpp:180-190
    ct = build_cluster_tree(np.zeros((1, 1)), 2)
    bt = build_block_tree(ct, ct, 1.0, Admissibility.weak)
    ah = scaled_identity(bt, 1.0)
    x0 = scaled_identity(bt, 0.5)
    u3 = unrolled_sampler(x0, ah, 3)
    assert abs(u3.apply(np.ones((1, 1)))[0, 0] - (1.0 - 0.5 ** 8)) < 1e-14


@pytest.mark.gpu
def test_residual_norm(cuda):   # test_inversion.cpp:192-204
    a = kernel_matrix(48)
    oa = DenseOperator(a, True)
    assert residual_norm(oa, DenseOperator(np.linalg.inv(a), True)) < 1e-10
    zero = make_operator(48, True, lambda x: 0.0 * x)
    assert abs(residual_norm(oa, zero) - 1.0) < 1e-8
    delta = 0.37
    assert abs(residual_norm(oa, DenseOperator((1 - delta) * np.linalg.inv(a), True)) - delta) <= 5e-3 * delta


@pytest.mark.gpu
def test_pnorm_inf_and_1_known_spectra(cuda):   # test_operator.cpp:32-45
    d = np.diag(np.arange(1.0, 11.0))
    op = DenseOperator(d, True)
    assert abs(pnorm_estimate(op, float("inf"))[0] - 10.0) < 1e-12
    assert abs(pnorm_estimate(op, 1)[0] - 10.0) < 1e-12
    assert abs(pnorm_estimate(op, 2)[0] - 10.0) <= 5e-3 * 10.0


@pytest.mark.gpu
def test_hierarchical_newton_schulz_matches_dense_inverse(cuda):   # test_inversion.cpp:206-228
    bt, ref = tree1d(256, 32)
    a = kernel_matrix(256)
    ah = compress_dense(a, bt, 1e-10)
    x0 = scaled_identity_start(ah)
    res = h_newton_schulz(ah, x0, ThresholdSchedule(), 1e-8, PeelConfig())
    assert res.trace.converged
    assert residual_norm(ah, res.X) <= 1e-8
    xd = np.linalg.inv(a)
    assert n2(dense(res.X, ref) - xd) <= 1e-6 * n2(xd)
    rows = res.trace.rows
    for i in range(1, len(rows)):
        if rows[i - 1].residual < 1.0:
            assert rows[i].residual < rows[i - 1].residual
        if rows[i - 1].residual < 0.1:
            assert rows[i].residual <= 2.0 * rows[i - 1].residual ** 2 + 1e-12


@pytest.mark.gpu
def test_one_peeled_ns_step_matches_dense_step(cuda):   # test_inversion.cpp:230-245
    bt, ref = tree1d(128, 16)
    a = kernel_matrix(128)
    ah = compress_dense(a, bt, 1e-12)
    x0 = scaled_identity_start(ah)
    x1 = peel_construct(ns_sampler(x0, ah), bt, PeelConfig(eps=1e-12)).matrix
    x0d = dense(x0, ref)
    step = (2.0 * np.eye(128) - x0d @ a) @ x0d
    assert n2(dense(x1, ref) - step) <= 1e-9 * n2(step)


@pytest.mark.gpu
def test_hyperpower_and_unrolled_converge(cuda):   # the inversion.hpp:288-311 drivers
    bt, ref = tree1d(256, 32)
    a = kernel_matrix(256)
    ah = compress_dense(a, bt, 1e-10)
    x0 = scaled_identity_start(ah)
    hp = h_hyperpower(ah, x0, 8, ThresholdSchedule(), 1e-8, PeelConfig())
    assert hp.trace.converged and residual_norm(ah, hp.X) <= 1e-8
    ns = h_newton_schulz(ah, x0, ThresholdSchedule(), 1e-8, PeelConfig())
    assert hp.trace.iterations() <= ns.trace.iterations()
    un = h_unrolled(ah, x0, 3, 1e-6, PeelConfig())
    assert len(un.trace.rows) == 1
    # three unrolled NS steps contract the residual like the scalar recurrence e^8
    e0 = residual_norm(ah, x0)
    assert un.trace.final_residual <= max(e0 ** 8 * 1.5, 1e-6) + 1e-9


@pytest.mark.gpu
def test_divergence_on_hopeless_start(cuda):   # test_inversion.cpp:300-308
    bt, _ = tree1d(64, 8)
    ah = scaled_identity(bt, 1.0)
    x0 = scaled_identity(bt, 3.0)
    with pytest.raises(divergence_error) as e:
        h_newton_schulz(ah, x0, ThresholdSchedule(), 1e-8, PeelConfig(), 20)
    assert e.value.trace is not None and len(e.value.trace.rows) >= 3


@pytest.mark.gpu
def test_dynamic_schedule_spends_fewer_samples(cuda):   # test_inversion.cpp:311-330
    bt, _ = tree1d(256, 32)
    a = kernel_matrix(256)
    ah = compress_dense(a, bt, 1e-8)
    x0 = scaled_identity_start(ah)
    rs = h_newton_schulz(ah, x0, ThresholdSchedule(), 1e-6, PeelConfig())
    rd = h_newton_schulz(ah, x0, ThresholdSchedule(dynamic=True), 1e-6, PeelConfig())
    assert rd.trace.converged
    assert rd.trace.total_samples() < rs.trace.total_samples()
    half = max(len(rd.trace.rows) // 2, 1)
    assert any(rd.trace.rows[i].samples < rs.trace.rows[i].samples for i in range(min(half, len(rs.trace.rows))))


@pytest.mark.gpu
@pytest.mark.parametrize("sym_update", [True, False])
def test_low_rank_update(cuda, sym_update):   # test_algebra.cpp:103-125 (update exact at eps = 0, contract at eps)
    bt, ref = tree1d(192, 16)
    ora = O.H2.random(ref, True, 6, 13)
    rr, cr = ora.ranks()
    m = H2Matrix.from_packed(bt, True, rr, cr, ora.export())
    a = ora.to_dense()
    X = O.gaussian(3, 192, 4)
    Y = X if sym_update else O.gaussian(4, 192, 4)
    up = low_rank_update(m, X, Y, 0.0)
    assert up.symmetric == sym_update
    target = a + X @ Y.T
    assert n2(dense(up, ref) - target) <= 1e-11 * n2(target)
    up2 = low_rank_update(m, X, Y, 1e-5)
    assert n2(dense(up2, ref) - target) <= 3e-5 * n2(target)


@pytest.mark.gpu
def test_desymmetrized_is_the_same_operator(cuda):   # test_core.cpp:123-132
    bt, ref = tree1d(160, 16)
    ora = O.H2.random(ref, True, 5, 21)
    rr, cr = ora.ranks()
    m = H2Matrix.from_packed(bt, True, rr, cr, ora.export())
    d = desymmetrized(m)
    assert not d.symmetric
    x = O.gaussian(5, 160, 3)
    assert np.allclose(d.matvec(x), m.matvec(x), rtol=0, atol=1e-13 * np.abs(m.matvec(x)).max())
    assert np.allclose(dense(d, ref), ora.to_dense(), rtol=0, atol=1e-14 * np.abs(ora.to_dense()).max())
