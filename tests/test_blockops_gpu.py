"""Block-level construction primitives and H^2 diagnostics on the B200 through
the C ABI, against the CPU restatement (oracle.pyoracle) and the reference's
own compiled code (oracle.pyref, oracle/_ref/libh2ref.so):

* sample_block_column / adaptive_block_factorization (construction.hpp:137-198)
  incl. the reference's known-answer tests (test_construction.cpp:39-108): the
  Gaussian panel Omega is BITWISE the reference's mt19937_64 normal stream;
* local_low_rank_update, frobenius_norm (algebra.hpp:119-137, 323-332);
* H2Matrix::to_dense / validate / storage / rank_profile (h2_matrix.hpp:128-196, 308-404).
"""
import os

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2003_10173_b200 import (Admissibility, DenseOperator, H2Matrix, PeelConfig, Rng,
                                   adaptive_block_factorization, build_block_tree, build_cluster_tree,
                                   frobenius_norm, local_low_rank_update, max_rank_error, orthogonalize,
                                   sample_block_column)

pytestmark = pytest.mark.gpu

_REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "libh2ref.so")
REFS = [O]
if os.path.exists(_REF):
    from oracle import pyref as R
    REFS.append(R)


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def n2(a):
    return np.linalg.norm(a, 2)


def gather_block(ct, a_user, t, s):
    rt = ct.perm[ct.begin[t]:ct.end[t]]
    rs = ct.perm[ct.begin[s]:ct.end[s]]
    return a_user[np.ix_(rt, rs)]


def root_children(ct):
    return int(ct.child0[0]), int(ct.child1[0])


# ---- sample_block_column (construction.hpp:137-148) --------------------------

@pytest.mark.parametrize("count", [1, 4, 16])
def test_sample_block_column_omega_bitwise_and_y(cuda, count):
    pts = O.grid2d(16, 16)
    ct = build_cluster_tree(pts, 16)
    a = O.gaussian(7, 256, 256)
    t, s = 3, int(ct.child1[0])
    om, y = sample_block_column(DenseOperator(a), ct, t, s, count, Rng(1234))
    for M in REFS:
        om_r, y_r = M.sample_block_column(M.Tree(pts, 16), a, False, t, s, count, 1234)
        assert np.array_equal(om, om_r), M.__name__      # the reference's mt19937_64 normal stream, bitwise
        assert rel(y, y_r) <= 1e-13
    assert rel(y, gather_block(ct, a, t, s) @ om) <= 1e-13


def test_sample_block_column_shares_the_stream(cuda):
    # consecutive draws continue one mt19937_64 (the reference passes rng by reference)
    pts = O.grid1d(64)
    ct = build_cluster_tree(pts, 8)
    op = DenseOperator(np.eye(64))
    rng = Rng(9)
    o1, _ = sample_block_column(op, ct, 1, 2, 3, rng)
    o2, _ = sample_block_column(op, ct, 1, 2, 3, rng)
    assert not np.array_equal(o1, o2)
    o0, _ = sample_block_column(op, ct, 1, 2, 3, Rng(9))
    assert np.array_equal(o0, o1)


def test_sample_block_column_known_answers(cuda):
    # test_construction.cpp:39-59
    pts = O.grid1d(64)
    ct = build_cluster_tree(pts, 8)
    t, s = root_children(ct)
    d = O.gaussian(51, 64, 1)[:, 0]
    diag = DenseOperator(np.diag(d), True)
    _, y0 = sample_block_column(diag, ct, t, s, 4, Rng(50))
    assert np.linalg.norm(y0) == 0.0
    a = O.gaussian(52, 64, 64)
    omega, y = sample_block_column(DenseOperator(a), ct, t, s, 6, Rng(50))
    assert rel(y, gather_block(ct, a, t, s) @ omega) < 1e-12
    _, y_all = sample_block_column(DenseOperator(a), ct, 0, 0, 3, Rng(50))
    assert y_all.shape[0] == 64
    with pytest.raises(ValueError):
        sample_block_column(DenseOperator(a), ct, t, s, 0, Rng(50))


# ---- adaptive_block_factorization (construction.hpp:156-198) -------------------

def test_adaptive_zero_block_one_increment(cuda):
    # test_construction.cpp:61-73: zero block -> rank 0 after exactly b columns
    pts = O.grid1d(64)
    ct = build_cluster_tree(pts, 8)
    t, s = root_children(ct)
    d = O.gaussian(52, 64, 1)[:, 0]
    op = DenseOperator(np.diag(d), True)
    cfg = PeelConfig()
    op.reset_counter()
    f = adaptive_block_factorization(op, ct, t, s, 1e-8, cfg)
    assert f.rank == 0 and op.columns_applied() == cfg.sample_block_size


def test_adaptive_exact_rank3(cuda):
    # test_construction.cpp:75-97
    pts = O.grid1d(64)
    ct = build_cluster_tree(pts, 8)
    t, s = root_children(ct)
    xf = np.zeros((64, 3))
    yf = np.zeros((64, 3))
    xf[ct.perm[ct.begin[t]:ct.end[t]]] = O.gaussian(53, int(ct.size(t)), 3)
    yf[ct.perm[ct.begin[s]:ct.end[s]]] = O.gaussian(54, int(ct.size(s)), 3)
    a = xf @ yf.T
    op = DenseOperator(a)
    cfg = PeelConfig(eps=1e-12)
    op.reset_counter()
    f = adaptive_block_factorization(op, ct, t, s, 1e-12, cfg)
    assert f.rank == 3
    assert op.columns_applied() <= 3 + cfg.sample_block_size + 3
    blk = gather_block(ct, a, t, s)
    assert n2(blk - f.u @ f.v.T) < 1e-12 * n2(blk)
    assert np.abs(f.u.T @ f.u - np.eye(3)).max() < 1e-13
    # the same decisions as the reference's own driver and the restatement
    for M in REFS:
        u, v, k, e, cols = M.adaptive_block_factorization(M.Tree(pts, 8), a, False, t, s, 1e-12)
        assert k == 3 and cols == op.columns_applied(), M.__name__
        assert rel(f.u @ f.v.T, u @ v.T) < 1e-12


def test_adaptive_max_rank_exhaustion(cuda):
    # test_construction.cpp:99-108
    pts = O.grid1d(64)
    ct = build_cluster_tree(pts, 8)
    t, s = root_children(ct)
    op = DenseOperator(O.gaussian(54, 64, 64))
    with pytest.raises(max_rank_error):
        adaptive_block_factorization(op, ct, t, s, 1e-10, PeelConfig(eps=1e-10, max_rank=2))


@pytest.mark.parametrize("eps", [1e-3, 1e-6, 1e-9])
def test_adaptive_kernel_block_matches_reference(cuda, eps):
    # a smooth kernel block: rank, err_est and the column count agree with the
    # reference's driver (same mt19937_64 panels, same stopping rule)
    pts = O.grid1d(256, -1, 1)
    x = pts[:, 0]
    a = np.exp(-np.abs(x[:, None] - x[None, :]) / 0.3)
    ct = build_cluster_tree(pts, 16)
    t, s = root_children(ct)
    op = DenseOperator(a, True)
    op.reset_counter()
    f = adaptive_block_factorization(op, ct, t, s, eps, PeelConfig())
    blk = gather_block(ct, a, t, s)
    assert n2(blk - f.u @ f.v.T) <= 3 * eps * n2(blk)
    for M in REFS:
        u, v, k, e, cols = M.adaptive_block_factorization(M.Tree(pts, 16), a, True, t, s, eps)
        assert (k, cols) == (f.rank, op.columns_applied()), M.__name__
        assert abs(e - f.err_est) <= 1e-9 * max(e, 1e-300) + 1e-15


# ---- algebra: local_low_rank_update, frobenius_norm --------------------------------

def pair(pts, leaf, weak, sym, kmax, seed):
    ref = O.Tree(pts, leaf, 1.0, weak)
    ora = O.H2.random(ref, sym, kmax, seed)
    ct = build_cluster_tree(pts, leaf)
    bt = build_block_tree(ct, ct, 1.0, Admissibility.weak if weak else Admissibility.strong)
    rr, cr = ora.ranks()
    return ora, H2Matrix.from_packed(bt, sym, rr, cr, ora.export()), bt, ref


def dense_of(m, ref):
    rr, cr = m.ranks()
    sym = m.symmetric
    return O.H2.from_packed(ref, sym, rr, None if sym else cr, m.download()).to_dense()


@pytest.mark.parametrize("case", ["sym-offdiag", "sym-diag-same", "sym-diag-diff", "nonsym"])
def test_local_low_rank_update_matches_oracle(cuda, case):
    pts = O.grid1d(160, -1, 1)
    sym = case != "nonsym"
    ora, m, bt, ref = pair(pts, 10, True, sym, 6, 31)
    ct = bt.tree
    c0, c1 = int(ct.child0[0]), int(ct.child1[0])
    t, s = {"sym-offdiag": (c0, c1), "sym-diag-same": (c0, c0), "sym-diag-diff": (c1, c1), "nonsym": (c1, c0)}[case]
    k = 3
    U = O.gaussian(5, int(ct.size(t)), k)
    V = U.copy() if case == "sym-diag-same" else O.gaussian(6, int(ct.size(s)), k)
    g = local_low_rank_update(m, t, s, U, V, 1e-12)
    go = ora.local_low_rank_update(t, s, U, V, 1e-12)
    ad = dense_of(g, ref)
    ao = go.to_dense()
    assert rel(ad, ao) <= 1e-10
    # the update landed exactly on the (t, s) region
    a0 = ora.to_dense()
    upd = np.zeros_like(a0)
    upd[np.ix_(ct.perm[ct.begin[t]:ct.end[t]], ct.perm[ct.begin[s]:ct.end[s]])] = U @ V.T
    if sym and t != s:
        upd = upd + upd.T
    assert rel(ad, a0 + upd) <= 1e-10
    assert g.symmetric == (sym and case != "sym-diag-diff")


def test_local_low_rank_update_zero_rank_is_a_copy(cuda):
    pts = O.grid1d(96, -1, 1)
    ora, m, bt, ref = pair(pts, 8, True, True, 5, 3)
    g = local_low_rank_update(m, 1, 2, np.zeros((int(bt.tree.size(1)), 0)), np.zeros((int(bt.tree.size(2)), 0)), 1e-8)
    assert np.array_equal(dense_of(g, ref), dense_of(m, ref))


@pytest.mark.parametrize("sym", [True, False])
def test_frobenius_norm(cuda, sym):
    # algebra.hpp:119-137 after orthogonalize; equals ||A||_F of the expansion
    pts = O.grid2d(20, 20)
    ora, m, bt, ref = pair(pts, 16, False, sym, 8, 17)
    with pytest.raises(ValueError):
        frobenius_norm(m)   # not orthonormal
    g = orthogonalize(m)
    f = frobenius_norm(g)
    assert abs(f - np.linalg.norm(ora.to_dense())) <= 1e-12 * f
    fo = ora.orthogonalize().frobenius_norm()
    assert abs(f - fo) <= 1e-12 * fo


# ---- diagnostics: to_dense, validate, storage, rank_profile ---------------------------

@pytest.mark.parametrize("sym", [True, False])
@pytest.mark.parametrize("case", ["1d-weak", "2d-strong"])
def test_to_dense_matches_reference(cuda, sym, case):
    pts, leaf, weak = (O.grid1d(300, -1, 1), 12, True) if case == "1d-weak" else (O.grid2d(24, 24), 16, False)
    ora, m, bt, ref = pair(pts, leaf, weak, sym, 9, 23)
    a = m.to_dense()
    for M in REFS:
        tr = M.Tree(pts, leaf, 1.0, weak)
        hr = M.H2.random(tr, sym, 9, 23)   # the same fixture (bitwise, test_ref_parity)
        assert rel(a, hr.to_dense()) <= 1e-13, M.__name__
    with pytest.raises(ValueError):
        m.to_dense(cap=pts.shape[0] - 1)


@pytest.mark.parametrize("sym", [True, False])
def test_validate_and_storage_match_reference(cuda, sym):
    pts = O.grid2d(24, 24)
    ora, m, bt, ref = pair(pts, 16, False, sym, 9, 29)
    rep = m.validate()
    assert rep.ok(), rep.violations
    nv, prof, st = ora.validate()
    assert nv == 0
    assert rep.level_max_rank == prof
    assert [rep.storage.dense_reals, rep.storage.leaf_basis_reals, rep.storage.transfer_reals,
            rep.storage.coupling_reals] == st
    assert rep.level_max_rank == m.rank_profile().tolist()


def test_validate_flags_false_orthonormal_claim(cuda):
    # random bases claimed orthonormal -> "row basis not orthonormal at node v"
    # (at most 8 reported, h2_matrix.hpp:376-399); orthogonalize() clears it
    pts = O.grid2d(16, 16)
    ora, m, bt, ref = pair(pts, 16, False, True, 6, 41)
    rr, cr = ora.ranks()
    bogus = H2Matrix.from_packed(bt, True, rr, cr, ora.export(), orthonormal=True)
    rep = bogus.validate()
    assert not rep.ok() and 1 <= len(rep.violations) <= 8
    assert all("not orthonormal" in v for v in rep.violations)
    assert bogus.validate(ortho_cap=10).ok()   # above the cap the claim is not checked
    assert orthogonalize(m).validate().ok()


@pytest.mark.parametrize("m,n", [(3000, 64), (3584, 128), (5000, 96), (900, 160), (2001, 40), (700, 170)])
def test_batched_qr_r_factor(cuda, m, n):
    """The batched QR's R factor (TSQR over shared-memory row chunks, then the pairwise
    structured combine of the chunk triangles for R-only problems with n <= 167, or the dense
    re-factorisation of the stacked R's above that) satisfies R^T R = A^T A and is upper
    triangular with Householder's sign convention (R_jj of the sign opposite to the pivot)."""
    import ctypes as C
    from paper_2003_10173_b200._lib import lib
    rng = np.random.default_rng(m * 7 + n)
    a = np.asfortranarray(rng.standard_normal((m, n)) * np.logspace(0, -8, n))
    r = np.zeros((n, n), order="F")
    assert lib.h2b_test_qr_r(a.ctypes.data_as(C.c_void_p), m, n, r.ctypes.data_as(C.c_void_p)) == 0
    assert np.all(np.tril(r, -1) == 0)
    g = a.T @ a
    assert np.linalg.norm(r.T @ r - g) <= 1e-13 * np.linalg.norm(g)
    # same R as a dense Householder QR up to the row signs
    rq = np.linalg.qr(a, mode="r")
    assert np.allclose(np.abs(r), np.abs(rq), rtol=0, atol=1e-12 * np.abs(rq).max())
