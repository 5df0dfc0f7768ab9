"""HARA and the H^2 algebra on the B200 vs the CPU oracle and the reference's
own construction / algebra tests (restated from test_construction.cpp and
test_algebra.cpp). The product path runs entirely through the C ABI; the
oracle is only the checker (dense expansion, oracle peel for parity)."""
import os

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2003_10173_b200 import (Admissibility, DenseOperator, H2Matrix, H2Operator, PeelConfig,
                                   build_block_tree, build_cluster_tree, estimate_relative_error,
                                   make_operator, orthogonalize, peel_construct, pnorm_estimate, recompress)

pytestmark = pytest.mark.gpu

_REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "libh2ref.so")
if os.path.exists(_REF):
    from oracle import pyref as R
else:
    R = None


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def n2(a):
    return np.linalg.norm(a, 2)


def trees(pts, leaf, weak):
    ct = build_cluster_tree(pts, leaf)
    bt = build_block_tree(ct, ct, 1.0, Admissibility.weak if weak else Admissibility.strong)
    return bt, O.Tree(pts, leaf, 1.0, weak)


def dense(m, ref_tree):
    """Expand a device H^2 exactly (through the oracle's to_dense, h2_matrix.hpp:128-163)."""
    rr, cr = m.ranks()
    sym = m.symmetric
    ora = O.H2.from_packed(ref_tree, sym, rr, None if sym else cr, m.download())
    return ora.to_dense()


def tree1d(n, leaf, weak=True):
    return trees(O.grid1d(n, -1, 1), leaf, weak)


# ---- algebra (test_algebra.cpp) -------------------------------------------

@pytest.mark.parametrize("sym", [True, False])
@pytest.mark.parametrize("case", ["1d-weak", "2d-strong"])
def test_orthogonalize_preserves_operator(cuda, sym, case):
    # test_algebra.cpp:24-43
    pts, leaf, weak = (O.grid1d(200, -1, 1), 12, True) if case == "1d-weak" else (O.grid2d(20, 20), 16, False)
    bt, ref = trees(pts, leaf, weak)
    ora = O.H2.random(ref, sym, 10, 11)
    rr, cr = ora.ranks()
    m = H2Matrix.from_packed(bt, sym, rr, cr, ora.export())
    g = orthogonalize(m)
    assert g.orthonormal
    a = ora.to_dense()
    assert rel(dense(g, ref), a) < 1e-12
    # orthonormal leaf bases
    parts = g.download()
    r2, _ = g.ranks()
    ct = bt.tree
    off = 0
    for v in ct.leaves:
        msz, k = ct.size(v), int(r2[v])
        U = parts["U"][off:off + msz * k].reshape((msz, k), order="F")
        off += msz * k
        if k:
            assert np.abs(U.T @ U - np.eye(k)).max() < 1e-13
    # ranks never exceed the oracle's orthogonalize ranks
    ro, _ = ora.orthogonalize().ranks()
    assert np.array_equal(r2, ro)


@pytest.mark.parametrize("sym", [True, False])
def test_recompress_contracts(cuda, sym):
    # test_algebra.cpp:66-101: eps=0 unchanged, ranks never increase, 2-norm contract <= 3 eps
    bt, ref = trees(O.grid2d(24, 24), 16, False)
    ora = O.H2.random(ref, sym, 12, 21)
    rr, cr = ora.ranks()
    m = H2Matrix.from_packed(bt, sym, rr, cr, ora.export())
    a = ora.to_dense()
    r0 = recompress(m, 0.0)
    assert rel(dense(r0, ref), a) < 1e-11
    assert np.all(r0.ranks()[0] <= rr)
    for eps in (1e-2, 1e-5):
        r = recompress(m, eps)
        assert n2(dense(r, ref) - a) <= 3 * eps * n2(a)
        # rank profile agrees with the oracle's recompress within +-2
        ro = ora.recompress(eps)
        assert np.abs(r.ranks()[0].astype(int) - ro.ranks()[0].astype(int)).max() <= 2
    with pytest.raises(ValueError):
        recompress(m, -1.0)


def test_recompress_idempotent_ranks(cuda):
    # test_algebra.cpp:93-101
    bt, ref = trees(O.grid1d(256, -1, 1), 16, True)
    ora = O.H2.random(ref, True, 8, 5)
    rr, cr = ora.ranks()
    m = H2Matrix.from_packed(bt, True, rr, cr, ora.export())
    r1 = recompress(m, 1e-3)
    r2 = recompress(r1, 1e-3)
    assert np.array_equal(r1.ranks()[0], r2.ranks()[0])


# ---- operators (test_operator.cpp) ------------------------------------------

def test_operator_counter_and_pnorm(cuda):
    # test_operator.cpp:10-19 (counter), :32-45 (identity and known spectra)
    d = np.diag(np.arange(1.0, 11.0))
    op = DenseOperator(d, True)
    x = np.random.default_rng(0).standard_normal((10, 3))
    assert rel(op.apply(x), d @ x) < 1e-15
    assert op.columns_applied() == 3
    op.reset_counter()
    v, it = pnorm_estimate(op)
    assert abs(v - 10.0) <= 5e-3 * 10.0
    assert op.columns_applied() == 3 * (2 * it - 1)
    ident = make_operator(50, True, lambda z: z)
    v1, it1 = pnorm_estimate(ident)
    assert abs(v1 - 1.0) < 1e-12 and it1 >= 1
    # same iteration count and value as the oracle's pnorm_estimate
    a = spd(3, 80)
    vo, ito = O.pnorm2_dense(a, True)
    vg, itg = pnorm_estimate(DenseOperator(a, True))
    assert itg == ito and abs(vg - vo) <= 1e-12 * vo


def test_nonsymmetric_operator_without_transpose_raises(cuda):
    op = make_operator(16, False, lambda z: 2 * z)
    with pytest.raises(NotImplementedError):
        op.apply_transpose(np.ones((16, 1)))


def test_h2_operator_adapter(cuda):
    # test_operator.cpp:61-70: the adapter is the hgemv and counts columns
    bt, ref = trees(O.grid1d(128, -1, 1), 16, True)
    ora = O.H2.random(ref, True, 6, 3)
    rr, cr = ora.ranks()
    m = H2Matrix.from_packed(bt, True, rr, cr, ora.export())
    op = H2Operator(m)
    x = O.gaussian(3, 128, 4)
    assert np.array_equal(op.apply(x), m.matvec(x))
    assert op.columns_applied() == 4


# ---- HARA (test_construction.cpp) -------------------------------------------

def test_peel_identity(cuda):
    # test_construction.cpp:112-124
    bt, ref = tree1d(128, 16)
    op = make_operator(128, True, lambda x: x)
    res = peel_construct(op, bt, PeelConfig(eps=1e-8))
    assert rel(dense(res.matrix, ref), np.eye(128)) < 1e-12
    assert np.all(res.matrix.ranks()[0] == 0)
    assert res.stats.consistent()
    assert res.stats.total == op.columns_applied()
    assert res.stats.levels[-1].samples == 16


def spd(seed, n):
    g = O.gaussian(seed, n, n)
    return g @ g.T + n * np.eye(n)


def test_peel_dense_spd_to_eps(cuda):
    # test_construction.cpp:126-144
    a = spd(55, 64)
    bt, ref = tree1d(64, 8)
    op = DenseOperator(a, True)
    res = peel_construct(op, bt, PeelConfig(eps=1e-6))
    assert n2(dense(res.matrix, ref) - a) <= 1e-6 * n2(a)
    assert res.matrix.symmetric
    tight = peel_construct(op, bt, PeelConfig(eps=1e-12))
    assert rel(dense(tight.matrix, ref), a) < 1e-11


def test_peel_rank5_plus_noise(cuda):
    # test_construction.cpp:146-159
    b5 = O.gaussian(56, 256, 5)
    noise = O.gaussian(57, 256, 256)
    a = b5 @ b5.T + 1e-8 * (noise + noise.T)
    bt, ref = tree1d(256, 32)
    res = peel_construct(DenseOperator(a, True), bt, PeelConfig(eps=1e-6))
    assert res.matrix.rank_profile().max() <= 5
    assert n2(dense(res.matrix, ref) - a) <= 3e-6 * n2(a)


def test_peel_deterministic(cuda):
    # test_construction.cpp:161-178: same seed => bitwise-identical payload, same sample count
    g = O.gaussian(57, 96, 96)
    a = g @ g.T
    bt, _ = tree1d(96, 12)
    cfg = PeelConfig(eps=1e-5, seed=1234)
    r1 = peel_construct(DenseOperator(a, True), bt, cfg)
    r2 = peel_construct(DenseOperator(a, True), bt, cfg)
    p1, p2 = r1.matrix.download(), r2.matrix.download()
    assert all(np.array_equal(p1[k], p2[k]) for k in p1)
    assert np.array_equal(r1.matrix.ranks()[0], r2.matrix.ranks()[0])
    assert r1.stats.total == r2.stats.total


def test_estimate_relative_error_below_eps(cuda):
    # test_construction.cpp:226-236
    g = O.gaussian(60, 96, 96)
    a = g @ g.T
    bt, _ = tree1d(96, 12)
    op = DenseOperator(a, True)
    pr = peel_construct(op, bt, PeelConfig(eps=1e-4))
    assert estimate_relative_error(op, pr.matrix) <= 1e-4


def test_peel_max_rank_error(cuda):
    # test_construction.cpp:100-110 (max_rank cap exceeded)
    from paper_2003_10173_b200 import max_rank_error
    a = O.gaussian(61, 64, 64)
    a = a + a.T
    bt, _ = tree1d(64, 8)
    with pytest.raises(max_rank_error):
        peel_construct(DenseOperator(a, True), bt, PeelConfig(eps=1e-12, max_rank=2))


# ---- parity with the oracle's peel_construct ---------------------------------

def kernel_matrix(pts, ell, kind="exp"):
    r = np.sqrt(((pts[:, None, :] - pts[None, :, :]) ** 2).sum(-1))
    return np.exp(-r / ell) if kind == "exp" else np.exp(-(r / ell) ** 2)


PARITY = {
    "1d-weak-spd": (lambda: O.grid1d(512, -1, 1), 16, True, True, 1e-6),
    "1d-weak-nonsym": (lambda: O.grid1d(256, -1, 1), 16, True, False, 1e-6),
    "2d-strong-kernel": (lambda: O.grid2d(32, 32), 32, False, True, 1e-5),
}


@pytest.mark.parametrize("case", list(PARITY))
def test_peel_matches_oracle(cuda, case):
    mk, leaf, weak, sym, eps = PARITY[case]
    pts = mk()
    n = pts.shape[0]
    a = kernel_matrix(pts, 0.2) + 0.5 * np.eye(n)   # test_inversion.cpp:18-25 style kernel matrix
    if not sym:
        a = a + 0.1 * np.triu(kernel_matrix(pts, 0.05), 1)
    bt, ref = trees(pts, leaf, weak)
    op = DenseOperator(a, sym)
    res = peel_construct(op, bt, PeelConfig(eps=eps))
    ora, st = O.peel_dense(ref, a, sym, eps=eps)
    ag = dense(res.matrix, ref)
    ao = ora.to_dense()
    # accuracy contract: ||A - H||_2 <= 3 eps ||A||_2, both paths
    assert n2(ag - a) <= 3 * eps * n2(a)
    assert n2(ao - a) <= 3 * eps * n2(a)
    # the two constructions agree with each other to the same order
    assert n2(ag - ao) <= 6 * eps * n2(a)
    # rng=0 (the default) draws the reference's mt19937_64 panels, so the
    # decisions are the reference's: identical per-level samples, per-level max
    # rank and per-node ranks, against the restatement AND the reference's own
    # compiled driver (oracle/_ref)
    gl = [lv.samples for lv in res.stats.levels]
    assert gl == st["level_samples"], (gl, st["level_samples"])
    assert [lv.max_rank for lv in res.stats.levels] == st["level_max_rank"]
    rr, _ = ora.ranks()
    assert np.array_equal(res.matrix.ranks()[0], rr)
    if R is not None:
        hr, sr = R.peel_dense(R.Tree(pts, leaf, 1.0, weak), a, sym, eps=eps)
        assert sr == st
        assert np.array_equal(hr.ranks()[0], rr)
    assert res.stats.consistent() and res.stats.total == op.columns_applied()


# ---- global randomized low-rank and hybrid (test_construction.cpp:180-224) -----

def test_randomized_lowrank_exact_rank8(cuda):
    from paper_2003_10173_b200 import randomized_lowrank
    b8 = O.gaussian(58, 100, 8)
    a = b8 @ b8.T
    op = DenseOperator(a, True)
    cfg = PeelConfig(norm_scale=n2(a))   # no estimation samples in this budget check
    op.reset_counter()
    lr = randomized_lowrank(op, 1e-10, 0, cfg)
    assert lr.factor.rank() == 8
    assert op.columns_applied() <= 8 + cfg.sample_block_size + cfg.oversampling
    assert not lr.max_rank_reached
    assert rel(lr.factor.X @ lr.factor.Y.T, a) < 1e-9
    assert lr.symmetric_form and np.array_equal(lr.factor.X, lr.factor.Y)


def test_randomized_lowrank_identity_stalls_at_max_rank(cuda):
    from paper_2003_10173_b200 import randomized_lowrank
    op = make_operator(64, True, lambda x: x)
    lr = randomized_lowrank(op, 1e-4, 16, PeelConfig(norm_scale=1.0))
    assert lr.max_rank_reached
    assert lr.factor.rank() <= 16
    assert abs(lr.residual_estimate - 1.0) <= 0.4 * 1.0 + 1e-12


def test_randomized_lowrank_nonsymmetric(cuda):
    from paper_2003_10173_b200 import randomized_lowrank
    u = O.gaussian(70, 90, 6)
    v = O.gaussian(71, 90, 6)
    a = u @ v.T
    lr = randomized_lowrank(DenseOperator(a, False), 1e-10, 0, PeelConfig())
    assert lr.factor.rank() == 6 and not lr.symmetric_form
    assert rel(lr.factor.X @ lr.factor.Y.T, a) < 1e-9


def test_hybrid_low_rank_operator(cuda):
    from paper_2003_10173_b200 import hybrid_construct
    b20 = O.gaussian(59, 128, 20)
    a = b20 @ b20.T
    bt, ref = tree1d(128, 16)
    cfg = PeelConfig(eps=1e-8)
    hy = hybrid_construct(DenseOperator(a, True), bt, cfg)
    assert hy.global_rank == 20
    assert n2(dense(hy.matrix, ref) - a) <= 3e-8 * n2(a)
    assert hy.stats.consistent()
    pr = peel_construct(DenseOperator(a, True), bt, cfg)
    assert hy.stats.total <= pr.stats.total


def test_peel_full_rank_blocks_above_256(cuda):
    # a full-rank SPD operator: the level-1 sibling blocks (320 x 320) are sampled
    # to rank 320, so the batched QR / Jacobi SVD of absorb_panel and recompress
    # run on more than 256 columns (the reference has no such limit either)
    n = 640
    g = O.gaussian(91, n, n)
    a = g @ g.T / n + np.eye(n)
    bt, ref = tree1d(n, 16)
    eps = 1e-8
    res = peel_construct(DenseOperator(a, True), bt, PeelConfig(eps=eps))
    assert max(res.matrix.rank_profile()) > 256
    assert n2(dense(res.matrix, ref) - a) <= 3 * eps * n2(a)
