"""Python mirror of the reference's operator and construction API
(linear_operator.hpp:20-178, algebra.hpp:72-226, construction.hpp:23-382)
over the C ABI. Every computation runs on the B200 (lib/libh2b200.so)."""
import ctypes as C
import dataclasses

import numpy as np

from ._lib import APPLY_FN, H, LevelStatsC, PeelConfigC, check, lib
from .h2 import H2Matrix


class LinearOperator:
    """Black-box operator handle (LinearOperator, linear_operator.hpp:20-55).
    apply / apply_transpose take host arrays in user ordering (n x b)."""

    def __init__(self, handle, n, symmetric, keep=None):
        self._h = handle
        self._n = int(n)
        self._sym = bool(symmetric)
        self._keep = keep   # keeps ctypes callbacks / source matrices alive

    def __del__(self):
        if getattr(self, "_h", None):
            lib.h2c_operator_destroy(self._h)
            self._h = None

    def dim(self):
        return self._n

    def symmetric(self):
        return self._sym

    def columns_applied(self):
        v = C.c_int64()
        check(lib.h2c_operator_columns_applied(self._h, C.byref(v)))
        return v.value

    def reset_counter(self):
        check(lib.h2c_operator_reset_counter(self._h))

    def _apply(self, x, transpose):
        import torch
        x = np.asarray(x, np.float64)
        vec = x.ndim == 1
        xm = x[:, None] if vec else x
        if xm.shape[0] != self._n:
            raise ValueError("operator apply: dimension mismatch")
        xd = torch.from_numpy(np.ascontiguousarray(xm.T)).cuda()
        yd = torch.empty_like(xd)
        check(lib.h2c_operator_apply(self._h, int(transpose), xm.shape[1], xd.data_ptr(), yd.data_ptr(), None))
        torch.cuda.synchronize()
        y = yd.cpu().numpy().T
        return y[:, 0] if vec else np.asfortranarray(y)

    def apply(self, x):
        return self._apply(x, False)

    def apply_transpose(self, x):
        return self._apply(x, True)


def DenseOperator(a, symmetric=False):
    """DenseOperator (linear_operator.hpp:86-101): the matrix is copied to HBM."""
    a = np.asfortranarray(a, np.float64)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError("dense operator: square only")
    h = H()
    check(lib.h2c_operator_dense(a.ctypes.data_as(C.c_void_p), a.shape[0], int(bool(symmetric)), C.byref(h)))
    return LinearOperator(h, a.shape[0], symmetric)


def H2Operator(m):
    """H2Operator (linear_operator.hpp:104-115): hgemv of a device H^2 matrix."""
    h = H()
    check(lib.h2c_operator_h2(m._h, C.byref(h)))
    return LinearOperator(h, m.tree.n, m.symmetric, keep=m)


def make_operator(n, symmetric, f, t=None):
    """make_operator (linear_operator.hpp:80-84): f(x) / t(x) act on host numpy
    arrays (n x b, user ordering); the library stages device <-> host copies."""
    def cb(ctx, transpose, b, x, y, stream):
        try:
            xa = np.ctypeslib.as_array(C.cast(x, C.POINTER(C.c_double)), shape=(b * n,)).reshape((n, b), order="F")
            ya = np.ctypeslib.as_array(C.cast(y, C.POINTER(C.c_double)), shape=(b * n,)).reshape((n, b), order="F")
            fn = t if transpose else f
            ya[...] = np.asarray(fn(xa), np.float64).reshape(n, b)
            return 0
        except Exception:   # reported as H2C_RUNTIME_ERROR by the library
            return 1
    fp = APPLY_FN(cb)
    h = H()
    check(lib.h2c_operator_host_callback(int(n), int(bool(symmetric)), int(t is not None), fp, None, C.byref(h)))
    return LinearOperator(h, n, symmetric, keep=fp)


def pnorm_estimate(op, p=2):
    """pnorm_estimate(op, p), p in {1, 2, inf} (linear_operator.hpp:127-178) -> (value, iterations)."""
    v, it = C.c_double(), C.c_int()
    check(lib.h2c_pnorm_estimate(op._h, float(p), C.byref(v), C.byref(it)))
    return v.value, it.value


def orthogonalize(m):
    """algebra.hpp:72-113 (new matrix)."""
    h = H()
    check(lib.h2c_orthogonalize(m._h, C.byref(h)))
    return H2Matrix(h, m.blocks)


def recompress(m, eps):
    """algebra.hpp:144-226 (new matrix)."""
    h = H()
    check(lib.h2c_recompress(m._h, float(eps), C.byref(h)))
    return H2Matrix(h, m.blocks)


@dataclasses.dataclass
class PeelConfig:   # construction.hpp:23-31
    eps: float = 1e-4
    sample_block_size: int = 16
    oversampling: int = 10
    max_rank: int = 0
    seed: int = 42
    norm_scale: float = 0.0
    crossover_rank_cap: int = 128
    rng: int = 0   # B200 extension: 0 reference host stream, 1 device Philox


@dataclasses.dataclass
class LevelStats:
    level: int
    blocks: int
    max_rank: int
    samples: int


@dataclasses.dataclass
class SampleStats:   # construction.hpp:40-59
    total: int
    levels: list

    def consistent(self):
        return sum(lv.samples for lv in self.levels) == self.total


@dataclasses.dataclass
class PeelResult:   # construction.hpp:295-298
    matrix: H2Matrix
    stats: SampleStats
    op_ms: float = 0.0
    total_ms: float = 0.0


def peel_construct(op, bt, cfg=None):
    """HARA (construction.hpp:300-382) on the B200."""
    cfg = cfg or PeelConfig()
    c = PeelConfigC(float(cfg.eps), int(cfg.sample_block_size), int(cfg.oversampling), int(cfg.max_rank),
                    int(cfg.seed), float(cfg.norm_scale), int(cfg.crossover_rank_cap), int(cfg.rng))
    h = H()
    tot = C.c_int64()
    lv = (LevelStatsC * 128)()
    nl = C.c_int()
    op_ms, tot_ms = C.c_double(), C.c_double()
    check(lib.h2c_peel_construct(op._h, bt._h, C.byref(c), C.byref(h), C.byref(tot), lv, 128, C.byref(nl),
                                 C.byref(op_ms), C.byref(tot_ms)))
    levels = [LevelStats(lv[i].level, lv[i].blocks, lv[i].max_rank, lv[i].samples) for i in range(nl.value)]
    return PeelResult(H2Matrix(h, bt), SampleStats(tot.value, levels), op_ms.value, tot_ms.value)


def estimate_relative_error(op, m, op_norm=0.0):
    """construction.hpp:537-546."""
    v = C.c_double()
    check(lib.h2c_estimate_relative_error(op._h, m._h, float(op_norm), C.byref(v)))
    return v.value


def frobenius_norm(m):
    """frobenius_norm(h) (algebra.hpp:119-137); needs orthonormal bases."""
    v = C.c_double()
    check(lib.h2c_frobenius_norm(m._h, C.byref(v)))
    return v.value


def local_low_rank_update(m, t, s, U, V, eps):
    """local_low_rank_update(h, t, s, U_blk, V_blk, eps) (algebra.hpp:323-332):
    U (|t| x k), V (|s| x k) host arrays in cluster (internal) row order."""
    import torch
    U = np.asarray(U, np.float64)
    V = np.asarray(V, np.float64)
    U = U[:, None] if U.ndim == 1 else U
    V = V[:, None] if V.ndim == 1 else V
    ct = m.blocks.tree
    if U.shape[0] != ct.size(t) or V.shape[0] != ct.size(s) or U.shape[1] != V.shape[1]:
        raise ValueError("local update: factor dimensions do not match clusters")
    k = U.shape[1]
    ud = torch.from_numpy(np.ascontiguousarray(U.T)).cuda()
    same = U.shape == V.shape and np.array_equal(U.view(np.uint64), V.view(np.uint64))
    vd = ud if same else torch.from_numpy(np.ascontiguousarray(V.T)).cuda()
    out = H()
    check(lib.h2c_local_low_rank_update(m._h, int(t), int(s), k, ud.data_ptr(), max(U.shape[0], 1), vd.data_ptr(),
                                        max(V.shape[0], 1), float(eps), C.byref(out)))
    torch.cuda.synchronize()
    return H2Matrix(out, m.blocks)


class Rng:
    """The std::mt19937_64 stream the reference threads through its samplers."""

    def __init__(self, seed):
        self._h = H()
        check(lib.h2c_rng_create(int(seed), C.byref(self._h)))

    def gaussian(self, rows, cols):
        """detail::fill_gaussian of a rows x cols block (construction.hpp:81-85)."""
        out = np.empty((int(rows), int(cols)), order="F")
        check(lib.h2c_rng_fill_gaussian(self._h, int(rows), int(cols), out.ctypes.data_as(C.c_void_p)))
        return out

    def __del__(self):
        if getattr(self, "_h", None):
            lib.h2c_rng_destroy(self._h)
            self._h = None


def sample_block_column(op, ct, t, s, count, rng):
    """sample_block_column(op, ct, t, s, count, rng) (construction.hpp:137-148) ->
    (Omega restricted to s, op(Omega) restricted to t), host arrays in cluster order."""
    import torch
    ms, mt = ct.size(s), ct.size(t)
    om = torch.empty((max(int(count), 0), ms), dtype=torch.float64, device="cuda")
    y = torch.empty((max(int(count), 0), mt), dtype=torch.float64, device="cuda")
    check(lib.h2c_sample_block_column(op._h, ct._h, int(t), int(s), int(count), rng._h, om.data_ptr(), y.data_ptr(),
                                      None))
    torch.cuda.synchronize()
    return om.cpu().numpy().T, y.cpu().numpy().T


@dataclasses.dataclass
class BlockFactor:   # construction.hpp:150-154
    u: np.ndarray
    v: np.ndarray
    rank: int
    err_est: float


def adaptive_block_factorization(op, ct, t, s, eps_block, cfg=None):
    """adaptive_block_factorization(op, ct, t, s, eps_block, cfg) (construction.hpp:156-198)."""
    cfg = cfg or PeelConfig()
    c = _cfg_c(cfg)
    h = H()
    check(lib.h2c_adaptive_block_factorization(op._h, ct._h, int(t), int(s), float(eps_block), C.byref(c),
                                               C.byref(h)))
    try:
        ru, rv, k, e = C.c_int64(), C.c_int64(), C.c_int64(), C.c_double()
        check(lib.h2c_block_factor_info(h, C.byref(ru), C.byref(rv), C.byref(k), C.byref(e)))
        u = np.empty((ru.value, k.value), order="F")
        v = np.empty((rv.value, k.value), order="F")
        check(lib.h2c_block_factor_download(h, u.ctypes.data_as(C.c_void_p), v.ctypes.data_as(C.c_void_p)))
    finally:
        lib.h2c_block_factor_destroy(h)
    return BlockFactor(u, v, int(k.value), float(e.value))


def _cfg_c(cfg):
    return PeelConfigC(float(cfg.eps), int(cfg.sample_block_size), int(cfg.oversampling), int(cfg.max_rank),
                       int(cfg.seed), float(cfg.norm_scale), int(cfg.crossover_rank_cap), int(cfg.rng))


@dataclasses.dataclass
class LowRankFactor:   # algebra.hpp:323-331 (LowRankFactor)
    X: np.ndarray
    Y: np.ndarray

    def rank(self):
        return self.X.shape[1]


@dataclasses.dataclass
class LowRankResult:   # construction.hpp:386-391
    factor: LowRankFactor
    stats: SampleStats
    residual_estimate: float
    max_rank_reached: bool
    symmetric_form: bool


def randomized_lowrank(op, eps, max_rank=0, cfg=None):
    """Adaptive global randomized range finder (construction.hpp:484-491) on the B200."""
    cfg = cfg or PeelConfig()
    c = _cfg_c(cfg)
    h = H()
    check(lib.h2c_randomized_lowrank(op._h, float(eps), int(max_rank), C.byref(c), C.byref(h)))
    try:
        n, k, tot = C.c_int64(), C.c_int64(), C.c_int64()
        sym, mr = C.c_int(), C.c_int()
        res = C.c_double()
        check(lib.h2c_lowrank_info(h, C.byref(n), C.byref(k), C.byref(sym), C.byref(res), C.byref(mr), C.byref(tot)))
        X = np.zeros((n.value, k.value), order="F")
        Y = np.zeros((n.value, k.value), order="F")
        if k.value:
            check(lib.h2c_lowrank_download(h, X.ctypes.data_as(C.c_void_p), Y.ctypes.data_as(C.c_void_p)))
    finally:
        lib.h2c_lowrank_destroy(h)
    return LowRankResult(LowRankFactor(X, Y), SampleStats(tot.value, [LevelStats(0, 1, k.value, tot.value)]),
                         res.value, bool(mr.value), bool(sym.value))


@dataclasses.dataclass
class HybridResult:   # construction.hpp:495-499
    matrix: H2Matrix
    stats: SampleStats
    global_rank: int


def hybrid_construct(op, bt, cfg=None):
    """Global low-rank capture, peel of the residual, global update back (construction.hpp:506-534)."""
    cfg = cfg or PeelConfig()
    c = _cfg_c(cfg)
    h = H()
    gr, tot = C.c_int64(), C.c_int64()
    lv = (LevelStatsC * 128)()
    nl = C.c_int()
    check(lib.h2c_hybrid_construct(op._h, bt._h, C.byref(c), C.byref(h), C.byref(gr), C.byref(tot), lv, 128,
                                   C.byref(nl)))
    levels = [LevelStats(lv[i].level, lv[i].blocks, lv[i].max_rank, lv[i].samples) for i in range(nl.value)]
    return HybridResult(H2Matrix(h, bt), SampleStats(tot.value, levels), gr.value)
