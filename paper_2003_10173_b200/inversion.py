"""Python mirror of the reference's iterative inversion API (inversion.hpp) and
low_rank_update (algebra.hpp:334-346) over the C ABI. Each hierarchical iterate
is rebuilt by HARA on the B200 from a sampler of device hgemvs."""
import ctypes as C
import dataclasses
import math

import numpy as np

from ._lib import H, PeelConfigC, TraceRowC, check, divergence_error, lib
from .construction import LinearOperator, PeelConfig
from .h2 import H2Matrix


@dataclasses.dataclass
class ThresholdSchedule:   # inversion.hpp:50-54
    dynamic: bool = False
    eps_initial: float = 1e-2


def threshold_schedule(residual, it, eps_final, sched):   # inversion.hpp:58-63
    if not sched.dynamic:
        return eps_final
    v = min(sched.eps_initial, residual * residual / 10.0)
    return min(max(v, eps_final), sched.eps_initial)


@dataclasses.dataclass
class TraceRow:
    iter: int
    residual: float
    eps_k: float
    samples: int
    wall_seconds: float


@dataclasses.dataclass
class ConvergenceTrace:   # inversion.hpp:27-39
    rows: list
    final_residual: float = 0.0
    converged: bool = False

    def iterations(self):
        return len(self.rows)

    def total_samples(self):
        return sum(r.samples for r in self.rows)


@dataclasses.dataclass
class HInverseResult:
    X: H2Matrix
    trace: ConvergenceTrace


def scaled_identity(bt, value):
    """H2Matrix::scaled_identity (h2_matrix.hpp:90-93)."""
    h = H()
    check(lib.h2c_scaled_identity(bt._h, float(value), C.byref(h)))
    return H2Matrix(h, bt)


def scaled_identity_start(a):
    """I / ||A||_inf (inversion.hpp:124-130)."""
    h = H()
    check(lib.h2c_scaled_identity_start(a._h, C.byref(h)))
    return H2Matrix(h, a.blocks)


def pnorm_estimate(op, p):
    """pnorm_estimate(op, p), p in {1, 2, inf} (linear_operator.hpp:127-178) -> (value, iterations)."""
    v, it = C.c_double(), C.c_int()
    check(lib.h2c_pnorm_estimate(op._h, float(p), C.byref(v), C.byref(it)))
    return v.value, it.value


def _sampler(xk, a, kind, arg):
    h = H()
    check(lib.h2c_sampler_operator(xk._h, a._h, int(kind), int(arg), C.byref(h)))
    return LinearOperator(h, a.tree.n, xk.symmetric and a.symmetric, keep=(xk, a))


def ns_sampler(xk, a):
    return _sampler(xk, a, 0, 0)


def hyperpower_sampler(xk, a, order):
    return _sampler(xk, a, 1, order)


def unrolled_sampler(x0, a, k):
    return _sampler(x0, a, 2, k)


def residual_norm(a, x):
    """||A X - I||_2 estimate (inversion.hpp:213-225); H2 matrices or LinearOperators."""
    v = C.c_double()
    if isinstance(a, LinearOperator):
        check(lib.h2c_residual_norm_op(a._h, x._h, C.byref(v)))
    else:
        check(lib.h2c_residual_norm(a._h, x._h, C.byref(v)))
    return v.value


def _inverse(a, x0, method, arg, sched, eps, cfg, max_iter):
    cfg = cfg or PeelConfig()
    sched = sched or ThresholdSchedule()
    c = PeelConfigC(float(cfg.eps), int(cfg.sample_block_size), int(cfg.oversampling), int(cfg.max_rank),
                    int(cfg.seed), float(cfg.norm_scale), int(cfg.crossover_rank_cap), int(cfg.rng))
    h = H()
    rows = (TraceRowC * 256)()
    nr, fr, cv = C.c_int(), C.c_double(), C.c_int()
    rc = lib.h2c_h_inverse(a._h, x0._h, int(method), int(arg), int(bool(sched.dynamic)), float(sched.eps_initial),
                           float(eps), C.byref(c), int(max_iter), C.byref(h), rows, 256, C.byref(nr), C.byref(fr),
                           C.byref(cv))
    trace = ConvergenceTrace([TraceRow(rows[i].iter, rows[i].residual, rows[i].eps_k, rows[i].samples,
                                       rows[i].wall_seconds) for i in range(min(nr.value, 256))],
                             fr.value, bool(cv.value))
    try:
        check(rc)
    except divergence_error as e:
        e.trace = trace
        raise
    return HInverseResult(H2Matrix(h, a.blocks), trace)


def h_newton_schulz(a, x0, sched=None, eps=1e-8, cfg=None, max_iter=64):
    """inversion.hpp:281-286."""
    return _inverse(a, x0, 0, 0, sched, eps, cfg, max_iter)


def h_hyperpower(a, x0, order, sched=None, eps=1e-8, cfg=None, max_iter=64):
    """inversion.hpp:288-295."""
    return _inverse(a, x0, 1, order, sched, eps, cfg, max_iter)


def h_unrolled(a, x0, k, eps, cfg=None):
    """inversion.hpp:303-311."""
    return _inverse(a, x0, 2, k, None, eps, cfg, 0)


def low_rank_update(h, X, Y, eps):
    """low_rank_update(h, {X, Y}, eps) (algebra.hpp:334-346); X, Y host n x k (user order)."""
    import torch
    X = np.asarray(X, np.float64)
    Y = np.asarray(Y, np.float64)
    if X.ndim == 1:
        X = X[:, None]
    if Y.ndim == 1:
        Y = Y[:, None]
    n = h.tree.n
    if X.shape[0] != n or Y.shape[0] != n or X.shape[1] != Y.shape[1]:
        raise ValueError("low_rank_update: factor dimensions do not match")
    k = X.shape[1]
    xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()
    same = np.array_equal(X.view(np.uint64), Y.view(np.uint64))
    yd = xd if same else torch.from_numpy(np.ascontiguousarray(Y.T)).cuda()
    out = H()
    check(lib.h2c_low_rank_update(h._h, k, xd.data_ptr(), yd.data_ptr(), float(eps), C.byref(out)))
    torch.cuda.synchronize()
    return H2Matrix(out, h.blocks)


def desymmetrized(h):
    """h2_matrix.hpp:200-216."""
    out = H()
    check(lib.h2c_desymmetrized(h._h, C.byref(out)))
    return H2Matrix(out, h.blocks)


_ = math
