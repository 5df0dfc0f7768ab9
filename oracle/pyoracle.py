"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes access to the CPU restatement of the reference (oracle/h2oracle.hpp,
built as oracle/build/liboracle.so). Used by tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference leg as the checker and the
CPU baseline — never by the product path.
"""
import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# oracle/pyref.py executes this same source with _LIB_OVERRIDE set to the
# reference-compiled library (oracle/_ref/libh2ref.so: the reference's own
# headers over the Eigen shim), which exports the same ora_* ABI.
_REF_BUILD = "_LIB_OVERRIDE" in globals()
LIB_PATH = globals().get("_LIB_OVERRIDE") or os.path.join(_HERE, "build", "liboracle.so")


def build():
    subprocess.run(["make", "-s", "-C", _HERE, "-j8"], check=True)


if not os.path.exists(LIB_PATH):
    if _REF_BUILD:
        subprocess.run(["make", "-s", "-C", _HERE, "ref"], check=True)
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built and /root/reference is absent")
    else:
        build()

_lib = C.CDLL(LIB_PATH)
vp, i32, i64, u64, f64 = C.c_void_p, C.c_int, C.c_int64, C.c_uint64, C.c_double
P = C.POINTER


# entries only one of the two builds exports: the diffusion oracle (restatement
# only) and the reference's own inversion drivers (oracle/_ref only)
_OPTIONAL = {"ora_h_inverse", "ora_residual_norm"}


def _sig(name, *args):
    if (_REF_BUILD or name in _OPTIONAL) and not hasattr(_lib, name):
        return
    f = getattr(_lib, name)
    f.restype = i32
    f.argtypes = list(args)


_lib.ora_last_error.restype = C.c_char_p
_sig("ora_tree_create", vp, i64, i32, i64, f64, i32, P(vp))
_lib.ora_tree_destroy.argtypes = [vp]
_lib.ora_tree_destroy.restype = None
_sig("ora_tree_info", vp, P(i64), P(i32), P(i32), P(i32), P(i32), P(i32))
_sig("ora_tree_arrays", vp, *([vp] * 12))
_sig("ora_tree_boxes", vp, vp, vp)
_sig("ora_h_inverse", vp, i32, i32, i32, f64, f64, u64, i32, P(vp), vp, i32, P(i32), P(f64), P(i32))
_sig("ora_residual_norm", vp, vp, P(f64))
_sig("ora_random_h2", vp, i32, i64, u64, P(vp))
_sig("ora_zero", vp, i32, P(vp))
_sig("ora_kernel_h2", vp, vp, i32, f64, i64, i32, P(vp))
_sig("ora_fixed_rank_h2", vp, i64, u64, i32, P(vp))
_lib.ora_h2_destroy.argtypes = [vp]
_lib.ora_h2_destroy.restype = None
_sig("ora_h2_info", vp, P(i32), P(i32), vp)
_sig("ora_h2_ranks", vp, vp, vp)
_sig("ora_h2_export", vp, *([vp] * 6))
_sig("ora_h2_import", vp, i32, i32, vp, vp, *([vp] * 6), P(vp))
_sig("ora_matvec", vp, i32, i32, i64, vp, vp, i32)
_sig("ora_to_dense", vp, vp)
_sig("ora_orthogonalize", vp, P(vp))
_sig("ora_recompress", vp, f64, P(vp))
_sig("ora_low_rank_update", vp, i64, vp, vp, f64, P(vp))
_sig("ora_frobenius_norm", vp, P(f64))
_sig("ora_peel_dense", vp, vp, i32, f64, i64, i64, i64, u64, f64, P(vp), P(i64), vp, vp, P(i32))
_sig("ora_peel_h2", vp, vp, f64, u64, f64, P(vp), P(i64))
_sig("ora_peel_dense_threads", vp, vp, i32, f64, u64, f64, i32, P(vp), P(i64), vp, vp, P(i32), P(f64))
_sig("ora_pnorm2_dense", vp, i64, i32, P(f64), P(i32))
_sig("ora_sample_block_column", vp, vp, i32, i32, i32, i64, u64, vp, vp)
_sig("ora_adaptive_block_factorization", vp, vp, i32, i32, i32, f64, i64, i64, i64, u64, vp, vp, P(i64), P(f64),
     P(i64))
_sig("ora_local_low_rank_update", vp, i32, i32, i64, vp, vp, f64, P(vp))
_sig("ora_validate", vp, i64, P(i32), vp, vp)
_sig("ora_gaussian", u64, i64, i64, vp)
_sig("ora_shuffle", i64, u64, vp)
_sig("ora_diff1d_create", i64, i64, f64, f64, f64, f64, f64, f64, f64, i32, vp, i64, P(vp))
if hasattr(_lib, "ora_diff1d_destroy"):
    _lib.ora_diff1d_destroy.argtypes = [vp]
    _lib.ora_diff1d_destroy.restype = None
_sig("ora_diff1d_info", vp, P(i64), P(i64), P(f64), P(f64), P(i64))
_sig("ora_diff1d_hessvec", vp, i64, vp, vp, i32, i32)
_sig("ora_diff1d_state", vp, i32, vp)
_sig("ora_peel_diff1d", vp, vp, i32, f64, u64, i32, P(vp), P(i64), P(f64), vp, vp, P(i32))


class OracleError(RuntimeError):
    pass


class OracleMaxRank(OracleError):
    pass


def _check(rc):
    if rc == 0:
        return
    msg = _lib.ora_last_error().decode()
    if rc == -1:
        raise ValueError(msg)
    if rc == -2:
        raise NotImplementedError(msg)
    if rc == -3:
        raise OracleMaxRank(msg)
    raise OracleError(msg)


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


PARTS = ("U", "E", "V", "F", "S", "D")


class Tree:
    """Cluster tree + block tree of the oracle (cluster_tree.hpp / block_tree.hpp)."""

    def __init__(self, points, leaf, eta=1.0, weak=False):
        pts = np.asarray(points, np.float64)
        if pts.ndim == 1:
            pts = pts[:, None]
        self.points = np.asfortranarray(pts)
        h = vp()
        _check(_lib.ora_tree_create(_p(self.points), pts.shape[0], pts.shape[1], int(leaf), float(eta), int(weak),
                                    C.byref(h)))
        self._h = h
        n, d, nn, nb, na, nd = i64(), i32(), i32(), i32(), i32(), i32()
        _check(_lib.ora_tree_info(h, C.byref(n), C.byref(d), C.byref(nn), C.byref(nb), C.byref(na), C.byref(nd)))
        self.n, self.depth, self.num_nodes, self.num_blocks = n.value, d.value, nn.value, nb.value
        self.perm = np.empty(self.n, np.int64)
        self.begin = np.empty(nn.value, np.int64)
        self.end = np.empty(nn.value, np.int64)
        self.level = np.empty(nn.value, np.int32)
        self.parent = np.empty(nn.value, np.int32)
        self.child0 = np.empty(nn.value, np.int32)
        self.child1 = np.empty(nn.value, np.int32)
        self.brow = np.empty(nb.value, np.int32)
        self.bcol = np.empty(nb.value, np.int32)
        self.btag = np.empty(nb.value, np.int32)
        self.adm = np.empty(na.value, np.int32)
        self.dense = np.empty(nd.value, np.int32)
        _check(_lib.ora_tree_arrays(h, *[_p(a) for a in (self.perm, self.begin, self.end, self.level, self.parent,
                                                          self.child0, self.child1, self.brow, self.bcol, self.btag,
                                                          self.adm, self.dense)]))

    def boxes(self):
        """(lo, hi), each num_nodes x 3 (unused axes 0)."""
        lo = np.zeros((self.num_nodes, 3))
        hi = np.zeros((self.num_nodes, 3))
        _check(_lib.ora_tree_boxes(self._h, _p(lo), _p(hi)))
        return lo, hi

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:   # (module globals may be gone at exit)
            _lib.ora_tree_destroy(self._h)
            self._h = None


class H2:
    """Oracle H2Matrix (h2_matrix.hpp:40-306)."""

    def __init__(self, handle, tree):
        self._h = handle
        self.tree = tree

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.ora_h2_destroy(self._h)
            self._h = None

    @staticmethod
    def random(tree, symmetric, kmax, seed):
        """Reference fixture random_h2 with mt19937_64(seed) (test_support.hpp:38-70)."""
        h = vp()
        _check(_lib.ora_random_h2(tree._h, int(symmetric), int(kmax), int(seed), C.byref(h)))
        return H2(h, tree)

    @staticmethod
    def fixed_rank(tree, k, seed=42, threads=1):
        """Symmetric fixed-rank content (CPU-only benchmark inputs)."""
        h = vp()
        _check(_lib.ora_fixed_rank_h2(tree._h, int(k), int(seed), int(threads), C.byref(h)))
        return H2(h, tree)

    @staticmethod
    def kernel(tree, kind="gaussian", ell=0.1, rank=32, threads=1):
        """Kernel-matrix H^2 (host restatement of the product's benchmark generator,
        csrc/matrix.cu make_kernel_h2): symmetric, Chebyshev interpolation."""
        kinds = {"exponential": 0, "gaussian": 1, "matern32": 2}
        h = vp()
        _check(_lib.ora_kernel_h2(tree._h, _p(tree.points), kinds[kind], float(ell), int(rank), int(threads),
                                  C.byref(h)))
        return H2(h, tree)

    @staticmethod
    def zero(tree, symmetric):
        h = vp()
        _check(_lib.ora_zero(tree._h, int(symmetric), C.byref(h)))
        return H2(h, tree)

    @staticmethod
    def from_packed(tree, symmetric, row_ranks, col_ranks, parts, orthonormal=False):
        rr = np.ascontiguousarray(row_ranks, np.int32)
        cr = np.ascontiguousarray(col_ranks if col_ranks is not None else row_ranks, np.int32)
        arrs = [np.ascontiguousarray(parts.get(k, np.zeros(0)), np.float64) for k in PARTS]
        h = vp()
        _check(_lib.ora_h2_import(tree._h, int(symmetric), int(orthonormal), _p(rr), _p(cr), *[_p(a) for a in arrs],
                                  C.byref(h)))
        return H2(h, tree)

    def info(self):
        s, o = i32(), i32()
        sizes = np.zeros(6, np.int64)
        _check(_lib.ora_h2_info(self._h, C.byref(s), C.byref(o), _p(sizes)))
        return bool(s.value), bool(o.value), [int(x) for x in sizes]

    @property
    def symmetric(self):
        return self.info()[0]

    def ranks(self):
        r = np.empty(self.tree.num_nodes, np.int32)
        c = np.empty(self.tree.num_nodes, np.int32)
        _check(_lib.ora_h2_ranks(self._h, _p(r), _p(c)))
        return r, c

    def export(self):
        sizes = self.info()[2]
        arrs = [np.empty(s, np.float64) for s in sizes]
        _check(_lib.ora_h2_export(self._h, *[_p(a) for a in arrs]))
        return dict(zip(PARTS, arrs))

    def matvec(self, x, transpose=False, ordering=0, threads=1):
        x = np.asarray(x, np.float64)
        vec = x.ndim == 1
        xf = np.asfortranarray(x[:, None] if vec else x)
        y = np.empty_like(xf, order="F")
        _check(_lib.ora_matvec(self._h, int(transpose), int(ordering), xf.shape[1], _p(xf), _p(y), int(threads)))
        return y[:, 0] if vec else y

    def to_dense(self):
        a = np.empty((self.tree.n, self.tree.n), order="F")
        _check(_lib.ora_to_dense(self._h, _p(a)))
        return a

    def orthogonalize(self):
        h = vp()
        _check(_lib.ora_orthogonalize(self._h, C.byref(h)))
        return H2(h, self.tree)

    def recompress(self, eps):
        h = vp()
        _check(_lib.ora_recompress(self._h, float(eps), C.byref(h)))
        return H2(h, self.tree)

    def low_rank_update(self, X, Y, eps):
        X = np.asfortranarray(X, np.float64)
        Y = np.asfortranarray(Y, np.float64)
        h = vp()
        _check(_lib.ora_low_rank_update(self._h, X.shape[1], _p(X), _p(Y), float(eps), C.byref(h)))
        return H2(h, self.tree)

    def local_low_rank_update(self, t, s, U, V, eps):
        U = np.asfortranarray(U, np.float64)
        V = np.asfortranarray(V, np.float64)
        h = vp()
        _check(_lib.ora_local_low_rank_update(self._h, int(t), int(s), U.shape[1], _p(U), _p(V), float(eps),
                                              C.byref(h)))
        return H2(h, self.tree)

    def validate(self, ortho_cap=4096):
        nv = i32()
        prof = np.zeros(self.tree.depth + 1, np.int64)
        st = np.zeros(4, np.int64)
        _check(_lib.ora_validate(self._h, int(ortho_cap), C.byref(nv), _p(prof), _p(st)))
        return nv.value, prof.tolist(), st.tolist()

    def h_inverse(self, eps, method=0, order=2, dynamic=True, eps_initial=1e-2, seed=42, max_iter=64):
        """oracle/_ref only: the reference's h_newton_schulz / h_hyperpower from
        scaled_identity_start -> (X, trace rows, final residual, converged)."""
        rows = np.zeros((512, 5))
        nr, fr, cv = i32(), f64(), i32()
        h = vp()
        _check(_lib.ora_h_inverse(self._h, int(method), int(order), int(dynamic), float(eps_initial), float(eps),
                                  int(seed), int(max_iter), C.byref(h), _p(rows), 512, C.byref(nr), C.byref(fr),
                                  C.byref(cv)))
        return H2(h, self.tree), rows[:min(nr.value, 512)], fr.value, bool(cv.value)

    def residual_norm(self, x):
        v = f64()
        _check(_lib.ora_residual_norm(self._h, x._h, C.byref(v)))
        return v.value

    def frobenius_norm(self):
        v = f64()
        _check(_lib.ora_frobenius_norm(self._h, C.byref(v)))
        return v.value


def peel_dense(tree, a, symmetric, eps=1e-4, b=16, p=10, max_rank=0, seed=42, norm_scale=0.0):
    """peel_construct(DenseOperator(a, symmetric), bt, cfg) (construction.hpp:300-382)."""
    a = np.asfortranarray(a, np.float64)
    h = vp()
    tot = i64()
    ls = np.zeros(64, np.int64)
    lr = np.zeros(64, np.int64)
    nl = i32()
    _check(_lib.ora_peel_dense(tree._h, _p(a), int(symmetric), float(eps), int(b), int(p), int(max_rank), int(seed),
                               float(norm_scale), C.byref(h), C.byref(tot), _p(ls), _p(lr), C.byref(nl)))
    return H2(h, tree), {"total": tot.value, "level_samples": ls[:nl.value].tolist(),
                         "level_max_rank": lr[:nl.value].tolist()}


def peel_dense_threads(tree, a, symmetric, eps=1e-4, seed=42, norm_scale=0.0, threads=1):
    """peel_construct over a dense black box applied on `threads` host threads ->
    (H2, stats, operator seconds)."""
    a = np.asfortranarray(a, np.float64)
    h = vp()
    tot = i64()
    ls = np.zeros(64, np.int64)
    lr = np.zeros(64, np.int64)
    nl = i32()
    ops = f64()
    _check(_lib.ora_peel_dense_threads(tree._h, _p(a), int(symmetric), float(eps), int(seed), float(norm_scale),
                                       int(threads), C.byref(h), C.byref(tot), _p(ls), _p(lr), C.byref(nl),
                                       C.byref(ops)))
    return H2(h, tree), {"total": tot.value, "level_samples": ls[:nl.value].tolist(),
                         "level_max_rank": lr[:nl.value].tolist()}, ops.value


def peel_h2(tree, src, eps=1e-4, seed=42, norm_scale=0.0):
    h = vp()
    tot = i64()
    _check(_lib.ora_peel_h2(tree._h, src._h, float(eps), int(seed), float(norm_scale), C.byref(h), C.byref(tot)))
    return H2(h, tree), tot.value


def sample_block_column(tree, a, symmetric, t, s, count, seed):
    """sample_block_column over DenseOperator(a) with a fresh mt19937_64(seed)."""
    a = np.asfortranarray(a, np.float64)
    ms = int(tree.end[s] - tree.begin[s])
    mt = int(tree.end[t] - tree.begin[t])
    om = np.empty((ms, count), order="F")
    y = np.empty((mt, count), order="F")
    _check(_lib.ora_sample_block_column(tree._h, _p(a), int(symmetric), int(t), int(s), int(count), int(seed),
                                        _p(om), _p(y)))
    return om, y


def adaptive_block_factorization(tree, a, symmetric, t, s, eps_block, b=16, p=10, max_rank=0, seed=42):
    """-> (u, v, rank, err_est, columns applied) (construction.hpp:156-198)."""
    a = np.asfortranarray(a, np.float64)
    ms = int(tree.end[s] - tree.begin[s])
    mt = int(tree.end[t] - tree.begin[t])
    kc = mt + b
    u = np.empty(mt * kc)
    v = np.empty(ms * kc)
    k, e, cols = i64(), f64(), i64()
    _check(_lib.ora_adaptive_block_factorization(tree._h, _p(a), int(symmetric), int(t), int(s), float(eps_block),
                                                 int(b), int(p), int(max_rank), int(seed), _p(u), _p(v), C.byref(k),
                                                 C.byref(e), C.byref(cols)))
    k = k.value
    return (u[:mt * k].reshape((mt, k), order="F"), v[:ms * k].reshape((ms, k), order="F"), k, e.value,
            cols.value)


def pnorm2_dense(a, symmetric):
    a = np.asfortranarray(a, np.float64)
    v, it = f64(), i32()
    _check(_lib.ora_pnorm2_dense(_p(a), a.shape[0], int(symmetric), C.byref(v), C.byref(it)))
    return v.value, it.value


def shuffle_indices(n, seed):
    """std::shuffle of 0..n-1 with std::mt19937_64(seed) (the reference's libstdc++ stream)."""
    out = np.empty(int(n), np.int64)
    _check(_lib.ora_shuffle(int(n), int(seed), _p(out)))
    return out


def gaussian(seed, r, c):
    """The reference's normal stream (fresh normal_distribution over mt19937_64(seed))."""
    out = np.empty((r, c), order="F")
    _check(_lib.ora_gaussian(int(seed), int(r), int(c), _p(out)))
    return out


def grid1d(n, a=0.0, b=1.0):
    """test_support.hpp:12-16."""
    return (a + (b - a) * np.arange(n) / max(n - 1, 1))[:, None]


def grid2d(nx, ny, a=0.0, b=1.0):
    """test_support.hpp:18-26 (row j*nx+i = (x_i, y_j))."""
    i = np.tile(np.arange(nx), ny)
    j = np.repeat(np.arange(ny), nx)
    return np.stack([a + (b - a) * i / max(nx - 1, 1), a + (b - a) * j / max(ny - 1, 1)], axis=1)


def grid3d(nx, ny, nz, a=0.0, b=1.0):
    i = np.tile(np.arange(nx), ny * nz)
    j = np.tile(np.repeat(np.arange(ny), nx), nz)
    k = np.repeat(np.arange(nz), nx * ny)
    s = lambda q, m: a + (b - a) * q / max(m - 1, 1)
    return np.stack([s(i, nx), s(j, ny), s(k, nz)], axis=1)


DIFF1D_DEFAULTS = dict(n=512, steps=512, T=30.0, tp=1.0, t0=0.0, amp=1000.0, alpha=3e-5, beta=1e-3, pad=0.5,
                       sources=(-0.5, 0.0, 0.5), receivers=8)


class Diff1D:
    """1D diffusion Hessian at the target density (oracle/diffusion1d.hpp,
    restating proj/include/h2/oracles/diffusion1d.hpp). Keys follow the
    reference registry overrides (registry.hpp:104-116)."""

    def __init__(self, **cfg):
        c = dict(DIFF1D_DEFAULTS)
        unknown = set(cfg) - set(c)
        if unknown:
            raise ValueError(f"unknown diffusion keys {sorted(unknown)}")
        c.update(cfg)
        self.cfg = c
        src = np.ascontiguousarray(c["sources"], np.float64)
        h = vp()
        _check(_lib.ora_diff1d_create(int(c["n"]), int(c["steps"]), float(c["T"]), float(c["tp"]), float(c["t0"]),
                                      float(c["amp"]), float(c["alpha"]), float(c["beta"]), float(c["pad"]),
                                      len(src), _p(src), int(c["receivers"]), C.byref(h)))
        self._h = h
        self.n = int(c["n"])

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.ora_diff1d_destroy(self._h)
            self._h = None

    def info(self):
        ns, npad, h, dt, m = i64(), i64(), f64(), f64(), i64()
        _check(_lib.ora_diff1d_info(self._h, C.byref(ns), C.byref(npad), C.byref(h), C.byref(dt), C.byref(m)))
        return dict(nstate=ns.value, npad=npad.value, h=h.value, dt=dt.value, marches=m.value)

    def hessvec(self, x, include_tv=True, threads=1):
        x = np.asarray(x, np.float64)
        vec = x.ndim == 1
        xf = np.asfortranarray(x[:, None] if vec else x)
        y = np.empty_like(xf, order="F")
        _check(_lib.ora_diff1d_hessvec(self._h, xf.shape[1], _p(xf), _p(y), int(include_tv), int(threads)))
        return y[:, 0] if vec else y

    def state(self, source):
        inf = self.info()
        u = np.empty((inf["nstate"], int(self.cfg["steps"]) + 1), order="F")
        _check(_lib.ora_diff1d_state(self._h, int(source), _p(u)))
        return u

    def peel(self, tree, eps=1e-6, seed=42, include_tv=True, threads=1):
        """peel_construct(hessian_operator(include_tv), bt, {eps, seed}) on the CPU:
        returns (H2, total samples, seconds spent in operator applies)."""
        h, tot, ops = vp(), i64(), f64()
        ls = np.zeros(64, np.int64)
        lr = np.zeros(64, np.int64)
        nl = i32()
        _check(_lib.ora_peel_diff1d(tree._h, self._h, int(include_tv), float(eps), int(seed), int(threads),
                                    C.byref(h), C.byref(tot), C.byref(ops), _p(ls), _p(lr), C.byref(nl)))
        self.last_stats = {"total": tot.value, "level_samples": ls[:nl.value].tolist(),
                           "level_max_rank": lr[:nl.value].tolist()}
        return H2(h, tree), tot.value, ops.value

    def points(self):
        """Grid1D(-1, 1, n).points() (grid.hpp:10-24)."""
        h = 2.0 / (self.n - 1)
        return (-1.0 + h * np.arange(self.n))[:, None]
