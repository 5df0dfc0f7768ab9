"""Python mirror of the reference H^2 API for the hot path, over the C ABI.

Names, argument meaning and error behaviour follow the reference headers:
  build_cluster_tree / ClusterTree     cluster_tree.hpp:18-188
  build_block_tree / BlockTree         block_tree.hpp:18-124
  H2Matrix (zero, matvec, ...)         h2_matrix.hpp:40-306
Matrices live on the B200 (HBM); host numpy arrays are accepted where the
reference takes an Eigen Matrix by value, device torch tensors where a
caller wants to stay on the GPU.
"""
import ctypes as C
import dataclasses
import enum

import numpy as np

from ._lib import H, check, lib


def col_major_geom(t):
    """(columns, leading dimension) of a column-major n x b tensor or a 1-D vector.

    A contiguous (n, 1) tensor has strides (1, 1); its leading dimension is n."""
    if t.dim() == 1:
        return 1, t.shape[0]
    if t.dim() != 2:
        raise ValueError("hgemv: tensors must be 1-D or 2-D")
    if t.shape[1] > 1 and t.stride(0) != 1:
        raise ValueError("hgemv: tensors must be column-major (stride(0) == 1)")
    if t.shape[1] == 1:
        return 1, max(t.stride(1), t.shape[0])
    return t.shape[1], t.stride(1)


class Admissibility(enum.IntEnum):
    strong = 0
    weak = 1


class Ordering(enum.IntEnum):
    user = 0
    internal = 1


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class ClusterTree:
    """KD cluster tree (cluster_tree.hpp:18-188); built in C++ on the host, or level by level on
    the device (device=True; the same tree bit for bit)."""

    def __init__(self, points, leaf_size, device=False):
        pts = np.asarray(points, dtype=np.float64)
        if pts.ndim == 1:
            pts = pts[:, None]
        if pts.shape[0] < 1:
            raise ValueError("PointSet: need at least one point")
        n, d = pts.shape
        coords = np.asfortranarray(pts)
        h = H()
        if device:
            check(lib.h2c_cluster_tree_create_device(coords.ctypes.data_as(C.c_void_p), n, d, int(leaf_size), None,
                                                     C.byref(h)))
        else:
            check(lib.h2c_cluster_tree_create(coords.ctypes.data_as(C.c_void_p), n, d, int(leaf_size), C.byref(h)))
        self._load(h, leaf_size)

    @classmethod
    def from_handle(cls, h, leaf_size=0):
        obj = cls.__new__(cls)
        obj._load(h, leaf_size)
        return obj

    def _load(self, h, leaf_size):
        self._h = h
        nn_, dim_, depth_, nodes_, leaves_ = C.c_int64(), C.c_int(), C.c_int(), C.c_int(), C.c_int()
        check(lib.h2c_cluster_tree_info(h, C.byref(nn_), C.byref(dim_), C.byref(depth_), C.byref(nodes_),
                                        C.byref(leaves_)))
        self.n, self.dim, self.depth, self.num_nodes = nn_.value, dim_.value, depth_.value, nodes_.value
        nn = self.num_nodes
        self.begin = np.empty(nn, np.int64)
        self.end = np.empty(nn, np.int64)
        self.level = np.empty(nn, np.int32)
        self.parent = np.empty(nn, np.int32)
        self.child0 = np.empty(nn, np.int32)
        self.child1 = np.empty(nn, np.int32)
        self.box_lo = np.empty((nn, 3))
        self.box_hi = np.empty((nn, 3))
        check(lib.h2c_cluster_tree_nodes(h, _ptr(self.begin), _ptr(self.end), _ptr(self.level), _ptr(self.parent),
                                         _ptr(self.child0), _ptr(self.child1), _ptr(self.box_lo),
                                         _ptr(self.box_hi)))
        self.perm = np.empty(self.n, np.int64)
        check(lib.h2c_cluster_tree_perm(h, _ptr(self.perm)))
        self.inv_perm = np.empty_like(self.perm)
        self.inv_perm[self.perm] = np.arange(self.n)
        self.leaves = np.nonzero(self.child0 < 0)[0].astype(np.int32)
        self.leaf_size = int(leaf_size) if leaf_size else int((self.end[self.leaves] - self.begin[self.leaves]).max())

    def __del__(self):
        if getattr(self, "_h", None):
            lib.h2c_cluster_tree_destroy(self._h)
            self._h = None

    def size(self, v):
        return int(self.end[v] - self.begin[v])

    def is_leaf(self, v):
        return self.child0[v] < 0

    def level_nodes(self, l):
        return np.nonzero(self.level == l)[0]

    def max_leaf_size(self):
        return int((self.end[self.leaves] - self.begin[self.leaves]).max())

    # cluster_tree.hpp:82-92 (host helpers)
    def to_internal(self, x_user):
        return np.asarray(x_user)[self.perm]

    def to_user(self, x_internal):
        out = np.empty_like(x_internal)
        out[self.perm] = x_internal
        return out


def build_cluster_tree(points, leaf_size, device=False):
    """build_cluster_tree (cluster_tree.hpp:186-188); device=True builds it on the B200."""
    return ClusterTree(points, leaf_size, device)


class BlockTree:
    """Block tree over (ct, ct) (block_tree.hpp:41-118)."""

    def __init__(self, ct, eta=1.0, mode=Admissibility.strong):
        h = H()
        check(lib.h2c_block_tree_create(ct._h, float(eta), int(mode == Admissibility.weak), C.byref(h)))
        self._load(h, ct, eta, mode)

    @classmethod
    def from_handle(cls, h):
        """Wrap a block tree handle returned by the library (e.g. by read_h2_file)."""
        ch = H()
        check(lib.h2c_block_tree_cluster_tree(h, C.byref(ch)))
        eta, weak = C.c_double(), C.c_int()
        check(lib.h2c_block_tree_params(h, C.byref(eta), C.byref(weak)))
        obj = cls.__new__(cls)
        obj._load(h, ClusterTree.from_handle(ch), eta.value, Admissibility.weak if weak.value else Admissibility.strong)
        return obj

    def _load(self, h, ct, eta, mode):
        self._h = h
        self.tree = ct
        self.eta = float(eta)
        self.mode = Admissibility(mode)
        nn, na, nd, ml = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        check(lib.h2c_block_tree_info(h, C.byref(nn), C.byref(na), C.byref(nd), C.byref(ml)))
        self.num_nodes, self.max_level = nn.value, ml.value
        n = nn.value
        self.row = np.empty(n, np.int32)
        self.col = np.empty(n, np.int32)
        self.blevel = np.empty(n, np.int32)
        self.bparent = np.empty(n, np.int32)
        self.tag = np.empty(n, np.int32)
        check(lib.h2c_block_tree_nodes(h, _ptr(self.row), _ptr(self.col), _ptr(self.blevel), _ptr(self.bparent),
                                       _ptr(self.tag)))
        self.admissible_leaves = np.empty(na.value, np.int32)
        self.dense_leaves = np.empty(nd.value, np.int32)
        check(lib.h2c_block_tree_leaves(h, _ptr(self.admissible_leaves), _ptr(self.dense_leaves)))

    def __del__(self):
        if getattr(self, "_h", None):
            lib.h2c_block_tree_destroy(self._h)
            self._h = None

    def n(self):
        return self.tree.n

    def canonical(self, b):
        return self.row[b] <= self.col[b]


def build_block_tree(rows, cols, eta, mode=Admissibility.strong):
    if rows is not cols:
        raise ValueError("block tree: the B200 path requires identical row and column trees")
    return BlockTree(rows, eta, mode)


_PARTS = ("U", "E", "V", "F", "S", "D")


@dataclasses.dataclass
class StorageReport:   # h2_matrix.hpp:25-31
    dense_reals: int
    leaf_basis_reals: int
    transfer_reals: int
    coupling_reals: int

    def total(self):
        return self.dense_reals + self.leaf_basis_reals + self.transfer_reals + self.coupling_reals


@dataclasses.dataclass
class ValidationReport:   # h2_matrix.hpp:33-38
    violations: list
    level_max_rank: list
    storage: StorageReport

    def ok(self):
        return not self.violations


class H2Matrix:
    """Device-resident H^2 matrix (h2_matrix.hpp:40-306)."""

    def __init__(self, handle, blocks):
        self._h = handle
        self.blocks = blocks
        self.tree = blocks.tree

    def __del__(self):
        if getattr(self, "_h", None):
            lib.h2c_matrix_destroy(self._h)
            self._h = None

    # ---- factories -------------------------------------------------------
    @staticmethod
    def zero(bt, symmetric):
        """H2Matrix::zero (h2_matrix.hpp:53-75)."""
        h = H()
        check(lib.h2c_matrix_create(bt._h, int(bool(symmetric)), None, None, C.byref(h)))
        return H2Matrix(h, bt)

    @staticmethod
    def from_packed(bt, symmetric, row_ranks, col_ranks, parts, orthonormal=False):
        """Build from packed payloads (layout of include/h2c.h)."""
        rr = np.ascontiguousarray(row_ranks, np.int32)
        cr = None if symmetric else np.ascontiguousarray(col_ranks, np.int32)
        h = H()
        check(lib.h2c_matrix_create(bt._h, int(bool(symmetric)), _ptr(rr), _ptr(cr), C.byref(h)))
        m = H2Matrix(h, bt)
        sizes = m.packed_sizes()
        arrs = []
        for name, sz in zip(_PARTS, sizes):
            a = parts.get(name) if isinstance(parts, dict) else None
            if a is None:
                arrs.append(None)
                continue
            a = _f64(a).ravel()
            if a.size != sz:
                raise ValueError(f"packed part {name}: {a.size} values, expected {sz}")
            arrs.append(a)
        check(lib.h2c_matrix_upload(h, *[_ptr(a) for a in arrs]))
        check(lib.h2c_matrix_set_orthonormal(h, int(bool(orthonormal))))
        return m

    @staticmethod
    def kernel(bt, points, kind="gaussian", ell=0.1, rank=32, shard=None):
        """Symmetric kernel matrix generated on the device (benchmark inputs).
        shard=(nranks, rank): only that row-subtree shard's payload (sharded hgemv only)."""
        kinds = {"exponential": 0, "gaussian": 1, "matern32": 2}
        pts = np.asfortranarray(np.asarray(points, np.float64).reshape(bt.tree.n, -1))
        h = H()
        if shard is None:
            check(lib.h2c_matrix_kernel(bt._h, pts.ctypes.data_as(C.c_void_p), kinds[kind], float(ell), int(rank),
                                        C.byref(h)))
        else:
            check(lib.h2c_matrix_kernel_sharded(bt._h, pts.ctypes.data_as(C.c_void_p), kinds[kind], float(ell),
                                                int(rank), int(shard[0]), int(shard[1]), C.byref(h)))
        return H2Matrix(h, bt)

    # ---- properties ------------------------------------------------------
    def _info(self):
        n, s, o = C.c_int64(), C.c_int(), C.c_int()
        check(lib.h2c_matrix_info(self._h, C.byref(n), C.byref(s), C.byref(o)))
        return n.value, bool(s.value), bool(o.value)

    def n(self):
        return self._info()[0]

    @property
    def symmetric(self):
        return self._info()[1]

    @property
    def orthonormal(self):
        return self._info()[2]

    def packed_sizes(self):
        s = np.zeros(6, np.int64)
        check(lib.h2c_matrix_sizes(self._h, _ptr(s)))
        return [int(x) for x in s]

    def ranks(self):
        nn = self.tree.num_nodes
        r = np.empty(nn, np.int32)
        c = np.empty(nn, np.int32)
        check(lib.h2c_matrix_ranks(self._h, _ptr(r), _ptr(c)))
        return r, c

    def rank_profile(self):
        """h2_matrix.hpp:190-195."""
        r, _ = self.ranks()
        prof = np.zeros(self.tree.depth + 1, np.int64)
        np.maximum.at(prof, self.tree.level, r)
        return prof

    def download(self):
        sizes = self.packed_sizes()
        arrs = [np.empty(s, np.float64) for s in sizes]
        check(lib.h2c_matrix_download(self._h, *[_ptr(a) for a in arrs]))
        return dict(zip(_PARTS, arrs))

    # ---- hgemv -----------------------------------------------------------
    def _host(self, x, transpose, ordering):
        x = np.asarray(x, np.float64)
        vec = x.ndim == 1
        xm = x[:, None] if vec else x
        if xm.shape[0] != self.tree.n:
            raise ValueError("matvec: dimension mismatch")
        if xm.shape[1] < 1:
            raise ValueError("matvec: need at least one column")
        xf = np.asfortranarray(xm)
        y = np.empty(xf.shape, np.float64, order="F")
        check(lib.h2c_matvec_host(self._h, int(transpose), int(ordering), xf.shape[0], xf.shape[1],
                                  xf.ctypes.data_as(C.c_void_p), y.ctypes.data_as(C.c_void_p)))
        return y[:, 0] if vec else y

    def matvec(self, x):
        """H2Matrix::matvec, user ordering (h2_matrix.hpp:112-115)."""
        return self._host(x, False, Ordering.user)

    def matvec_transpose(self, x):
        return self._host(x, True, Ordering.user)

    def matvec_internal(self, x):
        return self._host(x, False, Ordering.internal)

    def matvec_transpose_internal(self, x):
        return self._host(x, True, Ordering.internal)

    def hgemv(self, x, y, transpose=False, ordering=Ordering.user, alpha=1.0, beta=0.0, stream=None):
        """Device path: y = alpha op(H) x + beta y on CUDA tensors (column-major
        n x b, i.e. stride(0) == 1, or 1-D)."""
        geom = col_major_geom
        if x.dtype != y.dtype or str(x.dtype) != "torch.float64":
            raise ValueError("hgemv: float64 tensors required")
        b, ldx = geom(x)
        b2, ldy = geom(y)
        if b != b2 or x.shape[0] != y.shape[0]:
            raise ValueError("matvec: dimension mismatch")
        s = stream.cuda_stream if stream is not None else None
        check(lib.h2c_hgemv(self._h, int(transpose), int(ordering), x.shape[0], b, x.data_ptr(), ldx,
                            y.data_ptr(), ldy, float(alpha), float(beta), s))

    def to_dense(self, cap=8192):
        """H2Matrix::to_dense(cap) (h2_matrix.hpp:128-163): n x n, user ordering
        (computed on the device as the operator applied to identity panels)."""
        n = self.n()
        a = np.empty((n, n), order="F")
        check(lib.h2c_to_dense(self._h, int(cap), _ptr(a)))
        return a

    def validate(self, ortho_cap=4096):
        """H2Matrix::validate(ortho_cap) (h2_matrix.hpp:308-404) -> ValidationReport."""
        nv, nl = C.c_int(), C.c_int()
        buf = C.create_string_buffer(8192)
        prof = np.zeros(128, np.int64)
        st = np.zeros(4, np.int64)
        check(lib.h2c_validate(self._h, int(ortho_cap), C.byref(nv), buf, len(buf), _ptr(prof), len(prof),
                               C.byref(nl), _ptr(st)))
        msgs = [m for m in buf.value.decode().split("\n") if m] if nv.value else []
        return ValidationReport(msgs, prof[:nl.value].tolist(),
                                StorageReport(int(st[0]), int(st[1]), int(st[2]), int(st[3])))

    def storage(self):
        """H2Matrix::storage() (h2_matrix.hpp:167-187)."""
        return self.validate(ortho_cap=0).storage

    def add_diagonal(self, value):
        """In place H <- H + value I (diagonal dense leaves)."""
        check(lib.h2c_matrix_add_diagonal(self._h, float(value)))

    def launches(self, b, transpose=False):
        n = C.c_int()
        check(lib.h2c_hgemv_launches(self._h, int(transpose), int(b), C.byref(n)))
        return n.value


# ---- H2M1 container (serialize.hpp:110-322), byte-compatible with the reference ----

def serialize(m):
    """Bytes of the H2M1 container (serialize.hpp:110-182)."""
    n = C.c_int64()
    check(lib.h2c_serialize_size(m._h, C.byref(n)))
    buf = (C.c_char * n.value)()
    check(lib.h2c_serialize(m._h, buf, n.value))
    return bytes(buf)


def deserialize(data):
    """H2Matrix from H2M1 bytes (serialize.hpp:184-308); the block tree is rebuilt."""
    data = bytes(data)
    bt, h = H(), H()
    check(lib.h2c_deserialize(data, len(data), C.byref(bt), C.byref(h)))
    return H2Matrix(h, BlockTree.from_handle(bt))


def write_h2_file(m, path):
    check(lib.h2c_write_h2_file(m._h, str(path).encode()))


def read_h2_file(path):
    bt, h = H(), H()
    check(lib.h2c_read_h2_file(str(path).encode(), C.byref(bt), C.byref(h)))
    return H2Matrix(h, BlockTree.from_handle(bt))
