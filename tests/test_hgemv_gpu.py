"""hgemv parity: the B200 path (through the C ABI) vs the CPU oracle on the
reference's own fixture (random_h2, test_support.hpp:38-70) and on generated
kernel matrices. Tolerance: relative Frobenius error <= 1e-12,
the bound of test_core.cpp:40-53."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2003_10173_b200 import Admissibility, H2Matrix, build_block_tree, build_cluster_tree

pytestmark = pytest.mark.gpu
TOL = 1e-12


def rel(a, b):
    d = np.linalg.norm(b)
    return np.linalg.norm(a - b) / d if d else np.linalg.norm(a)


def pair(pts, leaf, weak, sym, kmax, seed):
    ref = O.Tree(pts, leaf, 1.0, weak)
    ora = O.H2.random(ref, sym, kmax, seed)
    ct = build_cluster_tree(pts, leaf)
    bt = build_block_tree(ct, ct, 1.0, Admissibility.weak if weak else Admissibility.strong)
    rr, cr = ora.ranks()
    m = H2Matrix.from_packed(bt, sym, rr, cr, ora.export())
    return ora, m, bt


TREES = {
    "1d-weak-96-8": (O.grid1d(96, -1, 1), 8, True),
    "1d-strong-70-6": (O.grid1d(70, -1, 1), 6, False),
    "2d-12-16": (O.grid2d(12, 12), 16, False),
    "rand3d-300-12": (O.gaussian(9, 300, 3), 12, False),
    "2d-64-64": (O.grid2d(64, 64), 64, False),
}


@pytest.mark.parametrize("tree", list(TREES))
@pytest.mark.parametrize("sym", [True, False])
@pytest.mark.parametrize("kmax", [4, 40])
def test_hgemv_matches_oracle(cuda, tree, sym, kmax):
    pts, leaf, weak = TREES[tree]
    kmax = min(kmax, leaf)
    ora, m, _ = pair(pts, leaf, weak, sym, kmax, seed=2)
    n = pts.shape[0]
    for b in (1, 5, 16, 32, 33, 64, 70):
        x = O.gaussian(100 + b, n, b)
        for transpose in (False, True):
            for ordering in (0, 1):
                y_ref = ora.matvec(x, transpose, ordering)
                y = m._host(x, transpose, ordering)
                assert rel(y, y_ref) <= TOL, (tree, sym, b, transpose, ordering, rel(y, y_ref))


def test_hgemv_large_ranks_and_leaves(cuda):
    # ranks and leaf sizes above one 64-row tile exercise the row tiling
    pts = O.gaussian(21, 2000, 2)
    ora, m, _ = pair(pts, 150, False, True, 90, seed=5)
    x = O.gaussian(22, 2000, 40)
    assert rel(m.matvec(x), ora.matvec(x)) <= TOL


def test_device_path_alpha_beta_and_strides(cuda):
    import torch
    pts = O.grid2d(40, 40)
    ora, m, _ = pair(pts, 32, False, True, 8, seed=3)
    n, b = 1600, 7
    x = O.gaussian(31, n, b)
    y0 = O.gaussian(32, n, b)
    # column-major device tensors with padded leading dimension
    X = torch.zeros(b, n + 3, dtype=torch.float64, device=cuda)
    Y = torch.zeros(b, n + 5, dtype=torch.float64, device=cuda)
    X[:, :n] = torch.from_numpy(x.T.copy())
    Y[:, :n] = torch.from_numpy(y0.T.copy())
    xv, yv = X[:, :n].T, Y[:, :n].T
    m.hgemv(xv, yv, alpha=-0.5, beta=2.0)
    torch.cuda.synchronize()
    expect = -0.5 * ora.matvec(x) + 2.0 * y0
    assert rel(yv.cpu().numpy(), expect) <= TOL
    assert torch.all(Y[:, n:] == 0)   # padding untouched


def test_residual_form(cuda):
    # y <- op(x) - H x, the HARA residual (construction.hpp:207-211) fused as alpha=-1, beta=1
    import torch
    pts = O.grid1d(256, -1, 1)
    ora, m, _ = pair(pts, 16, True, True, 6, seed=4)
    x = O.gaussian(41, 256, 16)
    opx = O.gaussian(42, 256, 16)
    X = torch.from_numpy(np.asfortranarray(x)).to(cuda).T.contiguous().T
    Y = torch.from_numpy(np.asfortranarray(opx)).to(cuda).T.contiguous().T
    m.hgemv(X, Y, alpha=-1.0, beta=1.0)
    assert rel(Y.cpu().numpy(), opx - ora.matvec(x)) <= TOL


def test_zero_and_rank_zero_nodes(cuda):
    pts = O.grid1d(128, -1, 1)
    ct = build_cluster_tree(pts, 16)
    bt = build_block_tree(ct, ct, 1.0, Admissibility.weak)
    z = H2Matrix.zero(bt, True)
    x = O.gaussian(1, 128, 3)
    assert np.all(z.matvec(x) == 0)
    # ranks 0 on a subset of nodes
    ref = O.Tree(pts, 16, 1.0, True)
    ora = O.H2.random(ref, False, 3, 9)
    rr, cr = ora.ranks()
    parts = ora.export()
    m = H2Matrix.from_packed(bt, False, rr, cr, parts)
    assert rel(m.matvec(x), ora.matvec(x)) <= TOL


def test_dimension_errors(cuda):
    pts = O.grid1d(64)
    ora, m, _ = pair(pts, 8, True, True, 3, seed=1)
    with pytest.raises(ValueError):
        m.matvec(np.zeros((63, 2)))
    with pytest.raises(ValueError):
        m.matvec(np.zeros((64, 0)))


def test_kernel_matrix_matches_oracle_on_same_payload(cuda):
    # device-generated Gaussian-kernel H^2 (bench input) downloaded into the oracle
    pts = O.grid2d(96, 96)
    ct = build_cluster_tree(pts, 64)
    bt = build_block_tree(ct, ct, 1.0)
    m = H2Matrix.kernel(bt, pts, "gaussian", 0.1, 32)
    ref = O.Tree(pts, 64, 1.0, False)
    rr, _ = m.ranks()
    ora = O.H2.from_packed(ref, True, rr, None, m.download())
    x = O.gaussian(7, pts.shape[0], 32)
    assert rel(m.matvec(x), ora.matvec(x)) <= TOL
    assert rel(m.matvec(x[:, :1]), ora.matvec(x[:, :1])) <= TOL


@pytest.mark.parametrize("kind,ell", [("gaussian", 0.1), ("exponential", 0.2), ("matern32", 0.1)])
def test_kernel_matrix_approximates_dense_kernel(cuda, kind, ell):
    # the Chebyshev-interpolation generator is a faithful kernel approximation
    pts = O.grid2d(48, 48)
    ct = build_cluster_tree(pts, 64)
    bt = build_block_tree(ct, ct, 1.0)
    m = H2Matrix.kernel(bt, pts, kind, ell, 32)
    r = np.sqrt(((pts[:, None, :] - pts[None, :, :]) ** 2).sum(-1))
    K = {"gaussian": np.exp(-(r / ell) ** 2), "exponential": np.exp(-r / ell),
         "matern32": (1 + np.sqrt(3) * r / ell) * np.exp(-np.sqrt(3) * r / ell)}[kind]
    x = O.gaussian(8, pts.shape[0], 4)
    assert rel(m.matvec(x), K @ x) < 1e-3


@pytest.mark.parametrize("b", [1, 2])
def test_few_vector_dense_overlap_bitwise(cuda, b):
    # symmetric b <= 2 path: the dense near-field block pass runs on a least-priority
    # stream beside the sweep chain (h2b_tune 8). Same kernels, same slot sums in a
    # fixed order, so eager and graph-replayed calls equal the serial path bit for bit
    import ctypes as C

    import torch
    from paper_2003_10173_b200._lib import lib
    lib.h2b_tune.argtypes = [C.c_int, C.c_int]
    lib.h2b_tune.restype = C.c_int
    pts = O.grid2d(48, 48)
    ora, m, _ = pair(pts, 16, False, True, 8, seed=9)
    n = pts.shape[0]
    x = O.gaussian(51, n, b)
    y0 = O.gaussian(52, n, b)
    X = torch.from_numpy(x.T.copy()).to(cuda).T
    out, keep = {}, []
    try:
        for ov in (0, 1):
            assert lib.h2b_tune(8, ov) == 0
            runs = []
            Y = torch.from_numpy(y0.T.copy()).to(cuda).T
            keep.append(Y)   # a new y pointer per setting: no graph replayed across settings
            for _ in range(4):   # 1st eager, 2nd captured, then graph replays
                Y.copy_(torch.from_numpy(y0.T.copy()).to(cuda).T)
                m.hgemv(X, Y, alpha=-0.75, beta=0.5)
                runs.append(Y.clone())
            torch.cuda.synchronize()
            for r in runs[1:]:
                assert torch.equal(r, runs[0])
            out[ov] = runs[0]
    finally:
        lib.h2b_tune(8, 1)
    assert torch.equal(out[0], out[1])
    expect = -0.75 * ora.matvec(x) + 0.5 * y0
    assert rel(out[1].cpu().numpy(), expect) <= TOL


def test_graph_cache_survives_workspace_resize(cuda):
    """b=1 twice (second call captures a graph), then b=64 on
    the same workspace (grows and frees its buffers), then b=1 again with the
    same x / y pointers must not replay the stale graph."""
    import torch
    pts = O.grid2d(48, 48)
    ora, m, _ = pair(pts, 32, False, True, 8, seed=4)
    n = pts.shape[0]
    X = torch.zeros(64, n, dtype=torch.float64, device=cuda)
    Y = torch.zeros(64, n, dtype=torch.float64, device=cuda)
    x64 = O.gaussian(41, n, 64)
    X[:, :] = torch.from_numpy(x64.T.copy())
    x1, y1 = X[:1].T, Y[:1].T          # (n, 1) views sharing the first column's storage
    xa, ya = X.T, Y.T
    for b, xv, yv in ((1, x1, y1), (1, x1, y1), (64, xa, ya), (1, x1, y1), (1, x1, y1)):
        yv.zero_()
        m.hgemv(xv, yv)
        torch.cuda.synchronize()
        expect = ora.matvec(x64[:, :b])
        assert rel(yv.cpu().numpy(), expect) <= TOL, b


def test_column_vector_tensor_leading_dimension(cuda):
    """A contiguous (n, 1) tensor has strides (1, 1); its leading dimension is n."""
    import torch
    pts = O.grid2d(20, 20)
    ora, m, _ = pair(pts, 16, False, True, 6, seed=6)
    n = pts.shape[0]
    x = O.gaussian(43, n, 1)
    xt = torch.from_numpy(x.copy()).to(cuda)
    assert xt.stride() == (1, 1)
    yt = torch.zeros(n, 1, dtype=torch.float64, device=cuda)
    m.hgemv(xt, yt)
    torch.cuda.synchronize()
    assert rel(yt.cpu().numpy(), ora.matvec(x)) <= TOL


def test_knob_toggle_does_not_replay_stale_graph(cuda):
    """the graph key includes the runtime knobs (dense overlap)."""
    import torch
    from paper_2003_10173_b200._lib import lib
    pts = O.grid2d(48, 48)
    ora, m, _ = pair(pts, 32, False, True, 8, seed=8)
    n = pts.shape[0]
    x = O.gaussian(44, n, 1)
    xt = torch.from_numpy(x.copy()).to(cuda)
    yt = torch.zeros(n, 1, dtype=torch.float64, device=cuda)
    outs = []
    try:
        for knob in (1, 1, 0, 0, 1):
            lib.h2b_tune(8, knob)
            yt.zero_()
            m.hgemv(xt, yt)
            torch.cuda.synchronize()
            outs.append(yt.cpu().numpy().copy())
    finally:
        lib.h2b_tune(8, 1)
    for o in outs:
        assert rel(o, ora.matvec(x)) <= TOL
        assert np.array_equal(o, outs[0])


_REF = __import__("os").path.join(__import__("os").path.dirname(__import__("os").path.dirname(
    __import__("os").path.abspath(__file__))), "oracle", "_ref", "libh2ref.so")


@pytest.mark.skipif(not __import__("os").path.exists(_REF), reason="oracle/_ref not built")
@pytest.mark.parametrize("tree", ["1d-weak-96-8", "2d-12-16", "rand3d-300-12", "2d-64-64"])
@pytest.mark.parametrize("sym", [True, False])
def test_hgemv_matches_reference_build(cuda, tree, sym):
    """The B200 hgemv against H2Matrix::matvec / matvec_transpose(_internal)
    executed by the reference's OWN code (h2_matrix.hpp:108-124, 246-305 compiled
    unchanged into oracle/_ref) on the reference's own fixture: the tree and the
    random_h2 payloads are built by the reference and uploaded as they are."""
    from oracle import pyref as R
    pts, leaf, weak = TREES[tree]
    rt = R.Tree(pts, leaf, 1.0, weak)
    rh = R.H2.random(rt, sym, min(12, leaf), 77)
    ct = build_cluster_tree(pts, leaf)
    bt = build_block_tree(ct, ct, 1.0, Admissibility.weak if weak else Admissibility.strong)
    rr, cr = rh.ranks()
    m = H2Matrix.from_packed(bt, sym, rr, cr, rh.export())
    n = pts.shape[0]
    for b in (1, 2, 16, 32, 64):
        x = O.gaussian(300 + b, n, b)
        for transpose in (False, True):
            for ordering in (0, 1):
                assert rel(m._host(x, transpose, ordering), rh.matvec(x, transpose, ordering)) <= TOL


@pytest.mark.parametrize("b", [1, 2])
def test_bulk_async_dense_pass_bitwise(cuda, b):
    """The few-vector dense block pass staged through the bulk-async smem ring
    (sym_tma64_kernel, used when there are >= 32 blocks per SM) is bitwise the
    register-streaming kernel, and both match the oracle."""
    import torch
    from paper_2003_10173_b200._lib import lib
    pts = O.grid2d(256, 256)
    ct = build_cluster_tree(pts, 64)
    bt = build_block_tree(ct, ct, 1.0)
    m = H2Matrix.kernel(bt, pts, "gaussian", 0.1, 16)
    n = pts.shape[0]
    ref = O.H2.from_packed(O.Tree(pts, 64), True, m.ranks()[0], None, m.download())
    x = O.gaussian(90 + b, n, b)
    xt = torch.from_numpy(x.T.copy()).to(cuda).t()
    outs = []
    try:
        for knob in (0, 1):
            lib.h2b_tune(10, knob)
            yt = torch.zeros(b, n, dtype=torch.float64, device=cuda).t()
            m.hgemv(xt, yt)
            torch.cuda.synchronize()
            outs.append(yt.cpu().numpy().copy())
    finally:
        lib.h2b_tune(10, 1)
    assert np.array_equal(outs[0], outs[1])
    assert rel(outs[1], ref.matvec(x)) <= TOL


@pytest.mark.parametrize("b", [3, 32])
def test_split_near_field_matches(cuda, b):
    """Stage-5 split on one GPU (near field into blocked partial sums on the side
    stream, added in the leaf-expansion epilogue) against the unsplit plan."""
    import torch
    from paper_2003_10173_b200._lib import lib
    pts = O.grid2d(64, 64)
    ora, m, _ = pair(pts, 32, False, True, 12, seed=14)
    n = pts.shape[0]
    x = O.gaussian(95, n, b)
    xt = torch.from_numpy(x.T.copy()).to(cuda).t()
    outs = []
    try:
        for knob in (0, 1, 1):
            lib.h2b_tune(9, knob)
            yt = torch.zeros(b, n, dtype=torch.float64, device=cuda).t()
            m.hgemv(xt, yt)
            torch.cuda.synchronize()
            outs.append(yt.cpu().numpy().copy())
    finally:
        lib.h2b_tune(9, 0)
    expect = ora.matvec(x)
    for o in outs:
        assert rel(o, expect) <= TOL
    assert np.array_equal(outs[1], outs[2])   # deterministic with the side stream


@pytest.mark.parametrize("sym,b,transpose", [(True, 3, False), (True, 32, False), (False, 32, True), (False, 1, False)])
def test_top_chain_matches(cuda, sym, b, transpose):
    """General plans with a top chain (h2b_tune 12: the levels with fewer nodes than the
    threshold run with their couplings on a side stream beside the deep coupling) are
    bitwise the single-stream plan, eagerly and through the captured graph."""
    import torch
    from paper_2003_10173_b200._lib import lib
    pts = O.grid2d(64, 64)
    ora, m, _ = pair(pts, 32, False, sym, 12, seed=21)
    n = pts.shape[0]
    x = O.gaussian(97, n, b)
    xt = torch.from_numpy(x.T.copy()).to(cuda).t()
    outs = []
    try:
        for knob in (0, 8, 8, 8, 8):   # eager, eager, captured, replayed
            lib.h2b_tune(12, knob)
            yt = torch.zeros(b, n, dtype=torch.float64, device=cuda).t()
            m.hgemv(xt, yt, transpose=transpose)
            torch.cuda.synchronize()
            outs.append(yt.cpu().numpy().copy())
    finally:
        lib.h2b_tune(12, 4096)
    expect = ora.matvec(x, transpose=transpose)
    assert rel(outs[0], expect) <= TOL
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


@pytest.mark.parametrize("b", [1, 32])
def test_kernel_launch_accounting(cuda, b):
    """h2b_kernel_launches counts every launch site, and a replayed CUDA graph adds its kernel
    nodes (captured launches are not counted twice): after a first call (eager, and the plan
    build's own U E product launch), 5 calls (1 captured and replayed, 4 replays) launch exactly
    5 x m.launches(b) kernels."""
    import ctypes as C
    import torch
    from paper_2003_10173_b200._lib import lib
    lib.h2b_kernel_launches.restype = C.c_longlong
    lib.h2b_kernel_launches.argtypes = [C.c_int]
    pts = O.grid2d(64, 64)
    ct = build_cluster_tree(pts, 32)
    bt = build_block_tree(ct, ct, 1.0)
    m = H2Matrix.kernel(bt, pts, "gaussian", 0.1, 12)
    n = pts.shape[0]
    xt = torch.randn(b, n, dtype=torch.float64, device=cuda).t()
    yt = torch.zeros(b, n, dtype=torch.float64, device=cuda).t()
    m.hgemv(xt, yt)
    torch.cuda.synchronize()
    lib.h2b_kernel_launches(1)
    for _ in range(5):
        m.hgemv(xt, yt)
    torch.cuda.synchronize()
    assert lib.h2b_kernel_launches(0) == 5 * m.launches(b)


@pytest.mark.parametrize("b", [1, 2])
@pytest.mark.parametrize("alpha,beta", [(-1.0, 1.0), (2.5, -0.5)])
def test_few_vector_alpha_beta_through_graph(cuda, b, alpha, beta):
    """The few-vector symmetric path (dense slot sums into blocked partial sums, added by the leaf
    expansion's epilogue before alpha / beta and the user-order scatter) with general alpha, beta,
    eagerly and through the captured-graph replays (4 identical calls)."""
    import torch
    pts = O.grid2d(48, 48)
    ora, m, _ = pair(pts, 24, False, True, 10, seed=31)
    n = pts.shape[0]
    x = O.gaussian(51 + b, n, b)
    y0 = O.gaussian(61 + b, n, b)
    expect = alpha * ora.matvec(x) + beta * y0
    xt = torch.from_numpy(x.T.copy()).to(cuda).t()
    for _ in range(4):
        yt = torch.from_numpy(y0.T.copy()).to(cuda).t()
        m.hgemv(xt, yt, alpha=alpha, beta=beta)
        torch.cuda.synchronize()
        assert rel(yt.cpu().numpy(), expect) <= TOL
