"""The reference's core hgemv properties (P/tests/test_core.cpp) restated on the
B200 path, plus the same size-independent properties at the full cfg2 size
(BASELINE.json configs[1], N=2^20, 32 vectors), where the CPU oracle is too slow
for a full comparison."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2003_10173_b200 import Admissibility, H2Matrix, build_block_tree, build_cluster_tree
from paper_2003_10173_b200.inversion import scaled_identity

pytestmark = pytest.mark.gpu


def rel(a, b):
    d = np.linalg.norm(b)
    return np.linalg.norm(a - b) / d if d else np.linalg.norm(a)


def fixture(pts, leaf, weak, sym, kmax, seed):
    """random_h2 (test_support.hpp:38-70) from the oracle, loaded into a device matrix."""
    ref = O.Tree(pts, leaf, 1.0, weak)
    ora = O.H2.random(ref, sym, kmax, seed)
    ct = build_cluster_tree(pts, leaf)
    bt = build_block_tree(ct, ct, 1.0, Admissibility.weak if weak else Admissibility.strong)
    rr, cr = ora.ranks()
    return ora, H2Matrix.from_packed(bt, sym, rr, cr, ora.export()), bt


def test_zero_and_scaled_identity_exact(cuda):   # test_core.cpp:24-38
    pts = O.grid1d(64, -1, 1)
    ct = build_cluster_tree(pts, 8)
    bt = build_block_tree(ct, ct, 1.0, Admissibility.weak)
    x = O.gaussian(1, 64, 3)
    z = H2Matrix.zero(bt, True)
    assert np.count_nonzero(z.matvec(x)) == 0
    ident = scaled_identity(bt, 0.5)
    assert rel(ident.matvec(x), 0.5 * x) < 1e-15
    shifted = H2Matrix.zero(bt, True)
    shifted.add_diagonal(0.5)
    assert rel(shifted.matvec(x), 0.5 * x) < 1e-15


def test_matvec_is_linear(cuda):   # test_core.cpp:55-64
    _, m, _ = fixture(O.grid1d(128, -1, 1), 16, True, True, 5, 3)
    x, z = O.gaussian(31, 128, 2), O.gaussian(32, 128, 2)
    alpha, beta = 0.37, -1.25
    assert rel(m.matvec(alpha * x + beta * z), alpha * m.matvec(x) + beta * m.matvec(z)) < 1e-12


def test_symmetric_bilinear_form(cuda):   # test_core.cpp:66-73
    _, m, _ = fixture(O.grid2d(10, 10), 8, False, True, 4, 4)
    x, y = O.gaussian(41, 100, 1), O.gaussian(42, 100, 1)
    a = float(x[:, 0] @ m.matvec(y)[:, 0])
    b = float(y[:, 0] @ m.matvec(x)[:, 0])
    assert abs(a - b) < 1e-12 * abs(a)


def test_ordering_tags(cuda):   # test_core.cpp:75-83
    _, m, bt = fixture(O.grid1d(32, -1, 1), 4, True, True, 3, 5)
    x = O.gaussian(51, 32, 2)
    ct = bt.tree
    y_user = m.matvec(x)
    y_int = ct.to_user(m.matvec_internal(ct.to_internal(x)))
    assert rel(y_user, y_int) < 1e-15


def test_full_size_cfg2_properties(cuda):
    """cfg2 (2D Gaussian kernel, N=2^20, leaf 64, rank 32, 32 vectors) on the device
    path: linearity, the symmetric bilinear form, and agreement of the user- and
    internal-ordering entry points."""
    import torch
    import bench
    cfg = bench.CONFIGS["cfg2"]
    pts = bench.grid_points(cfg["grid"])
    n, b = pts.shape[0], cfg["b"]
    ct = build_cluster_tree(pts, cfg["leaf"], device=True)
    bt = build_block_tree(ct, ct, 1.0)
    m = H2Matrix.kernel(bt, pts, cfg["kind"], cfg["ell"], cfg["rank"])
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randn(b, n, dtype=torch.float64, device="cuda", generator=g).t()
    z = torch.randn(b, n, dtype=torch.float64, device="cuda", generator=g).t()
    hx, hz, hs = (torch.empty(b, n, dtype=torch.float64, device="cuda").t() for _ in range(3))
    m.hgemv(x, hx)
    m.hgemv(z, hz)
    alpha, beta = 0.37, -1.25
    m.hgemv((alpha * x + beta * z).t().contiguous().t(), hs)
    lin = float(torch.linalg.norm(hs - (alpha * hx + beta * hz)) / torch.linalg.norm(hs))
    assert lin < 1e-12, lin
    # x^T (H z) = z^T (H x), column by column, relative to the Cauchy-Schwarz bound
    a = (x * hz).sum(0)
    c = (z * hx).sum(0)
    bound = torch.linalg.norm(x, dim=0) * torch.linalg.norm(hz, dim=0)
    assert float(((a - c).abs() / bound).max()) < 1e-12
    # accumulate form: y = 2 H x - y0 through alpha / beta equals the explicit combination
    y = z.clone()
    m.hgemv(x, y, alpha=2.0, beta=-1.0)
    acc = float(torch.linalg.norm(y - (2.0 * hx - z)) / torch.linalg.norm(y))
    assert acc < 1e-12, acc
    # user ordering vs internal ordering entry points
    perm = torch.as_tensor(ct.perm, device="cuda")
    xi = x[perm].t().contiguous().t()
    yi = torch.empty_like(xi)
    from paper_2003_10173_b200 import Ordering
    m.hgemv(xi, yi, ordering=Ordering.internal)
    yu = torch.empty_like(yi)
    yu[perm] = yi
    assert float(torch.linalg.norm(yu - hx) / torch.linalg.norm(hx)) < 1e-15


@pytest.mark.parametrize("kind,grid,rank", [("gaussian", (40, 40), 32), ("exponential", (32, 32), 16),
                                            ("matern32", (12, 12, 12), 32)])
def test_kernel_generator_matches_host_restatement(cuda, kind, grid, rank):
    """The benchmark payload (device generator, csrc/matrix.cu) equals its host
    restatement (oracle ora_kernel_h2) that the reference arm multiplies."""
    from paper_2003_10173_b200 import H2Matrix, build_block_tree, build_cluster_tree
    pts = O.grid2d(*grid) if len(grid) == 2 else O.grid3d(*grid)
    ct = build_cluster_tree(pts, 32)
    bt = build_block_tree(ct, ct, 1.0)
    m = H2Matrix.kernel(bt, pts, kind, 0.1, rank)
    h = O.H2.kernel(O.Tree(pts, 32), kind, 0.1, rank, threads=4)
    assert np.array_equal(m.ranks()[0], h.ranks()[0])
    dm, dh = m.download(), h.export()
    for k in ("U", "E", "S", "D"):
        assert dm[k].shape == dh[k].shape
        assert np.abs(dm[k] - dh[k]).max() <= 1e-12 * max(1.0, np.abs(dh[k]).max()), k
