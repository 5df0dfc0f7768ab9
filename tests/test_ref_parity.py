"""Parity against the reference's OWN code: oracle/_ref/libh2ref.so is the
unchanged reference headers (proj/include/h2, proj/tests/test_support.hpp)
compiled with the reference's Release flags over the Eigen-API shim
(oracle/Makefile `ref`). These tests pin the product's host trees and the CPU
restatement (oracle/h2oracle.hpp) to it:

* integer/index work is bit-exact: permutation, node ranges, boxes, block ids,
  tags, admissible/dense leaf lists (cluster_tree.hpp:122-176,
  block_tree.hpp:22-27, 77-109, point_set.hpp:72-86), at every BASELINE config's
  tree (cfg1 2D 128^2, cfg2 2D 1024^2, cfg3 1D weak 2^18, cfg4 3D 128^3);
* the reference's random_h2 fixture (test_support.hpp:38-70) is bitwise the
  restatement's (same libstdc++ streams);
* matvec and HARA control flow (samples per level, rank profile) agree.
"""
import os

import numpy as np
import pytest

from oracle import pyoracle as O

REF_LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "libh2ref.so")
if not os.path.exists(REF_LIB) and not os.path.isdir("/root/reference/proj/include/h2"):
    pytest.skip("oracle/_ref not built and the reference tree is absent", allow_module_level=True)
from oracle import pyref as R  # noqa: E402

from paper_2003_10173_b200 import Admissibility, build_block_tree, build_cluster_tree  # noqa: E402

SMALL = [
    ("1d-weak-96-8", O.grid1d(96, -1, 1), 8, True),
    ("1d-strong-70-6", O.grid1d(70, -1, 1), 6, False),
    ("2d-12x12-16", O.grid2d(12, 12), 16, False),
    ("rand2d-333-16", O.gaussian(7, 333, 2), 16, False),
    ("rand3d-257-10", O.gaussian(11, 257, 3), 10, False),
    ("rand3d-5000-16", O.gaussian(3, 5000, 3), 16, False),
    ("3d-16^3-64", O.grid3d(16, 16, 16), 64, False),
    ("3d-32^3-64", O.grid3d(32, 32, 32), 64, False),
    ("3d-20x12x7-8", O.grid3d(20, 12, 7), 8, False),
    ("leaf=n", O.grid1d(32), 32, False),
    ("ties", np.round(O.gaussian(5, 500, 2) * 2) / 2, 12, False),
    ("ties3d", np.round(O.gaussian(6, 700, 3) * 2) / 2, 9, False),
]
CONFIGS = [
    ("cfg1-2d-128^2", lambda: O.grid2d(128, 128), 64, False, (5692, 4692)),
    ("cfg2-2d-1024^2", lambda: O.grid2d(1024, 1024), 64, False, (556074, 338452)),
    ("cfg3-1d-2^18-weak", lambda: O.grid1d(2 ** 18, -1, 1), 32, True, (16382, 8192)),
    ("cfg4-3d-128^3", lambda: O.grid3d(128, 128, 128), 64, False, (5690728, 1866096)),
]


def assert_same_tree(ref, ct, bt):
    assert ct.n == ref.n and ct.depth == ref.depth and ct.num_nodes == ref.num_nodes
    np.testing.assert_array_equal(ct.perm, ref.perm)
    np.testing.assert_array_equal(ct.begin, ref.begin)
    np.testing.assert_array_equal(ct.end, ref.end)
    np.testing.assert_array_equal(ct.level, ref.level)
    np.testing.assert_array_equal(ct.parent, ref.parent)
    np.testing.assert_array_equal(ct.child0, ref.child0)
    np.testing.assert_array_equal(ct.child1, ref.child1)
    lo, hi = ref.boxes()
    d = ct.dim
    assert np.array_equal(ct.box_lo[:, :d], lo[:, :d]) and np.array_equal(ct.box_hi[:, :d], hi[:, :d])
    assert bt.num_nodes == ref.num_blocks
    np.testing.assert_array_equal(bt.row, ref.brow)
    np.testing.assert_array_equal(bt.col, ref.bcol)
    np.testing.assert_array_equal(bt.tag, ref.btag)
    np.testing.assert_array_equal(bt.admissible_leaves, ref.adm)
    np.testing.assert_array_equal(bt.dense_leaves, ref.dense)


def assert_same_oracle_tree(ref, ora):
    for k in ("perm", "begin", "end", "level", "parent", "child0", "child1", "brow", "bcol", "btag", "adm", "dense"):
        np.testing.assert_array_equal(getattr(ora, k), getattr(ref, k), err_msg=k)
    for a, b in zip(ora.boxes(), ref.boxes()):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("name,pts,leaf,weak", SMALL, ids=[c[0] for c in SMALL])
def test_small_trees_bitwise(name, pts, leaf, weak):
    ref = R.Tree(pts, leaf, 1.0, weak)
    ct = build_cluster_tree(pts, leaf)
    bt = build_block_tree(ct, ct, 1.0, Admissibility.weak if weak else Admissibility.strong)
    assert_same_tree(ref, ct, bt)
    assert_same_oracle_tree(ref, O.Tree(pts, leaf, 1.0, weak))


@pytest.mark.parametrize("eta", [0.5, 0.7071067811865476, 1.0, 1.4142135623730951, 2.0])
def test_eta_sweep_3d_grid_bitwise(eta):
    # exact-tie geometry: grid boxes make diam == eta * dist for many pairs
    pts = O.grid3d(24, 24, 24)
    ref = R.Tree(pts, 27, eta, False)
    ct = build_cluster_tree(pts, 27)
    bt = build_block_tree(ct, ct, eta)
    assert_same_tree(ref, ct, bt)


@pytest.mark.parametrize("name,make,leaf,weak,counts", CONFIGS, ids=[c[0] for c in CONFIGS])
def test_config_trees_bitwise(name, make, leaf, weak, counts):
    pts = make()
    ref = R.Tree(pts, leaf, 1.0, weak)
    assert (len(ref.adm), len(ref.dense)) == counts
    ct = build_cluster_tree(pts, leaf)
    bt = build_block_tree(ct, ct, 1.0, Admissibility.weak if weak else Admissibility.strong)
    assert_same_tree(ref, ct, bt)
    del ct, bt
    assert_same_oracle_tree(ref, O.Tree(pts, leaf, 1.0, weak))


@pytest.mark.parametrize("sym", [True, False])
def test_random_h2_fixture_bitwise(sym):
    pts = O.grid2d(20, 20)
    a, b = R.Tree(pts, 16), O.Tree(pts, 16)
    ha, hb = R.H2.random(a, sym, 7, 1234), O.H2.random(b, sym, 7, 1234)
    ra, rb = ha.ranks(), hb.ranks()
    assert np.array_equal(ra[0], rb[0]) and np.array_equal(ra[1], rb[1])
    ea, eb = ha.export(), hb.export()
    for k in O.PARTS:
        assert np.array_equal(ea[k], eb[k]), k


def test_gaussian_stream_bitwise():
    # fill_gaussian (construction.hpp:81-85) over mt19937_64(seed)
    assert np.array_equal(R.gaussian(42, 257, 5), O.gaussian(42, 257, 5))


@pytest.mark.parametrize("sym", [True, False])
@pytest.mark.parametrize("transpose", [False, True])
@pytest.mark.parametrize("ordering", [0, 1])
def test_matvec_matches_reference(sym, transpose, ordering):
    # h2_matrix.hpp:108-124, 246-305 run by the reference's own code
    pts = O.grid2d(24, 24)
    a, b = R.Tree(pts, 16), O.Tree(pts, 16)
    ha, hb = R.H2.random(a, sym, 8, 99), O.H2.random(b, sym, 8, 99)
    x = O.gaussian(5, pts.shape[0], 6)
    ya, yb = ha.matvec(x, transpose, ordering), hb.matvec(x, transpose, ordering)
    assert np.linalg.norm(ya - yb) <= 1e-13 * np.linalg.norm(ya)
    da = ha.to_dense()
    assert np.linalg.norm(da - hb.to_dense()) <= 1e-14 * np.linalg.norm(da)


def test_peel_dense_control_flow_matches_reference():
    # peel_construct (construction.hpp:300-382) of a dense kernel operator: the
    # same per-level samples and rank profile as the reference's own driver
    pts = O.grid1d(256, -1, 1)
    x = pts[:, 0]
    a = np.exp(-np.abs(x[:, None] - x[None, :]) / 0.3)
    ta, tb = R.Tree(pts, 16, 1.0, True), O.Tree(pts, 16, 1.0, True)
    ha, sa = R.peel_dense(ta, a, True, eps=1e-8)
    hb, sb = O.peel_dense(tb, a, True, eps=1e-8)
    assert sa == sb
    assert np.array_equal(ha.ranks()[0], hb.ranks()[0])
    ea = np.linalg.norm(ha.to_dense() - a, 2) / np.linalg.norm(a, 2)
    eb = np.linalg.norm(hb.to_dense() - a, 2) / np.linalg.norm(a, 2)
    assert ea <= 3e-8 and eb <= 3e-8


def test_peel_identity_known_answer_on_reference():
    # test_construction.cpp:112-124 on the reference's own driver and on the
    # restatement: ranks 0, dense leaves = I, the dense extraction costs one
    # leaf size (16) of indicator columns, and both drivers spend the same samples
    pts = O.grid1d(128, -1, 1)
    ta, tb = R.Tree(pts, 16, 1.0, True), O.Tree(pts, 16, 1.0, True)
    eye = np.eye(128)
    ha, sa = R.peel_dense(ta, eye, True, eps=1e-8)
    hb, sb = O.peel_dense(tb, eye, True, eps=1e-8)
    assert sa == sb and sa["level_samples"][-1] == 16
    assert not ha.ranks()[0].any() and not hb.ranks()[0].any()
    assert np.linalg.norm(ha.to_dense() - eye) < 1e-12 * np.sqrt(128)


@pytest.mark.parametrize("eps", [1e-4, 1e-6, 1e-10])
def test_peel_rank3_and_spd_match_reference(eps):
    # test_construction.cpp:126-159: a dense random SPD matrix; same samples and
    # rank profile from the reference's driver and the restatement
    g = O.gaussian(55, 64, 64)
    a = g @ g.T + 64.0 * np.eye(64)
    pts = O.grid1d(64, -1, 1)
    ta, tb = R.Tree(pts, 8, 1.0, True), O.Tree(pts, 8, 1.0, True)
    ha, sa = R.peel_dense(ta, a, True, eps=eps)
    hb, sb = O.peel_dense(tb, a, True, eps=eps)
    assert sa == sb
    assert np.array_equal(ha.ranks()[0], hb.ranks()[0])
    for h in (ha, hb):
        assert np.linalg.norm(h.to_dense() - a, 2) / np.linalg.norm(a, 2) <= 3 * eps


@pytest.mark.parametrize("seed", [0, 42, 1234, 0x9E3779B97F4A7C15])
def test_product_gaussian_stream_is_the_references(seed):
    # the product's host stream (csrc/refstream.cpp, compiled with FMA like the
    # reference's -march=native build) is bitwise the reference's; ~14% of the
    # normals would differ in the last bits without the polar method's FMA
    from paper_2003_10173_b200 import Rng
    r = Rng(seed)
    a, b = r.gaussian(3000, 5), r.gaussian(17, 3)
    ra = R.gaussian(seed, 3000, 5)
    assert np.array_equal(a, ra)
    assert not np.array_equal(b, R.gaussian(seed, 17, 3))   # the stream continues across calls
