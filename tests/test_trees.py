"""Product host tree builders vs the oracle: bit-exact permutation, node ranges,
block tree ids, tags and leaf ordinals (integer/index work -> exact parity).
Pins cluster_tree.hpp:122-176 and block_tree.hpp:22-27, 77-109."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2003_10173_b200 import Admissibility, build_block_tree, build_cluster_tree


def both(points, leaf, weak, eta=1.0):
    ref = O.Tree(points, leaf, eta, weak)
    ct = build_cluster_tree(points, leaf)
    bt = build_block_tree(ct, ct, eta, Admissibility.weak if weak else Admissibility.strong)
    return ref, ct, bt


CASES = [
    ("1d-weak-96-8", O.grid1d(96, -1, 1), 8, True),
    ("1d-strong-70-6", O.grid1d(70, -1, 1), 6, False),
    ("2d-12x12-16", O.grid2d(12, 12), 16, False),
    ("2d-32x32-64", O.grid2d(32, 32), 64, False),
    ("1d-2048-32-weak", O.grid1d(2048, -1, 1), 32, True),
    ("rand2d-333-16", O.gaussian(7, 333, 2), 16, False),
    ("rand3d-257-10", O.gaussian(11, 257, 3), 10, False),
    ("3d-16^3-64", O.grid3d(16, 16, 16), 64, False),
    ("leaf=n", O.grid1d(32), 32, False),
    ("ties", np.round(O.gaussian(5, 500, 2) * 2) / 2, 12, False),
    ("2d-128^2-64 (cfg1)", O.grid2d(128, 128), 64, False),
]


@pytest.mark.parametrize("name,pts,leaf,weak", CASES, ids=[c[0] for c in CASES])
def test_trees_match_oracle_bitwise(name, pts, leaf, weak):
    ref, ct, bt = both(pts, leaf, weak)
    assert ct.n == ref.n and ct.depth == ref.depth and ct.num_nodes == ref.num_nodes
    np.testing.assert_array_equal(ct.perm, ref.perm)
    np.testing.assert_array_equal(ct.begin, ref.begin)
    np.testing.assert_array_equal(ct.end, ref.end)
    np.testing.assert_array_equal(ct.level, ref.level)
    np.testing.assert_array_equal(ct.parent, ref.parent)
    np.testing.assert_array_equal(ct.child0, ref.child0)
    np.testing.assert_array_equal(ct.child1, ref.child1)
    assert bt.num_nodes == ref.num_blocks
    np.testing.assert_array_equal(bt.row, ref.brow)
    np.testing.assert_array_equal(bt.col, ref.bcol)
    np.testing.assert_array_equal(bt.tag, ref.btag)
    np.testing.assert_array_equal(bt.admissible_leaves, ref.adm)
    np.testing.assert_array_equal(bt.dense_leaves, ref.dense)


def test_cfg1_block_counts_match_survey():
    # cfg1 2D 128^2 leaf 64 eta 1 strong -> 511 nodes, depth 8,
    # 5,692 admissible (2,846 canonical) and 4,692 dense (2,474 canonical)
    ct = build_cluster_tree(O.grid2d(128, 128), 64)
    bt = build_block_tree(ct, ct, 1.0)
    assert ct.num_nodes == 511 and ct.depth == 8 and len(ct.leaves) == 256
    assert len(bt.admissible_leaves) == 5692 and len(bt.dense_leaves) == 4692
    canon = lambda leaves: int(np.sum(bt.row[leaves] <= bt.col[leaves]))
    assert canon(bt.admissible_leaves) == 2846 and canon(bt.dense_leaves) == 2474


def test_weak_tree_has_2_pow_l_blocks_per_level():
    # test_geometry.cpp:32-41
    ct = build_cluster_tree(O.grid1d(2048, -1, 1), 32)
    assert ct.depth == 6
    bt = build_block_tree(ct, ct, 1.0, Admissibility.weak)
    lv = bt.blevel[bt.admissible_leaves]
    for l in range(1, 7):
        assert int(np.sum(lv == l)) == 2 ** l


def test_tiling_and_permutation_roundtrip():
    pts = O.gaussian(3, 1000, 2)
    ct = build_cluster_tree(pts, 20)
    bt = build_block_tree(ct, ct, 1.0)
    sz = ct.end - ct.begin
    area = np.sum(sz[bt.row[bt.admissible_leaves]] * sz[bt.col[bt.admissible_leaves]])
    area += np.sum(sz[bt.row[bt.dense_leaves]] * sz[bt.col[bt.dense_leaves]])
    assert area == 1000 * 1000
    x = O.gaussian(4, 1000, 3)
    assert np.array_equal(ct.to_user(ct.to_internal(x)), x)
    assert sorted(ct.perm.tolist()) == list(range(1000))


@pytest.mark.slow
def test_cfg2_structure_counts():
    # 2D 1024^2 leaf 64 -> 32,767 nodes, depth 14, 556,074 adm / 338,452 dense
    ct = build_cluster_tree(O.grid2d(1024, 1024), 64)
    bt = build_block_tree(ct, ct, 1.0)
    assert ct.num_nodes == 32767 and ct.depth == 14
    assert len(bt.admissible_leaves) == 556074 and len(bt.dense_leaves) == 338452
