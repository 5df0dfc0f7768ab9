"""Device cluster-tree build against the host builder,
which the CPU suite pins to the reference rules (tests/test_trees.py): every
node range, level, link, bounding box and the permutation must be identical."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2003_10173_b200 import build_cluster_tree


def same_tree(a, b):
    assert a.num_nodes == b.num_nodes and a.depth == b.depth
    for f in ("begin", "end", "level", "parent", "child0", "child1", "perm"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert np.array_equal(a.box_lo, b.box_lo) and np.array_equal(a.box_hi, b.box_hi)


CASES = [
    ("grid1d", lambda: O.grid1d(1000, -1, 1), 32),
    ("grid2d_ties", lambda: O.grid2d(64, 48), 16),
    ("grid3d", lambda: O.grid3d(24, 20, 16), 64),
    ("random3d", lambda: np.random.default_rng(3).random((5000, 3)), 40),
    ("duplicates", lambda: np.repeat(np.random.default_rng(4).random((300, 2)), 3, axis=0), 8),
    ("tiny", lambda: np.random.default_rng(5).random((7, 2)), 2),
    ("single", lambda: np.zeros((1, 3)), 4),
    ("negative", lambda: np.random.default_rng(6).standard_normal((3000, 2)) * 1e3, 24),
]


@pytest.mark.gpu
@pytest.mark.parametrize("name,make,leaf", CASES, ids=[c[0] for c in CASES])
def test_device_tree_equals_host_tree(cuda, name, make, leaf):
    pts = make()
    same_tree(build_cluster_tree(pts, leaf, device=True), build_cluster_tree(pts, leaf))


@pytest.mark.gpu
def test_device_tree_at_bench_scale(cuda):   # cfg2 geometry, N = 2^20
    x = (np.arange(1024) / 1023.0)
    pts = np.stack([np.tile(x, 1024), np.repeat(x, 1024)], axis=1)
    same_tree(build_cluster_tree(pts, 64, device=True), build_cluster_tree(pts, 64))
