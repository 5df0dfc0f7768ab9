"""The C-ABI library loads and exports every symbol include/h2c.h declares (no GPU needed)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "h2c.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(h2c_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_all_declared_symbols():
    from paper_2003_10173_b200 import _lib
    names = declared_symbols()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(_lib.lib, n)]
    assert not missing, missing


def test_version_and_error_strings():
    from paper_2003_10173_b200 import _lib
    assert b"sm_100a" in _lib.lib.h2c_version()
    assert isinstance(_lib.lib.h2c_last_error(), bytes)


def test_invalid_arguments_map_to_value_error():
    import numpy as np
    import pytest
    from paper_2003_10173_b200 import build_cluster_tree
    with pytest.raises(ValueError):
        build_cluster_tree(np.zeros((10, 2)), 1)          # leaf_size < 2 (cluster_tree.hpp:33)
    with pytest.raises(ValueError):
        build_cluster_tree(np.zeros((10, 4)), 8)          # dim > 3 (point_set.hpp:26-27)
