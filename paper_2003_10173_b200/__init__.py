"""B200-native H^2 hot path (hgemv + HARA) for arXiv 2003.10173.

Host API mirrors the reference (proj/include/h2); compute runs in
lib/libh2b200.so (sm_100a CUDA kernels behind the C ABI in include/h2c.h).
"""
from .h2 import (Admissibility, BlockTree, ClusterTree, H2Matrix, Ordering, build_block_tree,
                 build_cluster_tree)
from ._lib import CudaError, LIB_PATH, max_rank_error

__all__ = ["Admissibility", "BlockTree", "ClusterTree", "H2Matrix", "Ordering", "build_block_tree",
           "build_cluster_tree", "CudaError", "LIB_PATH", "max_rank_error"]
