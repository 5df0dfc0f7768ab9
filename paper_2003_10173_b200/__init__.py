"""B200-native H^2 hot path (hgemv + HARA) for arXiv 2003.10173.

Host API mirrors the reference (proj/include/h2); compute runs in
lib/libh2b200.so (sm_100a CUDA kernels behind the C ABI in include/h2c.h).
"""
from .h2 import (Admissibility, BlockTree, ClusterTree, H2Matrix, Ordering, build_block_tree,
                 build_cluster_tree, deserialize, read_h2_file, serialize, write_h2_file)
from ._lib import CudaError, LIB_PATH, divergence_error, io_error, max_rank_error
from .construction import (BlockFactor, Rng, adaptive_block_factorization, frobenius_norm, local_low_rank_update,
                           sample_block_column)
from .h2 import StorageReport, ValidationReport
from .construction import (DenseOperator, H2Operator, HybridResult, LinearOperator, LowRankFactor, LowRankResult,
                           PeelConfig, PeelResult, SampleStats, estimate_relative_error, hybrid_construct,
                           make_operator, orthogonalize, peel_construct, pnorm_estimate, randomized_lowrank,
                           recompress)
from .pde import AdvDiff2D, Diffusion1D, MinimalSurface, Oracle, make_oracle
from .inversion import (ConvergenceTrace, HInverseResult, ThresholdSchedule, desymmetrized, h_hyperpower,
                        h_newton_schulz, h_unrolled, hyperpower_sampler, low_rank_update, ns_sampler,
                        residual_norm, scaled_identity, scaled_identity_start, threshold_schedule,
                        unrolled_sampler)

__all__ = ["Admissibility", "BlockTree", "ClusterTree", "H2Matrix", "Ordering", "build_block_tree",
           "build_cluster_tree", "CudaError", "LIB_PATH", "max_rank_error", "DenseOperator", "H2Operator",
           "LinearOperator", "PeelConfig", "PeelResult", "SampleStats", "estimate_relative_error", "make_operator",
           "orthogonalize", "peel_construct", "pnorm_estimate", "recompress", "divergence_error", "ConvergenceTrace",
           "HInverseResult", "ThresholdSchedule", "desymmetrized", "h_hyperpower", "h_newton_schulz", "h_unrolled",
           "hyperpower_sampler", "low_rank_update", "ns_sampler", "residual_norm", "scaled_identity",
           "scaled_identity_start", "threshold_schedule", "unrolled_sampler", "HybridResult", "LowRankFactor",
           "LowRankResult", "hybrid_construct", "randomized_lowrank", "serialize", "deserialize", "write_h2_file",
           "read_h2_file", "io_error", "BlockFactor", "Rng", "adaptive_block_factorization", "frobenius_norm",
           "local_low_rank_update", "sample_block_column", "StorageReport", "ValidationReport", "AdvDiff2D", "Diffusion1D", "MinimalSurface", "Oracle", "make_oracle"]
