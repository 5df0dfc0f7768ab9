"""ctypes binding of the C ABI (include/h2c.h) in lib/libh2b200.so.

The product path has no CPU fallback: if the shared library is missing the
import fails loudly (build it with `make -C paper_2003_10173_b200` or
`python -c "import __graft_entry__ as g; g.build()"`).
"""
import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libh2b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"paper_2003_10173_b200: native library {LIB_PATH} is missing; build it with "
        "`make -C paper_2003_10173_b200` (no CPU fallback exists)")

lib = C.CDLL(LIB_PATH)

i32, i64, f64, vp = C.c_int, C.c_int64, C.c_double, C.c_void_p
P = C.POINTER
H = C.c_void_p  # opaque handles

H2C_OK = 0
H2C_INVALID_ARGUMENT = -1
H2C_LOGIC_ERROR = -2
H2C_MAX_RANK_ERROR = -3
H2C_RUNTIME_ERROR = -4
H2C_CUDA_ERROR = -5
H2C_CALLBACK_ERROR = -6
H2C_DIVERGENCE_ERROR = -7


class CudaError(RuntimeError):
    pass


class max_rank_error(RuntimeError):
    """Mirror of h2::max_rank_error (construction.hpp:61-66)."""


class divergence_error(RuntimeError):
    """Mirror of h2::divergence_error (inversion.hpp:41-46); .trace holds the rows so far."""

    def __init__(self, msg, trace=None):
        super().__init__(msg)
        self.trace = trace


def _sig(name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_sig("h2c_last_error", C.c_char_p)
_sig("h2c_version", C.c_char_p)
_sig("h2c_cluster_tree_create", i32, vp, i64, i32, i64, P(H))
_sig("h2c_cluster_tree_create_device", i32, vp, i64, i32, i64, vp, P(H))
_sig("h2c_cluster_tree_destroy", None, H)
_sig("h2c_cluster_tree_info", i32, H, P(i64), P(i32), P(i32), P(i32), P(i32))
_sig("h2c_cluster_tree_nodes", i32, H, vp, vp, vp, vp, vp, vp, vp, vp)
_sig("h2c_cluster_tree_perm", i32, H, vp)
_sig("h2c_block_tree_create", i32, H, f64, i32, P(H))
_sig("h2c_block_tree_destroy", None, H)
_sig("h2c_block_tree_info", i32, H, P(i32), P(i32), P(i32), P(i32))
_sig("h2c_block_tree_nodes", i32, H, vp, vp, vp, vp, vp)
_sig("h2c_block_tree_leaves", i32, H, vp, vp)
_sig("h2c_block_tree_params", i32, H, P(f64), P(i32))
_sig("h2c_block_tree_cluster_tree", i32, H, P(H))
_sig("h2c_matrix_create", i32, H, i32, vp, vp, P(H))
_sig("h2c_matrix_destroy", None, H)
_sig("h2c_matrix_info", i32, H, P(i64), P(i32), P(i32))
_sig("h2c_matrix_set_orthonormal", i32, H, i32)
_sig("h2c_matrix_sizes", i32, H, vp)
_sig("h2c_matrix_ranks", i32, H, vp, vp)
_sig("h2c_matrix_upload", i32, H, vp, vp, vp, vp, vp, vp)
_sig("h2c_matrix_download", i32, H, vp, vp, vp, vp, vp, vp)
_sig("h2c_matrix_kernel", i32, H, vp, i32, f64, i32, P(H))
_sig("h2c_matrix_kernel_sharded", i32, H, vp, i32, f64, i32, i32, i32, P(H))
_sig("h2c_hgemv", i32, H, i32, i32, i64, i64, vp, i64, vp, i64, f64, f64, vp)
_sig("h2c_matvec_host", i32, H, i32, i32, i64, i64, vp, vp)
_sig("h2c_matvec_host_async", i32, H, i32, i32, i64, i64, vp, vp, vp)
_sig("h2c_hgemv_launches", i32, H, i32, i64, P(i32))

def check(rc):
    """Raise the Python mirror of the reference exception kind."""
    if rc == H2C_OK:
        return
    msg = lib.h2c_last_error().decode(errors="replace")
    if rc == H2C_INVALID_ARGUMENT:
        raise ValueError(msg)
    if rc == H2C_LOGIC_ERROR:
        raise NotImplementedError(msg)
    if rc == H2C_MAX_RANK_ERROR:
        raise max_rank_error(msg)
    if rc == H2C_DIVERGENCE_ERROR:
        raise divergence_error(msg)
    if rc == H2C_CUDA_ERROR:
        raise CudaError(msg)
    raise RuntimeError(f"h2c error {rc}: {msg}")


_sig("h2c_hgemv_stage_times", i32, H, i32, i32, i64, i64, vp, i64, vp, i64, vp, i32, P(i32), vp, vp, vp, vp)


class PeelConfigC(C.Structure):
    """h2c_peel_config (PeelConfig, construction.hpp:23-31)."""
    _fields_ = [("eps", C.c_double), ("sample_block_size", C.c_int64), ("oversampling", C.c_int64),
                ("max_rank", C.c_int64), ("seed", C.c_uint64), ("norm_scale", C.c_double),
                ("crossover_rank_cap", C.c_int64), ("rng", C.c_int)]


class LevelStatsC(C.Structure):
    _fields_ = [("level", C.c_int), ("blocks", C.c_int64), ("max_rank", C.c_int64), ("samples", C.c_int64)]


APPLY_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p)

_sig("h2c_operator_dense", i32, vp, i64, i32, P(H))
_sig("h2c_operator_h2", i32, H, P(H))
_sig("h2c_operator_device_callback", i32, i64, i32, i32, APPLY_FN, vp, P(H))
_sig("h2c_operator_host_callback", i32, i64, i32, i32, APPLY_FN, vp, P(H))
_sig("h2c_operator_destroy", None, H)
_sig("h2c_operator_apply", i32, H, i32, i64, vp, vp, vp)
_sig("h2c_operator_columns_applied", i32, H, P(i64))
_sig("h2c_operator_reset_counter", i32, H)
_sig("h2c_pnorm2_estimate", i32, H, P(f64), P(i32))
_sig("h2c_orthogonalize", i32, H, P(H))
_sig("h2c_recompress", i32, H, f64, P(H))
_sig("h2c_peel_config_default", None, P(PeelConfigC))
_sig("h2c_peel_construct", i32, H, H, P(PeelConfigC), P(H), P(i64), P(LevelStatsC), i32, P(i32), P(f64), P(f64))
_sig("h2c_estimate_relative_error", i32, H, H, f64, P(f64))

_sig("h2c_dist_plan_create", i32, H, i32, i32, i32, P(H))
_sig("h2c_dist_plan_destroy", None, H)
_sig("h2c_dist_plan_counts", i32, H, vp, vp, P(i64), P(i64))
_sig("h2c_dist_plan_launches", i32, H, P(i32))
_sig("h2c_dist_hgemv_begin", i32, H, i64, vp, i64, vp, vp)
_sig("h2c_dist_hgemv_local", i32, H, i64, vp)
_sig("h2c_dist_hgemv_begin_owned", i32, H, i64, vp, i64, vp, vp)
_sig("h2c_dist_hgemv_end_owned", i32, H, i64, vp, vp, i64, f64, f64, vp)
_sig("h2c_dist_hgemv_end", i32, H, i64, vp, vp, i64, f64, f64, vp)
_sig("h2c_dist_hgemv_nccl", i32, H, vp, i64, vp, i64, vp, i64, f64, f64, vp)
_sig("h2c_dist_hgemv_nccl_owned", i32, H, vp, i64, vp, i64, vp, i64, f64, f64, vp)
_sig("h2c_dist_peer_alloc", i32, H, i64)
_sig("h2c_dist_peer_export", i32, H, vp, vp)
_sig("h2c_dist_peer_import", i32, H, vp, vp)
_sig("h2c_dist_peer_link", i32, vp, i32)
_sig("h2c_partition_owner", i32, H, i32, vp)
_sig("h2c_partition_exchange", i32, H, i32, i32, vp, i32, i32, i32, P(i64), vp, vp, vp)


class TraceRowC(C.Structure):
    _fields_ = [("iter", C.c_int), ("residual", C.c_double), ("eps_k", C.c_double), ("samples", C.c_int64),
                ("wall_seconds", C.c_double)]


_sig("h2c_scaled_identity", i32, H, f64, P(H))
_sig("h2c_scaled_identity_start", i32, H, P(H))
_sig("h2c_matrix_add_diagonal", i32, H, f64)
_sig("h2c_pnorm_estimate", i32, H, f64, P(f64), P(i32))
_sig("h2c_sampler_operator", i32, H, H, i32, i32, P(H))
_sig("h2c_residual_norm", i32, H, H, P(f64))
_sig("h2c_residual_norm_op", i32, H, H, P(f64))
_sig("h2c_h_inverse", i32, H, H, i32, i32, i32, f64, f64, P(PeelConfigC), i32, P(H), P(TraceRowC), i32, P(i32),
     P(f64), P(i32))
_sig("h2c_low_rank_update", i32, H, i64, vp, vp, f64, P(H))
_sig("h2c_desymmetrized", i32, H, P(H))

_sig("h2c_randomized_lowrank", i32, H, f64, i64, P(PeelConfigC), P(H))
_sig("h2c_lowrank_info", i32, H, P(i64), P(i64), P(i32), P(f64), P(i32), P(i64))
_sig("h2c_lowrank_download", i32, H, vp, vp)
_sig("h2c_lowrank_destroy", None, H)
_sig("h2c_hybrid_construct", i32, H, H, P(PeelConfigC), P(H), P(i64), P(i64), P(LevelStatsC), i32, P(i32))

H2C_IO_ERROR = -8


class io_error(RuntimeError):
    """Mirror of h2::io_error (types.hpp:29-38); .kind in {bad_magic, version_mismatch, truncated, malformed}."""

    KINDS = ("bad_magic", "version_mismatch", "truncated", "malformed")

    def __init__(self, msg, kind):
        super().__init__(msg)
        self.kind = kind


_check_base = check


def check(rc):   # noqa: F811  (extends the mapping with io_error)
    if rc == H2C_IO_ERROR:
        k = lib.h2c_last_io_error_kind()
        raise io_error(lib.h2c_last_error().decode(errors="replace"),
                       io_error.KINDS[k] if 0 <= k < 4 else "malformed")
    _check_base(rc)


_sig("h2c_rng_create", i32, C.c_uint64, P(H))
_sig("h2c_rng_destroy", None, H)
_sig("h2c_rng_fill_gaussian", i32, H, i64, i64, vp)
_sig("h2c_rng_set_state", i32, H, C.c_char_p)
_sig("h2c_rng_get_state", i32, H, C.c_char_p, P(i64))
_sig("h2c_sample_block_column", i32, H, H, i32, i32, i64, H, vp, vp, vp)
_sig("h2c_adaptive_block_factorization", i32, H, H, i32, i32, f64, P(PeelConfigC), P(H))
_sig("h2c_block_factor_info", i32, H, P(i64), P(i64), P(i64), P(f64))
_sig("h2c_block_factor_download", i32, H, vp, vp)
_sig("h2c_block_factor_destroy", None, H)
_sig("h2c_local_low_rank_update", i32, H, i32, i32, i64, vp, i64, vp, i64, f64, P(H))
_sig("h2c_frobenius_norm", i32, H, P(f64))
_sig("h2c_to_dense", i32, H, i64, vp)
_sig("h2c_validate", i32, H, i64, P(i32), C.c_char_p, i64, vp, i32, P(i32), vp)
_sig("h2c_serialize_size", i32, H, P(i64))
_sig("h2c_serialize", i32, H, vp, i64)
_sig("h2c_deserialize", i32, vp, i64, P(H), P(H))
_sig("h2c_write_h2_file", i32, H, C.c_char_p)
_sig("h2c_read_h2_file", i32, C.c_char_p, P(H), P(H))
_sig("h2c_last_io_error_kind", i32)


class Diff1DConfigC(C.Structure):
    """h2c_diff1d_config (Diffusion1DConfig, diffusion1d.hpp:62-73)."""
    _fields_ = [("n", C.c_int64), ("steps", C.c_int64), ("final_time", C.c_double), ("t_p", C.c_double),
                ("t_0", C.c_double), ("source_amplitude", C.c_double), ("alpha", C.c_double), ("beta", C.c_double),
                ("pad", C.c_double), ("num_sources", C.c_int), ("source_positions", C.POINTER(C.c_double)),
                ("num_receivers", C.c_int64)]


_sig("h2c_diff1d_config_default", None, P(Diff1DConfigC))
_sig("h2c_diff1d_create", i32, P(Diff1DConfigC), vp, P(H))
_sig("h2c_diff1d_destroy", None, H)
_sig("h2c_diff1d_info", i32, H, P(i64), P(i64), P(f64), P(f64), P(i64))
_sig("h2c_diff1d_hessvec", i32, H, i32, i64, vp, vp, vp)
_sig("h2c_diff1d_state_field", i32, H, i32, vp)
_sig("h2c_diff1d_operator", i32, H, i32, P(H))
_sig("h2b_diff1d_tune", i32, i32, i32)
_sig("h2c_surface_create", i32, i64, f64, i32, P(H))
_sig("h2c_surface_destroy", None, H)
_sig("h2c_surface_info", i32, H, P(i64), P(i64), P(f64))
_sig("h2c_surface_state", i32, H, vp)
_sig("h2c_surface_hessvec", i32, H, i64, vp, vp, vp)
_sig("h2c_surface_operator", i32, H, P(H))


class AdvDiffConfigC(C.Structure):
    """h2c_advdiff_config (AdvDiff2DConfig, advdiff2d.hpp:21-28)."""
    _fields_ = [("grid", i64), ("kappa", f64), ("reaction", f64), ("num_observations", i64), ("noise_rel", f64),
                ("obs_seed", C.c_uint64)]


_sig("h2c_advdiff_config_default", None, P(AdvDiffConfigC))
_sig("h2c_advdiff_create", i32, P(AdvDiffConfigC), P(H))
_sig("h2c_advdiff_destroy", None, H)
_sig("h2c_advdiff_info", i32, H, P(i64), P(f64), P(i64), P(i64))
_sig("h2c_advdiff_observations", i32, H, vp)
_sig("h2c_advdiff_hessvec", i32, H, i64, vp, vp, vp)
_sig("h2c_advdiff_operator", i32, H, P(H))
