/*
 * h2c.h — C ABI of the B200-native H^2 hot path (hgemv + HARA).
 *
 * The reference (arxiv 2003.10173, /root/reference/proj) is a header-only
 * C++20/Eigen library with no FFI of its own; its boundary for this path is
 * the C++ API listed next to each entry point below. These functions are what
 * a binding of that API (the C++ wrapper include/h2b200.hpp, the Python
 * package paper_2003_10173_b200, a ctypes / cgo / JNI stub — INTEGRATION.md)
 * calls. Plain pointers and sizes only; every function returns H2C_OK (0) or
 * a negative status mirroring the reference's exception kinds, with the
 * message in h2c_last_error().
 *
 * Orderings: "user" = the caller's point order, "internal" = cluster-tree
 * order (reference types.hpp:19). Matrices are column-major FP64.
 * Device pointers are CUDA device addresses on the current device.
 */
#ifndef H2C_H
#define H2C_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes: reference exception kinds */
#define H2C_OK 0
#define H2C_INVALID_ARGUMENT (-1) /* std::invalid_argument  (e.g. h2_matrix.hpp:241-244) */
#define H2C_LOGIC_ERROR (-2)      /* std::logic_error       (linear_operator.hpp:46-48) */
#define H2C_MAX_RANK_ERROR (-3)   /* h2::max_rank_error     (construction.hpp:61-66) */
#define H2C_RUNTIME_ERROR (-4)    /* std::runtime_error */
#define H2C_CUDA_ERROR (-5)       /* CUDA failure (no reference counterpart) */
#define H2C_CALLBACK_ERROR (-6)   /* user operator callback returned non-zero */
#define H2C_DIVERGENCE_ERROR (-7) /* h2::divergence_error    (inversion.hpp:41-46) */
#define H2C_IO_ERROR (-8)         /* h2::io_error            (types.hpp:29-38); kind via h2c_last_io_error_kind */

typedef struct h2c_cluster_tree_s* h2c_cluster_tree;
typedef struct h2c_block_tree_s* h2c_block_tree;
typedef struct h2c_matrix_s* h2c_matrix;

/* thread-local message of the last failing call */
const char* h2c_last_error(void);
/* library version string */
const char* h2c_version(void);

/* ---- cluster tree: replaces ClusterTree(const PointSet&, Index leaf)
 *      (cluster_tree.hpp:31-47, build_cluster_tree :186-188) ------------- */
int h2c_cluster_tree_create(const double* coords /* n x dim, col-major */, int64_t n, int dim, int64_t leaf_size,
                            h2c_cluster_tree* out);
/* the same tree built on the device: bitwise-identical nodes, boxes and
 * permutation; coords on the host */
int h2c_cluster_tree_create_device(const double* coords, int64_t n, int dim, int64_t leaf_size, void* stream,
                                   h2c_cluster_tree* out);
void h2c_cluster_tree_destroy(h2c_cluster_tree t);
/* n(), dim(), depth(), num_nodes(), leaves().size()  (cluster_tree.hpp:49-58) */
int h2c_cluster_tree_info(h2c_cluster_tree t, int64_t* n, int* dim, int* depth, int* num_nodes, int* num_leaves);
/* node(v) fields (cluster_tree.hpp:18-27); any output may be NULL */
int h2c_cluster_tree_nodes(h2c_cluster_tree t, int64_t* begin, int64_t* end, int* level, int* parent, int* child0,
                           int* child1, double* box_lo /* 3 per node */, double* box_hi);
/* perm(): internal index i <-> user index perm[i] (cluster_tree.hpp:66-67) */
int h2c_cluster_tree_perm(h2c_cluster_tree t, int64_t* perm);

/* ---- block tree: replaces build_block_tree(rows, cols, eta, mode)
 *      (block_tree.hpp:120-124; rows == cols as in every reference use) ----- */
int h2c_block_tree_create(h2c_cluster_tree t, double eta, int weak, h2c_block_tree* out);
void h2c_block_tree_destroy(h2c_block_tree b);
int h2c_block_tree_info(h2c_block_tree b, int* num_nodes, int* num_admissible, int* num_dense, int* max_level);
/* node(b) fields; tag 0 interior, 1 admissible, 2 dense (block_tree.hpp:29-39) */
int h2c_block_tree_nodes(h2c_block_tree b, int* row, int* col, int* level, int* parent, int* tag);
/* eta(), mode() (block_tree.hpp:120-124) and the row/column cluster tree (new handle, shared tree) */
int h2c_block_tree_params(h2c_block_tree b, double* eta, int* weak);
int h2c_block_tree_cluster_tree(h2c_block_tree b, h2c_cluster_tree* out);
/* admissible_leaves(), dense_leaves() (block_tree.hpp:64-65) */
int h2c_block_tree_leaves(h2c_block_tree b, int* admissible, int* dense);

/* ---- H^2 matrix (device resident): replaces H2Matrix (h2_matrix.hpp:40-306)
 *
 * Packed payload layout (six parts U, E, V, F, S, D; V/F empty if symmetric):
 *   U: leaf bases m_t x k_t, leaves in id order        (BasisTree::leaf_basis)
 *   E: transfers k_v x k_parent, non-root nodes in id order (BasisTree::transfer)
 *   V, F: the same for the column basis (non-symmetric only)
 *   S: couplings k_row x k_col by admissible ordinal, stored blocks only
 *   D: dense blocks m_t x m_s by dense ordinal, stored blocks only
 * Symmetric matrices store canonical (row <= col) blocks only (h2_matrix.hpp:103).
 * ----------------------------------------------------------------------- */
/* H2Matrix::zero(bt, symmetric) when ranks are NULL; otherwise a zero matrix with the given ranks */
int h2c_matrix_create(h2c_block_tree b, int symmetric, const int* row_ranks, const int* col_ranks, h2c_matrix* out);
void h2c_matrix_destroy(h2c_matrix h);
int h2c_matrix_info(h2c_matrix h, int64_t* n, int* symmetric, int* orthonormal);
int h2c_matrix_set_orthonormal(h2c_matrix h, int orthonormal);
/* sizes[6] in doubles of U, E, V, F, S, D */
int h2c_matrix_sizes(h2c_matrix h, int64_t* sizes);
int h2c_matrix_ranks(h2c_matrix h, int* row_ranks, int* col_ranks /* may be NULL */);
/* host <-> device payload transfer; NULL parts are skipped */
int h2c_matrix_upload(h2c_matrix h, const double* U, const double* E, const double* V, const double* F,
                      const double* S, const double* D);
int h2c_matrix_download(h2c_matrix h, double* U, double* E, double* V, double* F, double* S, double* D);
/* symmetric kernel matrix generated on the device (benchmark inputs):
 * kind 0 exp(-r/ell), 1 exp(-r^2/ell^2), 2 Matern-3/2; Chebyshev-interpolation bases of rank `rank` */
int h2c_matrix_kernel(h2c_block_tree b, const double* coords /* user order, n x dim */, int kind, double ell,
                      int rank, h2c_matrix* out);

/* the same matrix, but only the payload rank `shard` of `nranks` needs for the
 * row-subtree sharded hgemv (h2c_dist_*): memory per rank ~ 1/nranks + top levels */
int h2c_matrix_kernel_sharded(h2c_block_tree b, const double* coords, int kind, double ell, int rank, int nranks,
                              int shard, h2c_matrix* out);

/* ---- hgemv: replaces H2Matrix::matvec / matvec_transpose (user ordering)
 *      and matvec_internal / matvec_transpose_internal (h2_matrix.hpp:108-124)
 *   y = alpha * op(H) x + beta * y  with x, y DEVICE pointers (n x b, col-major).
 *   ordering: 0 user, 1 internal. stream: cudaStream_t (NULL = legacy default).
 *   alpha = -1, beta = 1 with y preloaded by op(x) is the HARA residual
 *   (construction.hpp:207-216). Errors as check_dims (h2_matrix.hpp:241-244). */
int h2c_hgemv(h2c_matrix h, int transpose, int ordering, int64_t n, int64_t b, const double* x, int64_t ldx,
              double* y, int64_t ldy, double alpha, double beta, void* stream);
/* the same with HOST buffers: H2D copy, hgemv, D2H copy (the drop-in for the
 * by-value Matrix H2Matrix::matvec(const Matrix&)) */
int h2c_matvec_host(h2c_matrix h, int transpose, int ordering, int64_t n, int64_t b, const double* x, double* y);
/* asynchronous host-buffer matvec on `stream`: H2D of x (pinned host memory
 * for overlap), hgemv, D2H of y, all enqueued without waiting; the caller
 * synchronises the stream. Workspace is per stream, so successive calls on
 * alternating streams overlap one call's copies with another's compute. */
int h2c_matvec_host_async(h2c_matrix h, int transpose, int ordering, int64_t n, int64_t b, const double* x, double* y,
                          void* stream);
/* number of kernel launches one hgemv issues (gather + stage launches) */
int h2c_hgemv_launches(h2c_matrix h, int transpose, int64_t b, int* launches);
/* one hgemv (alpha 1, beta 0) with a CUDA event around every launch on `stream`:
 * per launch its stage (0 gather, 1 leaf upsweep, 2 transfer upsweep, 3 coupling,
 * 4 downsweep, 5 leaf expansion + dense near-field), duration in ms, and the
 * algorithmic flops / bytes it must do (the roofline numerators) */
int h2c_hgemv_stage_times(h2c_matrix h, int transpose, int ordering, int64_t n, int64_t b, const double* x,
                          int64_t ldx, double* y, int64_t ldy, void* stream, int max_records, int* count, int* stage,
                          double* ms, double* flops, double* bytes);

/* ---- black-box operators: replace LinearOperator and its adapters
 *      (linear_operator.hpp:20-115). Applications take / return DEVICE
 *      buffers in USER ordering (n x b, column-major, ld n) and add b to the
 *      operator's column counter (linear_operator.hpp:28-41). ------------- */
typedef struct h2c_operator_s* h2c_operator;
/* user callback: y = op(x) (transpose = 0) or op^T(x); return 0 on success */
typedef int (*h2c_apply_fn)(void* ctx, int transpose, int64_t b, const double* x, double* y, void* stream);
/* DenseOperator(a, symmetric) (linear_operator.hpp:86-101): a = n x n host matrix, copied to HBM */
int h2c_operator_dense(const double* a, int64_t n, int symmetric, h2c_operator* out);
/* H2Operator(h) (linear_operator.hpp:104-115): hgemv of a device H^2 matrix (h must outlive it) */
int h2c_operator_h2(h2c_matrix h, h2c_operator* out);
/* make_operator(n, sym, f, t) (linear_operator.hpp:80-84) with x, y DEVICE pointers */
int h2c_operator_device_callback(int64_t n, int symmetric, int has_transpose, h2c_apply_fn fn, void* ctx,
                                 h2c_operator* out);
/* the same with HOST pointers (the library stages x and y through host memory) */
int h2c_operator_host_callback(int64_t n, int symmetric, int has_transpose, h2c_apply_fn fn, void* ctx,
                               h2c_operator* out);
void h2c_operator_destroy(h2c_operator op);
/* LinearOperator::apply / apply_transpose on device buffers */
int h2c_operator_apply(h2c_operator op, int transpose, int64_t b, const double* x, double* y, void* stream);
/* the same on HOST buffers (n x b column-major; staged through HBM; returns when y is written):
 * the by-value LinearOperator::apply(const Matrix&) (linear_operator.hpp:28-39) */
int h2c_operator_apply_host(h2c_operator op, int transpose, int64_t b, const double* x, double* y);
/* columns_applied() / reset_counter() */
int h2c_operator_columns_applied(h2c_operator op, int64_t* cols);
int h2c_operator_reset_counter(h2c_operator op);
/* pnorm_estimate(op, 2) (linear_operator.hpp:127-153) */
int h2c_pnorm2_estimate(h2c_operator op, double* value, int* iterations);

/* ---- algebra (algebra.hpp:72-226): value semantics, new matrix out ------- */
int h2c_orthogonalize(h2c_matrix in, h2c_matrix* out);             /* algebra.hpp:72-113 */
int h2c_recompress(h2c_matrix in, double eps, h2c_matrix* out);    /* algebra.hpp:144-226 */

/* ---- HARA: replaces peel_construct(op, bt, cfg) (construction.hpp:300-382) */
typedef struct {
    double eps;                   /* 1e-4 */
    int64_t sample_block_size;    /* 16 */
    int64_t oversampling;         /* 10 */
    int64_t max_rank;             /* 0 = cap min(|t|,|s|) + b */
    uint64_t seed;                /* 42 */
    double norm_scale;            /* 0 = estimate ||op||_2 */
    int64_t crossover_rank_cap;   /* 128 */
    int rng;                      /* B200 extension: 0 = reference mt19937_64 normal stream (host,
                                     bit-compatible panels), 1 = Philox normals generated in HBM */
} h2c_peel_config;                /* PeelConfig (construction.hpp:23-31) */
typedef struct {
    int level;
    int64_t blocks, max_rank, samples;
} h2c_level_stats;                /* LevelStats (construction.hpp:33-38) */
void h2c_peel_config_default(h2c_peel_config* cfg);
/* stats: total columns (== op counter delta), per-level rows into `levels`
 * (up to max_levels; *num_levels = count); op_ms / total_ms: host wall time
 * spent in operator applies / in the whole build (any may be NULL) */
int h2c_peel_construct(h2c_operator op, h2c_block_tree bt, const h2c_peel_config* cfg, h2c_matrix* out,
                       int64_t* total_samples, h2c_level_stats* levels, int max_levels, int* num_levels,
                       double* op_ms, double* total_ms);
/* estimate_relative_error(op, h, op_norm) (construction.hpp:537-546) */
int h2c_estimate_relative_error(h2c_operator op, h2c_matrix h, double op_norm, double* out);

/* ---- block-level construction primitives (construction.hpp:137-198) ----
 * The reference threads one std::mt19937_64 through its samplers by reference;
 * h2c_rng is that stream (normals drawn exactly as detail::fill_gaussian). */
typedef struct h2c_rng_s* h2c_rng;
int h2c_rng_create(uint64_t seed, h2c_rng* out);
/* rows x cols normals from the stream, column-major host buffer (a fresh
 * normal_distribution per call, exactly detail::fill_gaussian; host only) */
int h2c_rng_fill_gaussian(h2c_rng r, int64_t rows, int64_t cols, double* out);
/* engine state as libstdc++ writes it (operator<< of std::mt19937_64): lets a
 * C++ caller lend its own std::mt19937_64 to a sampler and take it back
 * advanced, exactly as the reference's `std::mt19937_64& rng` arguments work.
 * get: *bytes = required size incl. the terminator; written when buf is large enough */
int h2c_rng_set_state(h2c_rng r, const char* state);
int h2c_rng_get_state(h2c_rng r, char* buf, int64_t* bytes);
void h2c_rng_destroy(h2c_rng r);
/* sample_block_column(op, ct, t, s, count, rng) (construction.hpp:137-148):
 * omega_s (|s| x count, ld |s|) and y_t = op(Omega) on the rows of t
 * (|t| x count, ld |t|); device buffers, cluster (internal) row order */
int h2c_sample_block_column(h2c_operator op, h2c_cluster_tree ct, int t, int s, int64_t count, h2c_rng rng,
                            double* omega_s, double* y_t, void* stream);
/* the same with host output buffers (synchronous) */
int h2c_sample_block_column_host(h2c_operator op, h2c_cluster_tree ct, int t, int s, int64_t count, h2c_rng rng,
                                 double* omega_s, double* y_t);
/* adaptive_block_factorization(op, ct, t, s, eps_block, cfg) (construction.hpp:156-198);
 * BlockFactor (:150-154): u (|t| x rank, orthonormal), v (|s| x rank), err_est.
 * A rank above cfg->max_rank returns H2C_MAX_RANK_ERROR (max_rank_error). */
typedef struct h2c_block_factor_s* h2c_block_factor;
int h2c_adaptive_block_factorization(h2c_operator op, h2c_cluster_tree ct, int t, int s, double eps_block,
                                     const h2c_peel_config* cfg, h2c_block_factor* out);
int h2c_block_factor_info(h2c_block_factor f, int64_t* rows_u, int64_t* rows_v, int64_t* rank, double* err_est);
/* u, v to host buffers (column-major, cluster row order) */
int h2c_block_factor_download(h2c_block_factor f, double* u, double* v);
void h2c_block_factor_destroy(h2c_block_factor f);

/* ---- algebra and diagnostics (algebra.hpp:119-137, 323-332; h2_matrix.hpp:128-196, 308-404) */
/* local_low_rank_update(h, t, s, U, V, eps): U (|t| x k, ld ldu), V (|s| x k, ld ldv)
 * device factors in cluster (internal) row order, added on the (t, s) region
 * (a block-tree node), then recompressed to eps */
int h2c_local_low_rank_update(h2c_matrix h, int t, int s, int64_t k, const double* U, int64_t ldu, const double* V,
                              int64_t ldv, double eps, h2c_matrix* out);
/* host-buffer forms of low_rank_update (X, Y: n x k user order) and
 * local_low_rank_update (U: |t| x k, V: |s| x k cluster order), ld = rows */
int h2c_low_rank_update_host(h2c_matrix h, int64_t k, const double* X, const double* Y, double eps, h2c_matrix* out);
int h2c_local_low_rank_update_host(h2c_matrix h, int t, int s, int64_t k, const double* U, const double* V, double eps,
                                   h2c_matrix* out);
/* frobenius_norm(h): requires orthonormal bases (H2C_INVALID_ARGUMENT otherwise) */
int h2c_frobenius_norm(h2c_matrix h, double* out);
/* H2Matrix::to_dense(cap): n x n host buffer, column-major, user ordering;
 * H2C_INVALID_ARGUMENT when n > cap */
int h2c_to_dense(h2c_matrix h, int64_t cap, double* a);
/* H2Matrix::validate(ortho_cap) -> ValidationReport: *num_violations, the
 * messages '\n'-separated into `messages` (truncated to message_bytes incl.
 * the terminator), rank_profile() into level_max_rank (up to max_levels;
 * *num_levels = depth + 1) and storage() as {dense, leaf_basis, transfer,
 * coupling} reals. Any output pointer may be NULL. */
int h2c_validate(h2c_matrix h, int64_t ortho_cap, int* num_violations, char* messages, int64_t message_bytes,
                 int64_t* level_max_rank, int max_levels, int* num_levels, int64_t* storage);

/* ---- row-subtree sharded hgemv (one process per GPU) ------
 * Rank r of P (power of two) owns the subtree under the r-th node of tree level
 * log2 P; levels above are replicated. One hgemv = begin (owned upsweep, pack
 * the send buffer) -> an all-to-all of send/recv buffers by the caller's
 * collective layer (NCCL via torch.distributed) -> end (unpack, couplings,
 * downsweep, near-field for the owned rows of y). Buffer sizes are rows per
 * vector column: send_rows[q] * b doubles go to peer q, peers in rank order. */
typedef struct h2c_dist_plan_s* h2c_dist_plan;
int h2c_dist_plan_create(h2c_matrix h, int transpose, int nranks, int rank, h2c_dist_plan* out);
void h2c_dist_plan_destroy(h2c_dist_plan p);
/* send_rows / recv_rows: nranks entries each; owned internal row range [begin, begin + rows) */
int h2c_dist_plan_counts(h2c_dist_plan p, int64_t* send_rows, int64_t* recv_rows, int64_t* owned_begin,
                         int64_t* owned_rows);
/* kernel launches of one sharded hgemv on this rank (begin + end) */
int h2c_dist_plan_launches(h2c_dist_plan p, int* launches);
/* x: full n x b user-order device matrix (only owned rows are read) */
int h2c_dist_hgemv_begin(h2c_dist_plan p, int64_t b, const double* x, int64_t ldx, double* sendbuf, void* stream);
/* y: full n x b user-order device matrix (only owned rows are written: y = alpha H x + beta y) */
/* optional, between begin and end while the caller's exchange is in flight:
 * the near-field products whose source rows this rank owns (kept in the plan's
 * workspace; end() runs them itself when this was not called) */
int h2c_dist_hgemv_local(h2c_dist_plan p, int64_t b, void* stream);
/* begin / end on this rank's OWN rows only: x and y hold the owned_rows rows
 * (h2c_dist_plan_counts) in cluster (internal) order, leading dimensions >=
 * owned_rows -- the layout of an application that keeps each rank's slice of
 * the vectors resident on its GPU */
int h2c_dist_hgemv_begin_owned(h2c_dist_plan p, int64_t b, const double* x_owned, int64_t ldx, double* sendbuf,
                               void* stream);
int h2c_dist_hgemv_end_owned(h2c_dist_plan p, int64_t b, const double* recvbuf, double* y_owned, int64_t ldy,
                             double alpha, double beta, void* stream);
int h2c_dist_hgemv_end(h2c_dist_plan p, int64_t b, const double* recvbuf, double* y, int64_t ldy, double alpha,
                       double beta, void* stream);
/* peer transport (opt-in; NVLink P2P, no collective library): after setup,
 * begin() with sendbuf == NULL writes each send item straight into the
 * destination rank's receive buffer and signals it (system-scope release), and
 * end() with recvbuf == NULL waits for the sources' signals, unpacks and
 * acknowledges them, so the exchange needs no host call between begin and end.
 * Setup, per rank: h2c_dist_peer_alloc (receive buffer for up to max_b columns
 * + a sync block, plain cudaMalloc), h2c_dist_peer_export (128 bytes of CUDA
 * IPC handles + this rank's nranks receive offsets), exchange those among the
 * ranks (e.g. an allgather), then h2c_dist_peer_import with every rank's
 * handles (nranks x 128 bytes, rank order) and offsets (nranks x nranks, row q
 * = rank q's). Plans of all ranks living in ONE process (tests) are linked with
 * h2c_dist_peer_link instead. Every rank must use the same max_b and call
 * begin/end the same number of times with the same b (the signals count calls). */
/* the whole sharded hgemv with the exchange done inside the library on the
 * caller's NCCL communicator (an ncclComm_t of nranks ranks whose rank order is
 * the plans' ranks; every rank calls it with the same b). NCCL is resolved at
 * run time from the process (the libnccl.so.2 already loaded, i.e. the instance
 * that created the communicator), so libh2b200 does not link NCCL; the grouped
 * send / receive runs on a side stream beside the local near field. */
int h2c_dist_hgemv_nccl(h2c_dist_plan p, void* nccl_comm, int64_t b, const double* x, int64_t ldx, double* y,
                        int64_t ldy, double alpha, double beta, void* stream);
int h2c_dist_hgemv_nccl_owned(h2c_dist_plan p, void* nccl_comm, int64_t b, const double* x_owned, int64_t ldx,
                              double* y_owned, int64_t ldy, double alpha, double beta, void* stream);
int h2c_dist_peer_alloc(h2c_dist_plan p, int64_t max_b);
int h2c_dist_peer_export(h2c_dist_plan p, void* handles, int64_t* recv_off);
int h2c_dist_peer_import(h2c_dist_plan p, const void* handles, const int64_t* recv_offs);
int h2c_dist_peer_link(h2c_dist_plan* plans, int n);
/* host-only partition metadata (no device needed): owner rank per cluster node
 * (-1 = replicated top level) and the exchange items rank dst receives from
 * rank src for a matrix with the given upsweep-basis ranks (arr 0 = x rows of
 * leaf `node`, 1 = x-hat of `node`; rows per vector column). Call with
 * arr == NULL to get *count. */
int h2c_partition_owner(h2c_block_tree b, int nranks, int* owner);
int h2c_partition_exchange(h2c_block_tree b, int symmetric, int transpose, const int* up_ranks, int nranks, int src,
                           int dst, int64_t* count, int* arr, int* node, int64_t* rows);

/* ---- iterative inversion (inversion.hpp; SURVEY §8(f) "next") ------------
 * Each iterate is rebuilt by h2c_peel_construct from a sampler of hgemvs. */
/* H2Matrix::scaled_identity(bt, value) (h2_matrix.hpp:90-93) */
int h2c_scaled_identity(h2c_block_tree b, double value, h2c_matrix* out);
/* in place: H <- H + value I (diagonal dense leaves; e.g. a Tikhonov shift of a Hessian) */
int h2c_matrix_add_diagonal(h2c_matrix h, double value);
/* scaled_identity_start(a) = I / ||A||_inf (inversion.hpp:124-130) */
int h2c_scaled_identity_start(h2c_matrix a, h2c_matrix* out);
/* pnorm_estimate(op, p) for p = 1, 2 or +inf (linear_operator.hpp:127-178) */
int h2c_pnorm_estimate(h2c_operator op, double p, double* value, int* iterations);
/* ns_sampler / hyperpower_sampler / unrolled_sampler (inversion.hpp:137-208) as operators:
 * kind 0 NS, 1 hyperpower (arg = order), 2 unrolled (arg = k); xk and a must outlive it */
int h2c_sampler_operator(h2c_matrix xk, h2c_matrix a, int kind, int arg, h2c_operator* out);
/* residual_norm(a, x) = ||A X - I||_2 estimate (inversion.hpp:213-225) */
int h2c_residual_norm(h2c_matrix a, h2c_matrix x, double* out);
/* the same for two black-box operators (inversion.hpp:213-220) */
int h2c_residual_norm_op(h2c_operator a, h2c_operator x, double* out);
typedef struct {
    int iter;
    double residual, eps_k;
    int64_t samples;
    double wall_seconds;
} h2c_trace_row;   /* TraceRow (inversion.hpp:19-25) */
/* h_newton_schulz (method 0), h_hyperpower (1, arg = order), h_unrolled (2, arg = k)
 * (inversion.hpp:281-311); schedule: dynamic 0/1 + eps_initial (ThresholdSchedule :50-54).
 * On H2C_DIVERGENCE_ERROR the trace so far is still returned. */
int h2c_h_inverse(h2c_matrix a, h2c_matrix x0, int method, int arg, int dynamic_schedule, double eps_initial,
                  double eps, const h2c_peel_config* cfg, int max_iter, h2c_matrix* out, h2c_trace_row* rows,
                  int max_rows, int* num_rows, double* final_residual, int* converged);
/* low_rank_update(h, {X, Y}, eps) (algebra.hpp:334-346); X, Y device n x k user order */
int h2c_low_rank_update(h2c_matrix h, int64_t k, const double* X, const double* Y, double eps, h2c_matrix* out);
/* desymmetrized() (h2_matrix.hpp:200-216) */
int h2c_desymmetrized(h2c_matrix h, h2c_matrix* out);

/* ---- global randomized low-rank and the hybrid constructor
 *      (construction.hpp:386-534; SURVEY §8(f) "next") ------------------ */
typedef struct h2c_lowrank_s* h2c_lowrank;
/* randomized_lowrank(op, eps, max_rank, cfg) (construction.hpp:484-491) */
int h2c_randomized_lowrank(h2c_operator op, double eps, int64_t max_rank, const h2c_peel_config* cfg,
                           h2c_lowrank* out);
int h2c_lowrank_info(h2c_lowrank f, int64_t* n, int64_t* rank, int* symmetric_form, double* residual_estimate,
                     int* max_rank_reached, int64_t* total_samples);
/* factor X Y^T to host buffers (n x rank, column-major, user ordering) */
int h2c_lowrank_download(h2c_lowrank f, double* X, double* Y);
void h2c_lowrank_destroy(h2c_lowrank f);
/* hybrid_construct(op, bt, cfg) (construction.hpp:506-534) */
int h2c_hybrid_construct(h2c_operator op, h2c_block_tree bt, const h2c_peel_config* cfg, h2c_matrix* out,
                         int64_t* global_rank, int64_t* total_samples, h2c_level_stats* levels, int max_levels,
                         int* num_levels);

/* ---- H2M1 container (serialize.hpp; SURVEY §8(f) "next"): byte-compatible
 *      with the reference's serialize / deserialize / write_h2_file / read_h2_file */
/* serialized size in bytes, then the bytes into a caller buffer of that size */
int h2c_serialize_size(h2c_matrix h, int64_t* bytes);
int h2c_serialize(h2c_matrix h, void* buf, int64_t bytes);
/* new block tree (rebuilt from the stored cluster tree and (eta, mode)) and matrix */
int h2c_deserialize(const void* buf, int64_t bytes, h2c_block_tree* bt_out, h2c_matrix* out);
int h2c_write_h2_file(h2c_matrix h, const char* path);
int h2c_read_h2_file(const char* path, h2c_block_tree* bt_out, h2c_matrix* out);
/* kind of the last H2C_IO_ERROR on this thread: 0 bad_magic, 1 version_mismatch, 2 truncated, 3 malformed */
int h2c_last_io_error_kind(void);

/* ---- Device black-box operator of cfg3: the 1D diffusion
 *      density-inversion Hessian at the target density, diffusion1d.hpp:62-354 */
typedef struct h2c_diff1d_s* h2c_diff1d;
typedef struct {
    int64_t n;                       /* parameter nodes on [-1, 1] */
    int64_t steps;
    double final_time, t_p, t_0, source_amplitude, alpha, beta, pad;
    int num_sources;                 /* source_positions NULL: the reference's {-0.5, 0, 0.5} */
    const double* source_positions;
    int64_t num_receivers;
} h2c_diff1d_config;                 /* Diffusion1DConfig (diffusion1d.hpp:62-73) */
void h2c_diff1d_config_default(h2c_diff1d_config* cfg);
/* Diffusion1D(cfg): stepper + cached state marches on `stream` (diffusion1d.hpp:77-112) */
int h2c_diff1d_create(const h2c_diff1d_config* cfg, void* stream, h2c_diff1d* out);
void h2c_diff1d_destroy(h2c_diff1d d);
int h2c_diff1d_info(h2c_diff1d d, int64_t* nstate, int64_t* npad, double* spacing, double* dt, int64_t* pde_solves);
/* hessvec_at_target (:173-175): y = H x, x and y n x b column-major DEVICE buffers (ld n) */
int h2c_diff1d_hessvec(h2c_diff1d d, int include_tv, int64_t b, const double* x, double* y, void* stream);
/* cached state field of one source at the physical nodes, n x (steps+1) column-major, to host */
int h2c_diff1d_state_field(h2c_diff1d d, int source, double* out);
/* hessian_operator(include_tv) (:177-181); the operator keeps the problem alive */
int h2c_diff1d_operator(h2c_diff1d d, int include_tv, h2c_operator* out);

/* ---- Device black-box operator "surface<N>" (registry.hpp:89-101): the exact
 *      minimal-surface Hessian (minimal_surface.hpp:100-140) at newton_state(steps) */
typedef struct h2c_surface_s* h2c_surface;
/* MinimalSurface(interior, rim) (minimal_surface.hpp:22-43) at newton_state(newton_steps) (:144-161) */
int h2c_surface_create(int64_t interior, double rim, int newton_steps, h2c_surface* out);
void h2c_surface_destroy(h2c_surface s);
/* n = interior^2 unknowns, nonzeros of the assembled Hessian, grid spacing h */
int h2c_surface_info(h2c_surface s, int64_t* n, int64_t* nnz, double* spacing);
/* the interior surface the Hessian is taken at (n doubles, host) */
int h2c_surface_state(h2c_surface s, double* out);
/* y = H x (hessian_operator, :163-167): x and y n x b column-major DEVICE buffers (ld n) */
int h2c_surface_hessvec(h2c_surface s, int64_t b, const double* x, double* y, void* stream);
/* hessian_operator (:163-167); the operator keeps the problem alive */
int h2c_surface_operator(h2c_surface s, h2c_operator* out);

/* ---- Device black-box operator "advdiff-<G>" (registry.hpp:125-150): the misfit
 *      Hessian of the stationary advection-diffusion source inversion (advdiff2d.hpp) */
typedef struct h2c_advdiff_s* h2c_advdiff;
typedef struct {
    int64_t grid;                    /* unknowns per side */
    double kappa, reaction;
    int64_t num_observations;
    double noise_rel;
    uint64_t obs_seed;
} h2c_advdiff_config;                /* AdvDiff2DConfig (advdiff2d.hpp:21-28) */
void h2c_advdiff_config_default(h2c_advdiff_config* cfg);
/* AdvDiff2D(cfg) (advdiff2d.hpp:35-40): operator, observation pick, noise calibration */
int h2c_advdiff_create(const h2c_advdiff_config* cfg, h2c_advdiff* out);
void h2c_advdiff_destroy(h2c_advdiff a);
/* n, sigma, number of observations, solves counted as the reference counts them */
int h2c_advdiff_info(h2c_advdiff a, int64_t* n, double* sigma, int64_t* num_observations, int64_t* solves);
/* the sorted observation nodes (num_observations int64, host) */
int h2c_advdiff_observations(h2c_advdiff a, int64_t* out);
/* misfit_hessvec (:54-64): y = H x, x and y n x b column-major DEVICE buffers (ld n) */
int h2c_advdiff_hessvec(h2c_advdiff a, int64_t b, const double* x, double* y, void* stream);
/* hessian_operator (:66-68); the operator keeps the problem alive */
int h2c_advdiff_operator(h2c_advdiff a, h2c_operator* out);

#ifdef __cplusplus
}
#endif

#endif /* H2C_H */
