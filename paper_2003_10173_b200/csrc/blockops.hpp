#pragma once
// Block-level construction primitives and H^2 diagnostics on the B200 -- the
// device counterparts of
//   sample_block_column            construction.hpp:137-148
//   adaptive_block_factorization   construction.hpp:156-198 (+ BlockFactor :150-154)
//   local_low_rank_update          algebra.hpp:323-332
//   frobenius_norm                 algebra.hpp:119-137
//   H2Matrix::to_dense             h2_matrix.hpp:128-163
//   H2Matrix::validate / storage / rank_profile   h2_matrix.hpp:167-196, 308-404
#include <random>
#include <string>
#include <vector>

#include "hara.hpp"
#include "la.hpp"

namespace h2b {

// Omega (|s| x count, i.i.d. N(0,1) from `rng`, the reference stream) on the
// rows of cluster s, zeros elsewhere; writes omega_s (|s| x count, ld |s|) and
// y_t = op(Omega) restricted to the rows of t (|t| x count, ld |t|), both device.
void sample_block_column(DevOperator& op, const ClusterTree& ct, int t, int s, int64_t count, std::mt19937_64& rng,
                         double* omega_s, double* y_t, cudaStream_t st);

struct BlockFactorDev {   // construction.hpp:150-154
    la::DBuf u, v;         // |t| x rank (orthonormal), |s| x rank; internal order of the clusters
    int64_t rank = 0;
    double err_est = 0;
};
BlockFactorDev adaptive_block_factorization(DevOperator& op, const ClusterTree& ct, int t, int s, double eps_block,
                                            const PeelConfig& cfg, cudaStream_t st);

// U_blk (|t| x k, ld ldu) V_blk^T (|s| x k) added on the (t, s) region, then
// recompressed to eps (value semantics; device factors in cluster order)
std::unique_ptr<H2Dev> local_low_rank_update(const H2Dev& h, int t, int s, int64_t k, const double* U, int64_t ldu,
                                             const double* V, int64_t ldv, double eps, cudaStream_t st);

double frobenius_norm(const H2Dev& h, cudaStream_t st);

// dense n x n expansion in USER ordering into host memory (column-major)
void to_dense(const H2Dev& h, int64_t cap, double* out_host, cudaStream_t st);

struct StorageReportDev {
    int64_t dense_reals = 0, leaf_basis_reals = 0, transfer_reals = 0, coupling_reals = 0;
};
struct ValidationReportDev {
    std::vector<std::string> violations;
    std::vector<int64_t> level_max_rank;
    StorageReportDev storage;
};
StorageReportDev storage_report(const H2Dev& h);
std::vector<int64_t> rank_profile(const H2Dev& h);
ValidationReportDev validate(const H2Dev& h, int64_t ortho_cap, cudaStream_t st);

}  // namespace h2b
