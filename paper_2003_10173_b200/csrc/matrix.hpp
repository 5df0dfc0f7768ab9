#pragma once
#include <memory>

#include "h2dev.hpp"

namespace h2b {

// zero-content matrix with the given per-node ranks (nullptr = all zero,
// which is the reference's H2Matrix::zero, h2_matrix.hpp:53-75)
std::unique_ptr<H2Dev> make_h2(std::shared_ptr<const BlockTree> bt, bool symmetric, const int* row_ranks,
                               const int* col_ranks);

// packed part sizes / transfer: U, E, V, F, S, D (see h2dev.hpp for the layout)
void packed_sizes(const H2Dev& h, int64_t sizes[6]);
void upload_packed(H2Dev& h, const double* const parts[6]);
void download_packed(const H2Dev& h, double* const parts[6]);

// symmetric kernel matrix K(x,y) (kind 0 exponential, 1 Gaussian, 2 Matern-3/2,
// length scale ell) with uniform rank, generated on the device by Chebyshev
// tensor interpolation; coords n x dim column-major in user ordering
// shard_nranks > 0: only the payload of rank `shard_rank`'s row-subtree shard
std::unique_ptr<H2Dev> make_kernel_h2(std::shared_ptr<const BlockTree> bt, const double* coords, int kind,
                                      double ell, int rank, int shard_nranks = 0, int shard_rank = -1);

}  // namespace h2b
