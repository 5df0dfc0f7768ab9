#pragma once
// The reference's Gaussian sample stream (detail::fill_gaussian,
// construction.hpp:81-85; pnorm_estimate's start block, linear_operator.hpp:
// 134-138): a fresh std::normal_distribution<double>(0, 1) per call over the
// caller's std::mt19937_64, filled column by column.
#include <cstdint>
#include <random>

namespace h2b {
// m: rows x cols, column-major with leading dimension ld (host memory)
void ref_fill_gaussian(double* m, int64_t rows, int64_t cols, int64_t ld, std::mt19937_64& rng);
}  // namespace h2b
