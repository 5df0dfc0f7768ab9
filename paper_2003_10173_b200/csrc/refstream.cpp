// The reference's Gaussian sample stream, bit for bit.
//
// libstdc++'s normal_distribution (Marsaglia polar method) is a header
// template, so its arithmetic is compiled into the caller. The reference's
// Release build (-O3 -march=native, proj/CMakeLists.txt:3-20) runs on FMA
// hardware, and GCC contracts the polar method's x*x + y*y into an FMA, which
// changes the last bit of some normals. This file is therefore compiled with
// -march=x86-64-v3 (FMA on; see the Makefile) so HARA's panels in rng=0 mode
// equal the reference's exactly; tests/test_blockops_gpu.py checks them
// bitwise against the reference's own compiled code (oracle/_ref).
#include "refstream.hpp"

namespace h2b {
void ref_fill_gaussian(double* m, int64_t rows, int64_t cols, int64_t ld, std::mt19937_64& rng) {
    std::normal_distribution<double> g(0, 1);
    for (int64_t j = 0; j < cols; ++j)
        for (int64_t i = 0; i < rows; ++i) m[i + j * ld] = g(rng);
}
}  // namespace h2b
