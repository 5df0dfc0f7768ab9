// Device advection-diffusion misfit Hessian (advdiff.hpp): the reference's
// upwind operator (proj/include/h2/oracles/advdiff2d.hpp:76-110), its
// observation pick (:112-124) and noise calibration (:126-139) on the host,
// the observation factor G in HBM, two batched GEMMs per application.
#include <algorithm>
#include <cmath>
#include <random>
#include <stdexcept>

#include "advdiff.hpp"
#include "la.hpp"

namespace h2b {

namespace {

// dense band storage of a matrix with lower / upper bandwidth w: entry (i, j),
// |i - j| <= w, at [i (2w+1) + (j - i + w)]
struct Band {
    int64_t n, w;
    std::vector<double> a;
    Band(int64_t n_, int64_t w_) : n(n_), w(w_), a(size_t(n_) * size_t(2 * w_ + 1), 0.0) {}
    double& at(int64_t i, int64_t j) { return a[size_t(i * (2 * w + 1) + (j - i + w))]; }
};

// in-place LU without pivoting (the matrix is diagonally dominant), L unit lower
void band_lu(Band& m) {
    for (int64_t k = 0; k < m.n; ++k) {
        const double piv = m.at(k, k);
        if (piv == 0.0) throw std::runtime_error("advdiff: forward operator factorization failed");
        const int64_t iend = std::min(m.n - 1, k + m.w);
        for (int64_t i = k + 1; i <= iend; ++i) {
            const double l = m.at(i, k) / piv;
            m.at(i, k) = l;
            if (l == 0.0) continue;
            for (int64_t j = k + 1; j <= std::min(m.n - 1, k + m.w); ++j) m.at(i, j) -= l * m.at(k, j);
        }
    }
}

void band_solve(Band& m, std::vector<double>& x) {
    for (int64_t i = 0; i < m.n; ++i) {   // L
        double s = x[size_t(i)];
        for (int64_t j = std::max<int64_t>(0, i - m.w); j < i; ++j) s -= m.at(i, j) * x[size_t(j)];
        x[size_t(i)] = s;
    }
    for (int64_t i = m.n - 1; i >= 0; --i) {   // U
        double s = x[size_t(i)];
        for (int64_t j = i + 1; j <= std::min(m.n - 1, i + m.w); ++j) s -= m.at(i, j) * x[size_t(j)];
        x[size_t(i)] = s / m.at(i, i);
    }
}

}  // namespace

AdvDiff2DDev::AdvDiff2DDev(const AdvDiffConfig& cfg) : c_(cfg) {
    if (c_.kappa <= 0) throw std::invalid_argument("advdiff: kappa must be positive");
    if (c_.grid < 4) throw std::invalid_argument("grid: need at least 4 nodes per side");   // grid.hpp:31-33
    const int64_t g = c_.grid, N = n();
    const double h = spacing(), h2 = h * h, k = c_.kappa;
    auto at = [&](int64_t i, int64_t j) { return (j - 1) * g + (i - 1); };   // grid.hpp:36
    // A^T in band form (A's entries, :76-103, placed transposed)
    Band at_t(N, g);
    for (int64_t j = 1; j <= g; ++j)
        for (int64_t i = 1; i <= g; ++i) {
            const int64_t row = at(i, j);
            const double v1 = h * double(i), v2 = h * double(j);
            double diag = 4.0 * k / (h * h) + (v1 + v2) / h + c_.reaction;
            if (i > 1) at_t.at(at(i - 1, j), row) = -k / (h * h) - v1 / h;
            if (i < g) at_t.at(at(i + 1, j), row) = -k / (h * h);
            else diag -= k / (h * h);
            if (j > 1) at_t.at(at(i, j - 1), row) = -k / (h * h) - v2 / h;
            if (j < g) at_t.at(at(i, j + 1), row) = -k / (h * h);
            else diag -= k / (h * h);
            at_t.at(row, row) = diag;
        }
    band_lu(at_t);
    // observation nodes: std::shuffle of the interior-interior nodes (:112-124)
    std::vector<int64_t> interior;
    for (int64_t j = 2; j < g; ++j)
        for (int64_t i = 2; i < g; ++i) interior.push_back(at(i, j));
    if (c_.num_observations > int64_t(interior.size()))
        throw std::invalid_argument("advdiff: more observations than interior nodes");
    if (c_.num_observations < 0) throw std::invalid_argument("advdiff: negative number of observations");
    std::mt19937_64 rng(c_.obs_seed);
    std::shuffle(interior.begin(), interior.end(), rng);
    obs_.assign(interior.begin(), interior.begin() + c_.num_observations);
    std::sort(obs_.begin(), obs_.end());
    // W = B A^{-1}: row r = (A^{-T} e_{o_r})^T
    const int64_t R = int64_t(obs_.size());
    std::vector<double> W(size_t(R * N));   // R x N column-major
    for (int64_t r = 0; r < R; ++r) {
        std::vector<double> e(size_t(N), 0.0);
        e[size_t(obs_[size_t(r)])] = 1.0;
        band_solve(at_t, e);
        for (int64_t c = 0; c < N; ++c) W[size_t(r + c * R)] = e[size_t(c)];
    }
    // sigma = max(noise_rel * peak |u(obs)|, 1e-12), u = A^{-1} (h^2 m_true) (:126-139)
    std::vector<double> mt(static_cast<size_t>(N));
    for (int64_t j = 1; j <= g; ++j)
        for (int64_t i = 1; i <= g; ++i) {
            const double dx = h * double(i) - 0.35, dy = h * double(j) - 0.7;
            mt[size_t(at(i, j))] = std::exp(-(dx * dx + dy * dy) / (2 * 0.08 * 0.08));
        }
    double peak = 0;
    for (int64_t r = 0; r < R; ++r) {
        double u = 0;
        for (int64_t c = 0; c < N; ++c) u += W[size_t(r + c * R)] * (h2 * mt[size_t(c)]);
        peak = std::max(peak, std::abs(u));
    }
    sigma_ = std::max(c_.noise_rel * peak, 1e-12);
    // G = (h^2 / sigma) W, so that H = G^T G
    const double sc = h2 / sigma_;
    for (double& v : W) v *= sc;
    G_.upload(W);
    H2B_CUDA(cudaDeviceSynchronize());
}

void AdvDiff2DDev::misfit_hessvec(int64_t b, const double* x, double* y, cudaStream_t s) {
    if (b < 1) throw std::invalid_argument("advdiff hessvec: dimension mismatch");
    const int64_t N = n(), R = int64_t(obs_.size());
    solves_ += 2;   // the reference's accounting: one forward and one adjoint solve (:54-64)
    if (R == 0) {   // no observations: the misfit Hessian is zero
        for (int64_t c = 0; c < b; ++c) H2B_CUDA(cudaMemsetAsync(y + c * N, 0, size_t(N) * sizeof(double), s));
        return;
    }
    DeviceArray<double> z(size_t(R * b), s);
    // z = G x, y = G^T z (two batched-GEMM launches, split-K over the n rows of the first)
    la::bgemm({la::GemmDesc{G_.data(), x, z.data(), int(R), int(b), int(N), int(R), int(N), int(R), 0, 0, 1.0, 0.0}}, s);
    la::bgemm({la::GemmDesc{G_.data(), z.data(), y, int(N), int(b), int(R), int(R), int(R), int(N), 1, 0, 1.0, 0.0}}, s);
}

std::unique_ptr<DevOperator> advdiff_hessian_operator(std::shared_ptr<AdvDiff2DDev> a) {
    const int64_t n = a->n();
    auto f = [a](bool, int64_t b, const double* x, double* y, cudaStream_t s) { a->misfit_hessvec(b, x, y, s); };
    return std::make_unique<FunctionDevOperator>(n, true, f, false);
}

}  // namespace h2b
