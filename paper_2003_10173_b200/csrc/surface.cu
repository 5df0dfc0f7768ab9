// Device minimal-surface Hessian operator (surface.hpp): host assembly of the
// reference's exact sparse Hessian (proj/include/h2/oracles/minimal_surface.hpp),
// CSR in HBM, one SpMV launch per application.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <stdexcept>

#include "surface.hpp"

namespace h2b {

namespace {

// y(:, c) = H x(:, c): one thread per (row, column); the row's entries are
// summed in ascending column order, a warp's rows are consecutive (coalesced
// x / y accesses within a column)
__global__ void csr_spmv_kernel(const int64_t* __restrict__ rp, const int* __restrict__ ci,
                                const double* __restrict__ val, int64_t n, const double* __restrict__ x,
                                double* __restrict__ y) {
    const int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (r >= n) return;
    const int64_t c = blockIdx.y;
    const double* xc = x + c * n;
    double acc = 0.0;
    for (int64_t k = rp[r]; k < rp[r + 1]; ++k) acc = fma(__ldg(val + k), __ldg(xc + ci[k]), acc);
    y[c * n + r] = acc;
}

// Cholesky solve with the lower band of an SPD matrix of half-bandwidth w
// (the Newton direction of newton_state, minimal_surface.hpp:149-152; the
// reference uses Eigen's SimplicialLLT: same factorization, other ordering)
std::vector<double> band_cholesky_solve(const std::vector<int64_t>& rp, const std::vector<int>& ci,
                                        const std::vector<double>& v, int64_t n, int64_t w,
                                        const std::vector<double>& rhs) {
    std::vector<double> L(size_t(n) * size_t(w + 1), 0.0);   // L(i, i - k) at [i (w+1) + k]
    auto at = [&](int64_t i, int64_t j) -> double& { return L[size_t(i * (w + 1) + (i - j))]; };
    for (int64_t i = 0; i < n; ++i)
        for (int64_t k = rp[size_t(i)]; k < rp[size_t(i) + 1]; ++k) {
            const int64_t j = ci[size_t(k)];
            if (j <= i) {
                if (i - j > w) throw std::runtime_error("minimal surface: Hessian wider than its band");
                at(i, j) = v[size_t(k)];
            }
        }
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t j = std::max<int64_t>(0, i - w); j <= i; ++j) {
            double s = at(i, j);
            for (int64_t k = std::max<int64_t>(std::max<int64_t>(0, i - w), j - w); k < j; ++k) s -= at(i, k) * at(j, k);
            if (i == j) {
                if (!(s > 0.0)) throw std::runtime_error("minimal surface: Hessian factorization failed");
                at(i, i) = std::sqrt(s);
            } else {
                at(i, j) = s / at(j, j);
            }
        }
    }
    std::vector<double> x(rhs);
    for (int64_t i = 0; i < n; ++i) {   // L z = b
        double s = x[size_t(i)];
        for (int64_t k = std::max<int64_t>(0, i - w); k < i; ++k) s -= at(i, k) * x[size_t(k)];
        x[size_t(i)] = s / at(i, i);
    }
    for (int64_t i = n - 1; i >= 0; --i) {   // L^T x = z
        double s = x[size_t(i)];
        for (int64_t k = i + 1; k <= std::min<int64_t>(n - 1, i + w); ++k) s -= at(k, i) * x[size_t(k)];
        x[size_t(i)] = s / at(i, i);
    }
    return x;
}

}  // namespace

MinimalSurfaceDev::MinimalSurfaceDev(int64_t interior, double rim, int newton_steps) : g_(interior), rim_(rim) {
    if (interior < 4) throw std::invalid_argument("grid: need at least 4 nodes per side");   // grid.hpp:31-33
    if (newton_steps < 0) throw std::invalid_argument("minimal surface: newton_steps must be >= 0");
    const int64_t nn = g_ + 2;
    boundary_.assign(size_t(nn * nn), 0.0);
    auto B = [&](int64_t i, int64_t j) -> double& { return boundary_[size_t(i + j * nn)]; };
    auto rim_at = [&](double s) { return rim_ * std::sin(2 * M_PI * s); };   // :28-29
    const double hh = spacing();
    for (int64_t i = 0; i < nn; ++i) {   // :30-35
        const double x = hh * double(i);
        B(i, 0) = rim_at(x / 4.0);
        B(i, nn - 1) = rim_at((2.0 + (1.0 - x)) / 4.0);
    }
    for (int64_t j = 0; j < nn; ++j) {   // :36-40
        const double y = hh * double(j);
        B(nn - 1, j) = rim_at((1.0 + y) / 4.0);
        B(0, j) = rim_at((3.0 + (1.0 - y)) / 4.0);
    }
    state_ = newton_state(newton_steps);
    hessian_csr(state_, rp_, ci_, val_);
    drp_.upload(rp_);
    dci_.upload(ci_);
    dval_.upload(val_);
}

std::vector<double> MinimalSurfaceDev::field(const std::vector<double>& m) const {
    if (int64_t(m.size()) != n()) throw std::invalid_argument("minimal surface: dimension mismatch");
    const int64_t nn = g_ + 2;
    std::vector<double> f(boundary_);
    for (int64_t j = 1; j <= g_; ++j)
        for (int64_t i = 1; i <= g_; ++i) f[size_t(i + j * nn)] = m[size_t((j - 1) * g_ + (i - 1))];
    return f;
}

double MinimalSurfaceDev::value(const std::vector<double>& m) const {   // :67-78
    const std::vector<double> f = field(m);
    const int64_t nn = g_ + 2;
    const double h = spacing();
    double j = 0;
    for (int64_t cy = 0; cy + 1 < nn; ++cy)
        for (int64_t cx = 0; cx + 1 < nn; ++cx) {
            const double f0 = f[size_t(cx + cy * nn)];
            const double gx = (f[size_t(cx + 1 + cy * nn)] - f0) / h;
            const double gy = (f[size_t(cx + (cy + 1) * nn)] - f0) / h;
            j += h * h * std::sqrt(1.0 + gx * gx + gy * gy);
        }
    return j;
}

std::vector<double> MinimalSurfaceDev::gradient(const std::vector<double>& m) const {   // :80-98
    const std::vector<double> f = field(m);
    const int64_t nn = g_ + 2;
    const double h = spacing();
    std::vector<double> g(size_t(nn * nn), 0.0);
    for (int64_t cy = 0; cy + 1 < nn; ++cy)
        for (int64_t cx = 0; cx + 1 < nn; ++cx) {
            const double f0 = f[size_t(cx + cy * nn)];
            const double gx = (f[size_t(cx + 1 + cy * nn)] - f0) / h;
            const double gy = (f[size_t(cx + (cy + 1) * nn)] - f0) / h;
            const double r = h / std::sqrt(1.0 + gx * gx + gy * gy);
            g[size_t(cx + 1 + cy * nn)] += r * gx;
            g[size_t(cx + cy * nn)] -= r * (gx + gy);
            g[size_t(cx + (cy + 1) * nn)] += r * gy;
        }
    std::vector<double> out(static_cast<size_t>(n()));
    for (int64_t j = 1; j <= g_; ++j)
        for (int64_t i = 1; i <= g_; ++i) out[size_t((j - 1) * g_ + (i - 1))] = g[size_t(i + j * nn)];
    return out;
}

void MinimalSurfaceDev::hessian_csr(const std::vector<double>& m, std::vector<int64_t>& rp, std::vector<int>& ci,
                                    std::vector<double>& v) const {   // :100-140
    const std::vector<double> f = field(m);
    const int64_t nn = g_ + 2;
    const double h = spacing();
    auto interior_index = [&](int64_t i, int64_t j) -> int64_t {
        if (i < 1 || i > g_ || j < 1 || j > g_) return -1;
        return (j - 1) * g_ + (i - 1);
    };
    struct Trip {
        int64_t r;
        int c;
        double v;
    };
    std::vector<Trip> trip;
    trip.reserve(size_t(9 * n()));
    const double gxd[3] = {-1.0 / h, 1.0 / h, 0.0};
    const double gyd[3] = {-1.0 / h, 0.0, 1.0 / h};
    for (int64_t cy = 0; cy + 1 < nn; ++cy)
        for (int64_t cx = 0; cx + 1 < nn; ++cx) {
            const double f0 = f[size_t(cx + cy * nn)];
            const double gx = (f[size_t(cx + 1 + cy * nn)] - f0) / h;
            const double gy = (f[size_t(cx + (cy + 1) * nn)] - f0) / h;
            const double f2 = 1.0 + gx * gx + gy * gy;
            const double fr = std::sqrt(f2);
            // d2/dg2 of sqrt(1+|g|^2): (f^2 I - g g^T) / f^3
            const double wxx = (f2 - gx * gx) / (f2 * fr);
            const double wyy = (f2 - gy * gy) / (f2 * fr);
            const double wxy = -gx * gy / (f2 * fr);
            const int64_t id[3] = {interior_index(cx, cy), interior_index(cx + 1, cy), interior_index(cx, cy + 1)};
            for (int a = 0; a < 3; ++a) {
                if (id[a] < 0) continue;
                for (int b = 0; b < 3; ++b) {
                    if (id[b] < 0) continue;
                    const double val = h * h *
                                       (wxx * gxd[a] * gxd[b] + wyy * gyd[a] * gyd[b] +
                                        wxy * (gxd[a] * gyd[b] + gyd[a] * gxd[b]));
                    if (val != 0.0) trip.push_back({id[a], int(id[b]), val});
                }
            }
        }
    // rows in order; within a row, columns ascending, duplicates summed in insertion order
    const int64_t N = n();
    std::vector<int64_t> cnt(size_t(N) + 1, 0);
    for (const Trip& t : trip) ++cnt[size_t(t.r) + 1];
    for (int64_t i = 0; i < N; ++i) cnt[size_t(i) + 1] += cnt[size_t(i)];
    std::vector<Trip> byrow(trip.size());
    std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
    for (const Trip& t : trip) byrow[size_t(fill[size_t(t.r)]++)] = t;
    rp.assign(size_t(N) + 1, 0);
    ci.clear();
    v.clear();
    for (int64_t i = 0; i < N; ++i) {
        auto b0 = byrow.begin() + cnt[size_t(i)], b1 = byrow.begin() + cnt[size_t(i) + 1];
        std::stable_sort(b0, b1, [](const Trip& a, const Trip& b) { return a.c < b.c; });
        for (auto it = b0; it != b1; ++it) {
            if (!ci.empty() && int64_t(ci.size()) > rp[size_t(i)] && ci.back() == it->c) v.back() += it->v;
            else {
                ci.push_back(it->c);
                v.push_back(it->v);
            }
        }
        rp[size_t(i) + 1] = int64_t(ci.size());
    }
}

std::vector<double> MinimalSurfaceDev::newton_state(int steps) const {   // :144-161
    std::vector<double> m(static_cast<size_t>(n()), 0.0);
    for (int it = 0; it < steps; ++it) {
        const std::vector<double> g = gradient(m);
        std::vector<int64_t> rp;
        std::vector<int> ci;
        std::vector<double> v;
        hessian_csr(m, rp, ci, v);
        const std::vector<double> dir = band_cholesky_solve(rp, ci, v, n(), g_, g);
        double alpha = 1.0;
        const double j0 = value(m);
        auto trial = [&](double a) {
            std::vector<double> t(m);
            for (size_t q = 0; q < t.size(); ++q) t[q] -= a * dir[q];
            return t;
        };
        while (alpha > 1e-6 && value(trial(alpha)) >= j0) alpha /= 2;
        m = trial(alpha);
    }
    return m;
}

void MinimalSurfaceDev::hessvec(int64_t b, const double* x, double* y, cudaStream_t s) const {
    if (b < 1) throw std::invalid_argument("hessvec: dimension mismatch");
    const int64_t N = n();
    for (int64_t c0 = 0; c0 < b; c0 += 65535) {   // grid.y limit
        const int64_t bc = std::min<int64_t>(65535, b - c0);
        csr_spmv_kernel<<<dim3(unsigned((N + 255) / 256), unsigned(bc)), 256, 0, s>>>(
            drp_.data(), dci_.data(), dval_.data(), N, x + c0 * N, y + c0 * N);
        H2B_LAUNCH();
    }
    ++applies_;
}

std::unique_ptr<DevOperator> surface_hessian_operator(std::shared_ptr<MinimalSurfaceDev> sfc) {
    const int64_t n = sfc->n();
    auto f = [sfc](bool, int64_t b, const double* x, double* y, cudaStream_t s) { sfc->hessvec(b, x, y, s); };
    return std::make_unique<FunctionDevOperator>(n, true, f, false);
}

}  // namespace h2b
