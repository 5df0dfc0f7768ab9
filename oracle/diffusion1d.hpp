#pragma once
// ORACLE — TEST INFRASTRUCTURE ONLY. CPU restatement of the reference's 1D
// diffusion density-inversion Hessian (proj/include/h2/oracles/diffusion1d.hpp)
// at the data-generating density: the black-box operator HARA compresses in
// BASELINE cfg3 ("diff1d-262144", registry.hpp:104-124). Used as the checker
// for the device operator (paper_2003_10173_b200/csrc/diffusion1d.cu) and as
// bench.py's CPU baseline of the operator leg. Never linked by the product.
//
// Semantics followed (reference file:line):
//   grid / padding / sources / receivers / target density  diffusion1d.hpp:77-98
//   Ricker source wavelet                                   ricker.hpp:12-19
//   A+ = M/dt + K/2 (LU without pivoting), A- = M/dt - K/2   diffusion1d.hpp:212-230,
//                                                            grid.hpp:53-73
//   forward state march                                     diffusion1d.hpp:237-255
//   Hessian at the target (adjoint fields vanish, :110-111) diffusion1d.hpp:279-342
//   TV second variation                                     diffusion1d.hpp:25-38
// With p == 0 the p-terms of hessvec_with_fields (:308, :322-324) add exact
// zeros; they are omitted here, which does not change a single bit.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <thread>
#include <vector>

namespace h2ora {

struct Diff1DConfig {   // diffusion1d.hpp:62-73
    int64_t n = 512;
    double pad = 0.5;
    double final_time = 30.0;
    int64_t steps = 512;
    double t_p = 1.0;
    double t_0 = 0.0;
    double source_amplitude = 1000.0;
    double alpha = 3e-5, beta = 1e-3;
    std::vector<double> source_positions{-0.5, 0.0, 0.5};
    int64_t num_receivers = 8;
};

inline double ricker_wavelet(double t, double t_p) {   // ricker.hpp:12-19
    if (t_p <= 0) throw std::invalid_argument("ricker: t_p must be positive");
    const double u = M_PI * (t - 1.4 * t_p) / t_p;
    const double a = u * u;
    return (a - 0.5) * std::exp(-a);
}

class Diff1DOracle {
public:
    explicit Diff1DOracle(Diff1DConfig cfg) : c_(std::move(cfg)) {
        if (c_.n < 8) throw std::invalid_argument("diffusion1d: n too small");
        h_ = 2.0 / double(c_.n - 1);
        npad_ = std::max<int64_t>(int64_t(std::lround(c_.pad / h_)), 2);
        ns_ = c_.n + 2 * npad_ - 2;
        dt_ = c_.final_time / double(c_.steps);
        for (double xs : c_.source_positions) src_.push_back(npad_ + nearest(xs) - 1);
        for (int64_t r = 0; r < c_.num_receivers; ++r)
            rcv_.push_back(npad_ + nearest(-0.875 + 1.75 * double(r) / double(c_.num_receivers - 1)) - 1);
        rho_.resize(size_t(c_.n));
        for (int64_t i = 0; i < c_.n; ++i) {
            // the reference's default build (-march=native, GNU dialect) contracts
            // -1.0 + h_ * double(i) (diffusion1d.hpp:96) into one FMA; the node at
            // x = -1/3 (n = 3m + 1) is classified by that rounding
            const double x = std::fma(h_, double(i), -1.0);
            rho_[size_t(i)] = x < -1.0 / 3.0 ? 1.0 : (x <= 1.0 / 3.0 ? 2.5 : 1.2);
        }
        build_stepper();
        march_states();
    }

    int64_t n() const { return c_.n; }
    int64_t nstate() const { return ns_; }
    int64_t npad() const { return npad_; }
    double spacing() const { return h_; }
    double dt() const { return dt_; }
    long pde_solves() const { return marches_; }
    const std::vector<double>& rho_target() const { return rho_; }
    // u(i, j) of one source, nstate x (steps + 1) column-major
    const std::vector<double>& state(size_t s) const { return u_[s]; }

    // y (n x b, column-major) = H x at the target, misfit (+ TV)
    void hessvec(int64_t b, const double* x, double* y, bool include_tv, int nthreads = 1) const {
        for (int64_t i = 0; i < c_.n * b; ++i) y[i] = 0.0;
        const size_t S = src_.size();
        // the reference accumulates out += c (acc_p + acc_q) source by source
        // (:336); columns are independent, so split them over threads
        auto work = [&](int64_t c0, int64_t c1) {
            const size_t nsz = static_cast<size_t>(ns_);
            std::vector<double> v(nsz), q(nsz), rhs(nsz);
            std::vector<double> vr(static_cast<size_t>((c_.steps + 1) * c_.num_receivers));
            std::vector<double> accq(static_cast<size_t>(c_.n));
            const double c = h_ / dt_;
            for (int64_t col = c0; col < c1; ++col) {
                const double* nu = x + col * c_.n;
                double* out = y + col * c_.n;
                for (size_t s = 0; s < S; ++s) {
                    const std::vector<double>& u = u_[s];
                    auto U = [&](int64_t i, int64_t j) { return u[size_t(i + j * ns_)]; };
                    // incremental state, forward (:297-313)
                    std::fill(v.begin(), v.end(), 0.0);
                    std::fill(vr.begin(), vr.end(), 0.0);
                    for (int64_t j = 0; j < c_.steps; ++j) {
                        apply_minus(v.data(), rhs.data());
                        for (int64_t k = 0; k < c_.n; ++k) {
                            const int64_t sk = npad_ + k - 1;
                            rhs[size_t(sk)] -= c * (nu[k] * (U(sk, j + 1) - U(sk, j)));
                        }
                        solve(rhs.data());
                        v.swap(rhs);
                        for (int64_t r = 0; r < c_.num_receivers; ++r)
                            vr[size_t((j + 1) * c_.num_receivers + r)] = v[size_t(rcv_[size_t(r)])];
                    }
                    // incremental adjoint, backward (:317-333)
                    std::fill(q.begin(), q.end(), 0.0);
                    std::fill(accq.begin(), accq.end(), 0.0);
                    for (int64_t j = c_.steps; j >= 1; --j) {
                        if (j == c_.steps)
                            std::fill(rhs.begin(), rhs.end(), 0.0);
                        else
                            apply_minus(q.data(), rhs.data());
                        for (int64_t r = 0; r < c_.num_receivers; ++r)
                            rhs[size_t(rcv_[size_t(r)])] -= quad_weight(j) * vr[size_t(j * c_.num_receivers + r)];
                        solve(rhs.data());
                        q.swap(rhs);
                        for (int64_t k = 0; k < c_.n; ++k) {
                            const int64_t sk = npad_ + k - 1;
                            accq[size_t(k)] += q[size_t(sk)] * (U(sk, j) - U(sk, j - 1));
                        }
                    }
                    for (int64_t k = 0; k < c_.n; ++k) out[k] += c * (0.0 + accq[size_t(k)]);
                }
                if (include_tv) tv_hessvec(nu, out);
            }
        };
        nthreads = int(std::max<int64_t>(1, std::min<int64_t>(nthreads, b)));
        if (nthreads == 1) {
            work(0, b);
        } else {
            std::vector<std::thread> th;
            for (int t = 0; t < nthreads; ++t)
                th.emplace_back(work, b * t / nthreads, b * (t + 1) / nthreads);
            for (auto& t : th) t.join();
        }
        marches_ += long(2 * S);
    }

private:
    int64_t nearest(double x) const {   // :184-186
        return std::clamp<int64_t>(int64_t(std::lround((x + 1.0) / h_)), 0, c_.n - 1);
    }
    double quad_weight(int64_t j) const { return (j == 0 || j == c_.steps) ? dt_ / 2 : dt_; }   // :188-190

    void build_stepper() {   // :212-230 and grid.hpp:53-64
        std::vector<double> re(size_t(ns_), 1.0);
        for (int64_t k = 0; k < c_.n; ++k) re[size_t(npad_ + k - 1)] = rho_[size_t(k)];
        const double koff = -1.0 / h_, kdiag = 2.0 / h_;
        off_ = koff / 2;
        mdiag_.resize(size_t(ns_));
        mult_.assign(size_t(ns_), 0.0);
        dfac_.resize(size_t(ns_));
        for (int64_t i = 0; i < ns_; ++i) {
            dfac_[size_t(i)] = h_ * re[size_t(i)] / dt_ + kdiag / 2;
            mdiag_[size_t(i)] = h_ * re[size_t(i)] / dt_ - kdiag / 2;
        }
        for (int64_t i = 1; i < ns_; ++i) {
            mult_[size_t(i)] = off_ / dfac_[size_t(i - 1)];
            dfac_[size_t(i)] = dfac_[size_t(i)] - mult_[size_t(i)] * off_;
            if (dfac_[size_t(i)] == 0) throw std::runtime_error("tridiagonal solve: singular matrix");
        }
        moff_ = -koff / 2;
    }
    void apply_minus(const double* x, double* y) const {   // Stepper::apply_minus :203-209
        for (int64_t i = 0; i < ns_; ++i) y[i] = mdiag_[size_t(i)] * x[i];
        for (int64_t i = 0; i + 1 < ns_; ++i) y[i] += moff_ * x[i + 1];
        for (int64_t i = 1; i < ns_; ++i) y[i] += moff_ * x[i - 1];
    }
    void solve(double* y) const {   // TridiagSolver::solve_in_place, grid.hpp:67-73
        for (int64_t i = 1; i < ns_; ++i) y[i] -= mult_[size_t(i)] * y[i - 1];
        y[ns_ - 1] /= dfac_[size_t(ns_ - 1)];
        for (int64_t i = ns_ - 2; i >= 0; --i) y[i] = (y[i] - off_ * y[i + 1]) / dfac_[size_t(i)];
    }
    double source_value(double t) const {   // :232-234
        return c_.source_amplitude * ricker_wavelet(t - c_.t_0, c_.t_p);
    }
    void march_states() {   // :237-255
        u_.assign(src_.size(), std::vector<double>(size_t(ns_ * (c_.steps + 1)), 0.0));
        std::vector<double> cur(static_cast<size_t>(ns_), 0.0), rhs(static_cast<size_t>(ns_));
        for (size_t s = 0; s < src_.size(); ++s) {
            std::fill(cur.begin(), cur.end(), 0.0);
            for (int64_t j = 0; j < c_.steps; ++j) {
                apply_minus(cur.data(), rhs.data());
                rhs[size_t(src_[s])] += 0.5 * (source_value(dt_ * double(j)) + source_value(dt_ * double(j + 1)));
                solve(rhs.data());
                cur.swap(rhs);
                std::copy(cur.begin(), cur.end(), u_[s].begin() + (j + 1) * ns_);
            }
            ++marches_;
        }
    }
    // out += tv_hessvec(rho, alpha, beta, nu, h) (:25-38, added per column at :338-340)
    void tv_hessvec(const double* nu, double* out) const {
        if (c_.beta <= 0) throw std::invalid_argument("tv_hessvec: beta must be positive");
        std::vector<double> t(static_cast<size_t>(c_.n), 0.0);
        for (int64_t i = 0; i + 1 < c_.n; ++i) {
            const double g = (rho_[size_t(i + 1)] - rho_[size_t(i)]) / h_;
            const double w = c_.alpha * c_.beta / (h_ * std::pow(g * g + c_.beta, 1.5));
            const double d = nu[i + 1] - nu[i];
            t[size_t(i)] -= w * d;
            t[size_t(i + 1)] += w * d;
        }
        for (int64_t i = 0; i < c_.n; ++i) out[i] += t[size_t(i)];
    }

    Diff1DConfig c_;
    int64_t npad_ = 0, ns_ = 0;
    double h_ = 0, dt_ = 0, off_ = 0, moff_ = 0;
    std::vector<int64_t> src_, rcv_;
    std::vector<double> rho_, mdiag_, mult_, dfac_;
    std::vector<std::vector<double>> u_;
    mutable long marches_ = 0;
};

}  // namespace h2ora
