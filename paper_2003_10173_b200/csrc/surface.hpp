#pragma once
// Device black-box operator "surface<N>" of the reference registry
// (proj/include/h2/oracles/minimal_surface.hpp, registry.hpp:89-101): the exact
// Hessian of the discrete minimal-surface area functional at a damped-Newton
// surface, applied on the B200 as a sparse matrix (the reference applies the
// assembled Eigen sparse matrix, minimal_surface.hpp:163-167). The Hessian
// depends only on the surface, so it is assembled once on the host (like the
// reference) and every application is one SpMV launch over b columns in HBM.
#include <memory>
#include <vector>

#include "hara.hpp"

namespace h2b {

class MinimalSurfaceDev {
public:
    // MinimalSurface(interior, rim) at newton_state(newton_steps) (registry.hpp:89-101)
    MinimalSurfaceDev(int64_t interior, double rim, int newton_steps);

    int64_t n() const { return g_ * g_; }
    int64_t interior() const { return g_; }
    double spacing() const { return 1.0 / double(g_ + 1); }
    int64_t nnz() const { return int64_t(val_.size()); }
    const std::vector<double>& state() const { return state_; }

    // host evaluations (setup and tests): J (minimal_surface.hpp:67-78), its gradient (:80-98)
    double value(const std::vector<double>& m) const;
    std::vector<double> gradient(const std::vector<double>& m) const;

    // y = H x (hessian_operator, :163-167); x, y: n x b column-major device buffers (ld n),
    // user ordering = grid index order (grid.hpp:36)
    void hessvec(int64_t b, const double* x, double* y, cudaStream_t s) const;
    long applies() const { return applies_; }

private:
    std::vector<double> field(const std::vector<double>& m) const;   // full_field (:59-65)
    // exact sparse Hessian (:100-140) in CSR: rows in grid order, columns ascending,
    // duplicate triplets summed in insertion order (as Eigen's setFromTriplets)
    void hessian_csr(const std::vector<double>& m, std::vector<int64_t>& rp, std::vector<int>& ci,
                     std::vector<double>& v) const;
    std::vector<double> newton_state(int steps) const;   // :144-161

    int64_t g_;
    double rim_;
    std::vector<double> boundary_;   // (g+2) x (g+2), column-major: boundary_(i, j) = [i + j (g+2)]
    std::vector<double> state_;
    std::vector<int64_t> rp_;
    std::vector<int> ci_;
    std::vector<double> val_;
    DeviceArray<int64_t> drp_;
    DeviceArray<int> dci_;
    DeviceArray<double> dval_;
    mutable long applies_ = 0;
};

// hessian_operator (minimal_surface.hpp:163-167): symmetric, no transpose
std::unique_ptr<DevOperator> surface_hessian_operator(std::shared_ptr<MinimalSurfaceDev> s);

}  // namespace h2b
