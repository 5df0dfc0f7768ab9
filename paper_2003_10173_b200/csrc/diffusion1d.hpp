#pragma once
// Device black-box operator of BASELINE cfg3: the Hessian of the 1D diffusion
// density inversion at the data-generating density
// (proj/include/h2/oracles/diffusion1d.hpp:165-181, 279-342; registry
// "diff1d-<n>", registry.hpp:104-124), so HARA's operator applies stay in HBM
// instead of crossing PCIe to a host callback.
//
// Every time step is a Crank-Nicolson update x' = A+^{-1}(A- x + f) with the
// reference's tridiagonal LU factors (grid.hpp:53-73). The solve runs as a
// chunked affine recurrence: each thread owns L rows of one column, solves
// them locally with zero boundary carries, and a per-column scan over the
// chunk boundaries supplies the exact carries (the LU recurrences are affine
// maps y_i = r_i - m_i y_{i-1}, x_i = y_i/d_i - beta_i x_{i+1}; splitting them
// into chunks is exact algebra, only the rounding order differs).
#include <memory>
#include <vector>

#include "hara.hpp"

namespace h2b {

struct Diff1DConfig {   // Diffusion1DConfig, diffusion1d.hpp:62-73
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

class Diffusion1DDev {
public:
    // builds the stepper and marches the cached state fields at the target
    // density on `s` (diffusion1d.hpp:77-112)
    Diffusion1DDev(const Diff1DConfig& cfg, cudaStream_t s);

    int64_t n() const { return c_.n; }
    int64_t nstate() const { return ns_; }
    int64_t npad() const { return npad_; }
    double spacing() const { return h_; }
    double dt() const { return dt_; }
    int num_sources() const { return int(src_.size()); }
    int num_receivers() const { return int(rcv_.size()); }
    const Diff1DConfig& config() const { return c_; }
    long pde_solves() const { return marches_; }   // diffusion1d.hpp:121
    const std::vector<double>& rho_target() const { return rho_; }

    // y = H x at the target (hessvec_at_target, :173-175); x, y: n x b
    // column-major device buffers (ld n), user ordering = grid order
    void hessvec(bool include_tv, int64_t b, const double* x, double* y, cudaStream_t s);
    // cached state field of one source at the physical nodes: n x (steps+1), column-major
    std::vector<double> state_field(int source, cudaStream_t s) const;

private:
    void march_states(cudaStream_t s);

    Diff1DConfig c_;
    int64_t npad_ = 0, ns_ = 0, P_ = 0;
    double h_ = 0, dt_ = 0, moff_ = 0;
    std::vector<int64_t> src_, rcv_;
    std::vector<double> rho_, srcval_;
    DeviceArray<double> coef_;      // per padded row: mdiag, cu, cl, mult, rdfac, beta, wg, hb
    DeviceArray<double> chunk_;     // per chunk: G, WG, HB
    DeviceArray<double> tvw_;       // TV second-variation weight per edge (:31-32)
    DeviceArray<int64_t> rows_;     // source rows then receiver rows
    DeviceArray<double> u_;         // state at physical nodes: [step][k][source]
    DeviceArray<double> du_;        // u_{j+1} - u_j: [step][k][source]
    long marches_ = 0;
};

// hessian_operator(include_tv) (diffusion1d.hpp:177-181): symmetric, no transpose
std::unique_ptr<DevOperator> diffusion_hessian_operator(std::shared_ptr<Diffusion1DDev> d, bool include_tv);

}  // namespace h2b
