#pragma once
// Device black-box operator "advdiff-<G>" of the reference registry
// (proj/include/h2/oracles/advdiff2d.hpp, registry.hpp:125-150): the misfit
// Hessian of the linear source inversion in stationary advection-diffusion,
// H = (1/sigma^2) C^T A^{-T} B^T B A^{-1} C with C = h^2 I and B the sampling at
// the observation nodes (advdiff2d.hpp:5-11).
//
// The reference applies H with one forward and one adjoint sparse LU solve per
// application (:54-64). H is parameter independent and has rank <= #observations,
// so the B200 build forms the observation factor G = (h / sigma)^... exactly once:
// G = (h^2 / sigma) B A^{-1} (#obs x n, one adjoint solve per observation row on
// the host, banded LU of the diagonally dominant upwind operator), and every
// application is two batched GEMMs in HBM: y = G^T (G x). Same operator in exact
// arithmetic; the solve counter keeps the reference's accounting (two per
// application).
#include <memory>
#include <vector>

#include "hara.hpp"

namespace h2b {

struct AdvDiffConfig {   // AdvDiff2DConfig, advdiff2d.hpp:21-28
    int64_t grid = 32;
    double kappa = 1e-3;
    double reaction = 0.5;
    int64_t num_observations = 100;
    double noise_rel = 0.01;
    uint64_t obs_seed = 7;
};

class AdvDiff2DDev {
public:
    explicit AdvDiff2DDev(const AdvDiffConfig& cfg);

    int64_t n() const { return c_.grid * c_.grid; }
    const AdvDiffConfig& config() const { return c_; }
    double sigma() const { return sigma_; }
    double spacing() const { return 1.0 / double(c_.grid + 1); }
    const std::vector<int64_t>& observation_nodes() const { return obs_; }
    long solves() const { return solves_; }

    // y = H x (misfit_hessvec, :54-64); x, y: n x b column-major device buffers (ld n)
    void misfit_hessvec(int64_t b, const double* x, double* y, cudaStream_t s);

private:
    AdvDiffConfig c_;
    std::vector<int64_t> obs_;
    double sigma_ = 1.0;
    DeviceArray<double> G_;   // #obs x n column-major
    long solves_ = 0;
};

// hessian_operator (:66-68): symmetric, no transpose
std::unique_ptr<DevOperator> advdiff_hessian_operator(std::shared_ptr<AdvDiff2DDev> a);

}  // namespace h2b
