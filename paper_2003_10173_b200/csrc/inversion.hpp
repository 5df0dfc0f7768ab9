#pragma once
// Iterative approximate inversion driven by HARA and hgemv on the B200
// (reference inversion.hpp:19-311, algebra.hpp:334-346): each iterate of
// Newton-Schulz / hyperpower / unrolled NS is rebuilt by peel_construct from a
// sampler that evaluates the iteration formula with a few device hgemvs.
#include <memory>
#include <string>
#include <vector>

#include "hara.hpp"

namespace h2b {

struct ThresholdSchedule {   // inversion.hpp:50-54
    bool dynamic = false;
    double eps_initial = 1e-2;
};
double threshold_schedule(double residual, int iter, double eps_final, const ThresholdSchedule& s);   // :58-63

struct TraceRow {   // inversion.hpp:19-25
    int iter = 0;
    double residual = 0, eps_k = 0;
    long samples = 0;
    double wall_seconds = 0;
};
struct ConvergenceTrace {   // inversion.hpp:27-39
    std::vector<TraceRow> rows;
    double final_residual = 0;
    bool converged = false;
    std::vector<std::string> notes;
};
class divergence_error : public std::runtime_error {   // inversion.hpp:41-46
public:
    divergence_error(const std::string& m, ConvergenceTrace t) : std::runtime_error(m), trace(std::move(t)) {}
    ConvergenceTrace trace;
};

// H2Matrix::diagonal / scaled_identity (h2_matrix.hpp:78-93)
std::unique_ptr<H2Dev> scaled_identity(std::shared_ptr<const BlockTree> bt, double value, cudaStream_t s);
// H <- H + value I on the diagonal dense leaves (regularisation shift; in place)
void add_diagonal(H2Dev& h, double value, cudaStream_t s);
// pnorm_estimate(op, 1 / inf) (linear_operator.hpp:155-178)
NormEstimate pnorm_1inf_estimate(DevOperator& op, bool inf, cudaStream_t s, int max_iter = 100);
// X0 = I / ||A||_inf (inversion.hpp:124-130)
std::unique_ptr<H2Dev> scaled_identity_start(const H2Dev& a, cudaStream_t s);

// samplers (inversion.hpp:137-208); xk / a must outlive the returned operator
std::unique_ptr<DevOperator> ns_sampler(const H2Dev& xk, const H2Dev& a);
std::unique_ptr<DevOperator> hyperpower_sampler(const H2Dev& xk, const H2Dev& a, int order);
std::unique_ptr<DevOperator> unrolled_sampler(const H2Dev& x0, const H2Dev& a, int k);

// |A X - I|_2 (inversion.hpp:213-225)
double residual_norm(DevOperator& a, DevOperator& x, cudaStream_t s);
double residual_norm(const H2Dev& a, const H2Dev& x, cudaStream_t s);

struct InverseResult {
    std::unique_ptr<H2Dev> X;
    ConvergenceTrace trace;
};
// kind 0 Newton-Schulz, 1 hyperpower (order), inversion.hpp:236-300
InverseResult h_iterative_inverse(const H2Dev& a, const H2Dev& x0, const ThresholdSchedule& sched, double eps,
                                  const PeelConfig& cfg, int kind, int order, int max_iter, cudaStream_t s);
InverseResult h_unrolled(const H2Dev& a, const H2Dev& x0, int k, double eps, const PeelConfig& cfg,
                         cudaStream_t s);   // inversion.hpp:303-311

// desymmetrized copy (h2_matrix.hpp:200-216): column basis = row basis, every block stored
std::unique_ptr<H2Dev> desymmetrized(const H2Dev& h, cudaStream_t s);
// low_rank_update(h, {X, Y}, eps) (algebra.hpp:334-346): H + X Y^T recompressed;
// X, Y: n x k device matrices in user ordering (ld n)
std::unique_ptr<H2Dev> low_rank_update(const H2Dev& h, const double* X, const double* Y, int k, double eps,
                                       cudaStream_t s);

}  // namespace h2b
