#pragma once
// HARA (adaptive randomized peeling construction) and the H^2 algebra it
// drives, on the B200: the device counterparts of
//   LinearOperator / DenseOperator / H2Operator / pnorm_estimate  linear_operator.hpp:20-178
//   orthogonalize / recompress / apply_local_update               algebra.hpp:31-316
//   PeelConfig / peel_construct / estimate_relative_error         construction.hpp:23-382, 537-546
// Control flow (loops, thresholds, stopping rules, RNG stream) follows the
// reference line by line; every array operation runs on the device as a
// batched launch over all nodes / blocks / pairs of one tree level. Only the
// scalar decisions (kept ranks, convergence flags) cross to the host.
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "h2dev.hpp"

namespace h2b {

// black-box operator on device buffers in USER ordering (x, y: n x b, ld n);
// mirrors LinearOperator (linear_operator.hpp:20-55) incl. the column counter
class DevOperator {
public:
    DevOperator(int64_t n, bool sym) : n_(n), sym_(sym) {}
    virtual ~DevOperator() = default;
    int64_t dim() const { return n_; }
    bool symmetric() const { return sym_; }
    // y = op(x) (:28-32)
    void apply(int64_t b, const double* x, double* y, cudaStream_t s) {
        cols_ += b;
        apply_impl(false, b, x, y, s);
    }
    // y = op^T(x) (:34-39): symmetric without transpose falls back to apply
    void apply_transpose(int64_t b, const double* x, double* y, cudaStream_t s) {
        cols_ += b;
        if (sym_ && !has_transpose()) return apply_impl(false, b, x, y, s);
        if (!has_transpose()) throw std::logic_error("operator: transpose application not available");
        apply_impl(true, b, x, y, s);
    }
    long columns_applied() const { return cols_; }
    void reset_counter() { cols_ = 0; }

protected:
    virtual void apply_impl(bool transpose, int64_t b, const double* x, double* y, cudaStream_t s) = 0;
    virtual bool has_transpose() const { return false; }

private:
    int64_t n_;
    bool sym_;
    long cols_ = 0;
};

// DenseOperator (linear_operator.hpp:86-101): the n x n matrix resident in HBM
class DenseDevOperator final : public DevOperator {
public:
    DenseDevOperator(const double* a_host, int64_t n, bool sym);
    const double* data() const { return a_.data(); }

protected:
    void apply_impl(bool transpose, int64_t b, const double* x, double* y, cudaStream_t s) override;
    bool has_transpose() const override { return true; }

private:
    DeviceArray<double> a_;
};

// H2Operator (linear_operator.hpp:104-115): hgemv of a device H^2 matrix
class H2DevOperator final : public DevOperator {
public:
    explicit H2DevOperator(const H2Dev& h);

protected:
    void apply_impl(bool transpose, int64_t b, const double* x, double* y, cudaStream_t s) override;
    bool has_transpose() const override { return true; }

private:
    const H2Dev* h_;
    Workspace ws_;
};

// make_operator (linear_operator.hpp:80-84) with a caller-supplied function
class FunctionDevOperator final : public DevOperator {
public:
    using Fn = std::function<void(bool transpose, int64_t b, const double* x, double* y, cudaStream_t s)>;
    FunctionDevOperator(int64_t n, bool sym, Fn f, bool has_t) : DevOperator(n, sym), f_(std::move(f)), t_(has_t) {}

protected:
    void apply_impl(bool transpose, int64_t b, const double* x, double* y, cudaStream_t s) override {
        f_(transpose, b, x, y, s);
    }
    bool has_transpose() const override { return t_; }

private:
    Fn f_;
    bool t_;
};

struct NormEstimate {
    double value = 0;
    int iterations = 0;
};
// pnorm_estimate(op, 2) (linear_operator.hpp:127-153)
NormEstimate pnorm2_estimate(DevOperator& op, cudaStream_t s, int max_iter = 100, double tol = 5e-3);

// value semantics, like the reference: inputs are not modified
std::unique_ptr<H2Dev> clone_h2(const H2Dev& h, cudaStream_t s);
std::unique_ptr<H2Dev> orthogonalize(const H2Dev& h, cudaStream_t s);              // algebra.hpp:72-113
std::unique_ptr<H2Dev> recompress(const H2Dev& h, double eps, cudaStream_t s);     // algebra.hpp:144-226

// apply_local_update (algebra.hpp:236-316) for a set of updates on disjoint
// regions (one sampled level group): X_i (|t_i| x k_i, ld ldx_i), Y_i (|s_i| x k_i)
struct LocalUpdate {
    int t, s, k;
    const double* X;
    int64_t ldx;
    const double* Y;
    int64_t ldy;
};
std::unique_ptr<H2Dev> apply_local_updates(const H2Dev& h, const std::vector<LocalUpdate>& ups, cudaStream_t s);

struct PeelConfig {   // construction.hpp:23-31
    double eps = 1e-4;
    int64_t sample_block_size = 16;
    int64_t oversampling = 10;
    int64_t max_rank = 0;
    uint64_t seed = 42;
    double norm_scale = 0;
    int64_t crossover_rank_cap = 128;
    // B200 extension: 0 = the reference's Gaussian stream (host mt19937_64 +
    // std::normal_distribution, construction.hpp:81-85; bit-compatible panels),
    // 1 = counter-based Philox4x32-10 normals generated in HBM (same accuracy
    // contract, no host RNG or PCIe upload on the sampling path)
    int rng = 0;
};
struct LevelStats {
    int level = 0;
    int64_t blocks = 0, max_rank = 0;
    long samples = 0;
};
struct SampleStats {   // construction.hpp:33-59
    long total = 0;
    std::vector<LevelStats> levels;
    void add_level(LevelStats l) {
        total += l.samples;
        levels.push_back(l);
    }
};
// construction.hpp:61-66
class max_rank_error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
struct PeelTimes {
    double op_ms = 0, total_ms = 0;   // host wall time in operator applies / whole build
};
struct PeelResult {
    std::unique_ptr<H2Dev> matrix;
    SampleStats stats;
    PeelTimes times;
};
// peel_construct (construction.hpp:300-382)
PeelResult peel_construct(DevOperator& op, std::shared_ptr<const BlockTree> bt, const PeelConfig& cfg,
                          cudaStream_t s);

// global randomized low-rank (construction.hpp:386-491): factor X Y^T (n x k
// device arrays, user ordering; X == Y for symmetric operators)
struct LowRankResultDev {
    int64_t rank = 0;
    std::shared_ptr<DeviceArray<double>> X, Y;   // Y aliases X for the symmetric form
    SampleStats stats;
    double residual_estimate = 0;
    bool max_rank_reached = false;
};
LowRankResultDev randomized_lowrank(DevOperator& op, double eps, int64_t max_rank, const PeelConfig& cfg,
                                    int stagnation_window, cudaStream_t s);
// hybrid_construct (construction.hpp:506-534): global low-rank capture, peel of
// the residual, global update back
struct HybridResultDev {
    std::unique_ptr<H2Dev> matrix;
    SampleStats stats;
    int64_t global_rank = 0;
};
HybridResultDev hybrid_construct(DevOperator& op, std::shared_ptr<const BlockTree> bt, const PeelConfig& cfg,
                                 cudaStream_t s);

// estimate_relative_error (construction.hpp:537-546)
double estimate_relative_error(DevOperator& op, const H2Dev& h, double op_norm, cudaStream_t s);

}  // namespace h2b
