// Global randomized low-rank range finder and the hybrid constructor on the
// B200 (reference construction.hpp:386-534). Control flow restates the
// reference; panels, projections, thin SVDs, the symmetric B B^T form and the
// residual operator all run on the device.
#include <algorithm>
#include <cmath>
#include <random>

#include <curand_kernel.h>

#include "hara.hpp"
#include "refstream.hpp"
#include "inversion.hpp"
#include "la.hpp"

namespace h2b {

using la::DBuf;

namespace {

// column 2-norms of an n x c matrix (one CTA per column, fixed reduction order)
__global__ void colnorm_kernel(const double* __restrict__ a, int64_t n, int64_t ld, double* __restrict__ out) {
    __shared__ double red[256];
    const double* col = a + int64_t(blockIdx.x) * ld;
    double acc = 0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc += col[i] * col[i];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = sqrt(red[0]);
}

std::vector<double> col_norms(const double* a, int64_t n, int64_t c, cudaStream_t s) {
    DBuf o(size_t(c), s);
    colnorm_kernel<<<unsigned(c), 256, 0, s>>>(a, n, n, o.data());
    H2B_LAUNCH();
    std::vector<double> h(static_cast<size_t>(c));
    H2B_CUDA(cudaMemcpyAsync(h.data(), o.data(), h.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    H2B_CUDA(cudaStreamSynchronize(s));
    return h;
}

__global__ void philox_panel_kernel(int64_t cnt, double* out, unsigned long long seed, unsigned long long panel) {
    for (int64_t e = 2 * (int64_t(blockIdx.x) * blockDim.x + threadIdx.x); e < cnt;
         e += 2 * int64_t(gridDim.x) * blockDim.x) {
        curandStatePhilox4_32_10_t st;
        curand_init(seed, panel, uint64_t(e), &st);
        const double2 g = curand_normal2_double(&st);
        out[e] = g.x;
        if (e + 1 < cnt) out[e + 1] = g.y;
    }
}

}  // namespace

LowRankResultDev randomized_lowrank(DevOperator& op, double eps, int64_t max_rank, const PeelConfig& cfg,
                                    int stagnation_window, cudaStream_t s) {   // construction.hpp:397-484
    std::mt19937_64 rng(cfg.seed);
    SampleStats stats;
    const long before = op.columns_applied();
    double norm_scale = cfg.norm_scale;
    if (norm_scale <= 0) norm_scale = std::max(pnorm2_estimate(op, s).value, 1e-300);
    const int64_t n = op.dim();
    const int64_t b = std::max<int64_t>(cfg.sample_block_size, 1);
    const int64_t probes = std::min<int64_t>(std::max<int64_t>(cfg.oversampling, 1), b);
    const double tol_abs = eps * norm_scale;

    int64_t cap = std::max<int64_t>(2 * b, 32), k = 0;
    DBuf Q(size_t(n * cap), s);
    bool converged = false, wants_full = true, capped = false;
    double err_est = 0;
    std::vector<double> panel_norms, omh;
    unsigned long long panel_id = 0;
    while (!converged) {
        const int64_t panel = wants_full ? b : probes;
        DBuf om(size_t(n * panel), s), y(size_t(n * panel), s);
        if (cfg.rng == 0) {   // fill_gaussian(omega, rng) (construction.hpp:81-85)
            omh.resize(size_t(n * panel));
            ref_fill_gaussian(omh.data(), n, panel, n, rng);
            H2B_CUDA(cudaMemcpyAsync(om.data(), omh.data(), omh.size() * sizeof(double), cudaMemcpyHostToDevice, s));
        } else {
            const int64_t cnt = n * panel;
            philox_panel_kernel<<<unsigned(std::min<int64_t>((cnt / 2 + 255) / 256, 4096)), 256, 0, s>>>(
                cnt, om.data(), cfg.seed, panel_id++);
            H2B_LAUNCH();
        }
        op.apply(panel, om.data(), y.data(), s);
        if (k > 0) {
            DBuf c(size_t(k * panel), s);
            for (int pass = 0; pass < 2; ++pass) {
                la::bgemm({la::GemmDesc{Q.data(), y.data(), c.data(), int(k), int(panel), int(n), int(n), int(n),
                                        int(k), 1, 0, 1.0, 0.0}}, s);
                la::bgemm({la::GemmDesc{Q.data(), c.data(), y.data(), int(n), int(panel), int(k), int(n), int(k),
                                        int(n), 0, 0, -1.0, 1.0}}, s);
            }
        }
        const std::vector<double> yn = col_norms(y.data(), n, panel, s), on = col_norms(om.data(), n, panel, s);
        double ratio = 0;
        for (int64_t j = 0; j < panel; ++j) ratio = std::max(ratio, yn[size_t(j)] / on[size_t(j)]);
        panel_norms.push_back(ratio);
        err_est = ratio;
        const int64_t p = std::min(n, panel);
        DBuf U(size_t(n * p), s), sg(size_t(p), s);
        la::bleft_svd({la::LeftSvdDesc{y.data(), int(n), int(panel), int(n), U.data(), int(n), sg.data(), nullptr, 0}},
                      s);
        std::vector<double> sv(static_cast<size_t>(p));
        H2B_CUDA(cudaMemcpyAsync(sv.data(), sg.data(), sv.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
        H2B_CUDA(cudaStreamSynchronize(s));
        const double keep_tol = 0.5 * tol_abs * std::sqrt(double(panel));
        int64_t kept_raw = 0;
        while (kept_raw < p && sv[size_t(kept_raw)] > keep_tol) ++kept_raw;
        int64_t kept = kept_raw;
        if (max_rank > 0) kept = std::min(kept, std::max<int64_t>(max_rank - k, 0));
        if (kept > 0) {
            if (k + kept > cap) {
                int64_t nc = cap;
                while (nc < k + kept) nc *= 2;
                DBuf q2(size_t(n * nc), s);
                if (k) H2B_CUDA(cudaMemcpyAsync(q2.data(), Q.data(), size_t(n * k) * sizeof(double),
                                                cudaMemcpyDeviceToDevice, s));
                Q = std::move(q2);
                cap = nc;
            }
            H2B_CUDA(cudaMemcpyAsync(Q.data() + n * k, U.data(), size_t(n * kept) * sizeof(double),
                                     cudaMemcpyDeviceToDevice, s));
            k += kept;
        }
        wants_full = kept_raw == panel;
        if (kept_raw < panel && (panel - kept_raw) >= probes) {
            converged = true;
            err_est = kept_raw < p ? sv[size_t(kept_raw)] / std::sqrt(double(panel)) : 0.0;
        }
        if (k >= n) converged = true;
        if (max_rank > 0 && k >= max_rank && !converged) {
            capped = true;
            break;
        }
        const size_t w = size_t(stagnation_window);
        if (stagnation_window > 0 && panel_norms.size() > w &&
            panel_norms.back() > 0.9 * panel_norms[panel_norms.size() - 1 - w]) {
            capped = true;   // stagnating spectrum: hand over to the peeler
            break;
        }
    }
    LowRankResultDev res;
    res.rank = k;
    res.X = std::make_shared<DeviceArray<double>>();
    if (k > 0) {
        DBuf y(size_t(n * k), s);
        op.apply_transpose(k, Q.data(), y.data(), s);
        if (op.symmetric()) {
            // Q (Q^T A Q) Q^T = B B^T with B = Q V sqrt(max(lambda, 0)) (symmetric eigen-form)
            DBuf t(size_t(k * k), s), ts(size_t(k * k), s), V(size_t(k * k), s), sg(size_t(k), s), W(size_t(k * k), s);
            la::bgemm({la::GemmDesc{Q.data(), y.data(), t.data(), int(k), int(k), int(n), int(n), int(n), int(k), 1, 0,
                                    1.0, 0.0}}, s);
            ts.zero();
            la::bcopy({la::CopyDesc{t.data(), ts.data(), int(k), int(k), int(k), int(k), 4}}, s);   // ts = (t + t^T) / 2
            la::bjacobi({la::SvdDesc{ts.data(), int(k), int(k), int(k), 0, sg.data(), V.data(), int(k)}}, s);
            la::bgemm({la::GemmDesc{ts.data(), V.data(), W.data(), int(k), int(k), int(k), int(k), int(k), int(k), 0, 0,
                                    1.0, 0.0}}, s);
            std::vector<double> hv(size_t(k * k)), hw(size_t(k * k));
            H2B_CUDA(cudaMemcpyAsync(hv.data(), V.data(), hv.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
            H2B_CUDA(cudaMemcpyAsync(hw.data(), W.data(), hw.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
            H2B_CUDA(cudaStreamSynchronize(s));
            // lambda_i = v_i^T sym(t) v_i; scale the eigenvector columns by sqrt(max(lambda, 0))
            std::vector<double> dsc(size_t(k * k), 0.0);
            for (int64_t i = 0; i < k; ++i) {
                double lam = 0;
                for (int64_t r = 0; r < k; ++r) lam += hv[size_t(r + i * k)] * hw[size_t(r + i * k)];
                dsc[size_t(i + i * k)] = std::sqrt(std::max(lam, 0.0));
            }
            DBuf D(size_t(k * k), s), VD(size_t(k * k), s);
            H2B_CUDA(cudaMemcpyAsync(D.data(), dsc.data(), dsc.size() * sizeof(double), cudaMemcpyHostToDevice, s));
            la::bgemm({la::GemmDesc{V.data(), D.data(), VD.data(), int(k), int(k), int(k), int(k), int(k), int(k), 0, 0,
                                    1.0, 0.0}}, s);
            res.X->resize(size_t(n * k), s);
            la::bgemm({la::GemmDesc{Q.data(), VD.data(), res.X->data(), int(n), int(k), int(k), int(n), int(k), int(n), 0,
                                    0, 1.0, 0.0}}, s);
            res.Y = res.X;
        } else {
            res.X->resize(size_t(n * k), s);
            H2B_CUDA(cudaMemcpyAsync(res.X->data(), Q.data(), size_t(n * k) * sizeof(double), cudaMemcpyDeviceToDevice, s));
            res.Y = std::make_shared<DeviceArray<double>>();
            res.Y->resize(size_t(n * k), s);
            H2B_CUDA(cudaMemcpyAsync(res.Y->data(), y.data(), size_t(n * k) * sizeof(double), cudaMemcpyDeviceToDevice, s));
        }
    } else {
        res.Y = res.X;
    }
    H2B_CUDA(cudaStreamSynchronize(s));
    res.max_rank_reached = capped;
    res.residual_estimate = norm_scale > 0 ? err_est / norm_scale : 0.0;
    stats.add_level({0, 1, k, op.columns_applied() - before});
    res.stats = std::move(stats);
    return res;
}

HybridResultDev hybrid_construct(DevOperator& op, std::shared_ptr<const BlockTree> bt, const PeelConfig& cfg,
                                 cudaStream_t s) {   // construction.hpp:506-534
    PeelConfig c = cfg;
    if (c.norm_scale <= 0) c.norm_scale = std::max(pnorm2_estimate(op, s).value, 1e-300);
    LowRankResultDev lr = randomized_lowrank(op, c.eps, c.crossover_rank_cap, c, 3, s);
    const int64_t n = op.dim(), k = lr.rank;
    const double* X = k ? lr.X->data() : nullptr;
    const double* Y = k ? lr.Y->data() : nullptr;
    FunctionDevOperator residual(
        n, op.symmetric(),
        [&](bool t, int64_t b, const double* x, double* y, cudaStream_t st) {
            if (t) op.apply_transpose(b, x, y, st);
            else op.apply(b, x, y, st);
            if (k == 0) return;
            DBuf tmp(size_t(k * b), st);   // y -= X (Y^T x)  (transpose: y -= Y (X^T x))
            const double* L = t ? Y : X;
            const double* Rm = t ? X : Y;
            la::bgemm({la::GemmDesc{Rm, x, tmp.data(), int(k), int(b), int(n), int(n), int(n), int(k), 1, 0, 1.0, 0.0}},
                      st);
            la::bgemm({la::GemmDesc{L, tmp.data(), y, int(n), int(b), int(k), int(n), int(k), int(n), 0, 0, -1.0, 1.0}},
                      st);
        },
        true);
    PeelResult pr = peel_construct(residual, bt, c, s);
    HybridResultDev res;
    res.global_rank = k;
    res.matrix = k > 0 ? low_rank_update(*pr.matrix, X, Y, int(k), c.eps, s) : std::move(pr.matrix);
    res.stats = lr.stats;
    for (const auto& l : pr.stats.levels) res.stats.add_level(l);
    return res;
}

}  // namespace h2b
