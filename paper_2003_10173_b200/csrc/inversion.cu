// Iterative inversion on the B200 (reference inversion.hpp, algebra.hpp:334-346).
// Control flow restates the reference; every vector operation, hgemv and
// construction runs on the device.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <unordered_map>

#include "inversion.hpp"
#include "la.hpp"
#include "matrix.hpp"

namespace h2b {

using la::DBuf;

double threshold_schedule(double residual, int, double eps_final, const ThresholdSchedule& s) {
    if (!s.dynamic) return eps_final;
    const double v = std::min(s.eps_initial, residual * residual / 10.0);
    return std::clamp(v, eps_final, s.eps_initial);
}

namespace {

constexpr int kRedBlocks = 256;

// y = a x + b z (n x c, contiguous)
__global__ void axpby_kernel(int64_t cnt, double a, const double* __restrict__ x, double b,
                             const double* __restrict__ z, double* __restrict__ y) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < cnt; i += int64_t(gridDim.x) * blockDim.x)
        y[i] = a * x[i] + (b == 0.0 ? 0.0 : b * z[i]);
}
void axpby(int64_t cnt, double a, const double* x, double b, const double* z, double* y, cudaStream_t s) {
    if (cnt == 0) return;
    const int64_t blocks = std::min<int64_t>((cnt + 255) / 256, 148 * 8);
    axpby_kernel<<<unsigned(blocks), 256, 0, s>>>(cnt, a, x, b, z, y);
    H2B_LAUNCH();
}

// per-block partials (fixed order): 0 sum |y|, 1 sum z x, plus (max |z|, first index)
__global__ void reduce_kernel(int64_t n, int what, const double* __restrict__ y, const double* __restrict__ x,
                              double* __restrict__ part, int64_t* __restrict__ arg) {
    __shared__ double sv[256];
    __shared__ int64_t si[256];
    double acc = 0;
    int64_t best = -1;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        if (what == 0) acc += fabs(y[i]);
        else if (what == 1) acc += y[i] * x[i];
        else if (best < 0 || fabs(y[i]) > acc) {
            acc = fabs(y[i]);
            best = i;
        }
    }
    sv[threadIdx.x] = acc;
    si[threadIdx.x] = best;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            if (what == 2) {
                const int64_t ib = si[threadIdx.x + w];
                const double vb = sv[threadIdx.x + w];
                const int64_t ia = si[threadIdx.x];
                if (ib >= 0 && (ia < 0 || vb > sv[threadIdx.x] || (vb == sv[threadIdx.x] && ib < ia))) {
                    sv[threadIdx.x] = vb;
                    si[threadIdx.x] = ib;
                }
            } else {
                sv[threadIdx.x] += sv[threadIdx.x + w];
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[blockIdx.x] = sv[0];
        if (arg) arg[blockIdx.x] = si[0];
    }
}

double reduce_sum(int64_t n, int what, const double* y, const double* x, cudaStream_t s) {
    DBuf part(kRedBlocks, s);
    reduce_kernel<<<kRedBlocks, 256, 0, s>>>(n, what, y, x, part.data(), nullptr);
    H2B_LAUNCH();
    std::vector<double> h(kRedBlocks);
    H2B_CUDA(cudaMemcpyAsync(h.data(), part.data(), kRedBlocks * sizeof(double), cudaMemcpyDeviceToHost, s));
    H2B_CUDA(cudaStreamSynchronize(s));
    double t = 0;
    for (double v : h) t += v;
    return t;
}

std::pair<double, int64_t> reduce_absmax(int64_t n, const double* z, cudaStream_t s) {
    DBuf part(kRedBlocks, s);
    int64_t* arg = nullptr;
    H2B_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&arg), kRedBlocks * sizeof(int64_t), s));
    reduce_kernel<<<kRedBlocks, 256, 0, s>>>(n, 2, z, nullptr, part.data(), arg);
    H2B_LAUNCH();
    std::vector<double> h(kRedBlocks);
    std::vector<int64_t> ha(kRedBlocks);
    H2B_CUDA(cudaMemcpyAsync(h.data(), part.data(), kRedBlocks * sizeof(double), cudaMemcpyDeviceToHost, s));
    H2B_CUDA(cudaMemcpyAsync(ha.data(), arg, kRedBlocks * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    H2B_CUDA(cudaStreamSynchronize(s));
    cudaFreeAsync(arg, s);
    double best = -1;
    int64_t bi = -1;
    for (int i = 0; i < kRedBlocks; ++i)
        if (ha[size_t(i)] >= 0 && (bi < 0 || h[size_t(i)] > best || (h[size_t(i)] == best && ha[size_t(i)] < bi))) {
            best = h[size_t(i)];
            bi = ha[size_t(i)];
        }
    return {best, bi};
}

__global__ void sign_kernel(int64_t n, const double* __restrict__ y, double* __restrict__ o) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        o[i] = y[i] >= 0 ? 1.0 : -1.0;
}
__global__ void fill_kernel(int64_t n, double v, double* __restrict__ o) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        o[i] = v;
}
// diagonal of the diagonal dense leaves: set to (add == 0) or add `value`
__global__ void diag_set_kernel(const int64_t* __restrict__ off, const int* __restrict__ m, double value,
                                double* __restrict__ D, int add) {
    const int64_t o = off[blockIdx.x];
    const int mm = m[blockIdx.x];
    for (int i = threadIdx.x; i < mm; i += blockDim.x) {
        double* p = D + o + int64_t(i) * mm + i;
        *p = add ? *p + value : value;
    }
}
void diag_apply(H2Dev& h, double value, int add, cudaStream_t s) {
    const BlockTree& bt = *h.bt;
    const ClusterTree& ct = *bt.tree;
    std::vector<int64_t> off;
    std::vector<int> m;
    for (size_t i = 0; i < bt.dense.size(); ++i) {
        const int b = bt.dense[i];
        if (h.d_off[i] < 0 || bt.row[size_t(b)] != bt.col[size_t(b)]) continue;
        off.push_back(h.d_off[i]);
        m.push_back(int(ct.size(bt.row[size_t(b)])));
    }
    if (off.empty()) return;
    DeviceArray<int64_t> doff;
    DeviceArray<int> dm;
    doff.upload(off, s);
    dm.upload(m, s);
    diag_set_kernel<<<unsigned(off.size()), 128, 0, s>>>(doff.data(), dm.data(), value, h.D.data(), add);
    H2B_LAUNCH();
}

// hgemv of one matrix with its own workspace (samplers own one per matrix)
struct Apply {
    const H2Dev* h;
    std::shared_ptr<Workspace> ws = std::make_shared<Workspace>();
    void operator()(bool t, int64_t b, const double* x, double* y, cudaStream_t s) const {
        const int64_t n = h->tree().n;
        hgemv(*h, t, true, n, b, x, n, y, n, 1.0, 0.0, s, *ws);
    }
};

}  // namespace

std::unique_ptr<H2Dev> scaled_identity(std::shared_ptr<const BlockTree> bt, double value, cudaStream_t s) {
    auto h = make_h2(bt, true, nullptr, nullptr);
    diag_apply(*h, value, 0, s);
    return h;
}

void add_diagonal(H2Dev& h, double value, cudaStream_t s) {
    diag_apply(h, value, 1, s);   // values only: plans (pointers, structure) stay valid
}

NormEstimate pnorm_1inf_estimate(DevOperator& op, bool inf, cudaStream_t s, int max_iter) {
    const int64_t n = op.dim();
    auto fwd = [&](const double* x, double* y) {
        if (inf) op.apply_transpose(1, x, y, s);
        else op.apply(1, x, y, s);
    };
    auto bwd = [&](const double* x, double* y) {
        if (inf) op.apply(1, x, y, s);
        else op.apply_transpose(1, x, y, s);
    };
    DBuf x(size_t(n), s), y(size_t(n), s), xi(size_t(n), s), z(size_t(n), s);
    const unsigned g = unsigned(std::min<int64_t>((n + 255) / 256, 148 * 8));
    fill_kernel<<<g, 256, 0, s>>>(n, 1.0 / double(n), x.data());
    H2B_LAUNCH();
    double est = 0;
    int it = 0;
    while (it < std::min(max_iter, 8)) {   // linear_operator.hpp:160-177
        ++it;
        fwd(x.data(), y.data());
        est = reduce_sum(n, 0, y.data(), nullptr, s);
        sign_kernel<<<g, 256, 0, s>>>(n, y.data(), xi.data());
        H2B_LAUNCH();
        bwd(xi.data(), z.data());
        const auto [zmax, j] = reduce_absmax(n, z.data(), s);
        const double ztx = reduce_sum(n, 1, z.data(), x.data(), s);
        if (zmax <= ztx) break;
        x.zero();
        const double one = 1.0;
        H2B_CUDA(cudaMemcpyAsync(x.data() + j, &one, sizeof(double), cudaMemcpyHostToDevice, s));
        H2B_CUDA(cudaStreamSynchronize(s));
    }
    return {est, it};
}

std::unique_ptr<H2Dev> scaled_identity_start(const H2Dev& a, cudaStream_t s) {
    H2DevOperator op(a);
    const double ninf = pnorm_1inf_estimate(op, true, s).value;
    if (ninf <= 0) throw std::invalid_argument("scaled_identity_start: zero operator");
    return scaled_identity(a.bt, 1.0 / ninf, s);
}

std::unique_ptr<DevOperator> ns_sampler(const H2Dev& xk, const H2Dev& a) {   // inversion.hpp:137-150
    if (xk.tree().n != a.tree().n) throw std::invalid_argument("ns_sampler: dimension mismatch");
    const int64_t n = a.tree().n;
    Apply X{&xk}, A{&a};
    auto f = [X, A, n](bool t, int64_t b, const double* w, double* y, cudaStream_t s) {
        DBuf t1(size_t(n * b), s), t2(size_t(n * b), s);
        if (!t) {   // Y = 2 X w - X (A (X w))
            X(false, b, w, t1.data(), s);
            A(false, b, t1.data(), t2.data(), s);
            X(false, b, t2.data(), y, s);
            axpby(n * b, 2.0, t1.data(), -1.0, y, y, s);
        } else {    // Y = X^T (2 w - A^T (X^T w))
            X(true, b, w, t1.data(), s);
            A(true, b, t1.data(), t2.data(), s);
            axpby(n * b, 2.0, w, -1.0, t2.data(), t2.data(), s);
            X(true, b, t2.data(), y, s);
        }
    };
    return std::make_unique<FunctionDevOperator>(n, xk.symmetric && a.symmetric, f, true);
}

std::unique_ptr<DevOperator> hyperpower_sampler(const H2Dev& xk, const H2Dev& a, int order) {   // :154-177
    if (order < 2 || order > 64) throw std::invalid_argument("hyperpower order must be in [2, 64]");
    const int64_t n = a.tree().n;
    Apply X{&xk}, A{&a};
    auto f = [X, A, n, order](bool t, int64_t b, const double* w, double* y, cudaStream_t s) {
        const size_t cnt = size_t(n * b);
        DBuf acc(cnt, s), r(cnt, s), t1(cnt, s), t2(cnt, s);
        if (!t) {   // y = X (w + r_1 + ... ), r_{i} = r_{i-1} - A X r_{i-1}
            H2B_CUDA(cudaMemcpyAsync(acc.data(), w, cnt * sizeof(double), cudaMemcpyDeviceToDevice, s));
            H2B_CUDA(cudaMemcpyAsync(r.data(), w, cnt * sizeof(double), cudaMemcpyDeviceToDevice, s));
            for (int i = 1; i < order; ++i) {
                X(false, b, r.data(), t1.data(), s);
                A(false, b, t1.data(), t2.data(), s);
                axpby(int64_t(cnt), 1.0, r.data(), -1.0, t2.data(), r.data(), s);
                axpby(int64_t(cnt), 1.0, acc.data(), 1.0, r.data(), acc.data(), s);
            }
            X(false, b, acc.data(), y, s);
        } else {    // u = X^T w; y = u + r_1 + ..., r_i = r_{i-1} - X^T A^T r_{i-1}
            X(true, b, w, acc.data(), s);
            H2B_CUDA(cudaMemcpyAsync(r.data(), acc.data(), cnt * sizeof(double), cudaMemcpyDeviceToDevice, s));
            for (int i = 1; i < order; ++i) {
                A(true, b, r.data(), t1.data(), s);
                X(true, b, t1.data(), t2.data(), s);
                axpby(int64_t(cnt), 1.0, r.data(), -1.0, t2.data(), r.data(), s);
                axpby(int64_t(cnt), 1.0, acc.data(), 1.0, r.data(), acc.data(), s);
            }
            H2B_CUDA(cudaMemcpyAsync(y, acc.data(), cnt * sizeof(double), cudaMemcpyDeviceToDevice, s));
        }
    };
    return std::make_unique<FunctionDevOperator>(n, xk.symmetric && a.symmetric, f, true);
}

std::unique_ptr<DevOperator> unrolled_sampler(const H2Dev& x0, const H2Dev& a, int k) {   // :197-208
    if (k < 0 || k > 6) throw std::invalid_argument("unrolled_sampler: k must be in [0, 6]");
    const int npow = 1 << k;
    std::vector<unsigned long long> row{1};   // binomial row C(npow, .) (inversion.hpp:183-192)
    for (int i = 1; i <= npow; ++i) {
        std::vector<unsigned long long> nx(size_t(i) + 1, 1);
        for (int j = 1; j < i; ++j) nx[size_t(j)] = row[size_t(j) - 1] + row[size_t(j)];
        row = std::move(nx);
    }
    const int64_t n = a.tree().n;
    Apply X{&x0}, A{&a};
    auto f = [X, A, n, npow, row](bool, int64_t b, const double* w, double* y, cudaStream_t s) {
        const size_t cnt = size_t(n * b);
        DBuf p(cnt, s), t1(cnt, s), t2(cnt, s);
        axpby(int64_t(cnt), double(row[size_t(npow)]), w, 0.0, nullptr, p.data(), s);
        for (int i = npow - 2; i >= 0; --i) {   // p = C(N, i+1) w - A X p
            X(false, b, p.data(), t1.data(), s);
            A(false, b, t1.data(), t2.data(), s);
            axpby(int64_t(cnt), double(row[size_t(i) + 1]), w, -1.0, t2.data(), p.data(), s);
        }
        X(false, b, p.data(), y, s);
    };
    // the reference defines no transpose for the unrolled sampler
    return std::make_unique<FunctionDevOperator>(n, x0.symmetric && a.symmetric, f, false);
}

double residual_norm(DevOperator& a, DevOperator& x, cudaStream_t s) {   // inversion.hpp:213-220
    if (a.dim() != x.dim()) throw std::invalid_argument("residual_norm: dimension mismatch");
    const int64_t n = a.dim();
    FunctionDevOperator composed(
        n, false,
        [&](bool t, int64_t b, const double* v, double* y, cudaStream_t st) {
            DBuf t1(size_t(n * b), st);
            if (!t) {
                x.apply(b, v, t1.data(), st);
                a.apply(b, t1.data(), y, st);
            } else {
                a.apply_transpose(b, v, t1.data(), st);
                x.apply_transpose(b, t1.data(), y, st);
            }
            axpby(n * b, 1.0, y, -1.0, v, y, st);
        },
        true);
    return pnorm2_estimate(composed, s).value;
}

double residual_norm(const H2Dev& a, const H2Dev& x, cudaStream_t s) {
    H2DevOperator oa(a), ox(x);
    return residual_norm(oa, ox, s);
}

InverseResult h_iterative_inverse(const H2Dev& a, const H2Dev& x0, const ThresholdSchedule& sched, double eps,
                                  const PeelConfig& cfg, int kind, int order, int max_iter, cudaStream_t s) {
    if (a.tree().n != x0.tree().n) throw std::invalid_argument("inverse: dimension mismatch");
    std::unique_ptr<H2Dev> x = clone_h2(x0, s);
    ConvergenceTrace trace;
    double prev_e = std::numeric_limits<double>::infinity();
    double prev_eps_k = std::numeric_limits<double>::infinity();
    int streak = 0;
    for (int k = 0;; ++k) {   // inversion.hpp:245-275
        const double e = residual_norm(a, *x, s);
        if (k == 0 && e >= 1.0) trace.notes.push_back("warm start residual >= 1; global convergence not guaranteed");
        if (e <= eps) {
            trace.final_residual = e;
            trace.converged = true;
            break;
        }
        streak = e > prev_e ? streak + 1 : 0;
        prev_e = e;
        if (streak >= 3) throw divergence_error("hierarchical inversion: residual increased 3 times", trace);
        if (k >= max_iter) throw divergence_error("hierarchical inversion: iteration limit", trace);
        const double eps_k = std::min(threshold_schedule(e, k, eps, sched), prev_eps_k);
        prev_eps_k = eps_k;
        PeelConfig step = cfg;
        step.eps = eps_k;
        step.seed = cfg.seed + 1000003ull * (unsigned long long)(k + 1);
        const auto t0 = std::chrono::steady_clock::now();
        auto sampler = kind == 0 ? ns_sampler(*x, a) : hyperpower_sampler(*x, a, order);
        PeelResult pr = peel_construct(*sampler, a.bt, step, s);
        const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        x = std::move(pr.matrix);
        trace.rows.push_back({k, e, eps_k, pr.stats.total, dt});
    }
    return {std::move(x), std::move(trace)};
}

InverseResult h_unrolled(const H2Dev& a, const H2Dev& x0, int k, double eps, const PeelConfig& cfg, cudaStream_t s) {
    auto sampler = unrolled_sampler(x0, a, k);
    PeelConfig step = cfg;
    step.eps = eps;
    const auto t0 = std::chrono::steady_clock::now();
    PeelResult pr = peel_construct(*sampler, a.bt, step, s);
    const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    InverseResult r;
    r.trace.rows.push_back({0, std::numeric_limits<double>::quiet_NaN(), eps, pr.stats.total, dt});
    r.X = std::move(pr.matrix);
    r.trace.final_residual = residual_norm(a, *r.X, s);
    r.trace.converged = r.trace.final_residual <= eps;
    return r;
}

std::unique_ptr<H2Dev> desymmetrized(const H2Dev& h, cudaStream_t s) {   // h2_matrix.hpp:200-216
    if (!h.symmetric) return clone_h2(h, s);
    const BlockTree& bt = *h.bt;
    const ClusterTree& ct = *bt.tree;
    auto out = make_h2(h.bt, false, h.row.rank.data(), h.row.rank.data());
    auto cp = [&](DeviceArray<double>& d, const DeviceArray<double>& src) {
        if (src.size())
            H2B_CUDA(cudaMemcpyAsync(d.data(), src.data(), src.size() * sizeof(double), cudaMemcpyDeviceToDevice, s));
    };
    cp(out->row.leaf, h.row.leaf);
    cp(out->row.xfer, h.row.xfer);
    cp(out->col.leaf, h.row.leaf);
    cp(out->col.xfer, h.row.xfer);
    // every block: the canonical one as stored, the mirrored one transposed
    std::vector<int64_t> canon_adm(bt.row.size(), -1), canon_dense(bt.row.size(), -1);
    for (size_t i = 0; i < bt.adm.size(); ++i) canon_adm[size_t(bt.adm[i])] = int64_t(i);
    for (size_t i = 0; i < bt.dense.size(); ++i) canon_dense[size_t(bt.dense[i])] = int64_t(i);
    std::vector<la::CopyDesc> cps;
    std::unordered_map<int64_t, int> mir;   // (row, col) -> block node, for the lookups below
    for (size_t q = 0; q < bt.row.size(); ++q)
        if (bt.tag[q] != 0) mir[(int64_t(bt.row[q]) << 32) | uint32_t(bt.col[q])] = int(q);
    for (size_t i = 0; i < bt.adm.size(); ++i) {
        const int b = bt.adm[i];
        const int r = bt.row[size_t(b)], c = bt.col[size_t(b)];
        const int kr = h.row.rank[size_t(r)], kc = h.row.rank[size_t(c)];
        if (kr == 0 || kc == 0) continue;
        double* dst = out->S.data() + out->s_off[i];
        if (h.s_off[i] >= 0) {
            cps.push_back(la::CopyDesc{h.S.data() + h.s_off[i], dst, kr, kc, kr, kr, 0});
        } else {
            const int mb = mir.at((int64_t(c) << 32) | uint32_t(r));
            const int64_t mi = canon_adm[size_t(mb)];
            cps.push_back(la::CopyDesc{h.S.data() + h.s_off[size_t(mi)], dst, kr, kc, kc, kr, 1});
        }
    }
    for (size_t i = 0; i < bt.dense.size(); ++i) {
        const int b = bt.dense[i];
        const int r = bt.row[size_t(b)], c = bt.col[size_t(b)];
        const int mr = int(ct.size(r)), mc = int(ct.size(c));
        double* dst = out->D.data() + out->d_off[i];
        if (h.d_off[i] >= 0) {
            cps.push_back(la::CopyDesc{h.D.data() + h.d_off[i], dst, mr, mc, mr, mr, 0});
        } else {
            const int mb = mir.at((int64_t(c) << 32) | uint32_t(r));
            const int64_t mi = canon_dense[size_t(mb)];
            cps.push_back(la::CopyDesc{h.D.data() + h.d_off[size_t(mi)], dst, mr, mc, mc, mr, 1});
        }
    }
    la::bcopy(cps, s);
    out->orthonormal = h.orthonormal;
    return out;
}

std::unique_ptr<H2Dev> low_rank_update(const H2Dev& h, const double* X, const double* Y, int k, double eps,
                                       cudaStream_t s) {   // algebra.hpp:334-346
    if (k < 0) throw std::invalid_argument("low_rank_update: factor dimensions do not match");
    if (k == 0) return clone_h2(h, s);
    const ClusterTree& ct = h.tree();
    const int64_t n = ct.n;
    // symmetric update iff X and Y are bitwise equal
    bool same = X == Y;
    if (!same) {
        std::vector<double> hx(size_t(n * k)), hy(size_t(n * k));
        H2B_CUDA(cudaMemcpyAsync(hx.data(), X, hx.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
        H2B_CUDA(cudaMemcpyAsync(hy.data(), Y, hy.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
        H2B_CUDA(cudaStreamSynchronize(s));
        same = std::memcmp(hx.data(), hy.data(), hx.size() * sizeof(double)) == 0;
    }
    std::unique_ptr<H2Dev> own;
    const H2Dev* g = &h;
    if (h.symmetric && !same) {
        own = desymmetrized(h, s);
        g = own.get();
    }
    DeviceArray<int> perm;
    perm.upload(std::vector<int>(ct.perm.begin(), ct.perm.end()), s);
    DBuf xi(size_t(n * k), s), yi(size_t(n * k), s);
    la::permute_rows(X, n, xi.data(), n, perm.data(), n, k, false, s);
    const double* yp = xi.data();
    if (!same) {
        la::permute_rows(Y, n, yi.data(), n, perm.data(), n, k, false, s);
        yp = yi.data();
    }
    const int root = ct.levels[0][0];
    auto upd = apply_local_updates(*g, {LocalUpdate{root, root, k, xi.data(), n, yp, n}}, s);
    return recompress(*upd, eps, s);
}

}  // namespace h2b
