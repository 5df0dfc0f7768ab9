// HARA on the B200: device-resident H^2 algebra (orthogonalize, recompress,
// local low-rank updates) and the peeling construction that drives it.
// Reference: algebra.hpp:31-316, construction.hpp:81-382, 537-546,
// linear_operator.hpp:86-153. Control flow mirrors the reference; every array
// operation is a batched launch over one tree level (la.hpp primitives).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

#include <curand_kernel.h>

#include "hara.hpp"
#include "la.hpp"
#include "matrix.hpp"
#include "refstream.hpp"
#include "blockops.hpp"
#include <string>

namespace h2b {

using la::bcopy;
using la::bgemm;
using la::bleft_svd;
using la::bjacobi;
using la::bqr;
using la::CopyDesc;
using la::DBuf;
using la::GemmDesc;
using la::LeftSvdDesc;
using la::QrDesc;
using la::SvdDesc;

namespace {

using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}
// host wall time per construction phase (stream synchronised at the phase end):
// 0 panel RNG, 1 operator applies, 2 residual hgemv of the partial matrix,
// 3 absorb_panel, 4 transposed-pass bookkeeping, 5 local updates, 6 recompress,
// 7 dense-leaf extraction
double g_phase_ms[16];   // 8 orthogonalize, 9 truncation bases, 10 projection (inside recompress)
// phase timers drain the stream only when enabled (h2b_hara_phase_sync): a
// synchronisation per phase would otherwise stall the device at every phase end
int g_phase_sync = 0;
const bool g_trace_absorb = std::getenv("H2_TRACE_ABSORB") != nullptr;
const bool g_trace_recompress = std::getenv("H2_TRACE_RECOMPRESS") != nullptr;
struct Phase {
    int id;
    cudaStream_t s;
    Clock::time_point t0;
    Phase(int i, cudaStream_t st) : id(i), s(st), t0(Clock::now()) {}
    ~Phase() {
        if (g_phase_sync) cudaStreamSynchronize(s);
        g_phase_ms[id] += ms_since(t0);
    }
};

int ld1(int64_t x) { return int(std::max<int64_t>(x, 1)); }

double* Up(const BasisDev& b, int v) { return const_cast<double*>(b.leaf.data()) + b.leaf_off[size_t(v)]; }
double* Ep(const BasisDev& b, int v) { return const_cast<double*>(b.xfer.data()) + b.xfer_off[size_t(v)]; }
double* Sp(const H2Dev& h, size_t i) { return const_cast<double*>(h.S.data()) + h.s_off[i]; }
double* Dp(const H2Dev& h, size_t i) { return const_cast<double*>(h.D.data()) + h.d_off[i]; }

// per-node offsets into one arena
struct Arena {
    std::vector<size_t> off;
    size_t total = 0;
    DBuf buf;
    void plan(const std::vector<size_t>& sizes) {
        off.resize(sizes.size());
        total = 0;
        for (size_t i = 0; i < sizes.size(); ++i) {
            off[i] = total;
            total += sizes[i];
        }
    }
    void alloc(cudaStream_t s) { buf.alloc(total, s); }
    double* at(size_t i) const { return buf.data() + off[i]; }
};

void copy_array(DeviceArray<double>& dst, const DeviceArray<double>& src, cudaStream_t s) {
    if (dst.size() != src.size()) throw std::logic_error("copy_array: size mismatch");
    if (src.size())
        H2B_CUDA(cudaMemcpyAsync(dst.data(), src.data(), src.size() * sizeof(double), cudaMemcpyDeviceToDevice, s));
}

const BasisDev& col_basis(const H2Dev& h) { return h.symmetric ? h.row : h.col; }

std::vector<int> int32_perm(const ClusterTree& ct) { return std::vector<int>(ct.perm.begin(), ct.perm.end()); }

// host-side reference normal stream (fill_gaussian, construction.hpp:81-85)
void fill_gaussian(double* m, int64_t rows, int64_t cols, int64_t ld, std::mt19937_64& rng) {
    ref_fill_gaussian(m, rows, cols, ld, rng);
}

// device Gaussian panel rows [r0, r0 + rows) x [0, cols) of an n-row matrix
// (Philox4x32-10, counter = (panel id, element index): deterministic for a seed)
struct RngSeg {
    int64_t r0, rows;
};
__global__ void philox_fill_kernel(const RngSeg* __restrict__ segs, int nseg, int64_t cols, int64_t n, double* out,
                                   unsigned long long seed, unsigned long long panel) {
    const RngSeg sg = segs[blockIdx.y];
    const int64_t total = sg.rows * cols;
    for (int64_t e = 2 * (int64_t(blockIdx.x) * blockDim.x + threadIdx.x); e < total;
         e += 2 * int64_t(gridDim.x) * blockDim.x) {
        curandStatePhilox4_32_10_t st;
        curand_init(seed, panel, uint64_t(sg.r0 * cols + e), &st);
        const double2 g = curand_normal2_double(&st);
        const int64_t i0 = e % sg.rows, j0 = e / sg.rows;
        out[sg.r0 + i0 + j0 * n] = g.x;
        if (e + 1 < total) {
            const int64_t i1 = (e + 1) % sg.rows, j1 = (e + 1) / sg.rows;
            out[sg.r0 + i1 + j1 * n] = g.y;
        }
    }
    (void)nseg;
}

}  // namespace

// ---------------------------------------------------------------------------
// operators
// ---------------------------------------------------------------------------
DenseDevOperator::DenseDevOperator(const double* a_host, int64_t n, bool sym) : DevOperator(n, sym) {
    a_.upload(a_host, size_t(n * n));
    H2B_CUDA(cudaDeviceSynchronize());
}

void DenseDevOperator::apply_impl(bool transpose, int64_t b, const double* x, double* y, cudaStream_t s) {
    const int n = int(dim());
    bgemm({GemmDesc{a_.data(), x, y, n, int(b), n, n, n, n, transpose ? 1 : 0, 0, 1.0, 0.0}}, s);
}

H2DevOperator::H2DevOperator(const H2Dev& h) : DevOperator(h.tree().n, h.symmetric), h_(&h) {}

void H2DevOperator::apply_impl(bool transpose, int64_t b, const double* x, double* y, cudaStream_t s) {
    hgemv(*h_, transpose, true, dim(), b, x, dim(), y, dim(), 1.0, 0.0, s, ws_);
}

namespace {
// sigma_max of an n x b device block (spectral_norm: thin SVD values)
double spectral_norm_dev(const double* y, int64_t n, int b, cudaStream_t s) {
    DBuf R(size_t(b) * b, s), sg(size_t(b), s);
    const int p = int(std::min<int64_t>(n, b));
    bqr({QrDesc{y, int(n), b, int(n), R.data(), p, nullptr, 0}}, s);
    bjacobi({SvdDesc{R.data(), p, b, p, 0, sg.data(), nullptr, 0}}, s);
    double v = 0;
    H2B_CUDA(cudaMemcpyAsync(&v, sg.data(), sizeof(double), cudaMemcpyDeviceToHost, s));
    H2B_CUDA(cudaStreamSynchronize(s));
    return v;
}
void thin_q_dev(const double* a, int64_t n, int b, double* q, cudaStream_t s) {
    bqr({QrDesc{a, int(n), b, int(n), nullptr, 0, q, int(n)}}, s);
}
}  // namespace

NormEstimate pnorm2_estimate(DevOperator& op, cudaStream_t s, int max_iter, double tol) {
    const int64_t n = op.dim();
    const int b = int(std::min<int64_t>(3, n));
    std::mt19937_64 rng(0x9E3779B97F4A7C15ull);
    std::vector<double> vh(size_t(n * b));
    ref_fill_gaussian(vh.data(), n, b, n, rng);   // linear_operator.hpp:134-138
    DBuf v0(size_t(n * b), s), v(size_t(n * b), s), y(size_t(n * b), s), z(size_t(n * b), s);
    H2B_CUDA(cudaMemcpyAsync(v0.data(), vh.data(), vh.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    thin_q_dev(v0.data(), n, b, v.data(), s);
    double est = 0, prev = -1;
    int it = 0;
    while (it < max_iter) {
        ++it;
        op.apply(b, v.data(), y.data(), s);
        est = spectral_norm_dev(y.data(), n, b, s);
        if (est == 0) return {0.0, it};
        if (prev > 0 && std::abs(est - prev) < tol * est) break;
        prev = est;
        op.apply_transpose(b, y.data(), z.data(), s);
        thin_q_dev(z.data(), n, b, v.data(), s);
    }
    return {est, it};
}

// ---------------------------------------------------------------------------
// algebra
// ---------------------------------------------------------------------------
std::unique_ptr<H2Dev> clone_h2(const H2Dev& h, cudaStream_t s) {
    auto out = make_h2(h.bt, h.symmetric, h.row.rank.data(), h.symmetric ? nullptr : h.col.rank.data());
    copy_array(out->row.leaf, h.row.leaf, s);
    copy_array(out->row.xfer, h.row.xfer, s);
    if (!h.symmetric) {
        copy_array(out->col.leaf, h.col.leaf, s);
        copy_array(out->col.xfer, h.col.xfer, s);
    }
    copy_array(out->S, h.S, s);
    copy_array(out->D, h.D, s);
    out->orthonormal = h.orthonormal;
    return out;
}

namespace {
// bottom-up thin-QR sweep of one basis tree (algebra.hpp:75-97): writes the
// orthonormal basis into `out` and returns the per-node R factors (kp_v x k_v)
Arena ortho_sweep(const ClusterTree& ct, const BasisDev& in, BasisDev& out, const std::vector<int>& kp,
                  cudaStream_t s) {
    const int nn = ct.num_nodes();
    Arena r, z, qz;
    std::vector<size_t> rs(static_cast<size_t>(nn)), zs(size_t(nn), 0), qs(size_t(nn), 0);
    for (int v = 0; v < nn; ++v) {
        rs[size_t(v)] = size_t(kp[size_t(v)]) * in.rank[size_t(v)];
        if (!ct.is_leaf(v)) {
            const int rows = kp[size_t(ct.child0[size_t(v)])] + kp[size_t(ct.child1[size_t(v)])];
            zs[size_t(v)] = size_t(rows) * in.rank[size_t(v)];
            qs[size_t(v)] = size_t(rows) * kp[size_t(v)];
        }
    }
    r.plan(rs);
    z.plan(zs);
    qz.plan(qs);
    r.alloc(s);
    z.alloc(s);
    qz.alloc(s);
    for (int l = ct.depth; l >= 0; --l) {
        std::vector<GemmDesc> gm;
        std::vector<QrDesc> qr;
        std::vector<CopyDesc> cp;
        for (int v : ct.levels[size_t(l)]) {
            const int k = in.rank[size_t(v)], kv = kp[size_t(v)];
            if (k == 0) continue;
            if (ct.is_leaf(v)) {
                const int m = int(ct.size(v));
                qr.push_back(QrDesc{Up(in, v), m, k, ld1(m), r.at(size_t(v)), ld1(kv), kv ? Up(out, v) : nullptr, ld1(m)});
                continue;
            }
            const int c0 = ct.child0[size_t(v)], c1 = ct.child1[size_t(v)];
            const int k0 = kp[size_t(c0)], k1 = kp[size_t(c1)], rows = k0 + k1;
            if (rows == 0) continue;
            double* Z = z.at(size_t(v));
            if (k0) gm.push_back(GemmDesc{r.at(size_t(c0)), Ep(in, c0), Z, k0, k, in.rank[size_t(c0)], k0,
                                          ld1(in.rank[size_t(c0)]), rows, 0, 0, 1.0, 0.0});
            if (k1) gm.push_back(GemmDesc{r.at(size_t(c1)), Ep(in, c1), Z + k0, k1, k, in.rank[size_t(c1)], k1,
                                          ld1(in.rank[size_t(c1)]), rows, 0, 0, 1.0, 0.0});
            qr.push_back(QrDesc{Z, rows, k, rows, r.at(size_t(v)), ld1(kv), qz.at(size_t(v)), rows});
            if (k0 && kv) cp.push_back(CopyDesc{qz.at(size_t(v)), Ep(out, c0), k0, kv, rows, k0, 0});
            if (k1 && kv) cp.push_back(CopyDesc{qz.at(size_t(v)) + k0, Ep(out, c1), k1, kv, rows, k1, 0});
        }
        bgemm(gm, s);
        bqr(qr, s);
        bcopy(cp, s);
    }
    return r;
}

std::vector<int> ortho_ranks(const ClusterTree& ct, const BasisDev& b) {
    std::vector<int> kp(size_t(ct.num_nodes()), 0);
    for (int l = ct.depth; l >= 0; --l)
        for (int v : ct.levels[size_t(l)]) {
            const int k = b.rank[size_t(v)];
            if (ct.is_leaf(v)) kp[size_t(v)] = int(std::min<int64_t>(ct.size(v), k));
            else kp[size_t(v)] = std::min(kp[size_t(ct.child0[size_t(v)])] + kp[size_t(ct.child1[size_t(v)])], k);
        }
    return kp;
}
}  // namespace

std::unique_ptr<H2Dev> orthogonalize(const H2Dev& h, cudaStream_t s) {
    NvtxRange nvtx("orthogonalize");
    Phase ph(8, s);
    const ClusterTree& ct = h.tree();
    const BlockTree& bt = *h.bt;
    const std::vector<int> kr = ortho_ranks(ct, h.row);
    const std::vector<int> kc = h.symmetric ? kr : ortho_ranks(ct, h.col);
    auto out = make_h2(h.bt, h.symmetric, kr.data(), h.symmetric ? nullptr : kc.data());
    Arena rr = ortho_sweep(ct, h.row, out->row, kr, s);
    Arena rc_store;
    if (!h.symmetric) rc_store = ortho_sweep(ct, h.col, out->col, kc, s);
    const Arena& rc = h.symmetric ? rr : rc_store;
    const BasisDev& vin = col_basis(h);
    // couplings S <- r_row S r_col^T (algebra.hpp:104-110)
    std::vector<size_t> ts;
    std::vector<size_t> idx;
    for (size_t i = 0; i < bt.adm.size(); ++i) {
        if (h.s_off[i] < 0) continue;
        const int b = bt.adm[i];
        idx.push_back(i);
        ts.push_back(size_t(kr[size_t(bt.row[size_t(b)])]) * vin.rank[size_t(bt.col[size_t(b)])]);
    }
    Arena t;
    t.plan(ts);
    t.alloc(s);
    std::vector<GemmDesc> g1, g2;
    for (size_t q = 0; q < idx.size(); ++q) {
        const size_t i = idx[q];
        const int b = bt.adm[i], r = bt.row[size_t(b)], c = bt.col[size_t(b)];
        const int krow = h.row.rank[size_t(r)], kcol = vin.rank[size_t(c)];
        const int pr = kr[size_t(r)], pc = kc[size_t(c)];
        if (pr == 0 || pc == 0) continue;
        g1.push_back(GemmDesc{rr.at(size_t(r)), Sp(h, i), t.at(q), pr, kcol, krow, ld1(pr), ld1(krow), ld1(pr), 0, 0,
                              1.0, 0.0});
        g2.push_back(GemmDesc{t.at(q), rc.at(size_t(c)), Sp(*out, i), pr, pc, kcol, ld1(pr), ld1(pc), ld1(pr), 0, 1,
                              1.0, 0.0});
    }
    bgemm(g1, s);
    bgemm(g2, s);
    copy_array(out->D, h.D, s);
    out->orthonormal = true;
    return out;
}

namespace {
struct Truncation {
    std::vector<int> rank;   // kept columns per node
    Arena U;                 // left singular vectors per node (k_v x min(k_v, cols_v), ld k_v)
};

// top-down truncation bases of one side (algebra.hpp:150-196)
Truncation truncation_bases(const H2Dev& g, bool row_side, double eps, double level_corr,
                            const std::vector<std::vector<size_t>>& by_row,
                            const std::vector<std::vector<size_t>>& by_col, cudaStream_t s) {
    NvtxRange nvtx("recompress truncation bases");
    const ClusterTree& ct = g.tree();
    const BlockTree& bt = *g.bt;
    const int nn = ct.num_nodes();
    const BasisDev& B = row_side ? g.row : g.col;
    const BasisDev& rowB = g.row;
    const BasisDev& colB = col_basis(g);
    // column counts of G_v and of P_v (structure only; no data dependence)
    std::vector<int> cols(size_t(nn), 0), pc(size_t(nn), 0);
    for (int l = 0; l <= ct.depth; ++l)
        for (int v : ct.levels[size_t(l)]) {
            const int k = B.rank[size_t(v)];
            int c = 0;
            if (row_side) {
                for (size_t i : by_row[size_t(v)]) c += colB.rank[size_t(bt.col[size_t(bt.adm[i])])];
                if (g.symmetric)
                    for (size_t i : by_col[size_t(v)])
                        if (bt.row[size_t(bt.adm[i])] != v) c += rowB.rank[size_t(bt.row[size_t(bt.adm[i])])];
            } else {
                for (size_t i : by_col[size_t(v)]) c += rowB.rank[size_t(bt.row[size_t(bt.adm[i])])];
            }
            const int par = ct.parent[size_t(v)];
            if (par >= 0 && pc[size_t(par)] > 0) c += pc[size_t(par)];
            if (c == 0 || k == 0) {
                cols[size_t(v)] = 0;
                pc[size_t(v)] = 0;
                continue;
            }
            cols[size_t(v)] = c;
            pc[size_t(v)] = c > k ? k : c;
        }
    Arena G, U, sg, P;
    std::vector<size_t> gs(static_cast<size_t>(nn)), us(static_cast<size_t>(nn)), ss(static_cast<size_t>(nn)), ps(static_cast<size_t>(nn));
    for (int v = 0; v < nn; ++v) {
        const size_t k = size_t(B.rank[size_t(v)]), c = size_t(cols[size_t(v)]);
        gs[size_t(v)] = k * c;
        us[size_t(v)] = k * std::min(k, c);
        ss[size_t(v)] = std::min(k, c);
        ps[size_t(v)] = c > k ? k * k : 0;   // when c <= k, P_v is G_v itself
    }
    G.plan(gs);
    U.plan(us);
    sg.plan(ss);
    P.plan(ps);
    G.alloc(s);
    U.alloc(s);
    sg.alloc(s);
    P.alloc(s);
    auto Pptr = [&](int v) { return cols[size_t(v)] > B.rank[size_t(v)] ? P.at(size_t(v)) : G.at(size_t(v)); };
    for (int l = 0; l <= ct.depth; ++l) {
        std::vector<CopyDesc> cp;
        std::vector<GemmDesc> gm;
        std::vector<LeftSvdDesc> sv;
        for (int v : ct.levels[size_t(l)]) {
            const int k = B.rank[size_t(v)], c = cols[size_t(v)];
            if (c == 0 || k == 0) continue;
            double* Gv = G.at(size_t(v));
            int at = 0;
            if (row_side) {
                for (size_t i : by_row[size_t(v)]) {
                    const int kc = colB.rank[size_t(bt.col[size_t(bt.adm[i])])];
                    if (kc) cp.push_back(CopyDesc{Sp(g, i), Gv + int64_t(at) * k, k, kc, k, k, 0});
                    at += kc;
                }
                if (g.symmetric)
                    for (size_t i : by_col[size_t(v)]) {
                        const int r = bt.row[size_t(bt.adm[i])];
                        if (r == v) continue;
                        const int kr = rowB.rank[size_t(r)];
                        if (kr) cp.push_back(CopyDesc{Sp(g, i), Gv + int64_t(at) * k, k, kr, ld1(kr), k, 1});
                        at += kr;
                    }
            } else {
                for (size_t i : by_col[size_t(v)]) {
                    const int kr = rowB.rank[size_t(bt.row[size_t(bt.adm[i])])];
                    if (kr) cp.push_back(CopyDesc{Sp(g, i), Gv + int64_t(at) * k, k, kr, ld1(kr), k, 1});
                    at += kr;
                }
            }
            const int par = ct.parent[size_t(v)];
            if (par >= 0 && pc[size_t(par)] > 0) {
                const int kpar = B.rank[size_t(par)];
                gm.push_back(GemmDesc{Ep(B, v), Pptr(par), Gv + int64_t(at) * k, k, pc[size_t(par)], kpar, k,
                                      ld1(kpar), k, 0, 0, 1.0, 0.0});
                at += pc[size_t(par)];
            }
            // columns 1000x below the smallest possible truncation threshold
            // (tau = eps sigma_0 / level_corr >= eps ||G||_F / (sqrt(min(k, c)) level_corr)) are
            // discarded, so the SVD need not converge among them (eps = 0: no such columns)
            const double skip = 1e-3 * eps / (std::sqrt(double(std::min(k, c))) * level_corr);
            sv.push_back(LeftSvdDesc{Gv, k, c, k, U.at(size_t(v)), k, sg.at(size_t(v)),
                                     c > k ? P.at(size_t(v)) : nullptr, k, skip});
        }
        const auto tl = Clock::now();
        bcopy(cp, s);
        bgemm(gm, s);
        bleft_svd(sv, s);
        if (g_trace_recompress && !sv.empty()) {   // diagnostics: per-level SVD batch shape and time
            H2B_CUDA(cudaStreamSynchronize(s));
            int km = 0, cm = 0;
            for (const auto& q : sv) {
                km = std::max(km, q.m);
                cm = std::max(cm, q.c);
            }
            std::fprintf(stderr, "trunc_level side=%d l=%d problems=%zu kmax=%d cmax=%d ms=%.3f\n", int(row_side), l,
                         sv.size(), km, cm, ms_since(tl));
        }
    }
    std::vector<double> sh(sg.total);
    if (sg.total)
        H2B_CUDA(cudaMemcpyAsync(sh.data(), sg.buf.data(), sg.total * sizeof(double), cudaMemcpyDeviceToHost, s));
    H2B_CUDA(cudaStreamSynchronize(s));
    Truncation tr;
    tr.rank.assign(size_t(nn), 0);
    for (int v = 0; v < nn; ++v) {
        const int k = B.rank[size_t(v)], c = cols[size_t(v)];
        if (c == 0 || k == 0) continue;
        const double* sv = sh.data() + sg.off[size_t(v)];
        const int ns = std::min(k, c);
        const double tau = eps * sv[0] / level_corr;
        int r = 0;
        while (r < ns && sv[r] > tau) ++r;
        tr.rank[size_t(v)] = r;
        if (g_trace_recompress)
            std::fprintf(stderr, "trunc side=%d v=%d k=%d c=%d s0=%.17g tau=%.17g r=%d lo=%.17g hi=%.17g\n",
                         int(row_side), v, k, c, sv[0], tau, r, r > 0 ? sv[r - 1] : -1.0, r < ns ? sv[r] : -1.0);
    }
    tr.U = std::move(U);
    return tr;
}

// w^T E w projection of one basis tree (algebra.hpp:203-221)
void project_basis(const ClusterTree& ct, const BasisDev& in, BasisDev& out, const Truncation& w, cudaStream_t s) {
    const int nn = ct.num_nodes();
    std::vector<size_t> ts(size_t(nn), 0);
    for (int v = 0; v < nn; ++v) {
        const int par = ct.parent[size_t(v)];
        if (par >= 0) ts[size_t(v)] = size_t(w.rank[size_t(v)]) * in.rank[size_t(par)];
    }
    Arena t;
    t.plan(ts);
    t.alloc(s);
    std::vector<GemmDesc> g1, g2;
    for (int v = 0; v < nn; ++v) {
        const int rv = w.rank[size_t(v)], kv = in.rank[size_t(v)];
        if (ct.is_leaf(v) && rv > 0) {
            const int m = int(ct.size(v));
            g2.push_back(GemmDesc{Up(in, v), w.U.at(size_t(v)), Up(out, v), m, rv, kv, ld1(m), ld1(kv), ld1(m), 0, 0,
                                  1.0, 0.0});
        }
        const int par = ct.parent[size_t(v)];
        if (par < 0) continue;
        const int kp = in.rank[size_t(par)], rp = w.rank[size_t(par)];
        if (rv == 0 || rp == 0) continue;
        g1.push_back(GemmDesc{w.U.at(size_t(v)), Ep(in, v), t.at(size_t(v)), rv, kp, kv, ld1(kv), ld1(kv), ld1(rv), 1,
                              0, 1.0, 0.0});
        g2.push_back(GemmDesc{t.at(size_t(v)), w.U.at(size_t(par)), Ep(out, v), rv, rp, kp, ld1(rv), ld1(kp), ld1(rv),
                              0, 0, 1.0, 0.0});
    }
    bgemm(g1, s);
    bgemm(g2, s);
}
}  // namespace

std::unique_ptr<H2Dev> recompress(const H2Dev& hin, double eps, cudaStream_t s) {
    NvtxRange nvtx("recompress");
    if (eps < 0) throw std::invalid_argument("recompress: eps must be >= 0");
    std::unique_ptr<H2Dev> own;
    const H2Dev* gp = &hin;
    if (!hin.orthonormal) {
        own = orthogonalize(hin, s);
        gp = own.get();
    }
    const H2Dev& g = *gp;
    const ClusterTree& ct = g.tree();
    const BlockTree& bt = *g.bt;
    const int nn = ct.num_nodes();
    const double level_corr = std::sqrt(double(std::max(ct.depth, 1)));
    std::vector<std::vector<size_t>> by_row(static_cast<size_t>(nn)), by_col(static_cast<size_t>(nn));
    for (size_t i = 0; i < bt.adm.size(); ++i) {
        if (g.s_off[i] < 0) continue;
        const int b = bt.adm[i];
        by_row[size_t(bt.row[size_t(b)])].push_back(i);
        by_col[size_t(bt.col[size_t(b)])].push_back(i);
    }
    Phase* ph9 = new Phase(9, s);
    Truncation wr = truncation_bases(g, true, eps, level_corr, by_row, by_col, s);
    Truncation wc_store;
    if (!g.symmetric) wc_store = truncation_bases(g, false, eps, level_corr, by_row, by_col, s);
    delete ph9;
    Phase* ph10 = new Phase(10, s);
    const Truncation& wc = g.symmetric ? wr : wc_store;
    auto out = make_h2(g.bt, g.symmetric, wr.rank.data(), g.symmetric ? nullptr : wc.rank.data());
    // couplings: S <- w_row^T S w_col
    const BasisDev& cin = col_basis(g);
    std::vector<size_t> ts, idx;
    for (size_t i = 0; i < bt.adm.size(); ++i) {
        if (g.s_off[i] < 0) continue;
        idx.push_back(i);
        const int b = bt.adm[i];
        ts.push_back(size_t(wr.rank[size_t(bt.row[size_t(b)])]) * cin.rank[size_t(bt.col[size_t(b)])]);
    }
    Arena t;
    t.plan(ts);
    t.alloc(s);
    std::vector<GemmDesc> g1, g2;
    for (size_t q = 0; q < idx.size(); ++q) {
        const size_t i = idx[q];
        const int b = bt.adm[i], r = bt.row[size_t(b)], c = bt.col[size_t(b)];
        const int kr = g.row.rank[size_t(r)], kc = cin.rank[size_t(c)];
        const int rr = wr.rank[size_t(r)], rc = wc.rank[size_t(c)];
        if (rr == 0 || rc == 0) continue;
        g1.push_back(GemmDesc{wr.U.at(size_t(r)), Sp(g, i), t.at(q), rr, kc, kr, ld1(kr), ld1(kr), ld1(rr), 1, 0, 1.0,
                              0.0});
        g2.push_back(GemmDesc{t.at(q), wc.U.at(size_t(c)), Sp(*out, i), rr, rc, kc, ld1(rr), ld1(kc), ld1(rr), 0, 0,
                              1.0, 0.0});
    }
    bgemm(g1, s);
    bgemm(g2, s);
    project_basis(ct, g.row, out->row, wr, s);
    if (!g.symmetric) project_basis(ct, g.col, out->col, wc, s);
    copy_array(out->D, g.D, s);
    out->orthonormal = false;
    delete ph10;
    return orthogonalize(*out, s);
}

// ---------------------------------------------------------------------------
// local low-rank updates (algebra.hpp:236-316), several disjoint regions at once
// ---------------------------------------------------------------------------
std::unique_ptr<H2Dev> apply_local_updates(const H2Dev& h, const std::vector<LocalUpdate>& ups, cudaStream_t s) {
    const ClusterTree& ct = h.tree();
    const BlockTree& bt = *h.bt;
    const int nn = ct.num_nodes();
    // region membership per basis: (update index, side 0 = X / t, 1 = Y / s)
    struct Mark {
        int u = -1, side = 0;
    };
    std::vector<Mark> mrow(static_cast<size_t>(nn)), mcol(static_cast<size_t>(nn));
    std::vector<char> in_t_any(size_t(nn), 0);
    auto mark = [&](std::vector<Mark>& m, int root, int u, int side) {
        std::vector<int> st{root};
        while (!st.empty()) {
            const int v = st.back();
            st.pop_back();
            if (m[size_t(v)].u >= 0) throw std::logic_error("local updates: overlapping regions");
            m[size_t(v)] = Mark{u, side};
            if (!ct.is_leaf(v)) {
                st.push_back(ct.child0[size_t(v)]);
                st.push_back(ct.child1[size_t(v)]);
            }
        }
    };
    for (size_t u = 0; u < ups.size(); ++u) {
        const LocalUpdate& up = ups[u];
        if (up.k == 0) continue;
        // a symmetric diagonal update (t == s) must have X == Y (algebra.hpp:242-243);
        // the caller guarantees it (low_rank_update desymmetrizes otherwise): the
        // region is augmented once with X and every (row, col) pair inside it
        // gets the identity coupling and X_r X_c^T dense contributions
        mark(mrow, up.t, int(u), 0);
        if (h.symmetric) {
            if (up.s != up.t) mark(mrow, up.s, int(u), 1);
        } else {
            mark(mcol, up.s, int(u), 1);
        }
    }
    std::vector<Mark>& mc = h.symmetric ? mrow : mcol;
    auto newr = [&](const BasisDev& b, const std::vector<Mark>& m) {
        std::vector<int> r(b.rank);
        for (int v = 0; v < nn; ++v)
            if (m[size_t(v)].u >= 0) r[size_t(v)] += ups[size_t(m[size_t(v)].u)].k;
        return r;
    };
    const std::vector<int> rr = newr(h.row, mrow);
    const std::vector<int> rc = h.symmetric ? rr : newr(h.col, mcol);
    auto out = make_h2(h.bt, h.symmetric, rr.data(), h.symmetric ? nullptr : rc.data());
    std::vector<CopyDesc> cp;
    std::vector<GemmDesc> gm;
    auto factor_rows = [&](const LocalUpdate& up, int side, int v) -> std::pair<const double*, int64_t> {
        const int root = side == 0 ? up.t : up.s;
        const int64_t off = ct.begin[size_t(v)] - ct.begin[size_t(root)];
        return side == 0 ? std::make_pair(up.X + off, up.ldx) : std::make_pair(up.Y + off, up.ldy);
    };
    auto augment = [&](const BasisDev& in, BasisDev& ob, const std::vector<Mark>& m) {
        for (int v = 0; v < nn; ++v) {
            const int k = in.rank[size_t(v)];
            const Mark mk = m[size_t(v)];
            if (ct.is_leaf(v)) {
                const int mm = int(ct.size(v));
                if (k) cp.push_back(CopyDesc{Up(in, v), Up(ob, v), mm, k, ld1(mm), ld1(mm), 0});
                if (mk.u >= 0) {
                    const LocalUpdate& up = ups[size_t(mk.u)];
                    auto f = factor_rows(up, mk.side, v);
                    cp.push_back(CopyDesc{f.first, Up(ob, v) + int64_t(k) * mm, mm, up.k, int(f.second), ld1(mm), 0});
                }
            }
            const int par = ct.parent[size_t(v)];
            if (par < 0) continue;
            const int kpar = in.rank[size_t(par)];
            const int knew = k + (mk.u >= 0 ? ups[size_t(mk.u)].k : 0);
            if (k && kpar) cp.push_back(CopyDesc{Ep(in, v), Ep(ob, v), k, kpar, ld1(k), ld1(knew), 0});
            if (mk.u >= 0 && m[size_t(par)].u == mk.u && m[size_t(par)].side == mk.side) {
                const int kp = ups[size_t(mk.u)].k;
                cp.push_back(CopyDesc{nullptr, Ep(ob, v) + k + int64_t(kpar) * knew, kp, kp, 1, ld1(knew), 2});
            }
        }
    };
    augment(h.row, out->row, mrow);
    if (!h.symmetric) augment(h.col, out->col, mcol);
    const BasisDev& vin = col_basis(h);
    for (size_t i = 0; i < bt.adm.size(); ++i) {
        if (h.s_off[i] < 0) continue;
        const int b = bt.adm[i], r = bt.row[size_t(b)], c = bt.col[size_t(b)];
        const int kr = h.row.rank[size_t(r)], kc = vin.rank[size_t(c)];
        const int nr = rr[size_t(r)];
        if (kr && kc) cp.push_back(CopyDesc{Sp(h, i), Sp(*out, i), kr, kc, ld1(kr), ld1(nr), 0});
        const Mark a = mrow[size_t(r)], bm = mc[size_t(c)];
        const bool self = a.u >= 0 && h.symmetric && ups[size_t(a.u)].t == ups[size_t(a.u)].s;
        const bool ident = a.u >= 0 && a.u == bm.u &&
                           (self || (a.side == 0 && bm.side == 1) || (h.symmetric && a.side == 1 && bm.side == 0));
        if (ident) {
            const int kp = ups[size_t(a.u)].k;
            cp.push_back(CopyDesc{nullptr, Sp(*out, i) + kr + int64_t(kc) * nr, kp, kp, 1, ld1(nr), 2});
        }
    }
    copy_array(out->D, h.D, s);
    for (size_t i = 0; i < bt.dense.size(); ++i) {
        if (h.d_off[i] < 0) continue;
        const int b = bt.dense[i], r = bt.row[size_t(b)], c = bt.col[size_t(b)];
        const Mark a = mrow[size_t(r)], bm = mc[size_t(c)];
        if (a.u < 0 || a.u != bm.u) continue;
        const LocalUpdate& up = ups[size_t(a.u)];
        const int mr = int(ct.size(r)), mcn = int(ct.size(c));
        const bool self = h.symmetric && up.t == up.s;
        if (self || (a.side == 0 && bm.side == 1)) {
            auto x = factor_rows(up, 0, r);
            auto y = factor_rows(up, 1, c);
            gm.push_back(GemmDesc{x.first, y.first, Dp(*out, i), mr, mcn, up.k, int(x.second), int(y.second), mr, 0, 1,
                                  1.0, 1.0});
        } else if (h.symmetric && a.side == 1 && bm.side == 0) {
            auto y = factor_rows(up, 1, r);
            auto x = factor_rows(up, 0, c);
            gm.push_back(GemmDesc{y.first, x.first, Dp(*out, i), mr, mcn, up.k, int(y.second), int(x.second), mr, 0, 1,
                                  1.0, 1.0});
        }
    }
    bcopy(cp, s);
    bgemm(gm, s);
    out->orthonormal = false;
    return out;
}

// ---------------------------------------------------------------------------
// peel_construct (construction.hpp:226-382)
// ---------------------------------------------------------------------------
namespace {


struct PeelContext {
    DevOperator& op;
    const H2Dev* partial = nullptr;   // residual = op - partial (ResidualOperator, :203-222)
    DeviceArray<int> perm;
    Workspace ws;
    cudaStream_t s;
    int64_t n;
    unsigned long long panel_counter = 0;

    PeelContext(DevOperator& o, const ClusterTree& ct, cudaStream_t st) : op(o), s(st), n(ct.n) {
        perm.upload(int32_perm(ct));
    }
    // y = residual(x) or residual^T(x), user ordering
    // operator time: bracketing events on the stream (summed once at the end of
    // the build), so timing the black box costs no synchronisation
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> op_events;
    ~PeelContext() {
        for (auto& e : op_events) {
            cudaEventDestroy(e.first);
            cudaEventDestroy(e.second);
        }
    }
    double op_device_ms() {
        double t = 0;
        for (auto& e : op_events) {
            float ms = 0;
            H2B_CUDA(cudaEventSynchronize(e.second));
            H2B_CUDA(cudaEventElapsedTime(&ms, e.first, e.second));
            t += ms;
        }
        return t;
    }
    void residual(bool transpose, int64_t b, const double* x, double* y) {
        const auto t0 = Clock::now();
        cudaEvent_t e0, e1;
        H2B_CUDA(cudaEventCreate(&e0));
        H2B_CUDA(cudaEventCreate(&e1));
        op_events.emplace_back(e0, e1);
        H2B_CUDA(cudaEventRecord(e0, s));
        if (transpose) op.apply_transpose(b, x, y, s);
        else op.apply(b, x, y, s);
        H2B_CUDA(cudaEventRecord(e1, s));
        if (g_phase_sync) H2B_CUDA(cudaStreamSynchronize(s));
        g_phase_ms[1] += ms_since(t0);
        if (partial) {
            Phase ph(2, s);
            hgemv(*partial, transpose, true, n, b, x, n, y, n, -1.0, 1.0, s, ws);
        }
    }
};

struct Range {
    int t = -1, s = -1;
    int rank = 0;
    bool converged = false, wants_full = true;
    double err_est = 0;
};

// sample_level_group (construction.hpp:226-291). Q factors live in one n x cap
// internal-order matrix (pair i on the rows of t_i); returns V factors in Wi.
std::vector<Range> sample_level_group(PeelContext& ctx, const ClusterTree& ct,
                                      const std::vector<std::pair<int, int>>& pairs, double tol_abs,
                                      const PeelConfig& cfg, std::mt19937_64& rng, DBuf& Qlev, int& cap, DBuf& Wi) {
    NvtxRange nvtx("sample_level_group");
    const int64_t n = ct.n;
    cudaStream_t s = ctx.s;
    std::vector<Range> ranges(pairs.size());
    for (size_t i = 0; i < pairs.size(); ++i) {
        ranges[i].t = pairs[i].first;
        ranges[i].s = pairs[i].second;
    }
    const int64_t b = std::max<int64_t>(cfg.sample_block_size, 1);
    const int64_t probes = std::min<int64_t>(std::max<int64_t>(cfg.oversampling, 1), b);
    cap = int(std::max<int64_t>(2 * b, 32));
    Qlev.alloc(size_t(n) * cap, s);
    Qlev.zero();
    std::vector<double> omh;
    DBuf om, omu, y, yi, ub, sg;
    bool all_done = false;
    while (!all_done) {
        int64_t panel = 0;
        for (const auto& r : ranges)
            if (!r.converged) panel = std::max(panel, r.wants_full ? b : probes);
        // Omega in internal order: Gaussians on each unconverged pair's s rows
        om.alloc(size_t(n * panel), s);
        omu.alloc(size_t(n * panel), s);
        y.alloc(size_t(n * panel), s);
        yi.alloc(size_t(n * panel), s);
        Phase* ph_rng = new Phase(0, s);
        if (cfg.rng == 0) {
            omh.assign(size_t(n * panel), 0.0);
            for (auto& r : ranges) {
                if (r.converged) continue;
                fill_gaussian(omh.data() + ct.begin[size_t(r.s)], ct.size(r.s), panel, n, rng);
            }
            H2B_CUDA(cudaMemcpyAsync(om.data(), omh.data(), omh.size() * sizeof(double), cudaMemcpyHostToDevice, s));
        } else {
            om.zero();
            std::vector<RngSeg> segs;
            for (auto& r : ranges)
                if (!r.converged) segs.push_back(RngSeg{ct.begin[size_t(r.s)], ct.size(r.s)});
            DeviceArray<RngSeg> dsegs;
            dsegs.upload(segs, s);
            int64_t maxrows = 0;
            for (const RngSeg& g : segs) maxrows = std::max(maxrows, g.rows);
            const int64_t bx = std::min<int64_t>((maxrows * panel / 2 + 255) / 256, 4096);
            philox_fill_kernel<<<dim3(unsigned(std::max<int64_t>(bx, 1)), unsigned(segs.size())), 256, 0, s>>>(
                dsegs.data(), int(segs.size()), panel, n, om.data(), cfg.seed, ctx.panel_counter++);
            H2B_LAUNCH();
        }
        la::permute_rows(om.data(), n, omu.data(), n, ctx.perm.data(), n, panel, true, s);
        delete ph_rng;
        ctx.residual(false, panel, omu.data(), y.data());
        Phase ph_absorb(3, s);
        la::permute_rows(y.data(), n, yi.data(), n, ctx.perm.data(), n, panel, false, s);
        const double keep_tol = 0.5 * tol_abs * std::sqrt(double(panel));
        // absorb_panel (construction.hpp:105-129), batched over the unconverged pairs
        std::vector<size_t> act;
        for (size_t i = 0; i < ranges.size(); ++i)
            if (!ranges[i].converged) act.push_back(i);
        Arena cbuf;
        std::vector<size_t> cs;
        for (size_t i : act) cs.push_back(size_t(ranges[i].rank) * panel);
        cbuf.plan(cs);
        cbuf.alloc(s);
        for (int pass = 0; pass < 2; ++pass) {
            std::vector<GemmDesc> g1, g2;
            for (size_t q = 0; q < act.size(); ++q) {
                const Range& r = ranges[act[q]];
                if (r.rank == 0) continue;
                const int m = int(ct.size(r.t));
                const double* Qt = Qlev.data() + ct.begin[size_t(r.t)];
                double* Yt = yi.data() + ct.begin[size_t(r.t)];
                g1.push_back(GemmDesc{Qt, Yt, cbuf.at(q), r.rank, int(panel), m, int(n), int(n), r.rank, 1, 0, 1.0, 0.0});
                g2.push_back(GemmDesc{Qt, cbuf.at(q), Yt, m, int(panel), r.rank, int(n), r.rank, int(n), 0, 0, -1.0, 1.0});
            }
            bgemm(g1, s);
            bgemm(g2, s);
        }
        Arena us, ss;
        std::vector<size_t> usz, ssz;
        for (size_t i : act) {
            const int64_t m = ct.size(ranges[i].t), p = std::min<int64_t>(m, panel);
            usz.push_back(size_t(m * p));
            ssz.push_back(size_t(p));
        }
        us.plan(usz);
        ss.plan(ssz);
        us.alloc(s);
        ss.alloc(s);
        std::vector<LeftSvdDesc> sv;
        for (size_t q = 0; q < act.size(); ++q) {
            const Range& r = ranges[act[q]];
            const int m = int(ct.size(r.t));
            sv.push_back(LeftSvdDesc{yi.data() + ct.begin[size_t(r.t)], m, int(panel), int(n), us.at(q), m, ss.at(q),
                                     nullptr, 0});
        }
        bleft_svd(sv, s);
        std::vector<double> sh(ss.total);
        if (ss.total)
            H2B_CUDA(cudaMemcpyAsync(sh.data(), ss.buf.data(), ss.total * sizeof(double), cudaMemcpyDeviceToHost, s));
        H2B_CUDA(cudaStreamSynchronize(s));
        // host decisions, then append the kept columns
        std::vector<int> kept(act.size(), 0);
        int need_cap = cap;
        for (size_t q = 0; q < act.size(); ++q) {
            Range& r = ranges[act[q]];
            const int64_t m = ct.size(r.t), p = std::min<int64_t>(m, panel);
            const double* sv = sh.data() + ss.off[q];
            int kk = 0;
            while (kk < p && sv[kk] > keep_tol) ++kk;
            const int64_t capr = std::min(ct.size(r.t), ct.size(r.s));
            const int64_t max_rank = cfg.max_rank > 0 ? cfg.max_rank : capr + b;
            if (max_rank > 0 && r.rank + kk > max_rank)
                throw max_rank_error("adaptive factorization: block rank exceeds max_rank");
            kept[q] = kk;
            need_cap = std::max(need_cap, r.rank + kk);
            if (g_trace_absorb)   // diagnostics (H2_TRACE_ABSORB): one line per absorbed panel
                std::fprintf(stderr, "absorb t=%d s=%d q=%d b=%ld tol=%.17g kept=%d lo=%.17g hi=%.17g\n", r.t, r.s,
                             r.rank, long(panel), keep_tol, kk, kk > 0 ? sv[kk - 1] : -1.0, kk < p ? sv[kk] : -1.0);
        }
        if (need_cap > cap) {
            int nc = cap;
            while (nc < need_cap) nc *= 2;
            DBuf q2(size_t(n) * nc, s);
            q2.zero();
            H2B_CUDA(cudaMemcpyAsync(q2.data(), Qlev.data(), size_t(n) * cap * sizeof(double), cudaMemcpyDeviceToDevice,
                                     s));
            Qlev = std::move(q2);
            cap = nc;
        }
        std::vector<CopyDesc> cp;
        all_done = true;
        for (size_t q = 0; q < act.size(); ++q) {
            Range& r = ranges[act[q]];
            const int m = int(ct.size(r.t));
            const int kk = kept[q];
            const int64_t p = std::min<int64_t>(m, panel);
            if (kk > 0)
                cp.push_back(CopyDesc{us.at(q), Qlev.data() + ct.begin[size_t(r.t)] + int64_t(r.rank) * n, m, kk, m,
                                      int(n), 0});
            r.rank += kk;
            r.wants_full = kk == panel;
            if (kk < panel && (panel - kk) >= probes) {
                r.converged = true;
                r.err_est = kk < p ? sh[ss.off[q] + size_t(kk)] : 0.0;
            }
            const int64_t capr = std::min(ct.size(r.t), ct.size(r.s));
            if (!r.converged && r.rank >= capr) {
                r.converged = true;
                r.err_est = 0;
            }
            all_done = all_done && r.converged;
        }
        bcopy(cp, s);
    }
    // transposed pass (:272-289): W = residual^T Z, Z = each pair's Q on its t rows
    Phase ph_t(4, s);
    int kmax = 0;
    for (const auto& r : ranges) kmax = std::max(kmax, r.rank);
    if (kmax > 0) {
        DBuf z(size_t(n) * kmax, s), w(size_t(n) * kmax, s);
        la::permute_rows(Qlev.data(), n, z.data(), n, ctx.perm.data(), n, kmax, true, s);
        ctx.residual(true, kmax, z.data(), w.data());
        Wi.alloc(size_t(n) * kmax, s);
        la::permute_rows(w.data(), n, Wi.data(), n, ctx.perm.data(), n, kmax, false, s);
    }
    return ranges;
}
}  // namespace

PeelResult peel_construct(DevOperator& op, std::shared_ptr<const BlockTree> bt, const PeelConfig& cfg,
                          cudaStream_t s) {
    NvtxRange nvtx("peel_construct");
    const auto t_start = Clock::now();
    const ClusterTree& ct = *bt->tree;
    if (ct.n != op.dim()) throw std::invalid_argument("peel_construct: dimension mismatch");
    std::mt19937_64 rng(cfg.seed);
    SampleStats stats;
    const bool sym = op.symmetric();
    long before = op.columns_applied();
    double norm_scale = cfg.norm_scale;
    if (norm_scale <= 0) norm_scale = std::max(pnorm2_estimate(op, s).value, 1e-300);
    stats.add_level({0, 0, 0, op.columns_applied() - before});
    const double tol_abs = 0.5 * cfg.eps * norm_scale;
    std::unique_ptr<H2Dev> partial = make_h2(bt, sym, nullptr, nullptr);
    PeelContext ctx(op, ct, s);
    for (int level = 1; level <= ct.depth; ++level) {
        std::vector<std::pair<int, int>> pairs;
        for (int v : ct.levels[size_t(level - 1)])
            if (!ct.is_leaf(v)) pairs.emplace_back(ct.child0[size_t(v)], ct.child1[size_t(v)]);
        if (pairs.empty()) continue;
        before = op.columns_applied();
        int64_t max_rank_seen = 0;
        auto group = [&](const std::vector<std::pair<int, int>>& prs) {
            DBuf Qlev, Wi;
            int cap = 0;
            ctx.partial = partial.get();
            auto ranges = sample_level_group(ctx, ct, prs, tol_abs, cfg, rng, Qlev, cap, Wi);
            std::vector<LocalUpdate> ups;
            for (const Range& r : ranges) {
                max_rank_seen = std::max<int64_t>(max_rank_seen, r.rank);
                if (r.rank > 0)
                    ups.push_back(LocalUpdate{r.t, r.s, r.rank, Qlev.data() + ct.begin[size_t(r.t)], ct.n,
                                              Wi.data() + ct.begin[size_t(r.s)], ct.n});
            }
            if (!ups.empty()) {
                Phase ph(5, s);
                partial = apply_local_updates(*partial, ups, s);
            }
        };
        group(pairs);
        if (!sym) {
            std::vector<std::pair<int, int>> mirrored;
            for (auto [t, u] : pairs) mirrored.emplace_back(u, t);
            group(mirrored);
        }
        auto dump = [&](const char* tag) {   // diagnostics (H2_PEEL_DUMP=prefix): dense partial per level
            const char* dp = std::getenv("H2_PEEL_DUMP");
            if (!dp) return;
            std::vector<double> a(size_t(ct.n * ct.n));
            to_dense(*partial, ct.n, a.data(), s);
            std::string f = std::string(dp) + "_gpu_" + tag + std::to_string(level) + ".bin";
            if (FILE* fp = std::fopen(f.c_str(), "wb")) {
                std::fwrite(a.data(), 8, a.size(), fp);
                std::fclose(fp);
            }
        };
        dump("u");
        {
            Phase ph(6, s);
            partial = recompress(*partial, 0.5 * cfg.eps, s);
        }
        dump("r");
        stats.add_level({level, int64_t(pairs.size()) * (sym ? 1 : 2), max_rank_seen, op.columns_applied() - before});
    }
    // dense diagonal leaves (:357-376): indicator columns, residual apply, symmetrise, add
    before = op.columns_applied();
    {
        Phase ph(7, s);
        const int64_t n = ct.n, m = ct.max_leaf_size();
        DBuf om(size_t(n * m), s), omu(size_t(n * m), s), y(size_t(n * m), s), yi(size_t(n * m), s);
        om.zero();
        std::vector<CopyDesc> id;
        for (int v : ct.leaves) {
            const int sz = int(ct.size(v));
            id.push_back(CopyDesc{nullptr, om.data() + ct.begin[size_t(v)], sz, sz, 1, int(n), 2});
        }
        bcopy(id, s);
        la::permute_rows(om.data(), n, omu.data(), n, ctx.perm.data(), n, m, true, s);
        ctx.partial = partial.get();
        ctx.residual(false, m, omu.data(), y.data());
        la::permute_rows(y.data(), n, yi.data(), n, ctx.perm.data(), n, m, false, s);
        std::vector<CopyDesc> add;
        for (size_t i = 0; i < bt->dense.size(); ++i) {
            if (partial->d_off[i] < 0) continue;
            const int b = bt->dense[i];
            const int r = bt->row[size_t(b)];
            if (r != bt->col[size_t(b)]) continue;
            const int sz = int(ct.size(r));
            add.push_back(CopyDesc{yi.data() + ct.begin[size_t(r)], Dp(*partial, i), sz, sz, int(n), sz, sym ? 4 : 3});
        }
        bcopy(add, s);
    }
    stats.add_level({ct.depth + 1, int64_t(ct.leaves.size()), 0, op.columns_applied() - before});
    PeelResult res;
    res.matrix = recompress(*partial, cfg.eps, s);
    res.stats = std::move(stats);
    H2B_CUDA(cudaStreamSynchronize(s));
    res.times.op_ms = ctx.op_device_ms();
    res.times.total_ms = ms_since(t_start);
    return res;
}

double estimate_relative_error(DevOperator& op, const H2Dev& h, double op_norm, cudaStream_t s) {
    Workspace ws;
    const int64_t n = op.dim();
    FunctionDevOperator diff(
        n, false,
        [&](bool transpose, int64_t b, const double* x, double* y, cudaStream_t st) {
            if (transpose) op.apply_transpose(b, x, y, st);
            else op.apply(b, x, y, st);
            hgemv(h, transpose, true, n, b, x, n, y, n, -1.0, 1.0, st, ws);
        },
        true);
    const double err = pnorm2_estimate(diff, s).value;
    const double base = op_norm > 0 ? op_norm : pnorm2_estimate(op, s).value;
    return base > 0 ? err / base : err;
}

}  // namespace h2b

// diagnostic hook (not part of the public ABI): per-phase host wall time of the last peel_construct
// diagnostics: 1 = drain the stream at every phase end so the phase timers are
// device-accurate (slower builds); 0 (default) = no timing synchronisation
extern "C" int h2b_hara_phase_sync(int on) {
    h2b::g_phase_sync = on;
    return 0;
}
// the phase timers accumulate across builds until reset (an inversion runs many)
extern "C" int h2b_hara_phase_reset() {
    std::fill(h2b::g_phase_ms, h2b::g_phase_ms + 16, 0.0);
    return 0;
}
extern "C" int h2b_hara_phase_ms(double* out, int n) {
    for (int i = 0; i < n && i < 16; ++i) out[i] = h2b::g_phase_ms[i];
    return 0;
}
