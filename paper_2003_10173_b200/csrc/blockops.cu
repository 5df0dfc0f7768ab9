// Block-level construction primitives and H^2 diagnostics on the B200
// (blockops.hpp). Everything the reference does per block row / per node runs
// as batched launches over HBM-resident payloads; only scalar decisions (kept
// ranks, convergence) and the diagnostics' results cross to the host.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "blockops.hpp"
#include "inversion.hpp"
#include "matrix.hpp"
#include "refstream.hpp"

namespace h2b {

using la::bcopy;
using la::bgemm;
using la::bleft_svd;
using la::CopyDesc;
using la::DBuf;
using la::GemmDesc;
using la::LeftSvdDesc;

namespace {

int ld1(int64_t x) { return int(std::max<int64_t>(x, 1)); }

void check_node(const ClusterTree& ct, int v, const char* what) {
    if (v < 0 || v >= ct.num_nodes()) throw std::invalid_argument(std::string(what) + ": cluster id out of range");
}

// the reference normal stream (construction.hpp:81-85), |rows| x cols packed
void fill_gaussian(double* m, int64_t rows, int64_t cols, std::mt19937_64& rng) {
    ref_fill_gaussian(m, rows, cols, rows, rng);
}

// dst[idx[i] + j * ldd] = src[i + j * lds]   (scatter = 1)
// dst[i + j * ldd] = src[idx[i] + j * lds]   (scatter = 0)
__global__ void rows_by_index_kernel(const double* __restrict__ src, int64_t lds, double* __restrict__ dst,
                                     int64_t ldd, const int* __restrict__ idx, int64_t rows, int64_t cols,
                                     int scatter) {
    const int64_t total = rows * cols;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = e % rows, j = e / rows;
        if (scatter) dst[idx[i] + j * ldd] = src[i + j * lds];
        else dst[i + j * ldd] = src[idx[i] + j * lds];
    }
}
void rows_by_index(const double* src, int64_t lds, double* dst, int64_t ldd, const int* idx, int64_t rows,
                   int64_t cols, bool scatter, cudaStream_t st) {
    if (rows <= 0 || cols <= 0) return;
    const int64_t blocks = std::min<int64_t>((rows * cols + 255) / 256, 148 * 16);
    rows_by_index_kernel<<<unsigned(blocks), 256, 0, st>>>(src, lds, dst, ldd, idx, rows, cols, scatter ? 1 : 0);
    H2B_LAUNCH();
}

// the user-order indices of cluster v's rows (perm[begin .. end))
DeviceArray<int> cluster_rows(const ClusterTree& ct, int v, cudaStream_t st) {
    std::vector<int> idx(size_t(ct.size(v)));
    for (int64_t i = 0; i < ct.size(v); ++i) idx[size_t(i)] = int(ct.perm[size_t(ct.begin[size_t(v)] + i)]);
    DeviceArray<int> d;
    d.upload(idx, st);
    return d;
}

// sigma of each panel (values only), copied to the host
std::vector<double> singular_values(const double* a, int m, int c, int lda, cudaStream_t st) {
    const int p = std::min(m, c);
    if (p == 0) return {};
    DBuf u(size_t(m) * p, st), sg(size_t(p), st);
    bleft_svd({LeftSvdDesc{a, m, c, lda, u.data(), m, sg.data(), nullptr, 0}}, st);
    std::vector<double> h(static_cast<size_t>(p));
    H2B_CUDA(cudaMemcpyAsync(h.data(), sg.data(), h.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
    H2B_CUDA(cudaStreamSynchronize(st));
    return h;
}

}  // namespace

// ---------------------------------------------------------------------------
// sample_block_column (construction.hpp:137-148)
// ---------------------------------------------------------------------------
void sample_block_column(DevOperator& op, const ClusterTree& ct, int t, int s, int64_t count, std::mt19937_64& rng,
                         double* omega_s, double* y_t, cudaStream_t st) {
    if (count < 1) throw std::invalid_argument("sample_block_column: count must be >= 1");
    check_node(ct, t, "sample_block_column");
    check_node(ct, s, "sample_block_column");
    const int64_t n = ct.n, ms = ct.size(s), mt = ct.size(t);
    std::vector<double> g(size_t(ms * count));
    fill_gaussian(g.data(), ms, count, rng);
    H2B_CUDA(cudaMemcpyAsync(omega_s, g.data(), g.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    DeviceArray<int> rs = cluster_rows(ct, s, st), rt = cluster_rows(ct, t, st);
    DBuf om(size_t(n * count), st), y(size_t(n * count), st);
    om.zero();
    rows_by_index(omega_s, ms, om.data(), n, rs.data(), ms, count, true, st);
    op.apply(count, om.data(), y.data(), st);
    rows_by_index(y.data(), n, y_t, ld1(mt), rt.data(), mt, count, false, st);
    // g is pageable: the upload above completed before cudaMemcpyAsync returned
}

// ---------------------------------------------------------------------------
// adaptive_block_factorization (construction.hpp:156-198) with absorb_panel
// (:105-129): one block, a fresh mt19937_64(cfg.seed), sample_block_column
// panels until the trailing directions prove convergence, then the row factor
// from one transposed application on the padded basis.
// ---------------------------------------------------------------------------
BlockFactorDev adaptive_block_factorization(DevOperator& op, const ClusterTree& ct, int t, int s, double eps_block,
                                            const PeelConfig& cfg, cudaStream_t st) {
    check_node(ct, t, "adaptive_block_factorization");
    check_node(ct, s, "adaptive_block_factorization");
    std::mt19937_64 rng(cfg.seed);
    const int64_t n = ct.n, mt = ct.size(t), ms = ct.size(s);
    const int64_t b = std::max<int64_t>(cfg.sample_block_size, 1);
    const int64_t probes = std::min<int64_t>(std::max<int64_t>(cfg.oversampling, 1), b);
    const int64_t dim_cap = std::min(mt, ms);
    const int64_t max_rank = cfg.max_rank > 0 ? cfg.max_rank : dim_cap + b;
    int64_t cap = std::max<int64_t>(2 * b, 32), rank = 0;
    DBuf q(size_t(mt * cap), st);
    bool converged = false, wants_full = true;
    double scale = 0, err_est = 0;
    DBuf om, y, c;
    while (!converged) {
        const int64_t panel = wants_full ? b : probes;
        om.alloc(size_t(ms * panel), st);
        y.alloc(size_t(mt * panel), st);
        sample_block_column(op, ct, t, s, panel, rng, om.data(), y.data(), st);
        // scale = max(scale, JacobiSVD(y).singularValues()(0)) on the raw panel
        const std::vector<double> s0 = singular_values(y.data(), int(mt), int(panel), ld1(mt), st);
        if (!s0.empty()) scale = std::max(scale, s0[0]);
        const double keep_tol = 0.5 * eps_block * scale;
        // two projection passes against the current basis
        if (rank > 0) {
            c.alloc(size_t(rank * panel), st);
            for (int pass = 0; pass < 2; ++pass) {
                bgemm({GemmDesc{q.data(), y.data(), c.data(), int(rank), int(panel), int(mt), ld1(mt), ld1(mt),
                                int(rank), 1, 0, 1.0, 0.0}},
                      st);
                bgemm({GemmDesc{q.data(), c.data(), y.data(), int(mt), int(panel), int(rank), ld1(mt), int(rank),
                                ld1(mt), 0, 0, -1.0, 1.0}},
                      st);
            }
        }
        const int64_t p = std::min(mt, panel);
        DBuf u(size_t(mt * std::max<int64_t>(p, 1)), st), sg(size_t(std::max<int64_t>(p, 1)), st);
        std::vector<double> sv(static_cast<size_t>(p));
        if (p > 0) {
            bleft_svd({LeftSvdDesc{y.data(), int(mt), int(panel), ld1(mt), u.data(), ld1(mt), sg.data(), nullptr, 0}},
                      st);
            H2B_CUDA(cudaMemcpyAsync(sv.data(), sg.data(), sv.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
            H2B_CUDA(cudaStreamSynchronize(st));
        }
        int64_t kept = 0;
        while (kept < p && sv[size_t(kept)] > keep_tol) ++kept;
        if (max_rank > 0 && rank + kept > max_rank)
            throw max_rank_error("adaptive factorization: block rank exceeds max_rank");
        if (kept > 0) {
            if (rank + kept > cap) {
                int64_t nc = cap;
                while (nc < rank + kept) nc *= 2;
                DBuf q2(size_t(mt * nc), st);
                if (rank)
                    H2B_CUDA(cudaMemcpyAsync(q2.data(), q.data(), size_t(mt * rank) * sizeof(double),
                                             cudaMemcpyDeviceToDevice, st));
                q = std::move(q2);
                cap = nc;
            }
            bcopy({CopyDesc{u.data(), q.data() + rank * mt, int(mt), int(kept), ld1(mt), ld1(mt), 0}}, st);
            rank += kept;
        }
        wants_full = kept == panel;
        if (kept < panel && (panel - kept) >= probes) {
            converged = true;
            err_est = kept < p ? sv[size_t(kept)] : 0.0;
        }
        if (!converged && rank >= dim_cap) {
            converged = true;   // full block captured
            err_est = 0;
        }
    }
    BlockFactorDev f;
    f.rank = rank;
    f.err_est = err_est;
    f.u.alloc(size_t(mt * rank), st);
    f.v.alloc(size_t(ms * rank), st);
    if (rank > 0) {
        H2B_CUDA(cudaMemcpyAsync(f.u.data(), q.data(), size_t(mt * rank) * sizeof(double), cudaMemcpyDeviceToDevice,
                                 st));
        DeviceArray<int> rt = cluster_rows(ct, t, st), rs = cluster_rows(ct, s, st);
        DBuf z(size_t(n * rank), st), w(size_t(n * rank), st);
        z.zero();
        rows_by_index(q.data(), mt, z.data(), n, rt.data(), mt, rank, true, st);
        op.apply_transpose(rank, z.data(), w.data(), st);
        rows_by_index(w.data(), n, f.v.data(), ld1(ms), rs.data(), ms, rank, false, st);
    }
    H2B_CUDA(cudaStreamSynchronize(st));
    return f;
}

// ---------------------------------------------------------------------------
// local_low_rank_update (algebra.hpp:323-332)
// ---------------------------------------------------------------------------
std::unique_ptr<H2Dev> local_low_rank_update(const H2Dev& h, int t, int s, int64_t k, const double* U, int64_t ldu,
                                             const double* V, int64_t ldv, double eps, cudaStream_t st) {
    const ClusterTree& ct = h.tree();
    check_node(ct, t, "local_low_rank_update");
    check_node(ct, s, "local_low_rank_update");
    if (k < 0) throw std::invalid_argument("local update: factor dimensions do not match clusters");
    if (k == 0) return clone_h2(h, st);   // `return h` (a copy, value semantics)
    const int64_t mt = ct.size(t), ms = ct.size(s);
    if (U == nullptr || V == nullptr || ldu < mt || ldv < ms)
        throw std::invalid_argument("local update: factor dimensions do not match clusters");
    // detail::bitwise_equal(u_blk, v_blk): same shape and identical bits
    bool same = U == V && ldu == ldv;
    if (!same && t == s && h.symmetric) {
        std::vector<double> hu(size_t(mt * k)), hv(size_t(ms * k));
        H2B_CUDA(cudaMemcpy2DAsync(hu.data(), size_t(mt) * sizeof(double), U, size_t(ldu) * sizeof(double),
                                   size_t(mt) * sizeof(double), size_t(k), cudaMemcpyDeviceToHost, st));
        H2B_CUDA(cudaMemcpy2DAsync(hv.data(), size_t(ms) * sizeof(double), V, size_t(ldv) * sizeof(double),
                                   size_t(ms) * sizeof(double), size_t(k), cudaMemcpyDeviceToHost, st));
        H2B_CUDA(cudaStreamSynchronize(st));
        same = std::memcmp(hu.data(), hv.data(), hu.size() * sizeof(double)) == 0;
    }
    std::unique_ptr<H2Dev> own;
    const H2Dev* g = &h;
    if (h.symmetric && t == s && !same) {
        own = desymmetrized(h, st);
        g = own.get();
    }
    auto upd = apply_local_updates(*g, {LocalUpdate{t, s, int(k), U, ldu, V, ldv}}, st);
    return recompress(*upd, eps, st);
}

// ---------------------------------------------------------------------------
// frobenius_norm (algebra.hpp:119-137): sum of squares of every stored
// coupling and dense block, off-diagonal blocks of a symmetric matrix counted
// twice. One CTA per block writes its weighted partial; a single CTA sums the
// partials in block order (deterministic).
// ---------------------------------------------------------------------------
namespace {
struct SqDesc {
    const double* p;
    int64_t size;
    double weight;
};
__global__ void block_sq_kernel(const SqDesc* __restrict__ d, int nd, double* __restrict__ partial) {
    const int i = blockIdx.x;
    if (i >= nd) return;
    const SqDesc q = d[i];
    double acc = 0;
    for (int64_t e = threadIdx.x; e < q.size; e += blockDim.x) acc = fma(q.p[e], q.p[e], acc);
    __shared__ double red[32];
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        acc = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
        if (threadIdx.x == 0) partial[i] = q.weight * acc;
    }
}
__global__ void sum_kernel(const double* __restrict__ v, int64_t n, double* __restrict__ out) {
    double acc = 0;
    for (int64_t e = threadIdx.x; e < n; e += blockDim.x) acc += v[e];
    __shared__ double red[32];
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        acc = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
        if (threadIdx.x == 0) *out = acc;
    }
}
}  // namespace

double frobenius_norm(const H2Dev& h, cudaStream_t st) {
    if (!h.orthonormal)
        throw std::invalid_argument("frobenius_norm: bases are not orthonormal; call orthogonalize");
    const BlockTree& bt = *h.bt;
    const BasisDev& vb = h.vbasis();
    std::vector<SqDesc> ds;
    for (size_t i = 0; i < bt.adm.size(); ++i) {
        if (h.s_off[i] < 0) continue;
        const int b = bt.adm[i], r = bt.row[size_t(b)], c = bt.col[size_t(b)];
        const int64_t sz = int64_t(h.row.rank[size_t(r)]) * vb.rank[size_t(c)];
        if (sz == 0) continue;
        ds.push_back(SqDesc{h.S.data() + h.s_off[i], sz, h.symmetric && r != c ? 2.0 : 1.0});
    }
    for (size_t i = 0; i < bt.dense.size(); ++i) {
        if (h.d_off[i] < 0) continue;
        const int b = bt.dense[i], r = bt.row[size_t(b)], c = bt.col[size_t(b)];
        const int64_t sz = h.tree().size(r) * h.tree().size(c);
        if (sz == 0) continue;
        ds.push_back(SqDesc{h.D.data() + h.d_off[i], sz, h.symmetric && r != c ? 2.0 : 1.0});
    }
    if (ds.empty()) return 0.0;
    DeviceArray<SqDesc> dd;
    dd.upload(ds, st);
    DBuf part(ds.size(), st), tot(1, st);
    block_sq_kernel<<<unsigned(ds.size()), 256, 0, st>>>(dd.data(), int(ds.size()), part.data());
    H2B_LAUNCH();
    sum_kernel<<<1, 1024, 0, st>>>(part.data(), int64_t(ds.size()), tot.data());
    H2B_LAUNCH();
    double sum = 0;
    H2B_CUDA(cudaMemcpyAsync(&sum, tot.data(), sizeof(double), cudaMemcpyDeviceToHost, st));
    H2B_CUDA(cudaStreamSynchronize(st));
    return std::sqrt(sum);
}

// ---------------------------------------------------------------------------
// to_dense (h2_matrix.hpp:128-163): the expansion is the operator applied to
// the identity, so it runs as hgemv over identity column panels (user
// ordering on both sides) and streams each panel to the host.
// ---------------------------------------------------------------------------
namespace {
__global__ void identity_panel_kernel(double* __restrict__ x, int64_t n, int64_t j0, int64_t w) {
    const int64_t total = n * w;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = e % n, j = e / n;
        x[e] = i == j0 + j ? 1.0 : 0.0;
    }
}
}  // namespace

void to_dense(const H2Dev& h, int64_t cap, double* out_host, cudaStream_t st) {
    const int64_t n = h.tree().n;
    if (n > cap) throw std::invalid_argument("to_dense: matrix size exceeds cap");
    if (h.shard_nranks > 0) throw std::invalid_argument("to_dense: this matrix holds one row-subtree shard");
    if (n == 0) return;
    const int64_t w = std::min<int64_t>(n, 256);
    DBuf x(size_t(n * w), st), y(size_t(n * w), st);
    Workspace ws;
    for (int64_t j0 = 0; j0 < n; j0 += w) {
        const int64_t wj = std::min(w, n - j0);
        const int64_t blocks = std::min<int64_t>((n * wj + 255) / 256, 148 * 16);
        identity_panel_kernel<<<unsigned(blocks), 256, 0, st>>>(x.data(), n, j0, wj);
        H2B_LAUNCH();
        hgemv(h, false, true, n, wj, x.data(), n, y.data(), n, 1.0, 0.0, st, ws);
        H2B_CUDA(cudaMemcpyAsync(out_host + j0 * n, y.data(), size_t(n * wj) * sizeof(double), cudaMemcpyDeviceToHost,
                                 st));
    }
    H2B_CUDA(cudaStreamSynchronize(st));
}

// ---------------------------------------------------------------------------
// storage / rank_profile / validate (h2_matrix.hpp:167-196, 308-404)
// ---------------------------------------------------------------------------
StorageReportDev storage_report(const H2Dev& h) {
    int64_t sz[6];
    packed_sizes(h, sz);
    StorageReportDev r;
    r.leaf_basis_reals = sz[0] + sz[2];
    r.transfer_reals = sz[1] + sz[3];
    r.coupling_reals = sz[4];
    r.dense_reals = sz[5];
    return r;
}

std::vector<int64_t> rank_profile(const H2Dev& h) {
    const ClusterTree& ct = h.tree();
    std::vector<int64_t> prof(size_t(ct.depth + 1), 0);
    for (int v = 0; v < ct.num_nodes(); ++v)
        prof[size_t(ct.level[size_t(v)])] = std::max<int64_t>(prof[size_t(ct.level[size_t(v)])], h.row.rank[size_t(v)]);
    return prof;
}

namespace {
// ||G - I||_F for each node's k x k Gram matrix G (k = ranks[v])
__global__ void gram_defect_kernel(const double* __restrict__ g, const int64_t* __restrict__ off,
                                   const int* __restrict__ k, int nn, double* __restrict__ out) {
    const int v = blockIdx.x;
    if (v >= nn) return;
    const int kk = k[v];
    double acc = 0;
    for (int e = threadIdx.x; e < kk * kk; e += blockDim.x) {
        const int i = e % kk, j = e / kk;
        const double d = g[off[v] + e] - (i == j ? 1.0 : 0.0);
        acc = fma(d, d, acc);
    }
    __shared__ double red[32];
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        acc = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
        if (threadIdx.x == 0) out[v] = sqrt(acc);
    }
}

// ||U_v^T U_v - I||_F for every node of a nested basis, U_v implicit
// (basis_tree.hpp:40-52): Gram matrices bottom-up, G_leaf = U^T U,
// G_v = sum_c E_c^T G_c E_c
std::vector<double> orthonormality_defects(const ClusterTree& ct, const BasisDev& b, cudaStream_t st) {
    const int nn = ct.num_nodes();
    std::vector<int64_t> off(static_cast<size_t>(nn));
    int64_t tot = 0, tmax = 0;
    for (int v = 0; v < nn; ++v) {
        off[size_t(v)] = tot;
        tot += int64_t(b.rank[size_t(v)]) * b.rank[size_t(v)];
    }
    DBuf g(size_t(std::max<int64_t>(tot, 1)), st);
    g.zero();
    for (int v = 0; v < nn; ++v)
        if (ct.parent[size_t(v)] >= 0)
            tmax = std::max<int64_t>(tmax, int64_t(b.rank[size_t(v)]) * b.rank[size_t(ct.parent[size_t(v)])]);
    for (int l = ct.depth; l >= 0; --l) {
        std::vector<GemmDesc> leaf, mid, up;
        std::vector<int> kids;
        for (int v : ct.levels[size_t(l)]) {
            const int k = b.rank[size_t(v)];
            if (k == 0) continue;
            if (ct.is_leaf(v)) {
                const int m = int(ct.size(v));
                const double* U = b.leaf.data() + b.leaf_off[size_t(v)];
                leaf.push_back(GemmDesc{U, U, g.data() + off[size_t(v)], k, k, m, ld1(m), ld1(m), k, 1, 0, 1.0, 0.0});
            } else {
                for (int c : {ct.child0[size_t(v)], ct.child1[size_t(v)]}) {
                    if (b.rank[size_t(c)] > 0) kids.push_back(c);
                }
            }
        }
        bgemm(leaf, st);
        if (kids.empty()) continue;
        // T_c = G_c E_c (k_c x k_v), then G_v += E_c^T T_c (children serialised per parent)
        DBuf tbuf(size_t(tmax) * kids.size(), st);
        for (size_t i = 0; i < kids.size(); ++i) {
            const int c = kids[i], v = ct.parent[size_t(c)];
            const int kc = b.rank[size_t(c)], kv = b.rank[size_t(v)];
            const double* E = b.xfer.data() + b.xfer_off[size_t(c)];
            mid.push_back(GemmDesc{g.data() + off[size_t(c)], E, tbuf.data() + size_t(tmax) * i, kc, kv, kc, kc, kc,
                                   kc, 0, 0, 1.0, 0.0});
        }
        bgemm(mid, st);
        for (int pass = 0; pass < 2; ++pass) {
            up.clear();
            for (size_t i = 0; i < kids.size(); ++i) {
                const int c = kids[i], v = ct.parent[size_t(c)];
                if ((c == ct.child0[size_t(v)]) != (pass == 0)) continue;
                const int kc = b.rank[size_t(c)], kv = b.rank[size_t(v)];
                const double* E = b.xfer.data() + b.xfer_off[size_t(c)];
                up.push_back(GemmDesc{E, tbuf.data() + size_t(tmax) * i, g.data() + off[size_t(v)], kv, kv, kc, kc,
                                      kc, kv, 1, 0, 1.0, 1.0});
            }
            bgemm(up, st);
        }
    }
    DeviceArray<int64_t> doff;
    doff.upload(off, st);
    DeviceArray<int> dk;
    dk.upload(b.rank, st);
    DBuf def(size_t(nn), st);
    gram_defect_kernel<<<unsigned(nn), 128, 0, st>>>(g.data(), doff.data(), dk.data(), nn, def.data());
    H2B_LAUNCH();
    std::vector<double> h(static_cast<size_t>(nn));
    H2B_CUDA(cudaMemcpyAsync(h.data(), def.data(), h.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
    H2B_CUDA(cudaStreamSynchronize(st));
    return h;
}
}  // namespace

ValidationReportDev validate(const H2Dev& h, int64_t ortho_cap, cudaStream_t st) {
    ValidationReportDev rep;
    auto bad = [&rep](const std::string& m) { rep.violations.push_back(m); };
    if (!h.bt || !h.bt->tree) {
        bad("missing cluster or block tree");
        return rep;
    }
    const ClusterTree& ct = h.tree();
    const BlockTree& bt = *h.bt;
    {   // permutation is a bijection
        std::vector<char> seen(size_t(ct.n), 0);
        for (int64_t i = 0; i < ct.n; ++i) {
            const int64_t p = ct.perm[size_t(i)];
            if (p < 0 || p >= ct.n || seen[size_t(p)]) {
                bad("permutation is not a bijection");
                break;
            }
            seen[size_t(p)] = 1;
        }
    }
    {   // block leaves tile the index square exactly (area accounting)
        int64_t area = 0;
        for (int b : bt.adm) area += ct.size(bt.row[size_t(b)]) * ct.size(bt.col[size_t(b)]);
        for (int b : bt.dense) area += ct.size(bt.row[size_t(b)]) * ct.size(bt.col[size_t(b)]);
        if (area != ct.n * ct.n) bad("block leaves do not tile the index square");
    }
    // basis shapes: payload slots are laid out from the ranks, so a shape
    // defect shows as a rank above the cluster size or a missing slot
    auto check_basis = [&](const BasisDev& b, const char* name) {
        if (int(b.rank.size()) != ct.num_nodes()) {
            bad(std::string(name) + ": wrong node count");
            return;
        }
        for (int v = 0; v < ct.num_nodes(); ++v) {
            if (b.rank[size_t(v)] > ct.size(v)) bad(std::string(name) + ": rank exceeds cluster size");
            if (ct.is_leaf(v)) {
                if (b.rank[size_t(v)] > 0 && b.leaf_off[size_t(v)] < 0)
                    bad(std::string(name) + ": leaf basis dimension mismatch");
            } else {
                for (int c : {ct.child0[size_t(v)], ct.child1[size_t(v)]})
                    if (int64_t(b.rank[size_t(c)]) * b.rank[size_t(v)] > 0 && b.xfer_off[size_t(c)] < 0)
                        bad(std::string(name) + ": transfer dimension mismatch");
            }
        }
    };
    check_basis(h.row, "row basis");
    if (!h.symmetric) check_basis(h.col, "col basis");
    const BasisDev& vb = h.vbasis();
    for (size_t i = 0; i < bt.adm.size(); ++i) {
        const int b = bt.adm[i];
        if (h.symmetric && !bt.canonical(b)) {
            if (h.s_off[i] >= 0) bad("coupling stored at non-canonical block of a symmetric matrix");
            continue;
        }
        const int64_t sz = int64_t(h.row.rank[size_t(bt.row[size_t(b)])]) * vb.rank[size_t(bt.col[size_t(b)])];
        if (sz > 0 && h.s_off[i] < 0)
            bad("coupling dimension mismatch at block (" + std::to_string(bt.row[size_t(b)]) + "," +
                std::to_string(bt.col[size_t(b)]) + ")");
    }
    for (size_t i = 0; i < bt.dense.size(); ++i) {
        const int b = bt.dense[i];
        if (!ct.is_leaf(bt.row[size_t(b)]) || !ct.is_leaf(bt.col[size_t(b)])) bad("dense block at non-leaf cluster pair");
        if (h.symmetric && !bt.canonical(b)) {
            if (h.d_off[i] >= 0) bad("dense block stored at non-canonical block of a symmetric matrix");
            continue;
        }
        if (h.d_off[i] < 0) bad("dense block dimension mismatch");
    }
    // orthonormality claim, at desk scale (the reference reconstructs each
    // basis explicitly; the Gram recursion measures the same defect)
    if (h.orthonormal && ct.n <= ortho_cap) {
        const std::vector<double> dr = orthonormality_defects(ct, h.row, st);
        std::vector<double> dc;
        if (!h.symmetric) dc = orthonormality_defects(ct, h.col, st);
        for (int v = 0; v < ct.num_nodes() && rep.violations.size() < 8; ++v) {
            const int ku = h.row.rank[size_t(v)];
            if (ku == 0) continue;
            if (dr[size_t(v)] > 1e-10 * std::sqrt(double(ku)))
                bad("row basis not orthonormal at node " + std::to_string(v));
            if (!h.symmetric) {
                const int kw = h.col.rank[size_t(v)];
                if (kw == 0) continue;
                if (dc[size_t(v)] > 1e-10 * std::sqrt(double(kw)))
                    bad("col basis not orthonormal at node " + std::to_string(v));
            }
        }
    }
    rep.level_max_rank = rank_profile(h);
    rep.storage = storage_report(h);
    return rep;
}

}  // namespace h2b
