// Device H^2 container: packed layout, host <-> device transfer, and the
// on-device generator of kernel-matrix H^2 content used by the benchmarks
// (Chebyshev tensor interpolation, SURVEY §8d option (ii)).
#include <algorithm>
#include <cmath>

#include "h2dev.hpp"
#include "matrix.hpp"

namespace h2b {

void BasisDev::layout(const ClusterTree& t) { layout(t, nullptr, nullptr); }

void BasisDev::layout(const ClusterTree& t, const std::vector<char>* need_leaf, const std::vector<char>* need_xfer) {
    const int nn = t.num_nodes();
    leaf_off.assign(size_t(nn), -1);
    xfer_off.assign(size_t(nn), -1);
    int64_t lo = 0, xo = 0;
    for (int v : t.leaves) {
        if (need_leaf && !(*need_leaf)[size_t(v)]) continue;
        leaf_off[size_t(v)] = lo;
        lo += t.size(v) * rank[size_t(v)];
    }
    for (int v = 0; v < nn; ++v) {
        if (t.parent[size_t(v)] < 0) continue;
        if (need_xfer && !(*need_xfer)[size_t(v)]) continue;
        xfer_off[size_t(v)] = xo;
        xo += int64_t(rank[size_t(v)]) * rank[size_t(t.parent[size_t(v)])];
    }
    leaf.resize(size_t(lo));
    xfer.resize(size_t(xo));
}

void H2Dev::layout_blocks() { layout_blocks(nullptr, nullptr); }

void H2Dev::layout_blocks(const std::vector<char>* need_s, const std::vector<char>* need_d) {
    const ClusterTree& t = tree();
    const BasisDev& vb = vbasis();
    s_off.assign(bt->adm.size(), -1);
    d_off.assign(bt->dense.size(), -1);
    int64_t so = 0, dof = 0;
    for (size_t i = 0; i < bt->adm.size(); ++i) {
        const int b = bt->adm[i];
        if (!stores(b) || (need_s && !(*need_s)[i])) continue;
        s_off[i] = so;
        so += int64_t(row.rank[size_t(bt->row[size_t(b)])]) * vb.rank[size_t(bt->col[size_t(b)])];
    }
    for (size_t i = 0; i < bt->dense.size(); ++i) {
        const int b = bt->dense[i];
        if (!stores(b) || (need_d && !(*need_d)[i])) continue;
        d_off[i] = dof;
        dof += t.size(bt->row[size_t(b)]) * t.size(bt->col[size_t(b)]);
    }
    S.resize(size_t(so));
    D.resize(size_t(dof));
}

std::unique_ptr<H2Dev> make_h2(std::shared_ptr<const BlockTree> bt, bool symmetric, const int* row_ranks,
                               const int* col_ranks) {
    auto h = std::make_unique<H2Dev>();
    h->bt = std::move(bt);
    h->symmetric = symmetric;
    const ClusterTree& t = h->tree();
    const int nn = t.num_nodes();
    auto set_ranks = [&](BasisDev& b, const int* r) {
        b.rank.assign(size_t(nn), 0);
        for (int v = 0; v < nn; ++v) {
            const int k = r ? r[v] : 0;
            if (k < 0) throw std::invalid_argument("negative rank");
            b.rank[size_t(v)] = k;
        }
        b.layout(t);
    };
    set_ranks(h->row, row_ranks);
    if (!symmetric) set_ranks(h->col, col_ranks ? col_ranks : row_ranks);
    h->layout_blocks();
    h->row.leaf.zero();
    h->row.xfer.zero();
    h->col.leaf.zero();
    h->col.xfer.zero();
    h->S.zero();
    h->D.zero();
    return h;
}

void packed_sizes(const H2Dev& h, int64_t sizes[6]) {
    sizes[0] = int64_t(h.row.leaf.size());
    sizes[1] = int64_t(h.row.xfer.size());
    sizes[2] = h.symmetric ? 0 : int64_t(h.col.leaf.size());
    sizes[3] = h.symmetric ? 0 : int64_t(h.col.xfer.size());
    sizes[4] = int64_t(h.S.size());
    sizes[5] = int64_t(h.D.size());
}

void upload_packed(H2Dev& h, const double* const parts[6]) {
    DeviceArray<double>* dst[6] = {&h.row.leaf, &h.row.xfer, &h.col.leaf, &h.col.xfer, &h.S, &h.D};
    for (int i = 0; i < 6; ++i) {
        if (h.symmetric && (i == 2 || i == 3)) continue;
        if (!parts[i] || dst[i]->size() == 0) continue;
        H2B_CUDA(cudaMemcpy(dst[i]->data(), parts[i], dst[i]->size() * sizeof(double), cudaMemcpyHostToDevice));
    }
    h.invalidate_plans();
}

void download_packed(const H2Dev& h, double* const parts[6]) {
    const DeviceArray<double>* src[6] = {&h.row.leaf, &h.row.xfer, &h.col.leaf, &h.col.xfer, &h.S, &h.D};
    for (int i = 0; i < 6; ++i) {
        if (h.symmetric && (i == 2 || i == 3)) continue;
        if (!parts[i] || src[i]->size() == 0) continue;
        H2B_CUDA(cudaMemcpy(parts[i], src[i]->data(), src[i]->size() * sizeof(double), cudaMemcpyDeviceToHost));
    }
}

// ---------------------------------------------------------------------------
// kernel-matrix generator
// ---------------------------------------------------------------------------
namespace {

struct NodeGrid {
    double lo[3], hi[3];
    int p[3];   // Chebyshev points per axis (product = rank)
};

__device__ __forceinline__ double kernel_eval(int kind, double ell, double r2) {
    if (kind == 1) return exp(-r2 / (ell * ell));   // Gaussian
    const double r = sqrt(r2);
    if (kind == 0) return exp(-r / ell);           // exponential
    const double a = 1.7320508075688772 * r / ell; // Matern nu = 3/2
    return (1.0 + a) * exp(-a);
}

__device__ __forceinline__ double cheb_node(const NodeGrid& g, int axis, int i) {
    const int p = g.p[axis];
    const double c = 0.5 * (g.lo[axis] + g.hi[axis]), h = 0.5 * (g.hi[axis] - g.lo[axis]);
    if (p == 1) return c;
    return c + h * cos(3.14159265358979323846 * (2 * i + 1) / (2.0 * p));
}

// tensor Lagrange basis function a of grid g evaluated at point x
__device__ double lagrange(const NodeGrid& g, int dim, int a, const double* x) {
    double v = 1.0;
    for (int d = 0; d < dim; ++d) {
        const int ia = a % g.p[d];
        a /= g.p[d];
        const double xa = cheb_node(g, d, ia);
        for (int j = 0; j < g.p[d]; ++j)
            if (j != ia) {
                const double xj = cheb_node(g, d, j);
                v *= (x[d] - xj) / (xa - xj);
            }
    }
    return v;
}

__device__ void grid_point(const NodeGrid& g, int dim, int a, double* x) {
    for (int d = 0; d < dim; ++d) {
        x[d] = cheb_node(g, d, a % g.p[d]);
        a /= g.p[d];
    }
}

__global__ void gen_leaf_kernel(const int* leaves, int nleaves, const int64_t* begin, const int64_t* end,
                                const int* rank, const int64_t* off, const NodeGrid* grids, const double* pts,
                                int dim, int64_t n, const int64_t* perm, double* U) {
    const int li = blockIdx.x;
    if (li >= nleaves) return;
    const int v = leaves[li];
    const int m = int(end[v] - begin[v]), k = rank[v];
    for (int idx = threadIdx.x; idx < m * k; idx += blockDim.x) {
        const int i = idx % m, a = idx / m;
        double x[3];
        const int64_t p = perm[begin[v] + i];
        for (int d = 0; d < dim; ++d) x[d] = pts[p + d * n];
        U[off[v] + idx] = lagrange(grids[v], dim, a, x);
    }
}

__global__ void gen_transfer_kernel(int nn, const int* parent, const int* rank, const int64_t* off,
                                    const NodeGrid* grids, int dim, double* E) {
    const int v = blockIdx.x;
    if (v >= nn || parent[v] < 0 || off[v] < 0) return;
    const int kc = rank[v], kp = rank[parent[v]];
    for (int idx = threadIdx.x; idx < kc * kp; idx += blockDim.x) {
        const int ac = idx % kc, ap = idx / kc;
        double x[3];
        grid_point(grids[v], dim, ac, x);
        E[off[v] + idx] = lagrange(grids[parent[v]], dim, ap, x);
    }
}

__global__ void gen_coupling_kernel(int nb, const int* rows, const int* cols, const int64_t* off, const int* rank,
                                    const NodeGrid* grids, int dim, int kind, double ell, double* S) {
    const int bi = blockIdx.x;
    if (bi >= nb) return;
    const int r = rows[bi], c = cols[bi];
    const int kr = rank[r], kc = rank[c];
    for (int idx = threadIdx.x; idx < kr * kc; idx += blockDim.x) {
        const int a = idx % kr, b = idx / kr;
        double x[3], y[3];
        grid_point(grids[r], dim, a, x);
        grid_point(grids[c], dim, b, y);
        double r2 = 0;
        for (int d = 0; d < dim; ++d) r2 += (x[d] - y[d]) * (x[d] - y[d]);
        S[off[bi] + idx] = kernel_eval(kind, ell, r2);
    }
}

__global__ void gen_dense_kernel(int nb, const int* rows, const int* cols, const int64_t* off, const int64_t* begin,
                                 const int64_t* end, const double* pts, int dim, int64_t n, const int64_t* perm,
                                 int kind, double ell, double* D) {
    const int bi = blockIdx.x;
    if (bi >= nb) return;
    const int r = rows[bi], c = cols[bi];
    const int mr = int(end[r] - begin[r]), mc = int(end[c] - begin[c]);
    for (int idx = threadIdx.x; idx < mr * mc; idx += blockDim.x) {
        const int i = idx % mr, j = idx / mr;
        const int64_t pi = perm[begin[r] + i], pj = perm[begin[c] + j];
        double r2 = 0;
        for (int d = 0; d < dim; ++d) {
            const double df = pts[pi + d * n] - pts[pj + d * n];
            r2 += df * df;
        }
        D[off[bi] + idx] = kernel_eval(kind, ell, r2);
    }
}

// per-axis point counts for rank k: all k points go to the longest axes
// first, e.g. 2D k=32 -> 8 x 4, 3D k=32 -> 4 x 4 x 2, k=64 -> 4 x 4 x 4
void axis_counts(int dim, int k, const double* ext, int* p) {
    int order[3] = {0, 1, 2};
    for (int i = 1; i < dim && i < 3; ++i)   // stable insertion sort of <= 3 axes, longest first
        for (int j = i; j > 0 && ext[order[j]] > ext[order[j - 1]]; --j) std::swap(order[j], order[j - 1]);
    for (int d = 0; d < 3; ++d) p[d] = 1;
    // factor k into dim factors as evenly as possible, biggest to longest axis
    int rem = k;
    std::vector<int> f(size_t(dim), 1);
    for (int d = dim - 1; d >= 0; --d) {
        int best = 1;
        const double target = std::pow(double(rem), 1.0 / double(d + 1));
        for (int q = 1; q <= rem; ++q)
            if (rem % q == 0 && std::abs(q - target) < std::abs(best - target)) best = q;
        f[size_t(d)] = best;
        rem /= best;
    }
    std::sort(f.begin(), f.end(), std::greater<int>());
    f[0] *= rem;
    for (int d = 0; d < dim; ++d) p[order[d]] = f[size_t(d)];
}

}  // namespace

std::unique_ptr<H2Dev> make_kernel_h2(std::shared_ptr<const BlockTree> bt, const double* coords, int kind,
                                      double ell, int rank, int shard_nranks, int shard_rank) {
    const ClusterTree& t = *bt->tree;
    const int nn = t.num_nodes(), dim = t.dim;
    std::vector<int> ranks(static_cast<size_t>(nn));
    for (int v = 0; v < nn; ++v) ranks[size_t(v)] = int(std::min<int64_t>(rank, t.size(v)));
    std::unique_ptr<H2Dev> h;
    if (shard_nranks > 0) {
        // only the payload this rank's sharded hgemv reads (see make_dist_plan):
        // owned leaves' bases, transfers of local nodes and of every partition
        // root, couplings touching a local node, dense blocks touching an owned leaf
        const DistSpec d = make_dist_spec(t, shard_nranks, shard_rank);
        auto own = [&](int v) { return d.owner[size_t(v)] == shard_rank; };
        auto local = [&](int v) { return d.owner[size_t(v)] == shard_rank || d.owner[size_t(v)] < 0; };
        std::vector<char> nl(size_t(nn), 0), nx(size_t(nn), 0), ns(bt->adm.size(), 0), nd(bt->dense.size(), 0);
        for (int v = 0; v < nn; ++v) {
            nl[size_t(v)] = own(v);
            nx[size_t(v)] = local(v) || t.level[size_t(v)] == d.lp;
        }
        for (size_t i = 0; i < bt->adm.size(); ++i) {
            const int b = bt->adm[i];
            ns[i] = local(bt->row[size_t(b)]) || local(bt->col[size_t(b)]);
        }
        for (size_t i = 0; i < bt->dense.size(); ++i) {
            const int b = bt->dense[i];
            nd[i] = own(bt->row[size_t(b)]) || own(bt->col[size_t(b)]);
        }
        h = std::make_unique<H2Dev>();
        h->bt = bt;
        h->symmetric = true;
        h->row.rank = ranks;
        h->row.layout(t, &nl, &nx);
        h->layout_blocks(&ns, &nd);
        h->shard_nranks = shard_nranks;
        h->shard_rank = shard_rank;
    } else {
        h = make_h2(bt, true, ranks.data(), nullptr);
    }
    std::vector<NodeGrid> grids(static_cast<size_t>(nn));
    for (int v = 0; v < nn; ++v) {
        NodeGrid& g = grids[size_t(v)];
        double ext[3] = {0, 0, 0}, diam = 0;
        for (int d = 0; d < 3; ++d) {
            g.lo[d] = t.lo[size_t(3 * v + d)];
            g.hi[d] = t.hi[size_t(3 * v + d)];
            ext[d] = d < dim ? g.hi[d] - g.lo[d] : 0;
            diam += ext[d] * ext[d];
        }
        diam = std::sqrt(diam);
        for (int d = 0; d < dim; ++d)
            if (ext[d] < 1e-9 * std::max(diam, 1e-300)) {   // degenerate axis: widen
                const double w = std::max(1e-3 * diam, 1e-12);
                g.lo[d] -= w;
                g.hi[d] += w;
                ext[d] = g.hi[d] - g.lo[d];
            }
        axis_counts(dim, ranks[size_t(v)], ext, g.p);
    }
    DeviceArray<NodeGrid> dgrids;
    dgrids.upload(grids);
    DeviceArray<double> dpts;
    dpts.upload(coords, size_t(t.n * dim));
    DeviceArray<int64_t> dperm, dbeg, dend, dloff, dxoff;
    DeviceArray<int> dleaves, drank, dpar;
    dperm.upload(t.perm);
    dbeg.upload(t.begin);
    dend.upload(t.end);
    std::vector<int> gl;
    for (int v : t.leaves)
        if (h->row.leaf_off[size_t(v)] >= 0) gl.push_back(v);
    dleaves.upload(gl);
    drank.upload(h->row.rank);
    dpar.upload(t.parent);
    dloff.upload(h->row.leaf_off);
    dxoff.upload(h->row.xfer_off);
    if (!gl.empty()) {
        gen_leaf_kernel<<<int(gl.size()), 256>>>(dleaves.data(), int(gl.size()), dbeg.data(), dend.data(),
                                                 drank.data(), dloff.data(), dgrids.data(), dpts.data(), dim, t.n,
                                                 dperm.data(), h->row.leaf.data());
        H2B_LAUNCH();
    }
    gen_transfer_kernel<<<nn, 256>>>(nn, dpar.data(), drank.data(), dxoff.data(), dgrids.data(), dim, h->row.xfer.data());
    H2B_LAUNCH();
    std::vector<int> sr, sc, dr, dc;
    std::vector<int64_t> so, dof;
    for (size_t i = 0; i < bt->adm.size(); ++i)
        if (h->s_off[i] >= 0) {
            sr.push_back(bt->row[size_t(bt->adm[i])]);
            sc.push_back(bt->col[size_t(bt->adm[i])]);
            so.push_back(h->s_off[i]);
        }
    for (size_t i = 0; i < bt->dense.size(); ++i)
        if (h->d_off[i] >= 0) {
            dr.push_back(bt->row[size_t(bt->dense[i])]);
            dc.push_back(bt->col[size_t(bt->dense[i])]);
            dof.push_back(h->d_off[i]);
        }
    DeviceArray<int> dsr, dsc, ddr, ddc;
    DeviceArray<int64_t> dso, ddo;
    dsr.upload(sr);
    dsc.upload(sc);
    dso.upload(so);
    ddr.upload(dr);
    ddc.upload(dc);
    ddo.upload(dof);
    if (!sr.empty()) {
        gen_coupling_kernel<<<int(sr.size()), 256>>>(int(sr.size()), dsr.data(), dsc.data(), dso.data(), drank.data(),
                                                     dgrids.data(), dim, kind, ell, h->S.data());
        H2B_LAUNCH();
    }
    if (!dr.empty()) {
        gen_dense_kernel<<<int(dr.size()), 256>>>(int(dr.size()), ddr.data(), ddc.data(), ddo.data(), dbeg.data(),
                                                  dend.data(), dpts.data(), dim, t.n, dperm.data(), kind, ell,
                                                  h->D.data());
        H2B_LAUNCH();
    }
    H2B_CUDA(cudaDeviceSynchronize());
    return h;
}

}  // namespace h2b
