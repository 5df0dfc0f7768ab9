// Cluster-tree construction on the B200: the same tree
// as build_cluster_tree (tree.cpp, restating cluster_tree.hpp:122-176), built
// level by level on the device.
//
// The node skeleton (ranges, levels, parents, children, preorder ids) depends
// only on the point count and the leaf size (mid = begin + size/2), so the host
// lays it out directly. What depends on the coordinates runs on the device, one
// tree level at a time for all nodes of the level at once:
//   * the bounding box of every node (segmented min/max over its range);
//   * the split axis (longest extent, first strictly larger wins) on the host;
//   * the reference's ordering of every split range: fully sorted by
//     (coordinate on the node's axis, user index). This is three stable LSD
//     radix passes over the whole permutation: by user index, by coordinate,
//     by node (ranges of leaves keep their order: their first key is their
//     position and their coordinate key is constant).
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>

#include "common.hpp"
#include "tree.hpp"

namespace h2b {

namespace {

int grid_for(int64_t n, int block) { return int((n + block - 1) / block); }

// order-preserving 64-bit key of a double (-0 and +0 compare equal, as with operator<)
__device__ __forceinline__ unsigned long long coord_key(double v) {
    if (v == 0.0) v = 0.0;
    const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(v));
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

// node id (level-local) of every position covered by a node of the level
__global__ void seg_fill_kernel(const int64_t* nb, const int64_t* ne, int nodes, int* seg) {
    for (int q = blockIdx.x; q < nodes; q += gridDim.x)
        for (int64_t i = nb[q] + threadIdx.x; i < ne[q]; i += blockDim.x) seg[i] = q;
}

// bounding box of every node of the level: one block per node
__global__ void bbox_kernel(const double* x, int64_t n, int dim, const int64_t* perm, const int64_t* nb,
                            const int64_t* ne, int nodes, double* lo, double* hi) {
    __shared__ double red[2][3][256];
    for (int q = blockIdx.x; q < nodes; q += gridDim.x) {
        double l[3] = {INFINITY, INFINITY, INFINITY}, h[3] = {-INFINITY, -INFINITY, -INFINITY};
        for (int64_t i = nb[q] + threadIdx.x; i < ne[q]; i += blockDim.x) {
            const int64_t p = perm[i];
            for (int a = 0; a < dim; ++a) {   // std::min / std::max semantics
                const double v = x[p + a * n];
                l[a] = v < l[a] ? v : l[a];
                h[a] = h[a] < v ? v : h[a];
            }
        }
        for (int a = 0; a < 3; ++a) {
            red[0][a][threadIdx.x] = l[a];
            red[1][a][threadIdx.x] = h[a];
        }
        __syncthreads();
        for (int st = blockDim.x / 2; st > 0; st >>= 1) {
            if (int(threadIdx.x) < st)
                for (int a = 0; a < 3; ++a) {
                    const double lo2 = red[0][a][threadIdx.x + st], hi2 = red[1][a][threadIdx.x + st];
                    if (lo2 < red[0][a][threadIdx.x]) red[0][a][threadIdx.x] = lo2;
                    if (red[1][a][threadIdx.x] < hi2) red[1][a][threadIdx.x] = hi2;
                }
            __syncthreads();
        }
        if (threadIdx.x == 0)
            for (int a = 0; a < 3; ++a) {
                lo[q * 3 + a] = a < dim ? red[0][a][0] : 0.0;
                hi[q * 3 + a] = a < dim ? red[1][a][0] : 0.0;
            }
        __syncthreads();
    }
}

// radix keys of the three passes for the element at original position vals[j]
__global__ void key_index_kernel(const int64_t* vals, const int* seg, const int* axis, const int64_t* perm, int64_t n,
                                 unsigned long long* key) {
    const int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (j >= n) return;
    const int64_t p = vals[j];
    const int q = seg[p];
    key[j] = (q < 0 || axis[q] < 0) ? static_cast<unsigned long long>(p) : static_cast<unsigned long long>(perm[p]);
}
__global__ void key_coord_kernel(const int64_t* vals, const int* seg, const int* axis, const int64_t* perm,
                                 const double* x, int64_t n, unsigned long long* key) {
    const int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (j >= n) return;
    const int64_t p = vals[j];
    const int q = seg[p];
    key[j] = (q < 0 || axis[q] < 0) ? 0ull : coord_key(x[perm[p] + axis[q] * n]);
}
// regroup by range: a node's elements key on its first position, a position no node of
// the level covers (inside a shallower leaf) keys on itself, so every range lands back in place
__global__ void key_range_kernel(const int64_t* vals, const int* seg, const int64_t* nb, int64_t n,
                                 unsigned long long* key) {
    const int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (j >= n) return;
    const int64_t p = vals[j];
    const int q = seg[p];
    key[j] = static_cast<unsigned long long>(q >= 0 ? nb[q] : p);
}
__global__ void apply_perm_kernel(const int64_t* vals, const int64_t* perm, int64_t n, int64_t* out) {
    const int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (j < n) out[j] = perm[vals[j]];
}
__global__ void iota_kernel(int64_t* v, int64_t n) {
    const int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (j < n) v[j] = j;
}

int bits_for(unsigned long long v) {
    int b = 1;
    while (b < 64 && (v >> b) != 0) ++b;
    return b;
}

// stable sort of (key, val) pairs on key bits [0, end_bit)
struct RadixSorter {
    DeviceArray<unsigned long long> k2;
    DeviceArray<int64_t> v2;
    DeviceArray<unsigned char> tmp;
    cudaStream_t s;
    int64_t n;
    RadixSorter(int64_t n_, cudaStream_t st) : k2(size_t(n_), st), v2(size_t(n_), st), s(st), n(n_) {}
    void sort(DeviceArray<unsigned long long>& k, DeviceArray<int64_t>& v, int end_bit) {
        cub::DoubleBuffer<unsigned long long> kb(k.data(), k2.data());
        cub::DoubleBuffer<int64_t> vb(v.data(), v2.data());
        size_t bytes = 0;
        H2B_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kb, vb, n, 0, end_bit, s));
        if (bytes > tmp.size()) tmp.resize(bytes, s);
        H2B_CUDA(cub::DeviceRadixSort::SortPairs(tmp.data(), bytes, kb, vb, n, 0, end_bit, s));
        if (kb.Current() != k.data()) std::swap(k, k2);
        if (vb.Current() != v.data()) std::swap(v, v2);
    }
};

}  // namespace

std::shared_ptr<ClusterTree> build_cluster_tree_device(const double* coords, int64_t n, int dim, int64_t leaf_size,
                                                       cudaStream_t s) {
    if (n < 1) throw std::invalid_argument("cluster tree: empty point set");
    if (dim < 1 || dim > 3) throw std::invalid_argument("PointSet: dimension must be 1, 2 or 3");
    if (leaf_size < 2) throw std::invalid_argument("cluster tree: leaf_size must be >= 2");
    if (n >= (int64_t(1) << 40)) throw std::invalid_argument("cluster tree: too many points");
    // skeleton in the host builder's preorder (tree.cpp: c0 = id + 1, c1 = c0 + #nodes(left subtree))
    auto t = std::make_shared<ClusterTree>();
    t->n = n;
    t->dim = dim;
    t->leaf_size = leaf_size;
    struct Item {
        int id;
        int64_t b, e;
        int lvl, par;
    };
    std::vector<Item> order;   // preorder
    {
        std::vector<Item> stack{{0, 0, n, 0, -1}};
        int next = 0;
        while (!stack.empty()) {
            Item it = stack.back();
            stack.pop_back();
            it.id = next++;
            order.push_back(it);
            if (it.e - it.b > leaf_size) {
                const int64_t mid = it.b + (it.e - it.b) / 2;
                stack.push_back({0, mid, it.e, it.lvl + 1, it.id});
                stack.push_back({0, it.b, mid, it.lvl + 1, it.id});
            }
        }
    }
    const size_t nn = order.size();
    t->begin.resize(nn);
    t->end.resize(nn);
    t->level.resize(nn);
    t->parent.resize(nn);
    t->child0.assign(nn, -1);
    t->child1.assign(nn, -1);
    t->lo.assign(3 * nn, 0.0);
    t->hi.assign(3 * nn, 0.0);
    for (const Item& it : order) {
        t->begin[size_t(it.id)] = it.b;
        t->end[size_t(it.id)] = it.e;
        t->level[size_t(it.id)] = it.lvl;
        t->parent[size_t(it.id)] = it.par;
        t->depth = std::max(t->depth, it.lvl);
        if (it.par >= 0) {
            if (t->child0[size_t(it.par)] < 0) t->child0[size_t(it.par)] = it.id;
            else t->child1[size_t(it.par)] = it.id;
        }
    }
    t->levels.assign(size_t(t->depth + 1), {});
    for (int v = 0; v < int(nn); ++v) {
        t->levels[size_t(t->level[size_t(v)])].push_back(v);
        if (t->is_leaf(v)) t->leaves.push_back(v);
    }

    // device passes, level by level
    DeviceArray<double> x(size_t(n) * dim, s);
    x.upload(coords, size_t(n) * dim, s);
    DeviceArray<int64_t> perm(size_t(n), s), perm2(size_t(n), s), vals(size_t(n), s);
    DeviceArray<unsigned long long> key(size_t(n), s);
    DeviceArray<int> seg(size_t(n), s);
    iota_kernel<<<grid_for(n, 256), 256, 0, s>>>(perm.data(), n);
    H2B_LAUNCH();
    RadixSorter sorter(n, s);
    const int ibits = bits_for(static_cast<unsigned long long>(n));
    for (int l = 0; l <= t->depth; ++l) {
        const std::vector<int>& lv = t->levels[size_t(l)];
        const int q = int(lv.size());
        std::vector<int64_t> nb(static_cast<size_t>(q)), ne(static_cast<size_t>(q));
        for (int i = 0; i < q; ++i) {
            nb[size_t(i)] = t->begin[size_t(lv[size_t(i)])];
            ne[size_t(i)] = t->end[size_t(lv[size_t(i)])];
        }
        DeviceArray<int64_t> dnb(size_t(q), s), dne(size_t(q), s);
        dnb.upload(nb, s);
        dne.upload(ne, s);
        DeviceArray<double> dlo(size_t(q) * 3, s), dhi(size_t(q) * 3, s);
        bbox_kernel<<<std::min(q, 148 * 8), 256, 0, s>>>(x.data(), n, dim, perm.data(), dnb.data(), dne.data(), q,
                                                         dlo.data(), dhi.data());
        H2B_LAUNCH();
        const std::vector<double> lo = dlo.download(s), hi = dhi.download(s);
        std::vector<int> axis(static_cast<size_t>(q), -1);
        bool split = false;
        for (int i = 0; i < q; ++i) {
            const int v = lv[size_t(i)];
            for (int a = 0; a < 3; ++a) {
                t->lo[size_t(3 * v + a)] = lo[size_t(3 * i + a)];
                t->hi[size_t(3 * v + a)] = hi[size_t(3 * i + a)];
            }
            if (t->is_leaf(v)) continue;
            int ax = 0;   // longest axis, first strictly larger extent wins (point_set.hpp:96-102)
            for (int a = 1; a < dim; ++a)
                if (hi[size_t(3 * i + a)] - lo[size_t(3 * i + a)] > hi[size_t(3 * i + ax)] - lo[size_t(3 * i + ax)]) ax = a;
            axis[size_t(i)] = ax;
            split = true;
        }
        if (!split) continue;
        DeviceArray<int> dax(size_t(q), s);
        dax.upload(axis, s);
        H2B_CUDA(cudaMemsetAsync(seg.data(), 0xff, sizeof(int) * size_t(n), s));   // -1: no node of this level
        seg_fill_kernel<<<std::min(q, 148 * 8), 256, 0, s>>>(dnb.data(), dne.data(), q, seg.data());
        H2B_LAUNCH();
        iota_kernel<<<grid_for(n, 256), 256, 0, s>>>(vals.data(), n);
        H2B_LAUNCH();
        key_index_kernel<<<grid_for(n, 256), 256, 0, s>>>(vals.data(), seg.data(), dax.data(), perm.data(), n, key.data());
        H2B_LAUNCH();
        sorter.sort(key, vals, ibits);
        key_coord_kernel<<<grid_for(n, 256), 256, 0, s>>>(vals.data(), seg.data(), dax.data(), perm.data(), x.data(), n,
                                                          key.data());
        H2B_LAUNCH();
        sorter.sort(key, vals, 64);
        key_range_kernel<<<grid_for(n, 256), 256, 0, s>>>(vals.data(), seg.data(), dnb.data(), n, key.data());
        H2B_LAUNCH();
        sorter.sort(key, vals, ibits);
        apply_perm_kernel<<<grid_for(n, 256), 256, 0, s>>>(vals.data(), perm.data(), n, perm2.data());
        H2B_LAUNCH();
        std::swap(perm, perm2);
    }
    t->perm = perm.download(s);
    t->inv_perm.resize(size_t(n));
    for (int64_t i = 0; i < n; ++i) t->inv_perm[size_t(t->perm[size_t(i)])] = i;
    return t;
}

}  // namespace h2b
