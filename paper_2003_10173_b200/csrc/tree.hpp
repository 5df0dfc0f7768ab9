#pragma once
// Host-side cluster tree and block tree for the B200 H^2 path.
//
// Same partition and numbering rules as the reference (cluster_tree.hpp:122-176,
// block_tree.hpp:22-27, 77-109) so node ids, the permutation and the
// admissible / dense leaf ordinals agree bit-for-bit with it, but built
// differently: structure-of-arrays storage, per-node subtree id ranges known
// up front (the split is by count, so a subtree's node count depends only on
// its size) which lets independent subtrees be built on separate host
// threads, and an explicit-stack block-tree traversal.
#include <array>
#include <cstdint>
#include <cuda_runtime.h>

#include <memory>
#include <vector>

namespace h2b {

struct ClusterTree {
    int64_t n = 0, leaf_size = 0;
    int dim = 0, depth = 0;
    // per node (preorder ids, child 0 first)
    std::vector<int64_t> begin, end;
    std::vector<int> level, parent, child0, child1;
    std::vector<double> lo, hi;   // 3 per node
    std::vector<int64_t> perm, inv_perm;   // internal i <-> user perm[i]
    std::vector<std::vector<int>> levels;  // node ids per level, id order
    std::vector<int> leaves;               // id order

    int num_nodes() const { return int(begin.size()); }
    bool is_leaf(int v) const { return child0[size_t(v)] < 0; }
    int64_t size(int v) const { return end[size_t(v)] - begin[size_t(v)]; }
    int64_t max_leaf_size() const;
    bool is_descendant(int u, int v) const {
        return begin[size_t(u)] >= begin[size_t(v)] && end[size_t(u)] <= end[size_t(v)] && level[size_t(u)] >= level[size_t(v)];
    }
    double diameter(int v) const;
    double distance(int v, int w) const;
};

// coords: n x dim column-major (user ordering)
std::shared_ptr<ClusterTree> build_cluster_tree(const double* coords, int64_t n, int dim, int64_t leaf_size);
// the same tree built on the device (tree_dev.cu); coords on the host
std::shared_ptr<ClusterTree> build_cluster_tree_device(const double* coords, int64_t n, int dim, int64_t leaf_size,
                                                       cudaStream_t s);

enum BlockTag : int { kInterior = 0, kAdmissible = 1, kDense = 2 };

struct BlockTree {
    std::shared_ptr<const ClusterTree> tree;   // row tree == col tree
    double eta = 1.0;
    bool weak = false;
    int max_level = 0;
    std::vector<int> row, col, level, parent, tag;
    std::vector<std::array<int, 4>> children;
    std::vector<int> adm, dense;             // leaf lists (creation order)
    std::vector<int> adm_ord, dense_ord;     // per block node, -1 if not that kind

    int num_nodes() const { return int(row.size()); }
    bool canonical(int b) const { return row[size_t(b)] <= col[size_t(b)]; }
};

std::shared_ptr<BlockTree> build_block_tree(std::shared_ptr<const ClusterTree> ct, double eta, bool weak);

// ClusterTree::restore (cluster_tree.hpp:95-117): a tree from stored nodes and permutation
std::shared_ptr<ClusterTree> restore_cluster_tree(int64_t n, int dim, int64_t leaf_size, std::vector<int64_t> begin,
                                                  std::vector<int64_t> end, std::vector<int> level,
                                                  std::vector<int> parent, std::vector<int> child0,
                                                  std::vector<int> child1, std::vector<double> lo,
                                                  std::vector<double> hi, std::vector<int64_t> perm);

}  // namespace h2b
