#pragma once
// ============================================================================
// ORACLE — TEST INFRASTRUCTURE ONLY (parity checker + CPU baseline).
// A CPU restatement of the reference H^2 library (/root/reference/proj/include/h2)
// for the hot path of SURVEY §8: trees, the H^2 value type and hgemv,
// orthogonalize / recompress / low-rank updates, the black-box operator
// contract, and HARA (peel_construct). Every function cites the reference
// file:line it restates. The reference itself cannot be compiled here (Eigen3
// and doctest are absent), so parity is pinned by restating the
// reference's own test suites against this file (tests/cpp/, tests/test_oracle*.py).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use it.
// ============================================================================
#include <array>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <limits>
#include <map>
#include <memory>
#include <random>
#include <string>

#include "la.hpp"

namespace h2 {
inline namespace oracle {

// ---- types.hpp:19-27 --------------------------------------------------------
enum class Ordering { user, internal };
struct VectorBlock {
    Matrix data;
    Ordering ordering = Ordering::user;
};

// ---- point_set.hpp:18-103 ----------------------------------------------------
class PointSet {
public:
    PointSet() = default;
    explicit PointSet(Matrix coords) : c_(std::move(coords)) {
        if (c_.rows() < 1) throw std::invalid_argument("PointSet: need at least one point");
        if (c_.cols() < 1 || c_.cols() > 3) throw std::invalid_argument("PointSet: dimension must be 1, 2 or 3");
    }
    Index size() const { return c_.rows(); }
    int dim() const { return int(c_.cols()); }
    double coord(Index i, int a) const { return c_(i, a); }
    const Matrix& coords() const { return c_; }

private:
    Matrix c_;
};

struct BBox {
    std::array<double, 3> lo{{0, 0, 0}}, hi{{0, 0, 0}};
    int dim = 0;
    double extent(int a) const { return hi[size_t(a)] - lo[size_t(a)]; }
    // point_set.hpp:72-76 / 79-86 as the reference's Release build evaluates
    // them (g++ 13 -O3 -march=native, proj/CMakeLists.txt:3-20, x86-64): the
    // d<=3 loop is vectorised two lanes wide, so the first two squares are
    // rounded and summed without contraction and a third is fused,
    // fma(x2, x2, x0^2 + x1^2). Pinned by compiling the reference's own
    // headers (oracle/_ref, tests/test_ref_parity.py); exact admissibility
    // ties on grids depend on it (cfg4: 5,690,728 admissible leaves).
    static double rsq(double x) {
        double p = x * x;
        asm("" : "+m"(p));   // keep the product rounded (no contraction into the add)
        return p;
    }
    static double release_sq_sum(const double* x, int d) {
        if (d == 1) return rsq(x[0]);
        double s = rsq(x[0]) + rsq(x[1]);
        if (d == 3) s = std::fma(x[2], x[2], s);
        return s;
    }
    double diameter() const {
        double e[3] = {0, 0, 0};
        for (int a = 0; a < dim; ++a) e[a] = extent(a);
        return std::sqrt(release_sq_sum(e, dim));
    }
    double distance(const BBox& o) const {
        double g[3] = {0, 0, 0};
        for (int a = 0; a < dim; ++a)
            g[a] = std::max({0.0, o.lo[size_t(a)] - hi[size_t(a)], lo[size_t(a)] - o.hi[size_t(a)]});
        return std::sqrt(release_sq_sum(g, dim));
    }
    int longest_axis() const {   // point_set.hpp:96-102 (strictly larger wins)
        int best = 0;
        for (int a = 1; a < dim; ++a)
            if (extent(a) > extent(best)) best = a;
        return best;
    }
};

// ---- cluster_tree.hpp:18-188 -------------------------------------------------
struct ClusterNode {
    Index begin = 0, end = 0;
    int level = 0, parent = -1;
    int child[2] = {-1, -1};
    BBox box;
    Index size() const { return end - begin; }
    bool is_leaf() const { return child[0] < 0; }
};

class ClusterTree {
public:
    ClusterTree(const PointSet& pts, Index leaf_size) {   // cluster_tree.hpp:31-47
        if (pts.size() < 1) throw std::invalid_argument("cluster tree: empty point set");
        if (leaf_size < 2) throw std::invalid_argument("cluster tree: leaf_size must be >= 2");
        n_ = pts.size();
        dim_ = pts.dim();
        leaf_ = leaf_size;
        perm_.resize(size_t(n_));
        std::iota(perm_.begin(), perm_.end(), Index(0));
        split(pts, 0, n_, 0, -1);
        finish();
    }
    Index n() const { return n_; }
    int dim() const { return dim_; }
    Index leaf_size() const { return leaf_; }
    int depth() const { return depth_; }
    int num_nodes() const { return int(nodes_.size()); }
    int root() const { return 0; }
    const ClusterNode& node(int v) const { return nodes_[size_t(v)]; }
    const std::vector<int>& leaves() const { return leaves_; }
    const std::vector<int>& level_nodes(int l) const { return levels_[size_t(l)]; }
    Index max_leaf_size() const {
        Index m = 0;
        for (int v : leaves_) m = std::max(m, node(v).size());
        return m;
    }
    const std::vector<Index>& perm() const { return perm_; }
    const std::vector<Index>& inv_perm() const { return inv_; }
    bool is_descendant(int u, int v) const {   // cluster_tree.hpp:59-63
        return node(u).begin >= node(v).begin && node(u).end <= node(v).end && node(u).level >= node(v).level;
    }
    Matrix gather_rows(const Matrix& xu, int v) const {   // cluster_tree.hpp:75-80
        const ClusterNode& t = node(v);
        Matrix out(t.size(), xu.cols());
        for (Index j = 0; j < xu.cols(); ++j)
            for (Index i = 0; i < t.size(); ++i) out(i, j) = xu(perm_[size_t(t.begin + i)], j);
        return out;
    }
    Matrix to_internal(const Matrix& xu) const {   // cluster_tree.hpp:82-86
        Matrix out(xu.rows(), xu.cols());
        for (Index j = 0; j < xu.cols(); ++j)
            for (Index i = 0; i < n_; ++i) out(i, j) = xu(perm_[size_t(i)], j);
        return out;
    }
    Matrix to_user(const Matrix& xi) const {   // cluster_tree.hpp:88-92
        Matrix out(xi.rows(), xi.cols());
        for (Index j = 0; j < xi.cols(); ++j)
            for (Index i = 0; i < n_; ++i) out(perm_[size_t(i)], j) = xi(i, j);
        return out;
    }

private:
    // cluster_tree.hpp:122-160: median-by-count split on the longest axis; ties
    // to the lower user index; both halves sorted with the same comparator
    int split(const PointSet& pts, Index b, Index e, int level, int parent) {
        const int id = int(nodes_.size());
        nodes_.emplace_back();
        nodes_.back().begin = b;
        nodes_.back().end = e;
        nodes_.back().level = level;
        nodes_.back().parent = parent;
        nodes_.back().box = box_of(pts, b, e);
        depth_ = std::max(depth_, level);
        if (e - b > leaf_) {
            const int ax = nodes_[size_t(id)].box.longest_axis();
            const Index mid = b + (e - b) / 2;
            auto less = [&](Index x, Index y) {
                const double cx = pts.coord(x, ax), cy = pts.coord(y, ax);
                return cx < cy || (cx == cy && x < y);
            };
            auto first = perm_.begin() + b, nth = perm_.begin() + mid, last = perm_.begin() + e;
            std::nth_element(first, nth, last, less);
            std::sort(first, nth, less);
            std::sort(nth, last, less);
            const int c0 = split(pts, b, mid, level + 1, id);
            const int c1 = split(pts, mid, e, level + 1, id);
            nodes_[size_t(id)].child[0] = c0;
            nodes_[size_t(id)].child[1] = c1;
        }
        return id;
    }
    BBox box_of(const PointSet& pts, Index b, Index e) const {   // cluster_tree.hpp:162-176
        BBox bb;
        bb.dim = pts.dim();
        for (int a = 0; a < bb.dim; ++a) {
            bb.lo[size_t(a)] = std::numeric_limits<double>::infinity();
            bb.hi[size_t(a)] = -std::numeric_limits<double>::infinity();
        }
        for (Index i = b; i < e; ++i)
            for (int a = 0; a < bb.dim; ++a) {
                const double x = pts.coord(perm_[size_t(i)], a);
                bb.lo[size_t(a)] = std::min(bb.lo[size_t(a)], x);
                bb.hi[size_t(a)] = std::max(bb.hi[size_t(a)], x);
            }
        return bb;
    }
    void finish() {
        inv_.resize(size_t(n_));
        for (Index i = 0; i < n_; ++i) inv_[size_t(perm_[size_t(i)])] = i;
        levels_.assign(size_t(depth_ + 1), {});
        for (int v = 0; v < num_nodes(); ++v) {
            levels_[size_t(node(v).level)].push_back(v);
            if (node(v).is_leaf()) leaves_.push_back(v);
        }
    }
    std::vector<ClusterNode> nodes_;
    std::vector<Index> perm_, inv_;
    std::vector<int> leaves_;
    std::vector<std::vector<int>> levels_;
    Index n_ = 0, leaf_ = 0;
    int dim_ = 0, depth_ = 0;
};

inline std::shared_ptr<const ClusterTree> build_cluster_tree(const PointSet& p, Index leaf) {
    return std::make_shared<const ClusterTree>(p, leaf);
}

// ---- block_tree.hpp:18-124 ---------------------------------------------------
enum class Admissibility { strong, weak };

inline bool is_admissible(const ClusterNode& t, const ClusterNode& s, double eta,
                          Admissibility mode = Admissibility::strong) {   // block_tree.hpp:22-27
    if (mode == Admissibility::weak) return t.begin != s.begin || t.end != s.end;
    return std::max(t.box.diameter(), s.box.diameter()) <= eta * t.box.distance(s.box);
}

struct BlockNode {
    enum class Tag { interior, admissible, dense };
    int row = -1, col = -1, level = 0, parent = -1;
    int child[4] = {-1, -1, -1, -1};
    Tag tag = Tag::interior;
    bool is_leaf() const { return tag != Tag::interior; }
};

class BlockTree {
public:
    BlockTree(std::shared_ptr<const ClusterTree> r, std::shared_ptr<const ClusterTree> c, double eta,
              Admissibility mode)
        : rows_(std::move(r)), cols_(std::move(c)), eta_(eta), mode_(mode) {
        if (rows_->n() != cols_->n()) throw std::invalid_argument("block tree: row/column trees have different sizes");
        subdivide(rows_->root(), cols_->root(), 0, -1);
    }
    const ClusterTree& row_tree() const { return *rows_; }
    const ClusterTree& col_tree() const { return *cols_; }
    std::shared_ptr<const ClusterTree> row_tree_ptr() const { return rows_; }
    double eta() const { return eta_; }
    Admissibility mode() const { return mode_; }
    Index n() const { return rows_->n(); }
    int num_nodes() const { return int(nodes_.size()); }
    const BlockNode& node(int b) const { return nodes_[size_t(b)]; }
    const std::vector<int>& admissible_leaves() const { return adm_; }
    const std::vector<int>& dense_leaves() const { return dense_; }
    int adm_ordinal(int b) const { return adm_ord_[size_t(b)]; }
    int dense_ordinal(int b) const { return dense_ord_[size_t(b)]; }
    bool canonical(int b) const { return node(b).row <= node(b).col; }   // block_tree.hpp:72
    int max_level() const { return max_level_; }

private:
    // block_tree.hpp:77-109: admissible first, then dense if both leaves, else
    // split the non-leaf side(s); children in row-major (t-child, s-child) order
    int subdivide(int t, int s, int level, int parent) {
        const int id = int(nodes_.size());
        nodes_.emplace_back();
        adm_ord_.push_back(-1);
        dense_ord_.push_back(-1);
        BlockNode& bn = nodes_.back();
        bn.row = t;
        bn.col = s;
        bn.level = level;
        bn.parent = parent;
        max_level_ = std::max(max_level_, level);
        const ClusterNode& tn = rows_->node(t);
        const ClusterNode& sn = cols_->node(s);
        if (is_admissible(tn, sn, eta_, mode_)) {
            nodes_[size_t(id)].tag = BlockNode::Tag::admissible;
            adm_ord_[size_t(id)] = int(adm_.size());
            adm_.push_back(id);
        } else if (tn.is_leaf() && sn.is_leaf()) {
            nodes_[size_t(id)].tag = BlockNode::Tag::dense;
            dense_ord_[size_t(id)] = int(dense_.size());
            dense_.push_back(id);
        } else {
            int ts[2] = {t, -1}, ss[2] = {s, -1};
            int nt = 1, ns = 1;
            if (!tn.is_leaf()) { ts[0] = tn.child[0]; ts[1] = tn.child[1]; nt = 2; }
            if (!sn.is_leaf()) { ss[0] = sn.child[0]; ss[1] = sn.child[1]; ns = 2; }
            int k = 0;
            for (int i = 0; i < nt; ++i)
                for (int j = 0; j < ns; ++j) {
                    const int c = subdivide(ts[i], ss[j], level + 1, id);
                    nodes_[size_t(id)].child[k++] = c;
                }
        }
        return id;
    }
    std::shared_ptr<const ClusterTree> rows_, cols_;
    std::vector<BlockNode> nodes_;
    std::vector<int> adm_, dense_, adm_ord_, dense_ord_;
    double eta_;
    Admissibility mode_;
    int max_level_ = 0;
};

inline std::shared_ptr<const BlockTree> build_block_tree(std::shared_ptr<const ClusterTree> r,
                                                         std::shared_ptr<const ClusterTree> c, double eta,
                                                         Admissibility mode) {
    return std::make_shared<const BlockTree>(std::move(r), std::move(c), eta, mode);
}

// ---- basis_tree.hpp:16-66 ----------------------------------------------------
class BasisTree {
public:
    BasisTree() = default;
    explicit BasisTree(const ClusterTree& ct)
        : rank_(size_t(ct.num_nodes()), 0), leaf_(size_t(ct.num_nodes())), transfer_(size_t(ct.num_nodes())) {
        for (int v = 0; v < ct.num_nodes(); ++v)
            if (ct.node(v).is_leaf()) leaf_[size_t(v)] = Matrix(ct.node(v).size(), 0);
    }
    Index rank(int v) const { return rank_[size_t(v)]; }
    void set_rank(int v, Index k) { rank_[size_t(v)] = k; }
    const Matrix& leaf_basis(int v) const { return leaf_[size_t(v)]; }
    Matrix& leaf_basis(int v) { return leaf_[size_t(v)]; }
    const Matrix& transfer(int v) const { return transfer_[size_t(v)]; }
    Matrix& transfer(int v) { return transfer_[size_t(v)]; }
    int num_nodes() const { return int(rank_.size()); }
    bool empty() const { return rank_.empty(); }
    Matrix reconstruct(const ClusterTree& ct, int v) const {   // basis_tree.hpp:42-53
        const ClusterNode& nd = ct.node(v);
        if (nd.is_leaf()) return leaf_[size_t(v)];
        Matrix out(nd.size(), rank_[size_t(v)]);
        Index row = 0;
        for (int c : nd.child) {
            Matrix uc = reconstruct(ct, c) * transfer_[size_t(c)];
            out.set_block(row, 0, uc);
            row += uc.rows();
        }
        return out;
    }

private:
    std::vector<Index> rank_;
    std::vector<Matrix> leaf_, transfer_;
};

// ---- h2_matrix.hpp:25-404 ----------------------------------------------------
struct StorageReport {
    Index dense_reals = 0, leaf_basis_reals = 0, transfer_reals = 0, coupling_reals = 0;
    Index total() const { return dense_reals + leaf_basis_reals + transfer_reals + coupling_reals; }
};
struct ValidationReport {
    std::vector<std::string> violations;
    std::vector<Index> level_max_rank;
    StorageReport storage;
    bool ok() const { return violations.empty(); }
};

class H2Matrix {
public:
    std::shared_ptr<const ClusterTree> tree;
    std::shared_ptr<const BlockTree> blocks;
    BasisTree row_basis, col_basis;
    std::vector<Matrix> coupling, dense;
    bool symmetric = false, orthonormal = false;

    static H2Matrix zero(std::shared_ptr<const BlockTree> bt, bool sym) {   // h2_matrix.hpp:53-75
        H2Matrix h;
        h.tree = bt->row_tree_ptr();
        h.blocks = std::move(bt);
        h.symmetric = sym;
        h.row_basis = BasisTree(*h.tree);
        if (!sym) h.col_basis = BasisTree(*h.tree);
        h.coupling.resize(h.blocks->admissible_leaves().size());
        h.dense.resize(h.blocks->dense_leaves().size());
        for (size_t i = 0; i < h.dense.size(); ++i) {
            const int b = h.blocks->dense_leaves()[i];
            if (!h.stores(b)) continue;
            const BlockNode& bn = h.blocks->node(b);
            h.dense[i] = Matrix(h.tree->node(bn.row).size(), h.tree->node(bn.col).size());
        }
        h.orthonormal = true;
        return h;
    }
    static H2Matrix diagonal(std::shared_ptr<const BlockTree> bt, const Vector& d) {   // :78-88
        H2Matrix h = zero(std::move(bt), true);
        for (int b : h.blocks->dense_leaves()) {
            const BlockNode& bn = h.blocks->node(b);
            if (bn.row != bn.col) continue;
            const ClusterNode& t = h.tree->node(bn.row);
            Matrix& blk = h.dense[size_t(h.blocks->dense_ordinal(b))];
            for (Index i = 0; i < t.size(); ++i) blk(i, i) = d[h.tree->perm()[size_t(t.begin + i)]];
        }
        return h;
    }
    static H2Matrix scaled_identity(std::shared_ptr<const BlockTree> bt, double v) {
        const Index m = bt->n();
        return diagonal(std::move(bt), Matrix::Constant(m, 1, v));
    }

    Index n() const { return tree ? tree->n() : 0; }
    const BasisTree& vbasis() const { return symmetric ? row_basis : col_basis; }
    BasisTree& vbasis() { return symmetric ? row_basis : col_basis; }
    const Matrix& coupling_of(int b) const { return coupling[size_t(blocks->adm_ordinal(b))]; }
    const Matrix& dense_of(int b) const { return dense[size_t(blocks->dense_ordinal(b))]; }
    bool stores(int b) const { return !symmetric || blocks->canonical(b); }   // :103

    Matrix matvec_internal(const Matrix& x) const { return apply_internal(x, false); }
    Matrix matvec_transpose_internal(const Matrix& x) const { return apply_internal(x, true); }
    Matrix matvec(const Matrix& xu) const {   // :112-115
        check_dims(xu);
        return tree->to_user(matvec_internal(tree->to_internal(xu)));
    }
    Matrix matvec_transpose(const Matrix& xu) const {
        check_dims(xu);
        return tree->to_user(matvec_transpose_internal(tree->to_internal(xu)));
    }
    VectorBlock matvec(const VectorBlock& x) const {
        if (x.ordering == Ordering::user) return {matvec(x.data), Ordering::user};
        return {matvec_internal(x.data), Ordering::internal};
    }

    Matrix to_dense(Index cap = 8192) const {   // :128-163
        if (n() > cap) throw std::invalid_argument("to_dense: matrix size exceeds cap");
        Matrix a(n(), n());
        std::vector<Matrix> ub(size_t(tree->num_nodes())), vbig;
        for (int v = 0; v < tree->num_nodes(); ++v) ub[size_t(v)] = row_basis.reconstruct(*tree, v);
        if (!symmetric) {
            vbig.resize(size_t(tree->num_nodes()));
            for (int v = 0; v < tree->num_nodes(); ++v) vbig[size_t(v)] = col_basis.reconstruct(*tree, v);
        }
        const auto& vb = symmetric ? ub : vbig;
        for (int b : blocks->admissible_leaves()) {
            if (!stores(b)) continue;
            const BlockNode& bn = blocks->node(b);
            const ClusterNode& t = tree->node(bn.row);
            const ClusterNode& s = tree->node(bn.col);
            Matrix blk = gemm(ub[size_t(bn.row)] * coupling_of(b), false, vb[size_t(bn.col)], true);
            a.add_block(t.begin, s.begin, blk);
            if (symmetric && bn.row != bn.col) a.add_block(s.begin, t.begin, blk.transpose());
        }
        for (int b : blocks->dense_leaves()) {
            if (!stores(b)) continue;
            const BlockNode& bn = blocks->node(b);
            const ClusterNode& t = tree->node(bn.row);
            const ClusterNode& s = tree->node(bn.col);
            a.add_block(t.begin, s.begin, dense_of(b));
            if (symmetric && bn.row != bn.col) a.add_block(s.begin, t.begin, dense_of(b).transpose());
        }
        Matrix out(n(), n());
        const auto& p = tree->perm();
        for (Index j = 0; j < n(); ++j)
            for (Index i = 0; i < n(); ++i) out(p[size_t(i)], p[size_t(j)]) = a(i, j);
        return out;
    }

    StorageReport storage() const {   // :167-188
        StorageReport r;
        for (const auto& m : dense) r.dense_reals += m.size();
        for (const auto& m : coupling) r.coupling_reals += m.size();
        auto basis = [&](const BasisTree& bt) {
            for (int v = 0; v < tree->num_nodes(); ++v) {
                const ClusterNode& nd = tree->node(v);
                if (nd.is_leaf()) r.leaf_basis_reals += bt.leaf_basis(v).size();
                else r.transfer_reals += bt.transfer(nd.child[0]).size() + bt.transfer(nd.child[1]).size();
            }
        };
        basis(row_basis);
        if (!symmetric) basis(col_basis);
        return r;
    }
    std::vector<Index> rank_profile() const {   // :190-195
        std::vector<Index> p(size_t(tree->depth() + 1), 0);
        for (int v = 0; v < tree->num_nodes(); ++v)
            p[size_t(tree->node(v).level)] = std::max(p[size_t(tree->node(v).level)], row_basis.rank(v));
        return p;
    }
    ValidationReport validate(Index ortho_cap = 4096) const;

    H2Matrix desymmetrized() const {   // :200-216
        if (!symmetric) return *this;
        H2Matrix g = *this;
        g.symmetric = false;
        g.col_basis = row_basis;
        for (int b : blocks->admissible_leaves()) {
            if (blocks->canonical(b)) continue;
            g.coupling[size_t(blocks->adm_ordinal(b))] = coupling[size_t(blocks->adm_ordinal(find_mirror(b)))].transpose();
        }
        for (int b : blocks->dense_leaves()) {
            if (blocks->canonical(b)) continue;
            g.dense[size_t(blocks->dense_ordinal(b))] = dense[size_t(blocks->dense_ordinal(find_mirror(b)))].transpose();
        }
        return g;
    }
    int find_mirror(int b) const {   // :220-239
        const BlockNode& bn = blocks->node(b);
        if (bn.row == bn.col) return b;
        if (mirror_.empty()) {
            std::map<std::pair<int, int>, int> where;
            for (int x = 0; x < blocks->num_nodes(); ++x) where[{blocks->node(x).row, blocks->node(x).col}] = x;
            mirror_.resize(size_t(blocks->num_nodes()));
            for (int x = 0; x < blocks->num_nodes(); ++x) {
                auto it = where.find({blocks->node(x).col, blocks->node(x).row});
                mirror_[size_t(x)] = it == where.end() ? -1 : it->second;
            }
        }
        return mirror_[size_t(b)];
    }

private:
    mutable std::vector<int> mirror_;
    void check_dims(const Matrix& x) const {   // :241-244
        if (x.rows() != n()) throw std::invalid_argument("matvec: dimension mismatch");
        if (x.cols() < 1) throw std::invalid_argument("matvec: need at least one column");
    }
    // h2_matrix.hpp:246-305, the four-stage hgemv
    Matrix apply_internal(const Matrix& x, bool transpose) const {
        const ClusterTree& ct = *tree;
        const Index b = x.cols();
        const BasisTree& up = transpose && !symmetric ? row_basis : vbasis();
        const BasisTree& down = transpose && !symmetric ? col_basis : row_basis;
        std::vector<Matrix> xh(size_t(ct.num_nodes())), yh(size_t(ct.num_nodes()));
        for (int l = ct.depth(); l >= 0; --l)   // stage 1 :253-261
            for (int v : ct.level_nodes(l)) {
                const ClusterNode& nd = ct.node(v);
                if (nd.is_leaf()) {
                    xh[size_t(v)] = Matrix(up.rank(v), b);
                    gemm_acc(up.leaf_basis(v), true, x.data() + nd.begin, x.rows(), b, xh[size_t(v)].data(), up.rank(v));
                } else {
                    xh[size_t(v)] = gemm(up.transfer(nd.child[0]), true, xh[size_t(nd.child[0])], false) +
                                    gemm(up.transfer(nd.child[1]), true, xh[size_t(nd.child[1])], false);
                }
            }
        for (int v = 0; v < ct.num_nodes(); ++v) yh[size_t(v)] = Matrix(down.rank(v), b);
        for (int blk : blocks->admissible_leaves()) {   // stage 2 :264-274
            if (!stores(blk)) continue;
            const BlockNode& bn = blocks->node(blk);
            const Matrix& s = coupling_of(blk);
            if (!transpose || symmetric) {
                Matrix& yr = yh[size_t(bn.row)];
                gemm_acc(s, false, xh[size_t(bn.col)].data(), s.cols(), b, yr.data(), yr.rows());
                if (symmetric && bn.row != bn.col) {
                    Matrix& yc = yh[size_t(bn.col)];
                    gemm_acc(s, true, xh[size_t(bn.row)].data(), s.rows(), b, yc.data(), yc.rows());
                }
            } else {
                Matrix& yc = yh[size_t(bn.col)];
                gemm_acc(s, true, xh[size_t(bn.row)].data(), s.rows(), b, yc.data(), yc.rows());
            }
        }
        Matrix y(x.rows(), b);
        for (int l = 0; l <= ct.depth(); ++l)   // stage 3 :277-286
            for (int v : ct.level_nodes(l)) {
                const ClusterNode& nd = ct.node(v);
                if (nd.is_leaf()) {
                    gemm_acc(down.leaf_basis(v), false, yh[size_t(v)].data(), down.rank(v), b, y.data() + nd.begin, y.rows());
                } else {
                    for (int c : nd.child) {
                        Matrix& yc = yh[size_t(c)];
                        gemm_acc(down.transfer(c), false, yh[size_t(v)].data(), down.rank(v), b, yc.data(), yc.rows());
                    }
                }
            }
        for (int blk : blocks->dense_leaves()) {   // stage 4 :288-303
            if (!stores(blk)) continue;
            const BlockNode& bn = blocks->node(blk);
            const ClusterNode& t = ct.node(bn.row);
            const ClusterNode& s = ct.node(bn.col);
            const Matrix& d = dense_of(blk);
            if (!transpose || symmetric) {
                gemm_acc(d, false, x.data() + s.begin, x.rows(), b, y.data() + t.begin, y.rows());
                if (symmetric && bn.row != bn.col)
                    gemm_acc(d, true, x.data() + t.begin, x.rows(), b, y.data() + s.begin, y.rows());
            } else {
                gemm_acc(d, true, x.data() + t.begin, x.rows(), b, y.data() + s.begin, y.rows());
            }
        }
        return y;
    }
};

inline ValidationReport H2Matrix::validate(Index ortho_cap) const {   // h2_matrix.hpp:308-404
    ValidationReport rep;
    auto bad = [&rep](const std::string& m) { rep.violations.push_back(m); };
    if (!tree || !blocks) {
        bad("missing cluster or block tree");
        return rep;
    }
    const ClusterTree& ct = *tree;
    {
        std::vector<char> seen(size_t(ct.n()), 0);
        for (Index i = 0; i < ct.n(); ++i) {
            const Index p = ct.perm()[size_t(i)];
            if (p < 0 || p >= ct.n() || seen[size_t(p)]) { bad("permutation is not a bijection"); break; }
            seen[size_t(p)] = 1;
        }
    }
    {
        Index area = 0;
        for (int b : blocks->admissible_leaves()) area += ct.node(blocks->node(b).row).size() * ct.node(blocks->node(b).col).size();
        for (int b : blocks->dense_leaves()) area += ct.node(blocks->node(b).row).size() * ct.node(blocks->node(b).col).size();
        if (area != ct.n() * ct.n()) bad("block leaves do not tile the index square");
    }
    auto check_basis = [&](const BasisTree& bt, const std::string& name) {
        if (bt.num_nodes() != ct.num_nodes()) { bad(name + ": wrong node count"); return; }
        for (int v = 0; v < ct.num_nodes(); ++v) {
            const ClusterNode& nd = ct.node(v);
            if (bt.rank(v) > nd.size()) bad(name + ": rank exceeds cluster size");
            if (nd.is_leaf()) {
                if (bt.leaf_basis(v).rows() != nd.size() || bt.leaf_basis(v).cols() != bt.rank(v))
                    bad(name + ": leaf basis dimension mismatch");
            } else {
                for (int c : nd.child)
                    if (bt.transfer(c).rows() != bt.rank(c) || bt.transfer(c).cols() != bt.rank(v))
                        bad(name + ": transfer dimension mismatch");
            }
        }
    };
    check_basis(row_basis, "row basis");
    if (!symmetric) check_basis(col_basis, "col basis");
    const BasisTree& vb = vbasis();
    for (int b : blocks->admissible_leaves()) {
        const BlockNode& bn = blocks->node(b);
        const Matrix& s = coupling[size_t(blocks->adm_ordinal(b))];
        if (symmetric && !blocks->canonical(b)) {
            if (s.size() != 0) bad("coupling stored at non-canonical block of a symmetric matrix");
            continue;
        }
        if (s.rows() != row_basis.rank(bn.row) || s.cols() != vb.rank(bn.col))
            bad("coupling dimension mismatch at block (" + std::to_string(bn.row) + "," + std::to_string(bn.col) + ")");
    }
    for (int b : blocks->dense_leaves()) {
        const BlockNode& bn = blocks->node(b);
        if (!ct.node(bn.row).is_leaf() || !ct.node(bn.col).is_leaf()) bad("dense block at non-leaf cluster pair");
        const Matrix& d = dense[size_t(blocks->dense_ordinal(b))];
        if (symmetric && !blocks->canonical(b)) {
            if (d.size() != 0) bad("dense block stored at non-canonical block of a symmetric matrix");
            continue;
        }
        if (d.rows() != ct.node(bn.row).size() || d.cols() != ct.node(bn.col).size()) bad("dense block dimension mismatch");
    }
    if (orthonormal && n() <= ortho_cap) {
        for (int v = 0; v < ct.num_nodes() && rep.violations.size() < 8; ++v) {
            for (int side = 0; side < (symmetric ? 1 : 2); ++side) {
                Matrix u = (side ? col_basis : row_basis).reconstruct(ct, v);
                if (u.cols() == 0) continue;
                const double err = (gemm(u, true, u, false) - Matrix::Identity(u.cols(), u.cols())).norm();
                if (err > 1e-10 * std::sqrt(double(u.cols())))
                    bad(std::string(side ? "col" : "row") + " basis not orthonormal at node " + std::to_string(v));
            }
        }
    }
    rep.level_max_rank = rank_profile();
    rep.storage = storage();
    return rep;
}

// ---- algebra.hpp -------------------------------------------------------------
struct LowRankFactor {
    Matrix X, Y;
    Index rank() const { return X.cols(); }
};

namespace detail {
inline std::pair<Matrix, Matrix> thin_qr(const Matrix& a) {   // algebra.hpp:31-38
    const Index m = a.rows(), k = a.cols(), kp = std::min(m, k);
    if (kp == 0) return {Matrix(m, 0), Matrix(0, k)};
    HouseholderQR qr(a);
    return {qr.thinQ(kp), qr.R(kp)};
}
inline Matrix lq_reduce(const Matrix& g) {   // algebra.hpp:42-46
    if (g.cols() <= g.rows()) return g;
    return thin_qr(g.transpose()).second.transpose();
}
struct LeafLists {
    std::vector<std::vector<int>> by_row, by_col;
};
inline LeafLists stored_leaf_lists(const H2Matrix& h) {   // algebra.hpp:53-63
    LeafLists ll;
    ll.by_row.resize(size_t(h.tree->num_nodes()));
    ll.by_col.resize(size_t(h.tree->num_nodes()));
    for (int b : h.blocks->admissible_leaves()) {
        if (!h.stores(b)) continue;
        ll.by_row[size_t(h.blocks->node(b).row)].push_back(b);
        ll.by_col[size_t(h.blocks->node(b).col)].push_back(b);
    }
    return ll;
}
}  // namespace detail

inline H2Matrix orthogonalize(const H2Matrix& h) {   // algebra.hpp:72-113
    H2Matrix g = h;
    const ClusterTree& ct = *g.tree;
    auto sweep = [&ct](BasisTree& b) {
        std::vector<Matrix> r(size_t(ct.num_nodes()));
        for (int l = ct.depth(); l >= 0; --l)
            for (int v : ct.level_nodes(l)) {
                const ClusterNode& nd = ct.node(v);
                if (nd.is_leaf()) {
                    auto qr = detail::thin_qr(b.leaf_basis(v));
                    b.leaf_basis(v) = std::move(qr.first);
                    r[size_t(v)] = std::move(qr.second);
                } else {
                    const int c0 = nd.child[0], c1 = nd.child[1];
                    Matrix z(r[size_t(c0)].rows() + r[size_t(c1)].rows(), b.rank(v));
                    z.set_block(0, 0, r[size_t(c0)] * b.transfer(c0));
                    z.set_block(r[size_t(c0)].rows(), 0, r[size_t(c1)] * b.transfer(c1));
                    auto qr = detail::thin_qr(z);
                    b.transfer(c0) = qr.first.topRows(r[size_t(c0)].rows());
                    b.transfer(c1) = qr.first.bottomRows(r[size_t(c1)].rows());
                    r[size_t(v)] = std::move(qr.second);
                }
                b.set_rank(v, r[size_t(v)].rows());
            }
        return r;
    };
    std::vector<Matrix> rr = sweep(g.row_basis), rc_store;
    if (!g.symmetric) rc_store = sweep(g.col_basis);
    const auto& rc = g.symmetric ? rr : rc_store;
    for (int b : g.blocks->admissible_leaves()) {
        if (!g.stores(b)) continue;
        const BlockNode& bn = g.blocks->node(b);
        Matrix& s = g.coupling[size_t(g.blocks->adm_ordinal(b))];
        s = gemm(rr[size_t(bn.row)] * s, false, rc[size_t(bn.col)], true);
    }
    g.orthonormal = true;
    return g;
}

inline double frobenius_norm(const H2Matrix& h) {   // algebra.hpp:119-136
    if (!h.orthonormal) throw std::invalid_argument("frobenius_norm: bases are not orthonormal; call orthogonalize");
    double sum = 0;
    for (int b : h.blocks->admissible_leaves()) {
        if (!h.stores(b)) continue;
        const double s2 = h.coupling_of(b).squaredNorm();
        sum += s2;
        if (h.symmetric && h.blocks->node(b).row != h.blocks->node(b).col) sum += s2;
    }
    for (int b : h.blocks->dense_leaves()) {
        if (!h.stores(b)) continue;
        const double d2 = h.dense_of(b).squaredNorm();
        sum += d2;
        if (h.symmetric && h.blocks->node(b).row != h.blocks->node(b).col) sum += d2;
    }
    return std::sqrt(sum);
}

inline H2Matrix recompress(const H2Matrix& h, double eps) {   // algebra.hpp:144-226
    if (eps < 0) throw std::invalid_argument("recompress: eps must be >= 0");
    H2Matrix g = h.orthonormal ? h : orthogonalize(h);
    const ClusterTree& ct = *g.tree;
    const double level_corr = std::sqrt(double(std::max(ct.depth(), 1)));
    detail::LeafLists ll = detail::stored_leaf_lists(g);
    auto truncation_bases = [&](bool row_side) {
        std::vector<Matrix> w(size_t(ct.num_nodes())), p(size_t(ct.num_nodes()));
        const BasisTree& basis = row_side ? g.row_basis : g.col_basis;
        for (int l = 0; l <= ct.depth(); ++l)
            for (int v : ct.level_nodes(l)) {
                const Index k = basis.rank(v);
                std::vector<Matrix> parts;
                auto add = [&parts](Matrix m) { if (m.cols() > 0) parts.push_back(std::move(m)); };
                if (row_side) {
                    for (int b : ll.by_row[size_t(v)]) add(g.coupling_of(b));
                    if (g.symmetric)
                        for (int b : ll.by_col[size_t(v)])
                            if (g.blocks->node(b).row != v) add(g.coupling_of(b).transpose());
                } else {
                    for (int b : ll.by_col[size_t(v)]) add(g.coupling_of(b).transpose());
                }
                const ClusterNode& nd = ct.node(v);
                if (nd.parent >= 0 && p[size_t(nd.parent)].cols() > 0) add(basis.transfer(v) * p[size_t(nd.parent)]);
                Index cols = 0;
                for (const auto& m : parts) cols += m.cols();
                if (cols == 0 || k == 0) {
                    w[size_t(v)] = Matrix(k, 0);
                    p[size_t(v)] = Matrix(k, 0);
                    continue;
                }
                Matrix gv(k, cols);
                Index at = 0;
                for (const auto& m : parts) {
                    gv.set_block(0, at, m);
                    at += m.cols();
                }
                ThinSVD svd(gv);
                const double tau = eps * svd.S[0] / level_corr;
                Index r = 0;
                while (r < Index(svd.S.size()) && svd.S[size_t(r)] > tau) ++r;
                if (std::getenv("H2_TRACE_RECOMPRESS"))
                    std::fprintf(stderr, "trunc side=%d v=%d k=%ld c=%ld s0=%.17g tau=%.17g r=%ld lo=%.17g hi=%.17g\n",
                                 int(row_side), v, long(k), long(cols), svd.S[0], tau, long(r),
                                 r > 0 ? svd.S[size_t(r - 1)] : -1.0,
                                 r < Index(svd.S.size()) ? svd.S[size_t(r)] : -1.0);
                w[size_t(v)] = svd.U.leftCols(r);
                p[size_t(v)] = detail::lq_reduce(gv);
            }
        return w;
    };
    std::vector<Matrix> wr = truncation_bases(true), wc_store;
    if (!g.symmetric) wc_store = truncation_bases(false);
    const auto& wc = g.symmetric ? wr : wc_store;
    for (int b : g.blocks->admissible_leaves()) {
        if (!g.stores(b)) continue;
        const BlockNode& bn = g.blocks->node(b);
        Matrix& s = g.coupling[size_t(g.blocks->adm_ordinal(b))];
        s = gemm(wr[size_t(bn.row)], true, s, false) * wc[size_t(bn.col)];
    }
    auto project = [&ct](BasisTree& b, const std::vector<Matrix>& w) {
        for (int l = ct.depth(); l >= 0; --l)
            for (int v : ct.level_nodes(l)) {
                const ClusterNode& nd = ct.node(v);
                if (!nd.is_leaf())
                    for (int c : nd.child) b.transfer(c) = gemm(w[size_t(c)], true, b.transfer(c), false) * w[size_t(v)];
                else
                    b.leaf_basis(v) = b.leaf_basis(v) * w[size_t(v)];
            }
        for (int v = 0; v < ct.num_nodes(); ++v) b.set_rank(v, w[size_t(v)].cols());
    };
    project(g.row_basis, wr);
    if (!g.symmetric) project(g.col_basis, wc);
    g.orthonormal = false;
    return orthogonalize(g);
}

namespace detail {
// algebra.hpp:236-316: add X Y^T on the (t, s) region in place
inline void apply_local_update(H2Matrix& h, int t, int s, const Matrix& x, const Matrix& y) {
    const ClusterTree& ct = *h.tree;
    const Index kp = x.cols();
    if (kp == 0) return;
    if (x.rows() != ct.node(t).size() || y.rows() != ct.node(s).size() || y.cols() != kp)
        throw std::invalid_argument("local update: factor dimensions do not match clusters");
    if (h.symmetric && t == s && !x.bitwise_equal(y))
        throw std::invalid_argument("local update: diagonal update on a symmetric matrix needs X == Y");
    std::vector<char> in_t(size_t(ct.num_nodes()), 0), in_s(size_t(ct.num_nodes()), 0);
    for (int v = 0; v < ct.num_nodes(); ++v) {
        in_t[size_t(v)] = ct.is_descendant(v, t);
        in_s[size_t(v)] = ct.is_descendant(v, s);
    }
    auto restrict_rows = [&ct](const Matrix& m, int region, int v) {
        return m.middleRows(ct.node(v).begin - ct.node(region).begin, ct.node(v).size());
    };
    auto augment = [&](BasisTree& b, const std::vector<char>& in_r, int region, const Matrix& f) {
        for (int v = 0; v < ct.num_nodes(); ++v) {
            if (!in_r[size_t(v)]) continue;
            const ClusterNode& nd = ct.node(v);
            const Index k_old = b.rank(v);
            if (nd.is_leaf()) {
                Matrix u(nd.size(), k_old + kp);
                u.set_block(0, 0, b.leaf_basis(v));
                u.set_block(0, k_old, restrict_rows(f, region, v));
                b.leaf_basis(v) = std::move(u);
            }
            if (nd.parent >= 0) {
                const bool parent_in = in_r[size_t(nd.parent)];
                Matrix& e = b.transfer(v);
                Matrix en(k_old + kp, parent_in ? e.cols() + kp : e.cols());
                en.set_block(0, 0, e);
                if (parent_in) en.set_block(k_old + kp - kp, e.cols(), Matrix::Identity(kp, kp));
                e = std::move(en);
            }
            b.set_rank(v, k_old + kp);
        }
    };
    if (h.symmetric) {
        augment(h.row_basis, in_t, t, x);
        if (s != t) augment(h.row_basis, in_s, s, y);
    } else {
        augment(h.row_basis, in_t, t, x);
        augment(h.col_basis, in_s, s, y);
    }
    const BasisTree& vb = h.vbasis();
    for (int b : h.blocks->admissible_leaves()) {
        if (!h.stores(b)) continue;
        const BlockNode& bn = h.blocks->node(b);
        const bool ra = h.symmetric ? (in_t[size_t(bn.row)] || in_s[size_t(bn.row)]) : bool(in_t[size_t(bn.row)]);
        const bool ca = h.symmetric ? (in_t[size_t(bn.col)] || in_s[size_t(bn.col)]) : bool(in_s[size_t(bn.col)]);
        if (!ra && !ca) continue;
        Matrix& sm = h.coupling[size_t(h.blocks->adm_ordinal(b))];
        Matrix sn(h.row_basis.rank(bn.row), vb.rank(bn.col));
        sn.set_block(0, 0, sm);
        if ((in_t[size_t(bn.row)] && in_s[size_t(bn.col)]) ||
            (h.symmetric && in_s[size_t(bn.row)] && in_t[size_t(bn.col)]))
            sn.set_block(sn.rows() - kp, sn.cols() - kp, Matrix::Identity(kp, kp));
        sm = std::move(sn);
    }
    for (int b : h.blocks->dense_leaves()) {
        if (!h.stores(b)) continue;
        const BlockNode& bn = h.blocks->node(b);
        Matrix& d = h.dense[size_t(h.blocks->dense_ordinal(b))];
        if (in_t[size_t(bn.row)] && in_s[size_t(bn.col)])
            d += gemm(restrict_rows(x, t, bn.row), false, restrict_rows(y, s, bn.col), true);
        else if (h.symmetric && in_s[size_t(bn.row)] && in_t[size_t(bn.col)])
            d += gemm(restrict_rows(y, s, bn.row), false, restrict_rows(x, t, bn.col), true);
    }
    h.orthonormal = false;
}
}  // namespace detail

inline H2Matrix local_low_rank_update(const H2Matrix& h, int t, int s, const Matrix& ub, const Matrix& vb,
                                      double eps) {   // algebra.hpp:323-331
    if (ub.cols() == 0) return h;
    H2Matrix g = (h.symmetric && t == s && !ub.bitwise_equal(vb)) ? h.desymmetrized() : h;
    detail::apply_local_update(g, t, s, ub, vb);
    return recompress(g, eps);
}

inline H2Matrix low_rank_update(const H2Matrix& h, const LowRankFactor& f, double eps) {   // algebra.hpp:334-346
    if (f.X.rows() != h.n() || f.Y.rows() != h.n() || f.X.cols() != f.Y.cols())
        throw std::invalid_argument("low_rank_update: factor dimensions do not match");
    if (f.rank() == 0) return h;
    const bool sym = f.X.bitwise_equal(f.Y);
    H2Matrix g = (h.symmetric && !sym) ? h.desymmetrized() : h;
    const Matrix xi = h.tree->to_internal(f.X);
    const Matrix yi = sym ? xi : h.tree->to_internal(f.Y);
    detail::apply_local_update(g, g.tree->root(), g.tree->root(), xi, yi);
    return recompress(g, eps);
}

// ---- linear_operator.hpp:20-178 ----------------------------------------------
class LinearOperator {
public:
    LinearOperator(Index n, bool sym) : n_(n), sym_(sym) {}
    virtual ~LinearOperator() = default;
    Index dim() const { return n_; }
    bool symmetric() const { return sym_; }
    Matrix apply(const Matrix& x) const {   // :28-32
        if (x.rows() != n_) throw std::invalid_argument("operator apply: dimension mismatch");
        cols_ += x.cols();
        return apply_impl(x);
    }
    Matrix apply_transpose(const Matrix& x) const {   // :34-39
        if (x.rows() != n_) throw std::invalid_argument("operator apply: dimension mismatch");
        cols_ += x.cols();
        if (sym_ && !has_transpose()) return apply_impl(x);
        return apply_transpose_impl(x);
    }
    long columns_applied() const { return cols_; }
    void reset_counter() const { cols_ = 0; }

protected:
    virtual Matrix apply_impl(const Matrix& x) const = 0;
    virtual Matrix apply_transpose_impl(const Matrix&) const {
        throw std::logic_error("operator: transpose application not available");
    }
    virtual bool has_transpose() const { return false; }

private:
    Index n_;
    bool sym_;
    mutable long cols_ = 0;
};

namespace detail {
class FunctionOperator final : public LinearOperator {
public:
    using Fn = std::function<Matrix(const Matrix&)>;
    FunctionOperator(Index n, bool sym, Fn f, Fn t) : LinearOperator(n, sym), f_(std::move(f)), t_(std::move(t)) {}

protected:
    Matrix apply_impl(const Matrix& x) const override { return f_(x); }
    Matrix apply_transpose_impl(const Matrix& x) const override {
        if (!t_) return LinearOperator::apply_transpose_impl(x);
        return t_(x);
    }
    bool has_transpose() const override { return bool(t_); }

private:
    Fn f_, t_;
};
}  // namespace detail

inline std::shared_ptr<LinearOperator> make_operator(Index n, bool sym, std::function<Matrix(const Matrix&)> f,
                                                     std::function<Matrix(const Matrix&)> t = nullptr) {
    return std::make_shared<detail::FunctionOperator>(n, sym, std::move(f), std::move(t));
}

class DenseOperator final : public LinearOperator {   // :86-101
public:
    explicit DenseOperator(Matrix a, bool sym = false) : LinearOperator(a.rows(), sym), a_(std::move(a)) {
        if (a_.rows() != a_.cols()) throw std::invalid_argument("dense operator: square only");
    }
    const Matrix& matrix() const { return a_; }

protected:
    Matrix apply_impl(const Matrix& x) const override { return a_ * x; }
    Matrix apply_transpose_impl(const Matrix& x) const override { return gemm(a_, true, x, false); }
    bool has_transpose() const override { return true; }

private:
    Matrix a_;
};

class H2Operator final : public LinearOperator {   // :104-115
public:
    explicit H2Operator(const H2Matrix& h) : LinearOperator(h.n(), h.symmetric), h_(&h) {}

protected:
    Matrix apply_impl(const Matrix& x) const override { return h_->matvec(x); }
    Matrix apply_transpose_impl(const Matrix& x) const override { return h_->matvec_transpose(x); }
    bool has_transpose() const override { return true; }

private:
    const H2Matrix* h_;
};

struct NormEstimate {
    double value = 0;
    int iterations = 0;
};

inline NormEstimate pnorm_estimate(const LinearOperator& op, double p, int max_iter = 100,
                                   double tol = 5e-3) {   // linear_operator.hpp:127-178
    const Index n = op.dim();
    if (p == 2.0) {
        const Index b = std::min<Index>(3, n);
        std::mt19937_64 rng(0x9E3779B97F4A7C15ull);
        std::normal_distribution<double> g(0, 1);
        Matrix v(n, b);
        for (Index j = 0; j < b; ++j)
            for (Index i = 0; i < n; ++i) v(i, j) = g(rng);
        v = HouseholderQR(v).thinQ(b);
        double est = 0, prev = -1;
        int it = 0;
        while (it < max_iter) {
            ++it;
            Matrix y = op.apply(v);
            est = spectral_norm(y);
            if (est == 0) return {0.0, it};
            if (prev > 0 && std::abs(est - prev) < tol * est) break;
            prev = est;
            Matrix z = op.apply_transpose(y);
            v = HouseholderQR(z).thinQ(b);
        }
        return {est, it};
    }
    if (p != 1.0 && !std::isinf(p)) throw std::invalid_argument("pnorm_estimate: p must be 1, 2 or inf");
    const bool want_inf = std::isinf(p);
    auto fwd = [&](const Matrix& x) { return want_inf ? op.apply_transpose(x) : op.apply(x); };
    auto bwd = [&](const Matrix& x) { return want_inf ? op.apply(x) : op.apply_transpose(x); };
    Matrix x = Matrix::Constant(n, 1, 1.0 / double(n));
    double est = 0;
    int it = 0;
    while (it < std::min(max_iter, 8)) {
        ++it;
        Matrix y = fwd(x);
        est = 0;
        for (Index i = 0; i < n; ++i) est += std::abs(y[i]);
        Matrix xi(n, 1);
        for (Index i = 0; i < n; ++i) xi[i] = y[i] >= 0 ? 1.0 : -1.0;
        Matrix z = bwd(xi);
        Index j = 0;
        double zmax = -1, ztx = 0;
        for (Index i = 0; i < n; ++i) {
            if (std::abs(z[i]) > zmax) { zmax = std::abs(z[i]); j = i; }
            ztx += z[i] * x[i];
        }
        if (zmax <= ztx) break;
        x.setZero();
        x[j] = 1.0;
    }
    return {est, it};
}

// ---- construction.hpp --------------------------------------------------------
struct PeelConfig {   // construction.hpp:23-31
    double eps = 1e-4;
    Index sample_block_size = 16;
    Index oversampling = 10;
    Index max_rank = 0;
    std::uint64_t seed = 42;
    double norm_scale = 0;
    Index crossover_rank_cap = 128;
};
struct LevelStats {
    int level = 0;
    Index blocks = 0, max_rank = 0;
    long samples = 0;
};
struct SampleStats {   // construction.hpp:40-59
    long total = 0;
    std::vector<LevelStats> levels;
    std::vector<long> per_iteration;
    void add_level(LevelStats ls) {
        total += ls.samples;
        levels.push_back(ls);
    }
    bool consistent() const {
        long s = 0;
        for (const auto& l : levels) s += l.samples;
        if (!per_iteration.empty()) {
            long t = 0;
            for (long x : per_iteration) t += x;
            return t == total;
        }
        return s == total;
    }
};
class max_rank_error : public std::runtime_error {
public:
    max_rank_error(std::string m, Matrix pu) : std::runtime_error(std::move(m)), partial_basis(std::move(pu)) {}
    Matrix partial_basis;
};

namespace detail {
inline void fill_gaussian(Matrix& m, std::mt19937_64& rng) {   // construction.hpp:81-85 (fresh distribution per call)
    std::normal_distribution<double> g(0, 1);
    for (Index j = 0; j < m.cols(); ++j)
        for (Index i = 0; i < m.rows(); ++i) m(i, j) = g(rng);
}
struct BlockRange {   // construction.hpp:88-96
    int t = -1, s = -1;
    Matrix q;
    bool converged = false, wants_full = true;
    double err_est = 0;
    Index rank() const { return q.cols(); }
};
// construction.hpp:105-129
inline void absorb_panel(BlockRange& blk, Matrix panel, double keep_tol, Index probes, Index max_rank) {
    if (blk.q.cols() > 0) {
        panel -= blk.q * gemm(blk.q, true, panel, false);
        panel -= blk.q * gemm(blk.q, true, panel, false);
    }
    const Index b = panel.cols();
    ThinSVD svd(panel);
    Index kept = 0;
    while (kept < Index(svd.S.size()) && svd.S[size_t(kept)] > keep_tol) ++kept;
    if (std::getenv("H2_TRACE_ABSORB"))   // diagnostics: one line per absorbed panel
        std::fprintf(stderr, "absorb t=%d s=%d q=%ld b=%ld tol=%.17g kept=%ld lo=%.17g hi=%.17g\n", blk.t, blk.s,
                     long(blk.q.cols()), long(b), keep_tol, long(kept),
                     kept > 0 ? svd.S[size_t(kept - 1)] : -1.0,
                     kept < Index(svd.S.size()) ? svd.S[size_t(kept)] : -1.0);
    if (max_rank > 0 && blk.q.cols() + kept > max_rank)
        throw max_rank_error("adaptive factorization: block rank exceeds max_rank", blk.q);
    if (kept > 0) {
        Matrix qn(blk.q.rows(), blk.q.cols() + kept);
        qn.set_block(0, 0, blk.q);
        qn.set_block(0, blk.q.cols(), svd.U.leftCols(kept));
        blk.q = std::move(qn);
    }
    blk.wants_full = kept == b;
    if (kept < b && (b - kept) >= probes) {
        blk.converged = true;
        blk.err_est = kept < Index(svd.S.size()) ? svd.S[size_t(kept)] : 0.0;
    }
}
}  // namespace detail

inline std::pair<Matrix, Matrix> sample_block_column(const LinearOperator& op, const ClusterTree& ct, int t, int s,
                                                     Index count, std::mt19937_64& rng) {   // construction.hpp:137-148
    if (count < 1) throw std::invalid_argument("sample_block_column: count must be >= 1");
    Matrix om(ct.node(s).size(), count);
    detail::fill_gaussian(om, rng);
    Matrix ou(ct.n(), count);
    const ClusterNode& sn = ct.node(s);
    for (Index j = 0; j < count; ++j)
        for (Index i = 0; i < sn.size(); ++i) ou(ct.perm()[size_t(sn.begin + i)], j) = om(i, j);
    Matrix y = op.apply(ou);
    return {std::move(om), ct.gather_rows(y, t)};
}

struct BlockFactor {
    Matrix u, v;
    Index rank = 0;
    double err_est = 0;
};

inline BlockFactor adaptive_block_factorization(const LinearOperator& op, const ClusterTree& ct, int t, int s,
                                                double eps_block, const PeelConfig& cfg) {   // :161-197
    std::mt19937_64 rng(cfg.seed);
    detail::BlockRange blk;
    blk.t = t;
    blk.s = s;
    blk.q = Matrix(ct.node(t).size(), 0);
    const Index b = std::max<Index>(cfg.sample_block_size, 1);
    const Index probes = std::min<Index>(std::max<Index>(cfg.oversampling, 1), b);
    const Index cap = std::min(ct.node(t).size(), ct.node(s).size());
    double scale = 0;
    while (!blk.converged) {
        const Index panel = blk.wants_full ? b : probes;
        auto sm = sample_block_column(op, ct, t, s, panel, rng);
        scale = std::max(scale, spectral_norm(sm.second));
        detail::absorb_panel(blk, std::move(sm.second), 0.5 * eps_block * scale, probes,
                             cfg.max_rank > 0 ? cfg.max_rank : cap + b);
        if (!blk.converged && blk.rank() >= cap) {
            blk.converged = true;
            blk.err_est = 0;
        }
    }
    BlockFactor f;
    f.rank = blk.rank();
    f.err_est = blk.err_est;
    if (f.rank > 0) {
        Matrix z(ct.n(), f.rank);
        const ClusterNode& tn = ct.node(t);
        for (Index j = 0; j < f.rank; ++j)
            for (Index i = 0; i < tn.size(); ++i) z(ct.perm()[size_t(tn.begin + i)], j) = blk.q(i, j);
        f.v = ct.gather_rows(op.apply_transpose(z), s);
    } else {
        f.v = Matrix(ct.node(s).size(), 0);
    }
    f.u = std::move(blk.q);
    return f;
}

namespace detail {
struct ResidualOperator final : LinearOperator {   // construction.hpp:203-222
    ResidualOperator(const LinearOperator& base, const H2Matrix* partial)
        : LinearOperator(base.dim(), base.symmetric()), base_(&base), partial_(partial) {}
    Matrix apply_impl(const Matrix& x) const override {
        Matrix y = base_->apply(x);
        if (partial_) y -= partial_->matvec(x);
        return y;
    }
    Matrix apply_transpose_impl(const Matrix& x) const override {
        Matrix y = base_->apply_transpose(x);
        if (partial_) y -= partial_->matvec_transpose(x);
        return y;
    }
    bool has_transpose() const override { return true; }

private:
    const LinearOperator* base_;
    const H2Matrix* partial_;
};

// construction.hpp:226-291
inline std::vector<BlockRange> sample_level_group(const LinearOperator& residual, const ClusterTree& ct,
                                                  const std::vector<std::pair<int, int>>& pairs, double tol_abs,
                                                  const PeelConfig& cfg, std::mt19937_64& rng,
                                                  std::vector<Matrix>& v_factors) {
    std::vector<BlockRange> ranges(pairs.size());
    for (size_t i = 0; i < pairs.size(); ++i) {
        ranges[i].t = pairs[i].first;
        ranges[i].s = pairs[i].second;
        ranges[i].q = Matrix(ct.node(pairs[i].first).size(), 0);
    }
    const Index b = std::max<Index>(cfg.sample_block_size, 1);
    const Index probes = std::min<Index>(std::max<Index>(cfg.oversampling, 1), b);
    bool all_done = false;
    while (!all_done) {
        Index panel = 0;
        for (const auto& r : ranges)
            if (!r.converged) panel = std::max(panel, r.wants_full ? b : probes);
        Matrix omega(ct.n(), panel);
        for (auto& r : ranges) {
            if (r.converged) continue;
            const ClusterNode& sn = ct.node(r.s);
            Matrix g(sn.size(), panel);
            fill_gaussian(g, rng);
            for (Index j = 0; j < panel; ++j)
                for (Index i = 0; i < sn.size(); ++i) omega(ct.perm()[size_t(sn.begin + i)], j) = g(i, j);
        }
        Matrix y = residual.apply(omega);
        const double keep_tol = 0.5 * tol_abs * std::sqrt(double(panel));
        all_done = true;
        for (auto& r : ranges) {
            if (r.converged) continue;
            const Index cap = std::min(ct.node(r.t).size(), ct.node(r.s).size());
            absorb_panel(r, ct.gather_rows(y, r.t), keep_tol, probes, cfg.max_rank > 0 ? cfg.max_rank : cap + b);
            if (!r.converged && r.rank() >= cap) {
                r.converged = true;
                r.err_est = 0;
            }
            all_done = all_done && r.converged;
        }
    }
    Index kmax = 0;
    for (const auto& r : ranges) kmax = std::max(kmax, r.rank());
    v_factors.assign(ranges.size(), Matrix());
    if (kmax > 0) {
        Matrix z(ct.n(), kmax);
        for (const auto& r : ranges) {
            const ClusterNode& tn = ct.node(r.t);
            for (Index j = 0; j < r.rank(); ++j)
                for (Index i = 0; i < tn.size(); ++i) z(ct.perm()[size_t(tn.begin + i)], j) = r.q(i, j);
        }
        Matrix w = residual.apply_transpose(z);
        for (size_t i = 0; i < ranges.size(); ++i) v_factors[i] = ct.gather_rows(w, ranges[i].s).leftCols(ranges[i].rank());
    } else {
        for (size_t i = 0; i < ranges.size(); ++i) v_factors[i] = Matrix(ct.node(ranges[i].s).size(), 0);
    }
    return ranges;
}
}  // namespace detail

struct PeelResult {
    H2Matrix matrix;
    SampleStats stats;
};

inline PeelResult peel_construct(const LinearOperator& op, std::shared_ptr<const BlockTree> bt,
                                 const PeelConfig& cfg) {   // construction.hpp:300-382
    if (bt->n() != op.dim()) throw std::invalid_argument("peel_construct: dimension mismatch");
    const ClusterTree& ct = bt->row_tree();
    std::mt19937_64 rng(cfg.seed);
    SampleStats stats;
    const bool sym = op.symmetric();
    long before = op.columns_applied();
    double norm_scale = cfg.norm_scale;
    if (norm_scale <= 0) norm_scale = std::max(pnorm_estimate(op, 2).value, 1e-300);
    stats.add_level({0, 0, 0, op.columns_applied() - before});
    const double tol_abs = 0.5 * cfg.eps * norm_scale;
    H2Matrix partial = H2Matrix::zero(bt, sym);
    for (int level = 1; level <= ct.depth(); ++level) {
        std::vector<std::pair<int, int>> pairs;
        for (int v : ct.level_nodes(level - 1))
            if (!ct.node(v).is_leaf()) pairs.emplace_back(ct.node(v).child[0], ct.node(v).child[1]);
        if (pairs.empty()) continue;
        before = op.columns_applied();
        Index max_rank_seen = 0;
        {
            detail::ResidualOperator residual(op, &partial);
            std::vector<Matrix> vf;
            auto ranges = detail::sample_level_group(residual, ct, pairs, tol_abs, cfg, rng, vf);
            for (size_t i = 0; i < ranges.size(); ++i) {
                max_rank_seen = std::max(max_rank_seen, ranges[i].rank());
                if (ranges[i].rank() > 0) detail::apply_local_update(partial, ranges[i].t, ranges[i].s, ranges[i].q, vf[i]);
            }
        }
        if (!sym) {
            std::vector<std::pair<int, int>> mirrored;
            for (auto [t, s] : pairs) mirrored.emplace_back(s, t);
            detail::ResidualOperator residual2(op, &partial);
            std::vector<Matrix> v2;
            auto ranges2 = detail::sample_level_group(residual2, ct, mirrored, tol_abs, cfg, rng, v2);
            for (size_t i = 0; i < ranges2.size(); ++i) {
                max_rank_seen = std::max(max_rank_seen, ranges2[i].rank());
                if (ranges2[i].rank() > 0) detail::apply_local_update(partial, ranges2[i].t, ranges2[i].s, ranges2[i].q, v2[i]);
            }
        }
        if (const char* dp = std::getenv("H2_PEEL_DUMP")) {   // diagnostics: dense partial per level
            Matrix a = partial.to_dense();
            std::string f = std::string(dp) + "_ora_u" + std::to_string(level) + ".bin";
            if (FILE* fp = std::fopen(f.c_str(), "wb")) { std::fwrite(a.data(), 8, size_t(a.size()), fp); std::fclose(fp); }
        }
        partial = recompress(partial, 0.5 * cfg.eps);
        if (const char* dp = std::getenv("H2_PEEL_DUMP")) {
            Matrix a = partial.to_dense();
            std::string f = std::string(dp) + "_ora_r" + std::to_string(level) + ".bin";
            if (FILE* fp = std::fopen(f.c_str(), "wb")) { std::fwrite(a.data(), 8, size_t(a.size()), fp); std::fclose(fp); }
        }
        stats.add_level({level, Index(pairs.size()) * (sym ? 1 : 2), max_rank_seen, op.columns_applied() - before});
    }
    before = op.columns_applied();
    const Index m = ct.max_leaf_size();
    {
        detail::ResidualOperator residual(op, &partial);
        Matrix omega(ct.n(), m);
        for (int v : ct.leaves()) {
            const ClusterNode& nd = ct.node(v);
            for (Index j = 0; j < nd.size(); ++j) omega(ct.perm()[size_t(nd.begin + j)], j) = 1.0;
        }
        Matrix y = residual.apply(omega);
        for (int b : bt->dense_leaves()) {
            if (!partial.stores(b)) continue;
            const BlockNode& bn = bt->node(b);
            if (bn.row != bn.col) continue;
            Matrix blk = ct.gather_rows(y, bn.row).leftCols(ct.node(bn.row).size());
            if (sym) blk = (blk + blk.transpose()) / 2;
            partial.dense[size_t(bt->dense_ordinal(b))] += blk;
        }
    }
    stats.add_level({ct.depth() + 1, Index(ct.leaves().size()), 0, op.columns_applied() - before});
    PeelResult res;
    res.matrix = recompress(partial, cfg.eps);
    res.stats = std::move(stats);
    return res;
}

inline double estimate_relative_error(const LinearOperator& op, const H2Matrix& h,
                                      double op_norm = 0) {   // construction.hpp:537-546
    auto diff = make_operator(
        op.dim(), false, [&](const Matrix& x) -> Matrix { return op.apply(x) - h.matvec(x); },
        [&](const Matrix& x) -> Matrix { return op.apply_transpose(x) - h.matvec_transpose(x); });
    const double err = pnorm_estimate(*diff, 2).value;
    const double base = op_norm > 0 ? op_norm : pnorm_estimate(op, 2).value;
    return base > 0 ? err / base : err;
}

}  // namespace oracle
}  // namespace h2
