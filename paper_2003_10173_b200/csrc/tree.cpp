// Host tree builders; see tree.hpp for the design and the reference rules.
#include "tree.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <thread>

namespace h2b {

namespace {

// nodes in a count-split subtree over m points (1 if a leaf)
int64_t subtree_nodes(int64_t m, int64_t leaf) {
    if (m <= leaf) return 1;
    const int64_t a = m / 2;
    return 1 + subtree_nodes(a, leaf) + subtree_nodes(m - a, leaf);
}

struct Builder {
    const double* x;
    int64_t n;
    int dim;
    int64_t leaf;
    ClusterTree& t;

    void box(int id) {
        double* lo = &t.lo[size_t(3 * id)];
        double* hi = &t.hi[size_t(3 * id)];
        for (int a = 0; a < 3; ++a) {
            lo[a] = a < dim ? std::numeric_limits<double>::infinity() : 0.0;
            hi[a] = a < dim ? -std::numeric_limits<double>::infinity() : 0.0;
        }
        for (int64_t i = t.begin[size_t(id)]; i < t.end[size_t(id)]; ++i) {
            const int64_t p = t.perm[size_t(i)];
            for (int a = 0; a < dim; ++a) {
                const double v = x[p + a * n];
                lo[a] = std::min(lo[a], v);
                hi[a] = std::max(hi[a], v);
            }
        }
    }

    // build the subtree whose root gets id `id`; ids of the subtree are
    // id .. id + subtree_nodes(e - b) - 1 in preorder
    void build(int id, int64_t b, int64_t e, int lvl, int par, int spawn_depth) {
        struct Item {
            int id;
            int64_t b, e;
            int lvl, par;
        };
        std::vector<Item> stack{{id, b, e, lvl, par}};
        std::vector<std::thread> workers;
        while (!stack.empty()) {
            Item it = stack.back();
            stack.pop_back();
            t.begin[size_t(it.id)] = it.b;
            t.end[size_t(it.id)] = it.e;
            t.level[size_t(it.id)] = it.lvl;
            t.parent[size_t(it.id)] = it.par;
            box(it.id);
            if (it.e - it.b <= leaf) continue;
            // longest axis, first strictly larger extent wins (point_set.hpp:96-102)
            int ax = 0;
            const double* lo = &t.lo[size_t(3 * it.id)];
            const double* hi = &t.hi[size_t(3 * it.id)];
            for (int a = 1; a < dim; ++a)
                if (hi[a] - lo[a] > hi[ax] - lo[ax]) ax = a;
            // the reference's nth_element + two sorts leave the range fully
            // sorted by (coordinate, user index): sort it directly
            const double* xa = x + ax * n;
            std::sort(t.perm.begin() + it.b, t.perm.begin() + it.e, [xa](int64_t p, int64_t q) {
                return xa[p] < xa[q] || (xa[p] == xa[q] && p < q);
            });
            const int64_t mid = it.b + (it.e - it.b) / 2;
            const int c0 = it.id + 1;
            const int c1 = c0 + int(subtree_nodes(mid - it.b, leaf));
            t.child0[size_t(it.id)] = c0;
            t.child1[size_t(it.id)] = c1;
            if (it.lvl < spawn_depth && (it.e - it.b) > 65536) {
                // disjoint perm ranges and id ranges: safe to build concurrently
                workers.emplace_back([this, c1, mid, it, spawn_depth] { build(c1, mid, it.e, it.lvl + 1, it.id, spawn_depth); });
                stack.push_back({c0, it.b, mid, it.lvl + 1, it.id});
            } else {
                stack.push_back({c1, mid, it.e, it.lvl + 1, it.id});
                stack.push_back({c0, it.b, mid, it.lvl + 1, it.id});
            }
        }
        for (auto& w : workers) w.join();
    }
};

}  // namespace

int64_t ClusterTree::max_leaf_size() const {
    int64_t m = 0;
    for (int v : leaves) m = std::max(m, size(v));
    return m;
}

namespace {
// x*x rounded to double and opaque to the optimiser, so no later add can be
// contracted into an FMA with it
inline double rounded_square(double x) {
    double p = x * x;
    asm("" : "+m"(p));
    return p;
}
// sum of squares of the (<= 3) box extents / gaps exactly as the reference's
// Release build evaluates point_set.hpp:72-76 / 79-86 (g++ 13 -O3
// -march=native on x86-64, proj/CMakeLists.txt:3-20): the loop is vectorised
// two lanes wide, so the first two squares are rounded and added without
// contraction, and a third term is fused as fma(x2, x2, x0^2 + x1^2).
// Verified against the reference headers compiled unchanged (oracle/_ref):
// cfg4's block tree then matches the reference's counts exactly.
inline double release_sq_sum(const double* x, int dim) {
    if (dim == 1) return rounded_square(x[0]);
    double s = rounded_square(x[0]) + rounded_square(x[1]);
    if (dim == 3) s = std::fma(x[2], x[2], s);
    return s;
}
}  // namespace

double ClusterTree::diameter(int v) const {
    double e[3] = {0, 0, 0};
    for (int a = 0; a < dim; ++a) e[a] = hi[size_t(3 * v + a)] - lo[size_t(3 * v + a)];
    return std::sqrt(release_sq_sum(e, dim));
}

double ClusterTree::distance(int v, int w) const {
    double g[3] = {0, 0, 0};
    for (int a = 0; a < dim; ++a)
        g[a] = std::max({0.0, lo[size_t(3 * w + a)] - hi[size_t(3 * v + a)], lo[size_t(3 * v + a)] - hi[size_t(3 * w + a)]});
    return std::sqrt(release_sq_sum(g, dim));
}

std::shared_ptr<ClusterTree> build_cluster_tree(const double* coords, int64_t n, int dim, int64_t leaf_size) {
    if (n < 1) throw std::invalid_argument("cluster tree: empty point set");
    if (dim < 1 || dim > 3) throw std::invalid_argument("PointSet: dimension must be 1, 2 or 3");
    if (leaf_size < 2) throw std::invalid_argument("cluster tree: leaf_size must be >= 2");
    auto t = std::make_shared<ClusterTree>();
    t->n = n;
    t->dim = dim;
    t->leaf_size = leaf_size;
    const int64_t nn = subtree_nodes(n, leaf_size);
    if (nn > std::numeric_limits<int>::max()) throw std::invalid_argument("cluster tree: too many nodes");
    t->begin.assign(size_t(nn), 0);
    t->end.assign(size_t(nn), 0);
    t->level.assign(size_t(nn), 0);
    t->parent.assign(size_t(nn), -1);
    t->child0.assign(size_t(nn), -1);
    t->child1.assign(size_t(nn), -1);
    t->lo.assign(size_t(3 * nn), 0.0);
    t->hi.assign(size_t(3 * nn), 0.0);
    t->perm.resize(size_t(n));
    std::iota(t->perm.begin(), t->perm.end(), int64_t(0));
    Builder bld{coords, n, dim, leaf_size, *t};
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    int spawn = 0;
    while ((1u << spawn) < hw && spawn < 6) ++spawn;
    bld.build(0, 0, n, 0, -1, spawn);
    t->inv_perm.resize(size_t(n));
    for (int64_t i = 0; i < n; ++i) t->inv_perm[size_t(t->perm[size_t(i)])] = i;
    for (int v = 0; v < int(nn); ++v) t->depth = std::max(t->depth, t->level[size_t(v)]);
    t->levels.assign(size_t(t->depth + 1), {});
    for (int v = 0; v < int(nn); ++v) {
        t->levels[size_t(t->level[size_t(v)])].push_back(v);
        if (t->is_leaf(v)) t->leaves.push_back(v);
    }
    return t;
}

std::shared_ptr<ClusterTree> restore_cluster_tree(int64_t n, int dim, int64_t leaf_size, std::vector<int64_t> begin,
                                                  std::vector<int64_t> end, std::vector<int> level,
                                                  std::vector<int> parent, std::vector<int> child0,
                                                  std::vector<int> child1, std::vector<double> lo,
                                                  std::vector<double> hi, std::vector<int64_t> perm) {
    const size_t nn = begin.size();
    if (end.size() != nn || level.size() != nn || parent.size() != nn || child0.size() != nn ||
        child1.size() != nn || lo.size() != 3 * nn || hi.size() != 3 * nn || perm.size() != size_t(n) || nn == 0)
        throw std::invalid_argument("cluster tree restore: inconsistent arrays");
    auto t = std::make_shared<ClusterTree>();
    t->n = n;
    t->dim = dim;
    t->leaf_size = leaf_size;
    t->begin = std::move(begin);
    t->end = std::move(end);
    t->level = std::move(level);
    t->parent = std::move(parent);
    t->child0 = std::move(child0);
    t->child1 = std::move(child1);
    t->lo = std::move(lo);
    t->hi = std::move(hi);
    t->perm = std::move(perm);
    t->inv_perm.assign(size_t(n), -1);
    for (int64_t i = 0; i < n; ++i) {
        const int64_t p = t->perm[size_t(i)];
        if (p < 0 || p >= n || t->inv_perm[size_t(p)] >= 0)
            throw std::invalid_argument("cluster tree restore: permutation is not a bijection");
        t->inv_perm[size_t(p)] = i;
    }
    for (int v = 0; v < int(nn); ++v) {
        const int c0 = t->child0[size_t(v)], c1 = t->child1[size_t(v)];
        if ((c0 < 0) != (c1 < 0) || c0 >= int(nn) || c1 >= int(nn) || t->begin[size_t(v)] > t->end[size_t(v)])
            throw std::invalid_argument("cluster tree restore: bad node");
        t->depth = std::max(t->depth, t->level[size_t(v)]);
    }
    t->levels.assign(size_t(t->depth + 1), {});
    for (int v = 0; v < int(nn); ++v) {
        t->levels[size_t(t->level[size_t(v)])].push_back(v);
        if (t->is_leaf(v)) t->leaves.push_back(v);
    }
    return t;
}

std::shared_ptr<BlockTree> build_block_tree(std::shared_ptr<const ClusterTree> ct, double eta, bool weak) {
    auto bt = std::make_shared<BlockTree>();
    bt->tree = ct;
    bt->eta = eta;
    bt->weak = weak;
    const ClusterTree& t = *ct;
    std::vector<double> diam(size_t(t.num_nodes()));
    for (int v = 0; v < t.num_nodes(); ++v) diam[size_t(v)] = t.diameter(v);
    // explicit-stack preorder traversal; a node's id is assigned when popped,
    // children pushed in reverse so (t0,s0),(t0,s1),(t1,s0),(t1,s1) come out
    // in the reference's row-major order
    struct Item {
        int r, c, lvl, par, slot;
    };
    std::vector<Item> stack{{0, 0, 0, -1, -1}};
    while (!stack.empty()) {
        const Item it = stack.back();
        stack.pop_back();
        const int id = bt->num_nodes();
        bt->row.push_back(it.r);
        bt->col.push_back(it.c);
        bt->level.push_back(it.lvl);
        bt->parent.push_back(it.par);
        bt->children.push_back({-1, -1, -1, -1});
        bt->adm_ord.push_back(-1);
        bt->dense_ord.push_back(-1);
        if (it.par >= 0) bt->children[size_t(it.par)][size_t(it.slot)] = id;
        bt->max_level = std::max(bt->max_level, it.lvl);
        bool admissible;
        if (weak) admissible = t.begin[size_t(it.r)] != t.begin[size_t(it.c)] || t.end[size_t(it.r)] != t.end[size_t(it.c)];
        else admissible = std::max(diam[size_t(it.r)], diam[size_t(it.c)]) <= eta * t.distance(it.r, it.c);
        if (admissible) {
            bt->tag.push_back(kAdmissible);
            bt->adm_ord[size_t(id)] = int(bt->adm.size());
            bt->adm.push_back(id);
            continue;
        }
        const bool rl = t.is_leaf(it.r), cl = t.is_leaf(it.c);
        if (rl && cl) {
            bt->tag.push_back(kDense);
            bt->dense_ord[size_t(id)] = int(bt->dense.size());
            bt->dense.push_back(id);
            continue;
        }
        bt->tag.push_back(kInterior);
        int rs[2] = {it.r, -1}, cs[2] = {it.c, -1};
        const int nr = rl ? 1 : 2, nc = cl ? 1 : 2;
        if (!rl) { rs[0] = t.child0[size_t(it.r)]; rs[1] = t.child1[size_t(it.r)]; }
        if (!cl) { cs[0] = t.child0[size_t(it.c)]; cs[1] = t.child1[size_t(it.c)]; }
        for (int k = nr * nc - 1; k >= 0; --k) stack.push_back({rs[k / nc], cs[k % nc], it.lvl + 1, id, k});
    }
    return bt;
}

}  // namespace h2b
