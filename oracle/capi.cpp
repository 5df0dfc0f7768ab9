// ORACLE — TEST INFRASTRUCTURE ONLY. extern "C" access to the CPU
// restatement for the Python parity tests and bench.py's cpu_baseline leg.
// The product library never links this.
#include <algorithm>
#include <chrono>
#include <random>
#include <cstring>
#include <string>
#include <thread>

#ifdef ORA_REFERENCE_HEADERS
// oracle/_ref build: the UNCHANGED reference headers (/root/reference/proj/
// include/h2 + tests/test_support.hpp, compiled where they lie) over the
// Eigen-API shim in oracle/eigen_shim. Same ora_* ABI as the restatement, so
// the Python checker can load either library.
#include "h2/algebra.hpp"
#include "h2/construction.hpp"
#include "h2/inversion.hpp"
#include "h2/serialize.hpp"
#include <test_support.hpp>   // the reference's, via -I$(REF)/tests (not ./test_support.hpp)
#else
#include "diffusion1d.hpp"
#include "test_support.hpp"
#endif

using namespace h2;

namespace {
thread_local std::string g_err;
template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const max_rank_error& e) {
        g_err = e.what();
        return -3;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return -1;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return -2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -4;
    }
}
Matrix wrap(const double* p, Index r, Index c) {
    Matrix m(r, c);
    if (r * c > 0) std::memcpy(m.data(), p, sizeof(double) * size_t(r * c));
    return m;
}
void out(const Matrix& m, double* p) {
    if (m.size()) std::memcpy(p, m.data(), sizeof(double) * size_t(m.size()));
}
}  // namespace

struct ora_tree {
    std::shared_ptr<const ClusterTree> ct;
    std::shared_ptr<const BlockTree> bt;
};
struct ora_h2 {
    H2Matrix h;
};

extern "C" {

const char* ora_last_error() { return g_err.c_str(); }

int ora_tree_create(const double* coords, int64_t n, int dim, int64_t leaf, double eta, int weak, ora_tree** o) {
    return guard([&] {
        auto ct = build_cluster_tree(PointSet(wrap(coords, n, dim)), leaf);
        auto bt = build_block_tree(ct, ct, eta, weak ? Admissibility::weak : Admissibility::strong);
        *o = new ora_tree{ct, bt};
    });
}
void ora_tree_destroy(ora_tree* t) { delete t; }

int ora_tree_info(ora_tree* t, int64_t* n, int* depth, int* num_nodes, int* num_blocks, int* n_adm, int* n_dense) {
    return guard([&] {
        *n = t->ct->n();
        *depth = t->ct->depth();
        *num_nodes = t->ct->num_nodes();
        *num_blocks = t->bt->num_nodes();
        *n_adm = int(t->bt->admissible_leaves().size());
        *n_dense = int(t->bt->dense_leaves().size());
    });
}

int ora_tree_arrays(ora_tree* t, int64_t* perm, int64_t* begin, int64_t* end, int* level, int* parent, int* child0,
                    int* child1, int* brow, int* bcol, int* btag, int* adm, int* dense) {
    return guard([&] {
        const auto& ct = *t->ct;
        for (Index i = 0; i < ct.n(); ++i) perm[i] = ct.perm()[size_t(i)];
        for (int v = 0; v < ct.num_nodes(); ++v) {
            begin[v] = ct.node(v).begin;
            end[v] = ct.node(v).end;
            level[v] = ct.node(v).level;
            parent[v] = ct.node(v).parent;
            child0[v] = ct.node(v).child[0];
            child1[v] = ct.node(v).child[1];
        }
        const auto& bt = *t->bt;
        for (int b = 0; b < bt.num_nodes(); ++b) {
            brow[b] = bt.node(b).row;
            bcol[b] = bt.node(b).col;
            btag[b] = int(bt.node(b).tag);
        }
        for (size_t i = 0; i < bt.admissible_leaves().size(); ++i) adm[i] = bt.admissible_leaves()[i];
        for (size_t i = 0; i < bt.dense_leaves().size(); ++i) dense[i] = bt.dense_leaves()[i];
    });
}

// per-node bounding boxes (point_set.hpp:68-70 BBox, cluster_tree.hpp:178-190), 3 per node
int ora_tree_boxes(ora_tree* t, double* lo, double* hi) {
    return guard([&] {
        const auto& ct = *t->ct;
        for (int v = 0; v < ct.num_nodes(); ++v)
            for (int a = 0; a < 3; ++a) {
                lo[3 * v + a] = ct.node(v).box.lo[size_t(a)];
                hi[3 * v + a] = ct.node(v).box.hi[size_t(a)];
            }
    });
}

// reference fixture random_h2 (test_support.hpp:38-70) from mt19937_64(seed)
int ora_random_h2(ora_tree* t, int symmetric, int64_t kmax, uint64_t seed, ora_h2** o) {
    return guard([&] {
        std::mt19937_64 rng(seed);
        *o = new ora_h2{testing::random_h2(t->bt, symmetric != 0, kmax, rng)};
    });
}
// fixed-rank symmetric content for CPU-only benchmark runs (SURVEY §8d option
// (i): cost and parity do not depend on the fill). Uniform(-1,1) values from a
// counter-based hash so blocks fill in parallel.
int ora_fixed_rank_h2(ora_tree* t, int64_t k, uint64_t seed, int nthreads, ora_h2** o) {
    return guard([&] {
        H2Matrix h = H2Matrix::zero(t->bt, true);
        const ClusterTree& ct = *h.tree;
        auto val = [seed](uint64_t a, uint64_t b) {
            uint64_t z = seed ^ (a * 0x9E3779B97F4A7C15ull) ^ (b * 0xC2B2AE3D27D4EB4Full);
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
            z ^= z >> 31;
            return double(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
        };
        auto fill = [&](Matrix& m, uint64_t tag) {
            for (Index i = 0; i < m.size(); ++i) m[i] = val(tag, uint64_t(i));
        };
        for (int v = 0; v < ct.num_nodes(); ++v) h.row_basis.set_rank(v, std::min(ct.node(v).size(), k));
        for (int v = 0; v < ct.num_nodes(); ++v) {
            const auto& nd = ct.node(v);
            if (nd.is_leaf()) {
                h.row_basis.leaf_basis(v) = Matrix(nd.size(), h.row_basis.rank(v));
                fill(h.row_basis.leaf_basis(v), uint64_t(v) << 2);
            }
            if (nd.parent >= 0) {
                h.row_basis.transfer(v) = Matrix(h.row_basis.rank(v), h.row_basis.rank(nd.parent));
                fill(h.row_basis.transfer(v), (uint64_t(v) << 2) | 1);
            }
        }
        const auto& bt = *t->bt;
        const int nt = std::max(1, nthreads);
        std::vector<std::thread> th;
        for (int w = 0; w < nt; ++w)
            th.emplace_back([&, w] {
                for (size_t i = size_t(w); i < bt.admissible_leaves().size(); i += size_t(nt)) {
                    const int b = bt.admissible_leaves()[i];
                    if (!h.stores(b)) continue;
                    h.coupling[i] = Matrix(h.row_basis.rank(bt.node(b).row), h.row_basis.rank(bt.node(b).col));
                    fill(h.coupling[i], (uint64_t(i) << 2) | 2);
                }
                for (size_t i = size_t(w); i < bt.dense_leaves().size(); i += size_t(nt)) {
                    const int b = bt.dense_leaves()[i];
                    if (!h.stores(b)) continue;
                    fill(h.dense[i], (uint64_t(i) << 2) | 3);
                }
            });
        for (auto& x : th) x.join();
        h.orthonormal = false;
        *o = new ora_h2{std::move(h)};
    });
}

// kernel-matrix H^2 content on the host: a CPU restatement of the product's
// benchmark generator (paper_2003_10173_b200/csrc/matrix.cu make_kernel_h2,
// SURVEY §8d option (ii)) so the reference arm multiplies the same payload as
// the B200 arm (to rounding: exp/cos on the host vs the device). Symmetric,
// rank min(k, |v|) per node: Chebyshev tensor grids, Lagrange leaf bases and
// transfers, S = K(grid_t, grid_s), D = K(x_t, x_s). kind 0 exponential,
// 1 Gaussian, 2 Matern-3/2.
}  // extern "C"
namespace {
struct KGrid {
    double lo[3], hi[3];
    int p[3];
};
double kval(int kind, double ell, double r2) {
    if (kind == 1) return std::exp(-r2 / (ell * ell));
    const double r = std::sqrt(r2);
    if (kind == 0) return std::exp(-r / ell);
    const double a = 1.7320508075688772 * r / ell;
    return (1.0 + a) * std::exp(-a);
}
double knode(const KGrid& g, int ax, int i) {
    const int p = g.p[ax];
    const double c = 0.5 * (g.lo[ax] + g.hi[ax]), h = 0.5 * (g.hi[ax] - g.lo[ax]);
    if (p == 1) return c;
    return c + h * std::cos(3.14159265358979323846 * (2 * i + 1) / (2.0 * p));
}
double klagrange(const KGrid& g, int dim, int a, const double* x) {
    double v = 1.0;
    for (int d = 0; d < dim; ++d) {
        const int ia = a % g.p[d];
        a /= g.p[d];
        const double xa = knode(g, d, ia);
        for (int j = 0; j < g.p[d]; ++j)
            if (j != ia) {
                const double xj = knode(g, d, j);
                v *= (x[d] - xj) / (xa - xj);
            }
    }
    return v;
}
void kgrid_point(const KGrid& g, int dim, int a, double* x) {
    for (int d = 0; d < dim; ++d) {
        x[d] = knode(g, d, a % g.p[d]);
        a /= g.p[d];
    }
}
void kaxis_counts(int dim, int k, const double* ext, int* p) {
    int order[3] = {0, 1, 2};
    for (int i = 1; i < dim && i < 3; ++i)
        for (int j = i; j > 0 && ext[order[j]] > ext[order[j - 1]]; --j) std::swap(order[j], order[j - 1]);
    for (int d = 0; d < 3; ++d) p[d] = 1;
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
template <class F>
void parallel_for(int64_t n, int nthreads, F&& f) {
    const int nt = std::max(1, nthreads);
    std::vector<std::thread> th;
    for (int w = 0; w < nt; ++w)
        th.emplace_back([&, w] {
            for (int64_t i = w; i < n; i += nt) f(i);
        });
    for (auto& t : th) t.join();
}
}  // namespace
extern "C" {

int ora_kernel_h2(ora_tree* t, const double* coords, int kind, double ell, int64_t rank, int nthreads, ora_h2** o) {
    return guard([&] {
        const ClusterTree& ct = *t->ct;
        const int nn = ct.num_nodes(), dim = ct.dim();
        const Index n = ct.n();
        H2Matrix h = H2Matrix::zero(t->bt, true);
        std::vector<KGrid> grids(static_cast<size_t>(nn));
        for (int v = 0; v < nn; ++v) {
            const auto& nd = ct.node(v);
            h.row_basis.set_rank(v, std::min<Index>(rank, nd.size()));
            KGrid& g = grids[size_t(v)];
            double ext[3] = {0, 0, 0}, diam = 0;
            for (int d = 0; d < 3; ++d) {
                g.lo[d] = d < dim ? nd.box.lo[size_t(d)] : 0.0;
                g.hi[d] = d < dim ? nd.box.hi[size_t(d)] : 0.0;
                ext[d] = d < dim ? g.hi[d] - g.lo[d] : 0;
                diam += ext[d] * ext[d];
            }
            diam = std::sqrt(diam);
            for (int d = 0; d < dim; ++d)
                if (ext[d] < 1e-9 * std::max(diam, 1e-300)) {
                    const double w = std::max(1e-3 * diam, 1e-12);
                    g.lo[d] -= w;
                    g.hi[d] += w;
                    ext[d] = g.hi[d] - g.lo[d];
                }
            kaxis_counts(dim, int(h.row_basis.rank(v)), ext, g.p);
        }
        auto pt = [&](Index user, double* x) {
            for (int d = 0; d < dim; ++d) x[d] = coords[user + d * n];
        };
        for (int v : ct.leaves()) {
            const auto& nd = ct.node(v);
            const Index m = nd.size(), k = h.row_basis.rank(v);
            Matrix u(m, k);
            for (Index a = 0; a < k; ++a)
                for (Index i = 0; i < m; ++i) {
                    double x[3];
                    pt(ct.perm()[size_t(nd.begin + i)], x);
                    u(i, a) = klagrange(grids[size_t(v)], dim, int(a), x);
                }
            h.row_basis.leaf_basis(v) = std::move(u);
        }
        for (int v = 0; v < nn; ++v) {
            const int par = ct.node(v).parent;
            if (par < 0) continue;
            const Index kc = h.row_basis.rank(v), kp = h.row_basis.rank(par);
            Matrix e(kc, kp);
            for (Index ap = 0; ap < kp; ++ap)
                for (Index ac = 0; ac < kc; ++ac) {
                    double x[3];
                    kgrid_point(grids[size_t(v)], dim, int(ac), x);
                    e(ac, ap) = klagrange(grids[size_t(par)], dim, int(ap), x);
                }
            h.row_basis.transfer(v) = std::move(e);
        }
        const auto& adm = t->bt->admissible_leaves();
        parallel_for(int64_t(adm.size()), nthreads, [&](int64_t i) {
            const int b = adm[size_t(i)];
            if (!h.stores(b)) return;
            const auto& bn = t->bt->node(b);
            const Index kr = h.row_basis.rank(bn.row), kc = h.row_basis.rank(bn.col);
            Matrix sm(kr, kc);
            for (Index c = 0; c < kc; ++c)
                for (Index a = 0; a < kr; ++a) {
                    double x[3], y[3], r2 = 0;
                    kgrid_point(grids[size_t(bn.row)], dim, int(a), x);
                    kgrid_point(grids[size_t(bn.col)], dim, int(c), y);
                    for (int d = 0; d < dim; ++d) r2 += (x[d] - y[d]) * (x[d] - y[d]);
                    sm(a, c) = kval(kind, ell, r2);
                }
            h.coupling[size_t(i)] = std::move(sm);
        });
        const auto& den = t->bt->dense_leaves();
        parallel_for(int64_t(den.size()), nthreads, [&](int64_t i) {
            const int b = den[size_t(i)];
            if (!h.stores(b)) return;
            const auto& bn = t->bt->node(b);
            const auto &tr = ct.node(bn.row), &tc = ct.node(bn.col);
            Matrix dm(tr.size(), tc.size());
            for (Index j = 0; j < tc.size(); ++j)
                for (Index r = 0; r < tr.size(); ++r) {
                    double x[3], y[3], r2 = 0;
                    pt(ct.perm()[size_t(tr.begin + r)], x);
                    pt(ct.perm()[size_t(tc.begin + j)], y);
                    for (int d = 0; d < dim; ++d) r2 += (x[d] - y[d]) * (x[d] - y[d]);
                    dm(r, j) = kval(kind, ell, r2);
                }
            h.dense[size_t(i)] = std::move(dm);
        });
        h.orthonormal = false;
        *o = new ora_h2{std::move(h)};
    });
}

// H2Matrix::zero (h2_matrix.hpp:53-75)
int ora_zero(ora_tree* t, int symmetric, ora_h2** o) {
    return guard([&] { *o = new ora_h2{H2Matrix::zero(t->bt, symmetric != 0)}; });
}
void ora_h2_destroy(ora_h2* h) { delete h; }

int ora_h2_info(ora_h2* h, int* symmetric, int* orthonormal, int64_t sizes[6]) {
    return guard([&] {
        const H2Matrix& m = h->h;
        *symmetric = m.symmetric;
        *orthonormal = m.orthonormal;
        const ClusterTree& ct = *m.tree;
        for (int i = 0; i < 6; ++i) sizes[i] = 0;
        auto basis = [&](const BasisTree& b, int64_t& su, int64_t& se) {
            for (int v : ct.leaves()) su += b.leaf_basis(v).size();
            for (int v = 0; v < ct.num_nodes(); ++v)
                if (ct.node(v).parent >= 0) se += b.transfer(v).size();
        };
        basis(m.row_basis, sizes[0], sizes[1]);
        if (!m.symmetric) basis(m.col_basis, sizes[2], sizes[3]);
        for (size_t i = 0; i < m.coupling.size(); ++i)
            if (m.stores(m.blocks->admissible_leaves()[i])) sizes[4] += m.coupling[i].size();
        for (size_t i = 0; i < m.dense.size(); ++i)
            if (m.stores(m.blocks->dense_leaves()[i])) sizes[5] += m.dense[i].size();
    });
}

int ora_h2_ranks(ora_h2* h, int* row, int* col) {
    return guard([&] {
        for (int v = 0; v < h->h.tree->num_nodes(); ++v) {
            row[v] = int(h->h.row_basis.rank(v));
            if (col) col[v] = int(h->h.vbasis().rank(v));
        }
    });
}

// packed export in the layout of include/h2c.h
int ora_h2_export(ora_h2* h, double* U, double* E, double* V, double* F, double* S, double* D) {
    return guard([&] {
        const H2Matrix& m = h->h;
        const ClusterTree& ct = *m.tree;
        auto basis = [&](const BasisTree& b, double* pu, double* pe) {
            for (int v : ct.leaves()) {
                out(b.leaf_basis(v), pu);
                pu += b.leaf_basis(v).size();
            }
            for (int v = 0; v < ct.num_nodes(); ++v)
                if (ct.node(v).parent >= 0) {
                    out(b.transfer(v), pe);
                    pe += b.transfer(v).size();
                }
        };
        basis(m.row_basis, U, E);
        if (!m.symmetric) basis(m.col_basis, V, F);
        for (size_t i = 0; i < m.coupling.size(); ++i)
            if (m.stores(m.blocks->admissible_leaves()[i])) {
                out(m.coupling[i], S);
                S += m.coupling[i].size();
            }
        for (size_t i = 0; i < m.dense.size(); ++i)
            if (m.stores(m.blocks->dense_leaves()[i])) {
                out(m.dense[i], D);
                D += m.dense[i].size();
            }
    });
}

int ora_h2_import(ora_tree* t, int symmetric, int orthonormal, const int* row_ranks, const int* col_ranks,
                  const double* U, const double* E, const double* V, const double* F, const double* S,
                  const double* D, ora_h2** o) {
    return guard([&] {
        H2Matrix m = H2Matrix::zero(t->bt, symmetric != 0);
        const ClusterTree& ct = *m.tree;
        auto basis = [&](BasisTree& b, const int* ranks, const double* pu, const double* pe) {
            for (int v = 0; v < ct.num_nodes(); ++v) b.set_rank(v, ranks[v]);
            for (int v : ct.leaves()) {
                b.leaf_basis(v) = wrap(pu, ct.node(v).size(), ranks[v]);
                pu += ct.node(v).size() * ranks[v];
            }
            for (int v = 0; v < ct.num_nodes(); ++v)
                if (ct.node(v).parent >= 0) {
                    b.transfer(v) = wrap(pe, ranks[v], ranks[ct.node(v).parent]);
                    pe += Index(ranks[v]) * ranks[ct.node(v).parent];
                }
        };
        basis(m.row_basis, row_ranks, U, E);
        if (!m.symmetric) basis(m.col_basis, col_ranks, V, F);
        for (size_t i = 0; i < m.coupling.size(); ++i) {
            const int b = m.blocks->admissible_leaves()[i];
            if (!m.stores(b)) continue;
            const Index kr = m.row_basis.rank(m.blocks->node(b).row), kc = m.vbasis().rank(m.blocks->node(b).col);
            m.coupling[i] = wrap(S, kr, kc);
            S += kr * kc;
        }
        for (size_t i = 0; i < m.dense.size(); ++i) {
            const int b = m.blocks->dense_leaves()[i];
            if (!m.stores(b)) continue;
            const Index mr = ct.node(m.blocks->node(b).row).size(), mc = ct.node(m.blocks->node(b).col).size();
            m.dense[i] = wrap(D, mr, mc);
            D += mr * mc;
        }
        m.orthonormal = orthonormal != 0;
        *o = new ora_h2{std::move(m)};
    });
}

// y = op(H) x, n x b column-major; ordering 0 user, 1 internal. With
// nthreads > 1 the columns are split across host threads (each thread runs
// the reference's four-stage product on its own columns).
int ora_matvec(ora_h2* h, int transpose, int ordering, int64_t b, const double* x, double* y, int nthreads) {
    return guard([&] {
        const H2Matrix& m = h->h;
        const Index n = m.n();
        auto run = [&](const Matrix& xx) {
            if (ordering == 0) return transpose ? m.matvec_transpose(xx) : m.matvec(xx);
            return transpose ? m.matvec_transpose_internal(xx) : m.matvec_internal(xx);
        };
        const int nt = int(std::max<int64_t>(1, std::min<int64_t>(nthreads, b)));
        if (nt == 1) {
            out(run(wrap(x, n, b)), y);
            return;
        }
        std::vector<std::thread> th;
        std::vector<std::string> errs(static_cast<size_t>(nt));
        for (int i = 0; i < nt; ++i) {
            th.emplace_back([&, i] {
                try {
                    const Index c0 = b * i / nt, c1 = b * (i + 1) / nt;
                    Matrix yy = run(wrap(x + c0 * n, n, c1 - c0));
                    out(yy, y + c0 * n);
                } catch (const std::exception& e) {
                    errs[size_t(i)] = e.what();
                }
            });
        }
        for (auto& t : th) t.join();
        for (auto& e : errs)
            if (!e.empty()) throw std::runtime_error(e);
    });
}

int ora_to_dense(ora_h2* h, double* a) {
    return guard([&] { out(h->h.to_dense(), a); });
}
int ora_orthogonalize(ora_h2* h, ora_h2** o) {
    return guard([&] { *o = new ora_h2{orthogonalize(h->h)}; });
}
int ora_recompress(ora_h2* h, double eps, ora_h2** o) {
    return guard([&] { *o = new ora_h2{recompress(h->h, eps)}; });
}
int ora_low_rank_update(ora_h2* h, int64_t k, const double* X, const double* Y, double eps, ora_h2** o) {
    return guard([&] {
        const Index n = h->h.n();
        *o = new ora_h2{low_rank_update(h->h, LowRankFactor{wrap(X, n, k), wrap(Y, n, k)}, eps)};
    });
}
int ora_frobenius_norm(ora_h2* h, double* v) {
    return guard([&] { *v = frobenius_norm(h->h); });
}

// peel_construct over a DenseOperator(a, symmetric) (construction.hpp:300-382)
int ora_peel_dense(ora_tree* t, const double* a, int symmetric, double eps, int64_t b, int64_t p, int64_t max_rank,
                   uint64_t seed, double norm_scale, ora_h2** o, int64_t* total_samples, int64_t* level_samples,
                   int64_t* level_max_rank, int* nlevels) {
    return guard([&] {
        const Index n = t->ct->n();
        DenseOperator op(wrap(a, n, n), symmetric != 0);
        PeelConfig cfg;
        cfg.eps = eps;
        cfg.sample_block_size = b;
        cfg.oversampling = p;
        cfg.max_rank = max_rank;
        cfg.seed = seed;
        cfg.norm_scale = norm_scale;
        PeelResult r = peel_construct(op, t->bt, cfg);
        *total_samples = r.stats.total;
        *nlevels = int(r.stats.levels.size());
        for (size_t i = 0; i < r.stats.levels.size(); ++i) {
            level_samples[i] = r.stats.levels[i].samples;
            level_max_rank[i] = r.stats.levels[i].max_rank;
        }
        *o = new ora_h2{std::move(r.matrix)};
    });
}

// peel_construct over a dense black box applied by `nthreads` host threads
// (y = A x rows split across threads, A^T x output rows = columns of A): the
// reference's construction code, single-threaded as it is, around a threaded
// user operator. *op_seconds = wall time inside the operator.
int ora_peel_dense_threads(ora_tree* t, const double* a, int symmetric, double eps, uint64_t seed, double norm_scale,
                           int nthreads, ora_h2** o, int64_t* total_samples, int64_t* level_samples,
                           int64_t* level_max_rank, int* nlevels, double* op_seconds) {
    return guard([&] {
        const Index n = t->ct->n();
        const int nt = std::max(1, nthreads);
        double op_s = 0;
        auto apply = [&](const Matrix& x, bool trans) {
            const auto t0 = std::chrono::steady_clock::now();
            const Index b = x.cols();
            Matrix y(n, b);
            const double* xp = x.data();
            double* yp = y.data();
            std::vector<std::thread> th;
            for (int w = 0; w < nt; ++w)
                th.emplace_back([&, w] {
                    const Index r0 = n * w / nt, r1 = n * (w + 1) / nt;
                    if (!trans) {   // y[r0:r1, :] = A[r0:r1, :] x  (A column-major: stream each column's slice)
                        for (Index j = 0; j < b; ++j)
                            for (Index i = r0; i < r1; ++i) yp[i + j * n] = 0.0;
                        for (Index k = 0; k < n; ++k) {
                            const double* ac = a + k * n;
                            for (Index j = 0; j < b; ++j) {
                                const double xk = xp[k + j * n];
                                double* yc = yp + j * n;
                                for (Index i = r0; i < r1; ++i) yc[i] += ac[i] * xk;
                            }
                        }
                    } else {        // y[i, :] = A[:, i]^T x for i in [r0, r1)
                        for (Index i = r0; i < r1; ++i) {
                            const double* ac = a + i * n;
                            for (Index j = 0; j < b; ++j) {
                                const double* xc = xp + j * n;
                                double acc = 0;
                                for (Index k = 0; k < n; ++k) acc += ac[k] * xc[k];
                                yp[i + j * n] = acc;
                            }
                        }
                    }
                });
            for (auto& x2 : th) x2.join();
            op_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            return y;
        };
        auto op = make_operator(n, symmetric != 0, [&](const Matrix& x) { return apply(x, false); },
                                [&](const Matrix& x) { return apply(x, true); });
        PeelConfig cfg;
        cfg.eps = eps;
        cfg.seed = seed;
        cfg.norm_scale = norm_scale;
        PeelResult r = peel_construct(*op, t->bt, cfg);
        *total_samples = r.stats.total;
        *nlevels = int(r.stats.levels.size());
        for (size_t i = 0; i < r.stats.levels.size(); ++i) {
            level_samples[i] = r.stats.levels[i].samples;
            level_max_rank[i] = r.stats.levels[i].max_rank;
        }
        *op_seconds = op_s;
        *o = new ora_h2{std::move(r.matrix)};
    });
}

// peel_construct over an H2Operator of another oracle matrix
int ora_peel_h2(ora_tree* t, ora_h2* src, double eps, uint64_t seed, double norm_scale, ora_h2** o,
                int64_t* total_samples) {
    return guard([&] {
        H2Operator op(src->h);
        PeelConfig cfg;
        cfg.eps = eps;
        cfg.seed = seed;
        cfg.norm_scale = norm_scale;
        PeelResult r = peel_construct(op, t->bt, cfg);
        *total_samples = r.stats.total;
        *o = new ora_h2{std::move(r.matrix)};
    });
}

// sample_block_column(DenseOperator(a), ct, t, s, count, mt19937_64(seed))
// (construction.hpp:137-148): omega_s |s| x count, y_t |t| x count
int ora_sample_block_column(ora_tree* t, const double* a, int symmetric, int tt, int ss, int64_t count, uint64_t seed,
                            double* omega_s, double* y_t) {
    return guard([&] {
        const Index n = t->ct->n();
        DenseOperator op(wrap(a, n, n), symmetric != 0);
        std::mt19937_64 rng(seed);
        auto [om, y] = sample_block_column(op, *t->ct, tt, ss, count, rng);
        out(om, omega_s);
        out(y, y_t);
    });
}

// adaptive_block_factorization(DenseOperator(a), ct, t, s, eps_block, cfg)
// (construction.hpp:156-198); u, v sized |t| x (|t| + b), |s| x (|t| + b) by
// the caller; *cols = columns the operator applied
int ora_adaptive_block_factorization(ora_tree* t, const double* a, int symmetric, int tt, int ss, double eps_block,
                                     int64_t b, int64_t p, int64_t max_rank, uint64_t seed, double* u, double* v,
                                     int64_t* rank, double* err_est, int64_t* cols) {
    return guard([&] {
        const Index n = t->ct->n();
        DenseOperator op(wrap(a, n, n), symmetric != 0);
        PeelConfig cfg;
        cfg.sample_block_size = b;
        cfg.oversampling = p;
        cfg.max_rank = max_rank;
        cfg.seed = seed;
        op.reset_counter();
        BlockFactor f = adaptive_block_factorization(op, *t->ct, tt, ss, eps_block, cfg);
        *rank = f.rank;
        *err_est = f.err_est;
        *cols = op.columns_applied();
        out(f.u, u);
        out(f.v, v);
    });
}

// local_low_rank_update(h, t, s, U, V, eps) (algebra.hpp:323-332); U |t| x k, V |s| x k
int ora_local_low_rank_update(ora_h2* h, int tt, int ss, int64_t k, const double* U, const double* V, double eps,
                              ora_h2** o) {
    return guard([&] {
        const auto& ct = *h->h.tree;
        *o = new ora_h2{local_low_rank_update(h->h, tt, ss, wrap(U, ct.node(tt).size(), k),
                                              wrap(V, ct.node(ss).size(), k), eps)};
    });
}

// H2Matrix::validate(ortho_cap) (h2_matrix.hpp:308-404): violation count,
// rank_profile (depth + 1 entries) and storage {dense, leaf, transfer, coupling}
int ora_validate(ora_h2* h, int64_t ortho_cap, int* num_violations, int64_t* level_max_rank, int64_t* storage) {
    return guard([&] {
        auto rep = h->h.validate(ortho_cap);
        *num_violations = int(rep.violations.size());
        for (size_t i = 0; i < rep.level_max_rank.size(); ++i) level_max_rank[i] = rep.level_max_rank[i];
        storage[0] = rep.storage.dense_reals;
        storage[1] = rep.storage.leaf_basis_reals;
        storage[2] = rep.storage.transfer_reals;
        storage[3] = rep.storage.coupling_reals;
    });
}

// pnorm_estimate(op, 2) of a dense operator (linear_operator.hpp:127-153)
int ora_pnorm2_dense(const double* a, int64_t n, int symmetric, double* v, int* iters) {
    return guard([&] {
        DenseOperator op(wrap(a, n, n), symmetric != 0);
        NormEstimate e = pnorm_estimate(op, 2);
        *v = e.value;
        *iters = e.iterations;
    });
}

// reference normal stream (fill_gaussian, construction.hpp:81-85): one
// fresh distribution over mt19937_64(seed), column-major r x c
int ora_gaussian(uint64_t seed, int64_t r, int64_t c, double* outp) {
    return guard([&] {
        std::mt19937_64 rng(seed);
        Matrix m(r, c);
        detail::fill_gaussian(m, rng);
        out(m, outp);
    });
}

// std::shuffle of 0..n-1 with std::mt19937_64(seed): the observation pick of
// AdvDiff2D::pick_observations (advdiff2d.hpp:112-124), with the same libstdc++
int ora_shuffle(int64_t n, uint64_t seed, int64_t* outp) {
    return guard([&] {
        std::vector<int64_t> v(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) v[size_t(i)] = i;
        std::mt19937_64 rng(seed);
        std::shuffle(v.begin(), v.end(), rng);
        std::memcpy(outp, v.data(), v.size() * sizeof(int64_t));
    });
}

#ifndef ORA_REFERENCE_HEADERS
// ---- diffusion1d Hessian at the target (oracle/diffusion1d.hpp) ----
struct ora_diff1d {
    h2ora::Diff1DOracle d;
};
int ora_diff1d_create(int64_t n, int64_t steps, double final_time, double t_p, double t_0, double amp,
                      double alpha, double beta, double pad, int nsrc, const double* src_pos, int64_t nrcv,
                      ora_diff1d** o) {
    return guard([&] {
        h2ora::Diff1DConfig c;
        c.n = n;
        c.steps = steps;
        c.final_time = final_time;
        c.t_p = t_p;
        c.t_0 = t_0;
        c.source_amplitude = amp;
        c.alpha = alpha;
        c.beta = beta;
        c.pad = pad;
        if (nsrc >= 0) c.source_positions.assign(src_pos, src_pos + nsrc);
        c.num_receivers = nrcv;
        *o = new ora_diff1d{h2ora::Diff1DOracle(c)};
    });
}
void ora_diff1d_destroy(ora_diff1d* d) { delete d; }
int ora_diff1d_info(ora_diff1d* d, int64_t* nstate, int64_t* npad, double* h, double* dt, int64_t* marches) {
    return guard([&] {
        *nstate = d->d.nstate();
        *npad = d->d.npad();
        *h = d->d.spacing();
        *dt = d->d.dt();
        *marches = d->d.pde_solves();
    });
}
int ora_diff1d_hessvec(ora_diff1d* d, int64_t b, const double* x, double* y, int include_tv, int nthreads) {
    return guard([&] { d->d.hessvec(b, x, y, include_tv != 0, nthreads); });
}
int ora_diff1d_state(ora_diff1d* d, int source, double* u) {
    return guard([&] {
        const auto& v = d->d.state(size_t(source));
        std::memcpy(u, v.data(), sizeof(double) * v.size());
    });
}

// peel_construct over the diffusion Hessian at the target (registry "diff1d-<n>"
// with hessian_operator(include_tv), diffusion1d.hpp:177-181); the operator
// applies run on `nthreads` host threads (columns are independent)
int ora_peel_diff1d(ora_tree* t, ora_diff1d* d, int include_tv, double eps, uint64_t seed, int nthreads, ora_h2** o,
                    int64_t* total_samples, double* op_seconds, int64_t* level_samples, int64_t* level_max_rank,
                    int* nlevels) {
    return guard([&] {
        const Index n = d->d.n();
        double op_s = 0;
        auto op = make_operator(n, true, [&](const Matrix& x) {
            Matrix y(n, x.cols());
            const auto t0 = std::chrono::steady_clock::now();
            d->d.hessvec(x.cols(), x.data(), y.data(), include_tv != 0, nthreads);
            op_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            return y;
        });
        PeelConfig cfg;
        cfg.eps = eps;
        cfg.seed = seed;
        PeelResult r = peel_construct(*op, t->bt, cfg);
        *total_samples = r.stats.total;
        *op_seconds = op_s;
        *nlevels = int(r.stats.levels.size());
        for (size_t i = 0; i < r.stats.levels.size(); ++i) {
            level_samples[i] = r.stats.levels[i].samples;
            level_max_rank[i] = r.stats.levels[i].max_rank;
        }
        *o = new ora_h2{std::move(r.matrix)};
    });
}

#endif  // ORA_REFERENCE_HEADERS

#ifdef ORA_REFERENCE_HEADERS
// The reference's own hierarchical inversion drivers (inversion.hpp:137-311),
// oracle/_ref only: h_newton_schulz (method 0) / h_hyperpower (1, arg = order)
// from X0 = scaled_identity_start(A) (:124-130) with a fixed (dynamic = 0) or
// dynamic threshold schedule. rows: (iter, residual, eps_k, samples, seconds)
// per rebuild, up to max_rows. Returns the divergence status in *converged
// (1 converged, 0 divergence_error) instead of throwing, keeping the trace.
int ora_h_inverse(ora_h2* a, int method, int arg, int dynamic, double eps_initial, double eps, uint64_t seed,
                  int max_iter, ora_h2** x_out, double* rows, int max_rows, int* num_rows, double* final_residual,
                  int* converged) {
    return guard([&] {
        H2Matrix x0 = scaled_identity_start(a->h);
        ThresholdSchedule sched;
        sched.mode = dynamic ? ThresholdSchedule::Mode::dynamic : ThresholdSchedule::Mode::fixed;
        sched.eps_initial = eps_initial;
        PeelConfig cfg;
        cfg.eps = eps;
        cfg.seed = seed;
        ConvergenceTrace tr;
        H2Matrix x;
        try {
            HInverseResult r = method == 0 ? h_newton_schulz(a->h, x0, sched, eps, cfg, max_iter)
                                           : h_hyperpower(a->h, x0, arg, sched, eps, cfg, max_iter);
            tr = std::move(r.trace);
            x = std::move(r.X);
            *converged = tr.converged ? 1 : 0;
        } catch (const divergence_error& e) {
            tr = e.trace;
            x = x0;
            *converged = 0;
        }
        *num_rows = int(tr.rows.size());
        for (int i = 0; i < *num_rows && i < max_rows; ++i) {
            rows[5 * i + 0] = tr.rows[size_t(i)].iter;
            rows[5 * i + 1] = tr.rows[size_t(i)].residual;
            rows[5 * i + 2] = tr.rows[size_t(i)].eps_k;
            rows[5 * i + 3] = double(tr.rows[size_t(i)].samples);
            rows[5 * i + 4] = tr.rows[size_t(i)].wall_seconds;
        }
        *final_residual = tr.final_residual;
        *x_out = new ora_h2{std::move(x)};
    });
}
int ora_residual_norm(ora_h2* a, ora_h2* x, double* out) {   // inversion.hpp:222-225
    return guard([&] { *out = residual_norm(a->h, x->h); });
}
#endif

}  // extern "C"

