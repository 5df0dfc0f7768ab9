// The reference's own test cases, restated against the B200 C++ host API
// (include/h2b200.hpp -> include/h2c.h -> libh2b200.so on the GPU). Reads like
// proj/tests/test_core.cpp / test_construction.cpp / test_operator.cpp.
#include <cmath>
#include <random>

#include <cuda_runtime.h>

#include "../../include/h2b200.hpp"
#include "mini_test.hpp"

using namespace h2;

namespace {

PointSet grid1d(Index n, double a, double b) {   // test_support.hpp:12-16
    std::vector<double> c(static_cast<size_t>(n));
    for (Index i = 0; i < n; ++i) c[size_t(i)] = a + (b - a) * double(i) / double(std::max<Index>(n - 1, 1));
    return PointSet(n, 1, c);
}

Matrix random_matrix(Index r, Index c, std::mt19937_64& rng) {   // test_support.hpp:28-34
    std::normal_distribution<double> g(0, 1);
    Matrix m(r, c);
    for (Index j = 0; j < c; ++j)
        for (Index i = 0; i < r; ++i) m(i, j) = g(rng);
    return m;
}

Matrix mul(const Matrix& a, const Matrix& b, bool tb = false) {
    const Index k = a.cols(), n = tb ? b.rows() : b.cols();
    Matrix c(a.rows(), n);
    for (Index j = 0; j < n; ++j)
        for (Index p = 0; p < k; ++p) {
            const double bv = tb ? b(j, p) : b(p, j);
            for (Index i = 0; i < a.rows(); ++i) c(i, j) += a(i, p) * bv;
        }
    return c;
}

double fro(const Matrix& a) {
    double s = 0;
    for (Index j = 0; j < a.cols(); ++j)
        for (Index i = 0; i < a.rows(); ++i) s += a(i, j) * a(i, j);
    return std::sqrt(s);
}

double rel_err(const Matrix& a, const Matrix& b) {
    Matrix d(a.rows(), a.cols());
    for (Index j = 0; j < a.cols(); ++j)
        for (Index i = 0; i < a.rows(); ++i) d(i, j) = a(i, j) - b(i, j);
    return fro(d) / fro(b);
}

std::shared_ptr<const BlockTree> tree1d(Index n, Index leaf, Admissibility mode) {
    auto ct = build_cluster_tree(grid1d(n, -1, 1), leaf);
    return build_block_tree(ct, ct, 1.0, mode);
}

}  // namespace

TEST_CASE("peel of the identity: zero couplings, identity dense leaves") {   // test_construction.cpp:112-124
    auto bt = tree1d(128, 16, Admissibility::weak);
    auto op = make_operator(128, true, [](const Matrix& x) { return x; });
    PeelConfig cfg;
    cfg.eps = 1e-8;
    auto r = peel_construct(op, bt, cfg);
    const Matrix id = Matrix::Identity(128, 128);
    CHECK(rel_err(r.matrix.matvec(id), id) < 1e-12);
    for (int k : r.matrix.row_ranks()) CHECK(k == 0);
    CHECK(r.stats.consistent());
    CHECK(r.stats.total == op.columns_applied());
    CHECK(r.stats.levels.back().samples == 16);
}

TEST_CASE("peel reconstructs a dense random SPD matrix to eps; hgemv matches A x") {   // :126-144
    std::mt19937_64 rng(55);
    Matrix g = random_matrix(64, 64, rng);
    Matrix a = mul(g, g, true);
    for (Index i = 0; i < 64; ++i) a(i, i) += 64.0;
    auto op = DenseOperator(a, true);
    auto bt = tree1d(64, 8, Admissibility::weak);
    PeelConfig tight;
    tight.eps = 1e-12;
    auto r = peel_construct(op, bt, tight);
    CHECK(r.matrix.symmetric());
    Matrix x = random_matrix(64, 5, rng);
    CHECK(rel_err(r.matrix.matvec(x), mul(a, x)) < 1e-11);
    CHECK(rel_err(r.matrix.matvec_transpose(x), mul(a, x)) < 1e-11);   // symmetric
    CHECK(estimate_relative_error(op, r.matrix) < 1e-11);
    // recompress at eps keeps the 2-norm contract (test_algebra.cpp:78-91, estimated)
    auto c = recompress(r.matrix, 1e-4);
    CHECK(estimate_relative_error(op, c) <= 3e-4);
}

TEST_CASE("operator contract: counter, transpose fallback, errors") {   // test_operator.cpp:10-30
    auto op = make_operator(16, false, [](const Matrix& x) { return x; });
    CHECK(op.columns_applied() == 0);
    CHECK(pnorm_estimate(make_operator(50, true, [](const Matrix& x) { return x; }), 2).value > 0.999999999999);
    auto bt = tree1d(16, 4, Admissibility::weak);
    CHECK_THROWS_AS(peel_construct(op, bt, PeelConfig{}), std::logic_error);   // no transpose, not symmetric
    auto z = H2Matrix::zero(bt, true);
    CHECK_THROWS_AS(z.matvec(Matrix(15, 2)), std::invalid_argument);           // h2_matrix.hpp:241-244
    CHECK_THROWS_AS(build_cluster_tree(grid1d(10, 0, 1), 1), std::invalid_argument);   // cluster_tree.hpp:33
}

TEST_CASE("max_rank_error is raised with the reference's exception type") {   // test_construction.cpp:100-110
    std::mt19937_64 rng(61);
    Matrix g = random_matrix(64, 64, rng);
    Matrix a(64, 64);
    for (Index j = 0; j < 64; ++j)
        for (Index i = 0; i < 64; ++i) a(i, j) = g(i, j) + g(j, i);
    auto bt = tree1d(64, 8, Admissibility::weak);
    PeelConfig cfg;
    cfg.eps = 1e-12;
    cfg.max_rank = 2;
    CHECK_THROWS_AS(peel_construct(DenseOperator(a, true), bt, cfg), max_rank_error);
}

TEST_CASE("sample_block_column hits exactly the requested block; rng advances like the reference's") {   // test_construction.cpp:39-59
    std::mt19937_64 rng(50), op_rng(51);
    auto ct = build_cluster_tree(grid1d(64, 0, 1), 8);
    Matrix d = random_matrix(64, 1, op_rng);
    Matrix dg(64, 64);
    for (Index i = 0; i < 64; ++i) dg(i, i) = d(i, 0);
    std::vector<int64_t> b(static_cast<size_t>(ct->num_nodes())), e(b.size());
    std::vector<int> lv(b.size()), par(b.size()), c0(b.size()), c1(b.size());
    detail::check(h2c_cluster_tree_nodes(ct->handle(), b.data(), e.data(), lv.data(), par.data(), c0.data(), c1.data(),
                                         nullptr, nullptr));
    const int t = c0[0], s = c1[0];
    auto y0 = sample_block_column(DenseOperator(dg, true), *ct, t, s, 4, rng).second;
    CHECK(fro(y0) == 0.0);
    // the reference's stream: omega = fill_gaussian over the same engine, which the call advanced
    std::mt19937_64 mirror(50);
    Matrix skip = random_matrix(e[size_t(s)] - b[size_t(s)], 4, mirror);   // what the first call consumed
    (void)skip;
    Matrix a = random_matrix(64, 64, op_rng);
    auto [omega, y] = sample_block_column(DenseOperator(a, false), *ct, t, s, 6, rng);
    Matrix expect_omega = random_matrix(e[size_t(s)] - b[size_t(s)], 6, mirror);
    CHECK(rel_err(omega, expect_omega) == 0.0);
    std::vector<int64_t> perm(64);
    detail::check(h2c_cluster_tree_perm(ct->handle(), perm.data()));
    Matrix blk(e[size_t(t)] - b[size_t(t)], e[size_t(s)] - b[size_t(s)]);
    for (Index i = 0; i < blk.rows(); ++i)
        for (Index j = 0; j < blk.cols(); ++j) blk(i, j) = a(perm[size_t(b[size_t(t)] + i)], perm[size_t(b[size_t(s)] + j)]);
    CHECK(rel_err(y, mul(blk, omega)) < 1e-12);
}

TEST_CASE("adaptive factorization: zero block in one increment, exact rank 3, max_rank") {   // test_construction.cpp:61-108
    std::mt19937_64 op_rng(52);
    auto ct = build_cluster_tree(grid1d(64, 0, 1), 8);
    std::vector<int64_t> b(static_cast<size_t>(ct->num_nodes())), e(b.size());
    std::vector<int> lv(b.size()), par(b.size()), c0(b.size()), c1(b.size());
    detail::check(h2c_cluster_tree_nodes(ct->handle(), b.data(), e.data(), lv.data(), par.data(), c0.data(), c1.data(),
                                         nullptr, nullptr));
    std::vector<int64_t> perm(64);
    detail::check(h2c_cluster_tree_perm(ct->handle(), perm.data()));
    const int t = c0[0], s = c1[0];
    Matrix d = random_matrix(64, 1, op_rng), dg(64, 64);
    for (Index i = 0; i < 64; ++i) dg(i, i) = d(i, 0);
    auto diag = DenseOperator(dg, true);
    PeelConfig cfg;
    diag.reset_counter();
    BlockFactor f0 = adaptive_block_factorization(diag, *ct, t, s, 1e-8, cfg);
    CHECK(f0.rank == 0);
    CHECK(diag.columns_applied() == cfg.sample_block_size);
    Matrix xf(64, 3), yf(64, 3);
    for (Index i = b[size_t(t)]; i < e[size_t(t)]; ++i) {
        Matrix r = random_matrix(1, 3, op_rng);
        for (Index j = 0; j < 3; ++j) xf(perm[size_t(i)], j) = r(0, j);
    }
    for (Index i = b[size_t(s)]; i < e[size_t(s)]; ++i) {
        Matrix r = random_matrix(1, 3, op_rng);
        for (Index j = 0; j < 3; ++j) yf(perm[size_t(i)], j) = r(0, j);
    }
    Matrix a = mul(xf, yf, true);
    auto op = DenseOperator(a, false);
    PeelConfig tight;
    tight.eps = 1e-12;
    op.reset_counter();
    BlockFactor f = adaptive_block_factorization(op, *ct, t, s, 1e-12, tight);
    CHECK(f.rank == 3);
    CHECK(op.columns_applied() <= 3 + tight.sample_block_size + 3);
    Matrix blk(e[size_t(t)] - b[size_t(t)], e[size_t(s)] - b[size_t(s)]);
    for (Index i = 0; i < blk.rows(); ++i)
        for (Index j = 0; j < blk.cols(); ++j) blk(i, j) = a(perm[size_t(b[size_t(t)] + i)], perm[size_t(b[size_t(s)] + j)]);
    CHECK(rel_err(mul(f.u, f.v, true), blk) < 1e-12);
    PeelConfig capped;
    capped.eps = 1e-10;
    capped.max_rank = 2;
    CHECK_THROWS_AS(adaptive_block_factorization(DenseOperator(random_matrix(64, 64, op_rng), false), *ct, t, s,
                                                 1e-10, capped),
                    max_rank_error);
}

TEST_CASE("to_dense, validate, frobenius_norm, low-rank updates") {   // h2_matrix.hpp:128-163, 308-404; algebra.hpp:119-137, 323-346
    std::mt19937_64 rng(57);
    Matrix g = random_matrix(96, 96, rng);
    Matrix a = mul(g, g, true);
    for (Index i = 0; i < 96; ++i) a(i, i) += 96.0;
    auto op = DenseOperator(a, true);
    auto bt = tree1d(96, 12, Admissibility::weak);
    PeelConfig tight;
    tight.eps = 1e-12;
    auto h = peel_construct(op, bt, tight).matrix;
    const Matrix dense = h.to_dense();
    CHECK(rel_err(dense, a) < 1e-11);
    CHECK_THROWS_AS(h.to_dense(50), std::invalid_argument);
    auto rep = h.validate();
    CHECK(rep.ok());
    CHECK(rep.level_max_rank.size() == 4u);   // 96 points, leaf 12: depth 3
    CHECK(rep.storage.total() > 0);
    CHECK(h.orthonormal());
    const double fn = frobenius_norm(h);
    CHECK(std::abs(fn - fro(a)) <= 1e-10 * fro(a));
    // global update A + x x^T keeps symmetric storage
    LowRankFactor f{random_matrix(96, 2, rng), Matrix()};
    f.Y = f.X;
    auto h2 = low_rank_update(h, f, 1e-12);
    CHECK(h2.symmetric());
    CHECK(rel_err(h2.to_dense(), [&] {
              Matrix r = a;
              Matrix xx = mul(f.X, f.X, true);
              for (Index j = 0; j < 96; ++j)
                  for (Index i = 0; i < 96; ++i) r(i, j) += xx(i, j);
              return r;
          }()) < 1e-10);
    // local update on the root's sibling pair (cluster order factors)
    std::vector<int64_t> b(static_cast<size_t>(bt->row_tree().num_nodes())), e(b.size());
    std::vector<int> lv(b.size()), par(b.size()), c0(b.size()), c1(b.size());
    detail::check(h2c_cluster_tree_nodes(bt->row_tree().handle(), b.data(), e.data(), lv.data(), par.data(), c0.data(),
                                         c1.data(), nullptr, nullptr));
    const int t = c0[0], s = c1[0];
    Matrix u = random_matrix(e[size_t(t)] - b[size_t(t)], 2, rng), v = random_matrix(e[size_t(s)] - b[size_t(s)], 2, rng);
    auto h3 = local_low_rank_update(h, t, s, u, v, 1e-12);
    const Matrix d3 = h3.to_dense();
    std::vector<int64_t> perm(96);
    detail::check(h2c_cluster_tree_perm(bt->row_tree().handle(), perm.data()));
    Matrix expect = a;
    const Matrix uv = mul(u, v, true);
    for (Index i = 0; i < uv.rows(); ++i)
        for (Index j = 0; j < uv.cols(); ++j) {
            expect(perm[size_t(b[size_t(t)] + i)], perm[size_t(b[size_t(s)] + j)]) += uv(i, j);
            expect(perm[size_t(b[size_t(s)] + j)], perm[size_t(b[size_t(t)] + i)]) += uv(i, j);   // symmetric mirror
        }
    CHECK(rel_err(d3, expect) < 1e-10);
}

MINI_MAIN

TEST_CASE("diffusion oracle: registry, symmetric PSD Hessian, two marches per source") {   // test_oracles.cpp:205-238, 321-331
    auto o = oracles::make_oracle("diff1d-64", {{"steps", "32"}, {"leaf", "16"}});
    CHECK(o.op->dim() == 64);
    CHECK(o.leaf == 16);
    CHECK(o.mode == Admissibility::weak);
    CHECK(o.diffusion->config().steps == 32);
    std::mt19937_64 rng(85);
    Matrix x = random_matrix(64, 1, rng), y = random_matrix(64, 1, rng);
    const Matrix hx = o.op->apply(x), hy = o.op->apply(y);
    double a = 0, b = 0, q = 0;
    for (Index i = 0; i < 64; ++i) {
        a += x(i, 0) * hy(i, 0);
        b += y(i, 0) * hx(i, 0);
        q += x(i, 0) * hx(i, 0);
    }
    CHECK(std::abs(a - b) <= 1e-10 * std::abs(b));
    CHECK(q >= 0.0);
    const long before = o.diffusion->pde_solves();
    o.op->apply(x);
    CHECK(o.diffusion->pde_solves() - before == 6);
    bool threw = false;
    try {
        oracles::make_oracle("nonsense");
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    CHECK(threw);
    auto ad = oracles::make_oracle("advdiff-16-k1e-2-obs50");   // test_oracles.cpp:333-336
    CHECK(ad.op->dim() == 256);
    CHECK(ad.advdiff->config().kappa == 1e-2);
    CHECK(ad.advdiff->config().num_observations == 50);
    const long s0 = ad.advdiff->solves();
    ad.op->apply(random_matrix(256, 2, rng));
    CHECK(ad.advdiff->solves() - s0 == 2);
    auto s = oracles::make_oracle("surface16");   // test_oracles.cpp:321-324
    CHECK(s.op->dim() == 256);
    CHECK(s.mode == Admissibility::strong);
    CHECK(s.leaf == 64);
    Matrix e = random_matrix(256, 2, rng);
    const Matrix se = s.op->apply(e);
    double sa = 0, sb = 0;
    for (Index i = 0; i < 256; ++i) {
        sa += e(i, 0) * se(i, 1);
        sb += e(i, 1) * se(i, 0);
    }
    CHECK(std::abs(sa - sb) <= 1e-12 * std::abs(sb));
    // HARA on the device operator (the cfg3 pipeline at desk scale)
    auto res = peel_construct(*o.op, o.default_block_tree(), PeelConfig{1e-6});
    CHECK(estimate_relative_error(*o.op, res.matrix) <= 3e-6);
}

TEST_CASE("sharded hgemv through the C++ mirror: collective buffers and peer transport") {
    // two ranks held by this process on one GPU: the collective exchange is done by
    // device copies in rank order; the peer transport links the plans directly and
    // enqueues both begins before either end (nothing waits on work that has not run)
    std::mt19937_64 rng(77);
    const Index n = 256, b = 3;
    Matrix g = random_matrix(n, n, rng);
    Matrix a = mul(g, g, true);
    for (Index i = 0; i < n; ++i) a(i, i) += double(n);
    auto op = DenseOperator(a, true);
    PeelConfig tight;
    tight.eps = 1e-10;
    auto h = peel_construct(op, tree1d(n, 16, Admissibility::weak), tight).matrix;
    Matrix x = random_matrix(n, b, rng);
    const Matrix y_ref = h.matvec(x);
    double *dx = nullptr, *dy = nullptr;
    CHECK(cudaMalloc(reinterpret_cast<void**>(&dx), sizeof(double) * n * b) == cudaSuccess);
    CHECK(cudaMalloc(reinterpret_cast<void**>(&dy), sizeof(double) * n * b) == cudaSuccess);
    cudaMemcpy(dx, x.data(), sizeof(double) * n * b, cudaMemcpyHostToDevice);
    std::vector<ShardedPlan> plans{ShardedPlan(h, 2, 0), ShardedPlan(h, 2, 1)};
    CHECK(plans[0].owned_rows() + plans[1].owned_rows() == n);
    // collective layout: rank r receives, in source order, what each q sends to r
    std::vector<double*> send(2), recv(2);
    for (int r = 0; r < 2; ++r) {
        int64_t ns = 0, nr = 0;
        for (int q = 0; q < 2; ++q) {
            ns += plans[size_t(r)].send_rows()[size_t(q)];
            nr += plans[size_t(r)].recv_rows()[size_t(q)];
        }
        cudaMalloc(reinterpret_cast<void**>(&send[size_t(r)]), sizeof(double) * std::max<int64_t>(ns * b, 1));
        cudaMalloc(reinterpret_cast<void**>(&recv[size_t(r)]), sizeof(double) * std::max<int64_t>(nr * b, 1));
    }
    for (int r = 0; r < 2; ++r) plans[size_t(r)].begin(b, dx, n, send[size_t(r)]);
    for (int r = 0; r < 2; ++r) {
        int64_t at = 0;
        for (int q = 0; q < 2; ++q) {
            int64_t off = 0;
            for (int s = 0; s < r; ++s) off += plans[size_t(q)].send_rows()[size_t(s)];
            const int64_t rows = plans[size_t(q)].send_rows()[size_t(r)];
            CHECK(rows == plans[size_t(r)].recv_rows()[size_t(q)]);
            cudaMemcpy(recv[size_t(r)] + at * b, send[size_t(q)] + off * b, sizeof(double) * rows * b,
                       cudaMemcpyDeviceToDevice);
            at += rows;
        }
        plans[size_t(r)].end(b, recv[size_t(r)], dy, n);
    }
    Matrix y(n, b);
    cudaMemcpy(y.data(), dy, sizeof(double) * n * b, cudaMemcpyDeviceToHost);
    CHECK(rel_err(y, y_ref) < 1e-12);
    // peer transport, twice (epochs and acknowledgements): bitwise the collective result
    for (ShardedPlan& p : plans) p.peer_alloc(4);
    ShardedPlan::peer_link({&plans[0], &plans[1]});
    for (int call = 0; call < 2; ++call) {
        cudaMemset(dy, 0, sizeof(double) * n * b);
        for (ShardedPlan& p : plans) {
            p.begin(b, dx, n, nullptr);
            p.local(b);
        }
        for (ShardedPlan& p : plans) p.end(b, nullptr, dy, n);
        Matrix yp(n, b);
        cudaMemcpy(yp.data(), dy, sizeof(double) * n * b, cudaMemcpyDeviceToHost);
        CHECK(rel_err(yp, y) == 0.0);
    }
    for (double* p : send) cudaFree(p);
    for (double* p : recv) cudaFree(p);
    cudaFree(dx);
    cudaFree(dy);
}
