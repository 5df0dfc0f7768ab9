// The reference's own test cases, restated against the B200 C++ host API
// (include/h2b200.hpp -> include/h2c.h -> libh2b200.so on the GPU). Reads like
// proj/tests/test_core.cpp / test_construction.cpp / test_operator.cpp.
#include <cmath>
#include <random>

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
