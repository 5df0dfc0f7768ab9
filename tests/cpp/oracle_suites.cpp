// The reference's doctest suites (proj/tests/test_{geometry,core,algebra,
// operator,construction}.cpp) restated against the CPU oracle. Passing them is
// what pins the oracle to the reference's behaviour: the
// reference publishes no golden vectors, only these property / known-answer
// tests, and its fixtures (random_h2, random_matrix) draw from the same
// libstdc++ mt19937_64 stream, so the inputs here are the reference's inputs.
#include "../../oracle/test_support.hpp"
#include "mini_test.hpp"

using namespace h2;
using namespace h2::testing;

namespace {
std::shared_ptr<const BlockTree> tree1d(Index n, Index leaf, Admissibility mode) {
    auto ct = build_cluster_tree(grid1d(n, -1, 1), leaf);
    return build_block_tree(ct, ct, 1.0, mode);
}
std::shared_ptr<const BlockTree> tree2d(Index g, Index leaf) {
    auto ct = build_cluster_tree(grid2d(g, g), leaf);
    return build_block_tree(ct, ct, 1.0, Admissibility::strong);
}
Matrix diag_of(const Matrix& d) {
    Matrix m(d.rows(), d.rows());
    for (Index i = 0; i < d.rows(); ++i) m(i, i) = d[i];
    return m;
}
Matrix gather_block(const ClusterTree& ct, const Matrix& a, int t, int s) {
    const auto& tn = ct.node(t);
    const auto& sn = ct.node(s);
    Matrix blk(tn.size(), sn.size());
    for (Index i = 0; i < tn.size(); ++i)
        for (Index j = 0; j < sn.size(); ++j) blk(i, j) = a(ct.perm()[size_t(tn.begin + i)], ct.perm()[size_t(sn.begin + j)]);
    return blk;
}
bool same_payload(const H2Matrix& a, const H2Matrix& b) {
    if (a.symmetric != b.symmetric || a.coupling.size() != b.coupling.size()) return false;
    for (size_t i = 0; i < a.coupling.size(); ++i)
        if (!a.coupling[i].bitwise_equal(b.coupling[i])) return false;
    for (size_t i = 0; i < a.dense.size(); ++i)
        if (!a.dense[i].bitwise_equal(b.dense[i])) return false;
    for (int v = 0; v < a.tree->num_nodes(); ++v) {
        if (a.row_basis.rank(v) != b.row_basis.rank(v)) return false;
        if (a.tree->node(v).is_leaf() && !a.row_basis.leaf_basis(v).bitwise_equal(b.row_basis.leaf_basis(v))) return false;
        if (v != 0 && !a.row_basis.transfer(v).bitwise_equal(b.row_basis.transfer(v))) return false;
    }
    return true;
}
}  // namespace

// ---------------- test_geometry.cpp ----------------
TEST_CASE("geometry: median split on a sorted line") {
    Matrix c(4, 1);
    for (int i = 0; i < 4; ++i) c(i, 0) = i;
    ClusterTree ct(PointSet(c), 2);
    const auto& root = ct.node(ct.root());
    REQUIRE(!root.is_leaf());
    CHECK(root.begin == 0);
    CHECK(root.end == 4);
    CHECK(ct.node(root.child[0]).end == 2);
    CHECK(ct.node(root.child[1]).begin == 2);
}
TEST_CASE("geometry: empty point set is rejected") { CHECK_THROWS(PointSet{Matrix(0, 1)}); }
TEST_CASE("geometry: 1d grid n=2048 leaf 32 gives 6 levels, 2^l weak blocks per level") {
    auto ct = build_cluster_tree(grid1d(2048, -1, 1), 32);
    CHECK(ct->depth() == 6);
    for (int v : ct->leaves()) CHECK(ct->node(v).size() <= 32);
    auto bt = build_block_tree(ct, ct, 1.0, Admissibility::weak);
    std::vector<int> count(size_t(bt->max_level() + 1), 0);
    for (int b : bt->admissible_leaves()) count[size_t(bt->node(b).level)]++;
    for (int l = 1; l <= 6; ++l) CHECK(count[size_t(l)] == (1 << l));
}
TEST_CASE("geometry: children partition the parent's range; depth near log2(n/leaf)") {
    std::mt19937_64 rng(7);
    Matrix c = random_matrix(333, 2, rng);
    ClusterTree ct(PointSet(c), 16);
    for (int v = 0; v < ct.num_nodes(); ++v) {
        const auto& nd = ct.node(v);
        if (nd.is_leaf()) continue;
        CHECK(ct.node(nd.child[0]).begin == nd.begin);
        CHECK(ct.node(nd.child[0]).end == ct.node(nd.child[1]).begin);
        CHECK(ct.node(nd.child[1]).end == nd.end);
    }
    CHECK(ct.depth() >= 5);
    CHECK(ct.depth() <= 6);
}
TEST_CASE("geometry: n = leaf_size gives a single dense leaf") {
    auto ct = build_cluster_tree(grid1d(32), 32);
    auto bt = build_block_tree(ct, ct, 1.0, Admissibility::strong);
    CHECK(bt->admissible_leaves().empty());
    REQUIRE(bt->dense_leaves().size() == 1);
}
TEST_CASE("geometry: strong block tree tiles the square exactly (2d 32x32)") {
    auto ct = build_cluster_tree(grid2d(32, 32), 64);
    auto bt = build_block_tree(ct, ct, 1.0, Admissibility::strong);
    Index area = 0;
    for (int b : bt->admissible_leaves()) area += ct->node(bt->node(b).row).size() * ct->node(bt->node(b).col).size();
    for (int b : bt->dense_leaves()) area += ct->node(bt->node(b).row).size() * ct->node(bt->node(b).col).size();
    CHECK(area == Index(1024) * 1024);
}
TEST_CASE("geometry: permutation round trip is the identity") {
    std::mt19937_64 rng(11);
    Matrix pts = random_matrix(257, 3, rng);
    ClusterTree ct(PointSet(pts), 10);
    Matrix x = random_matrix(257, 4, rng);
    CHECK((ct.to_user(ct.to_internal(x)) - x).norm() == 0.0);
    CHECK((ct.to_internal(ct.to_user(x)) - x).norm() == 0.0);
}

// ---------------- test_core.cpp ----------------
TEST_CASE("core: zero and diagonal factories expand exactly") {
    auto bt = tree1d(64, 8, Admissibility::weak);
    H2Matrix z = H2Matrix::zero(bt, true);
    CHECK(z.to_dense().norm() == 0.0);
    std::mt19937_64 rng(1);
    Matrix d = random_matrix(64, 1, rng);
    H2Matrix dm = H2Matrix::diagonal(bt, d);
    CHECK((dm.to_dense() - diag_of(d)).norm() == 0.0);
    H2Matrix id = H2Matrix::scaled_identity(bt, 0.5);
    Matrix x = random_matrix(64, 3, rng);
    CHECK(rel_err(id.matvec(x), 0.5 * x) < 1e-15);
}
TEST_CASE("core: matvec agrees with the dense expansion") {
    std::mt19937_64 rng(2);
    for (bool sym : {true, false})
        for (auto bt : {tree1d(96, 8, Admissibility::weak), tree1d(70, 6, Admissibility::strong), tree2d(12, 16)}) {
            H2Matrix h = random_h2(bt, sym, 4, rng);
            Matrix a = h.to_dense();
            Matrix x = random_matrix(h.n(), 5, rng);
            CHECK(rel_err(h.matvec(x), a * x) < 1e-12);
            CHECK(rel_err(h.matvec_transpose(x), gemm(a, true, x, false)) < 1e-12);
            if (sym) CHECK((a - a.transpose()).norm() < 1e-13 * a.norm());
        }
}
TEST_CASE("core: matvec is linear") {
    std::mt19937_64 rng(3);
    auto bt = tree1d(128, 16, Admissibility::weak);
    H2Matrix h = random_h2(bt, true, 5, rng);
    Matrix x = random_matrix(128, 2, rng), z = random_matrix(128, 2, rng);
    const double al = 0.37, be = -1.25;
    CHECK(rel_err(h.matvec(al * x + be * z), al * h.matvec(x) + be * h.matvec(z)) < 1e-12);
}
TEST_CASE("core: symmetric matvec satisfies x'(Hy) = y'(Hx)") {
    std::mt19937_64 rng(4);
    auto bt = tree2d(10, 8);
    H2Matrix h = random_h2(bt, true, 4, rng);
    Matrix x = random_matrix(h.n(), 1, rng), y = random_matrix(h.n(), 1, rng);
    const double a = gemm(x, true, h.matvec(y), false)(0, 0), b = gemm(y, true, h.matvec(x), false)(0, 0);
    CHECK(std::abs(a - b) < 1e-12 * std::abs(a));
}
TEST_CASE("core: vector block ordering tags") {
    std::mt19937_64 rng(5);
    auto bt = tree1d(32, 4, Admissibility::weak);
    H2Matrix h = random_h2(bt, true, 3, rng);
    Matrix x = random_matrix(32, 2, rng);
    VectorBlock u{x, Ordering::user};
    VectorBlock i{h.tree->to_internal(x), Ordering::internal};
    CHECK(rel_err(h.matvec(u).data, h.tree->to_user(h.matvec(i).data)) < 1e-15);
}
TEST_CASE("core: to_dense rejects matrices above the cap") {
    auto bt = tree1d(128, 16, Admissibility::weak);
    H2Matrix h = H2Matrix::zero(bt, true);
    CHECK_THROWS_AS(h.to_dense(64), std::invalid_argument);
}
TEST_CASE("core: validate: fresh instance is clean, corrupted coupling is flagged") {
    std::mt19937_64 rng(6);
    auto bt = tree1d(64, 8, Admissibility::weak);
    H2Matrix h = random_h2(bt, true, 4, rng);
    CHECK(h.validate().ok());
    for (auto& s : h.coupling)
        if (s.size() > 0) {
            s = Matrix(s.rows() + 1, s.cols());
            break;
        }
    ValidationReport bad = h.validate();
    CHECK_FALSE(bad.ok());
    bool found = false;
    for (const auto& v : bad.violations) found |= v.find("coupling dimension") != std::string::npos;
    CHECK(found);
}
TEST_CASE("core: desymmetrized matrix represents the same operator") {
    std::mt19937_64 rng(8);
    auto bt = tree2d(8, 8);
    H2Matrix h = random_h2(bt, true, 3, rng);
    H2Matrix g = h.desymmetrized();
    CHECK_FALSE(g.symmetric);
    CHECK(rel_err(g.to_dense(), h.to_dense()) < 1e-14);
    Matrix x = random_matrix(h.n(), 3, rng);
    CHECK(rel_err(g.matvec(x), h.matvec(x)) < 1e-13);
}

// ---------------- test_algebra.cpp ----------------
TEST_CASE("algebra: orthogonalize preserves the operator and yields orthonormal bases") {
    std::mt19937_64 rng(21);
    for (bool sym : {true, false}) {
        auto bt = tree1d(96, 8, Admissibility::weak);
        H2Matrix h = random_h2(bt, sym, 4, rng);
        Matrix a = h.to_dense();
        H2Matrix g = orthogonalize(h);
        CHECK(g.orthonormal);
        CHECK(rel_err(g.to_dense(), a) < 1e-12);
        Matrix x = random_matrix(h.n(), 4, rng);
        CHECK(rel_err(g.matvec(x), h.matvec(x)) < 1e-12);
        for (int v = 0; v < g.tree->num_nodes(); ++v) {
            Matrix u = g.row_basis.reconstruct(*g.tree, v);
            if (u.cols() == 0) continue;
            CHECK((gemm(u, true, u, false) - Matrix::Identity(u.cols(), u.cols())).norm() < 1e-12);
        }
        CHECK(g.validate().ok());
    }
}
TEST_CASE("algebra: orthogonalize is idempotent up to floating point") {
    std::mt19937_64 rng(22);
    auto bt = tree2d(8, 8);
    H2Matrix g = orthogonalize(random_h2(bt, true, 3, rng));
    H2Matrix g2 = orthogonalize(g);
    Matrix x = random_matrix(g.n(), 3, rng);
    CHECK(rel_err(g2.matvec(x), g.matvec(x)) < 1e-14);
}
TEST_CASE("algebra: frobenius norm exact against the dense expansion") {
    std::mt19937_64 rng(23);
    auto bt = tree1d(80, 8, Admissibility::strong);
    H2Matrix h = random_h2(bt, true, 4, rng);
    CHECK_THROWS_AS(frobenius_norm(h), std::invalid_argument);
    H2Matrix g = orthogonalize(h);
    CHECK(frobenius_norm(g) == mini::Approx(g.to_dense().norm()).epsilon(1e-10));
    CHECK(frobenius_norm(H2Matrix::zero(bt, true)) == 0.0);
}
TEST_CASE("algebra: recompress with eps=0 leaves the operator unchanged") {
    std::mt19937_64 rng(24);
    auto bt = tree1d(96, 8, Admissibility::weak);
    H2Matrix h = random_h2(bt, true, 4, rng);
    H2Matrix g = recompress(h, 0.0);
    Matrix x = random_matrix(h.n(), 3, rng);
    CHECK(rel_err(g.matvec(x), h.matvec(x)) < 1e-12);
    for (int v = 0; v < h.tree->num_nodes(); ++v) CHECK(g.row_basis.rank(v) <= h.row_basis.rank(v));
}
TEST_CASE("algebra: recompress meets the 2-norm contract with 3x slack") {
    std::mt19937_64 rng(25);
    for (auto bt : {tree1d(96, 8, Admissibility::weak), tree2d(10, 8)}) {
        H2Matrix h = random_h2(bt, true, 6, rng);
        Matrix a = h.to_dense();
        const double na = dense_2norm(a);
        for (double eps : {1e-2, 1e-5}) {
            H2Matrix g = recompress(h, eps);
            CHECK(dense_2norm(g.to_dense() - a) <= 3 * eps * na);
            CHECK(g.validate().ok());
        }
    }
}
TEST_CASE("algebra: recompress is idempotent in the ranks") {
    std::mt19937_64 rng(26);
    auto bt = tree1d(128, 16, Admissibility::weak);
    H2Matrix h = random_h2(bt, true, 8, rng);
    H2Matrix g1 = recompress(h, 1e-4);
    H2Matrix g2 = recompress(g1, 1e-4);
    for (int v = 0; v < h.tree->num_nodes(); ++v) CHECK(g2.row_basis.rank(v) == g1.row_basis.rank(v));
}
TEST_CASE("algebra: global low-rank update exact at eps = 0") {
    std::mt19937_64 rng(27);
    for (bool sym : {true, false}) {
        auto bt = tree1d(64, 8, Admissibility::weak);
        H2Matrix h = random_h2(bt, sym, 3, rng);
        Matrix a = h.to_dense();
        LowRankFactor f{random_matrix(64, 2, rng), random_matrix(64, 2, rng)};
        H2Matrix g = low_rank_update(h, f, 0.0);
        CHECK(rel_err(g.to_dense(), a + gemm(f.X, false, f.Y, true)) < 1e-12);
        CHECK(g.validate().ok());
    }
}
TEST_CASE("algebra: global low-rank update with truncation meets its tolerance") {
    std::mt19937_64 rng(28);
    auto bt = tree2d(8, 8);
    H2Matrix h = random_h2(bt, true, 4, rng);
    Matrix a = h.to_dense();
    LowRankFactor f{random_matrix(h.n(), 1, rng), random_matrix(h.n(), 1, rng)};
    Matrix target = a + gemm(f.X, false, f.Y, true);
    H2Matrix g = low_rank_update(h, f, 1e-6);
    CHECK(dense_2norm(g.to_dense() - target) <= 3e-6 * dense_2norm(target));
}
TEST_CASE("algebra: update with zero-rank factors returns the input unchanged") {
    std::mt19937_64 rng(29);
    auto bt = tree1d(32, 4, Admissibility::weak);
    H2Matrix h = orthogonalize(random_h2(bt, true, 3, rng));
    const double before = frobenius_norm(h);
    H2Matrix g = low_rank_update(h, LowRankFactor{Matrix(32, 0), Matrix(32, 0)}, 1e-8);
    CHECK(frobenius_norm(g) == before);
}
TEST_CASE("algebra: symmetric update keeps the flag; asymmetric update drops it") {
    std::mt19937_64 rng(31);
    auto bt = tree1d(64, 8, Admissibility::weak);
    H2Matrix h = random_h2(bt, true, 3, rng);
    Matrix b = random_matrix(64, 2, rng);
    H2Matrix gs = low_rank_update(h, LowRankFactor{b, b}, 1e-10);
    CHECK(gs.symmetric);
    CHECK(rel_err(gs.to_dense(), h.to_dense() + gemm(b, false, b, true)) < 1e-9);
    H2Matrix ga = low_rank_update(h, LowRankFactor{b, random_matrix(64, 2, rng)}, 1e-10);
    CHECK_FALSE(ga.symmetric);
}
TEST_CASE("algebra: local update zero outside the block, equivalent to padded global update") {
    std::mt19937_64 rng(33);
    auto ct = build_cluster_tree(grid1d(64, -1, 1), 8);
    auto bt = build_block_tree(ct, ct, 1.0, Admissibility::weak);
    H2Matrix h = random_h2(bt, true, 3, rng);
    Matrix a = h.to_dense();
    const int t = ct->node(0).child[0], s = ct->node(0).child[1];
    Matrix ub = random_matrix(ct->node(t).size(), 2, rng), vb = random_matrix(ct->node(s).size(), 2, rng);
    H2Matrix g = local_low_rank_update(h, t, s, ub, vb, 0.0);
    Matrix xf(64, 2), yf(64, 2);
    for (Index i = 0; i < ct->node(t).size(); ++i)
        for (int j = 0; j < 2; ++j) xf(ct->perm()[size_t(ct->node(t).begin + i)], j) = ub(i, j);
    for (Index i = 0; i < ct->node(s).size(); ++i)
        for (int j = 0; j < 2; ++j) yf(ct->perm()[size_t(ct->node(s).begin + i)], j) = vb(i, j);
    Matrix target = a + gemm(xf, false, yf, true) + gemm(yf, false, xf, true);
    CHECK(rel_err(g.to_dense(), target) < 1e-12);
    H2Matrix g2 = local_low_rank_update(h, t, s, ub, Matrix(ct->node(s).size(), 2), 0.0);
    CHECK((g2.to_dense() - a).norm() < 1e-12);
    H2Matrix hd = h.desymmetrized();
    H2Matrix gl = local_low_rank_update(hd, t, s, ub, vb, 0.0);
    H2Matrix gg = low_rank_update(hd, LowRankFactor{xf, yf}, 0.0);
    CHECK(rel_err(gl.to_dense(), gg.to_dense()) < 1e-12);
}
TEST_CASE("algebra: frobenius dominates the spectral norm") {
    std::mt19937_64 rng(34);
    auto bt = tree1d(96, 8, Admissibility::weak);
    H2Matrix g = orthogonalize(random_h2(bt, true, 4, rng));
    CHECK(frobenius_norm(g) >= dense_2norm(g.to_dense()) * (1 - 1e-12));
}

// ---------------- test_operator.cpp ----------------
TEST_CASE("operator: counter increases by the number of columns") {
    auto op = make_operator(10, true, [](const Matrix& x) { return 2.0 * x; });
    CHECK(op->columns_applied() == 0);
    op->apply(Matrix::Constant(10, 3, 1.0));
    CHECK(op->columns_applied() == 3);
    op->apply(Matrix::Constant(10, 5, 1.0));
    CHECK(op->columns_applied() == 8);
    op->reset_counter();
    CHECK(op->columns_applied() == 0);
}
TEST_CASE("operator: symmetric operators default apply_transpose to apply") {
    Matrix a(3, 3);
    const double v[9] = {1, 2, 0, 2, 5, 1, 0, 1, 3};
    for (int i = 0; i < 9; ++i) a[i] = v[i];
    auto op = make_operator(3, true, [a](const Matrix& x) { return a * x; });
    CHECK((op->apply_transpose(Matrix::Identity(3, 3)) - a).norm() == 0.0);
    auto asym = make_operator(3, false, [a](const Matrix& x) { return a * x; });
    CHECK_THROWS_AS(asym->apply_transpose(Matrix::Identity(3, 3)), std::logic_error);
}
TEST_CASE("operator: pnorm estimate on identity and known spectra") {
    auto id = make_operator(50, true, [](const Matrix& x) { return x; });
    NormEstimate e2 = pnorm_estimate(*id, 2);
    CHECK(e2.value == mini::Approx(1.0).epsilon(1e-12));
    CHECK(e2.iterations >= 1);
    Matrix d(10, 1);
    for (int i = 0; i < 10; ++i) d[i] = i + 1;
    DenseOperator diag{diag_of(d), true};
    CHECK(pnorm_estimate(diag, 2).value == mini::Approx(10.0).epsilon(5e-3));
    CHECK(pnorm_estimate(diag, std::numeric_limits<double>::infinity()).value == mini::Approx(10.0));
    CHECK(pnorm_estimate(diag, 1).value == mini::Approx(10.0));
}
TEST_CASE("operator: pnorm estimate of a non-symmetric dense operator") {
    std::mt19937_64 rng(40);
    Matrix a = random_matrix(40, 40, rng);
    DenseOperator op(a);
    const double exact = dense_2norm(a);
    NormEstimate est = pnorm_estimate(op, 2);
    CHECK(est.value <= exact * (1 + 1e-10));
    CHECK(est.value >= exact * 0.9);
}
TEST_CASE("operator: h2 operator adapter matches the matrix") {
    std::mt19937_64 rng(41);
    auto ct = build_cluster_tree(grid1d(64), 8);
    auto bt = build_block_tree(ct, ct, 1.0, Admissibility::weak);
    H2Matrix h = random_h2(bt, true, 3, rng);
    H2Operator op(h);
    Matrix x = random_matrix(64, 2, rng);
    CHECK(rel_err(op.apply(x), h.matvec(x)) == 0.0);
    CHECK(op.columns_applied() == 2);
}

// ---------------- test_construction.cpp ----------------
TEST_CASE("construction: sample_block_column hits exactly the requested block") {
    std::mt19937_64 rng(50), op_rng(51);
    auto ct = build_cluster_tree(grid1d(64), 8);
    Matrix d = random_matrix(64, 1, op_rng);
    DenseOperator diag{diag_of(d), true};
    const int t = ct->node(0).child[0], s = ct->node(0).child[1];
    auto r0 = sample_block_column(diag, *ct, t, s, 4, rng);
    CHECK(r0.second.norm() == 0.0);
    Matrix a = random_matrix(64, 64, op_rng);
    DenseOperator op(a);
    auto r1 = sample_block_column(op, *ct, t, s, 6, rng);
    CHECK(rel_err(r1.second, gather_block(*ct, a, t, s) * r1.first) < 1e-12);
}
TEST_CASE("construction: zero block converges after one increment") {
    std::mt19937_64 op_rng(52);
    auto ct = build_cluster_tree(grid1d(64), 8);
    Matrix d = random_matrix(64, 1, op_rng);
    DenseOperator diag{diag_of(d), true};
    const int t = ct->node(0).child[0], s = ct->node(0).child[1];
    PeelConfig cfg;
    BlockFactor f = adaptive_block_factorization(diag, *ct, t, s, 1e-8, cfg);
    CHECK(f.rank == 0);
    CHECK(diag.columns_applied() == cfg.sample_block_size);
}
TEST_CASE("construction: exact rank-3 block within 3+b samples") {
    std::mt19937_64 op_rng(53);
    auto ct = build_cluster_tree(grid1d(64), 8);
    const int t = ct->node(0).child[0], s = ct->node(0).child[1];
    Matrix xf(64, 3), yf(64, 3);
    for (Index i = 0; i < ct->node(t).size(); ++i) {
        Matrix r = random_matrix(1, 3, op_rng);
        for (int j = 0; j < 3; ++j) xf(ct->perm()[size_t(ct->node(t).begin + i)], j) = r[j];
    }
    for (Index i = 0; i < ct->node(s).size(); ++i) {
        Matrix r = random_matrix(1, 3, op_rng);
        for (int j = 0; j < 3; ++j) yf(ct->perm()[size_t(ct->node(s).begin + i)], j) = r[j];
    }
    Matrix a = gemm(xf, false, yf, true);
    DenseOperator op(a);
    PeelConfig cfg;
    cfg.eps = 1e-12;
    BlockFactor f = adaptive_block_factorization(op, *ct, t, s, 1e-12, cfg);
    CHECK(f.rank == 3);
    CHECK(op.columns_applied() <= 3 + cfg.sample_block_size + 3);
    Matrix blk = gather_block(*ct, a, t, s);
    CHECK(dense_2norm(blk - gemm(f.u, false, f.v, true)) < 1e-12 * dense_2norm(blk));
}
TEST_CASE("construction: max_rank exhaustion throws") {
    std::mt19937_64 op_rng(54);
    auto ct = build_cluster_tree(grid1d(64), 8);
    const int t = ct->node(0).child[0], s = ct->node(0).child[1];
    DenseOperator op(random_matrix(64, 64, op_rng));
    PeelConfig cfg;
    cfg.eps = 1e-10;
    cfg.max_rank = 2;
    CHECK_THROWS_AS(adaptive_block_factorization(op, *ct, t, s, 1e-10, cfg), max_rank_error);
}
TEST_CASE("construction: peel of the identity") {
    auto bt = tree1d(128, 16, Admissibility::weak);
    auto op = make_operator(128, true, [](const Matrix& x) { return x; });
    PeelConfig cfg;
    cfg.eps = 1e-8;
    PeelResult r = peel_construct(*op, bt, cfg);
    CHECK(rel_err(r.matrix.to_dense(), Matrix::Identity(128, 128)) < 1e-12);
    for (int v = 0; v < r.matrix.tree->num_nodes(); ++v) CHECK(r.matrix.row_basis.rank(v) == 0);
    CHECK(r.stats.consistent());
    CHECK(r.stats.total == op->columns_applied());
    CHECK(r.stats.levels.back().samples == 16);
}
TEST_CASE("construction: peel reconstructs a dense random SPD matrix to eps") {
    std::mt19937_64 op_rng(55);
    Matrix g = random_matrix(64, 64, op_rng);
    Matrix a = gemm(g, false, g, true) + 64.0 * Matrix::Identity(64, 64);
    DenseOperator op(a, true);
    auto bt = tree1d(64, 8, Admissibility::weak);
    PeelConfig cfg;
    cfg.eps = 1e-6;
    PeelResult r = peel_construct(op, bt, cfg);
    CHECK(dense_2norm(r.matrix.to_dense() - a) <= 1e-6 * dense_2norm(a));
    CHECK(r.matrix.symmetric);
    CHECK(r.matrix.validate().ok());
    PeelConfig tight;
    tight.eps = 1e-12;
    PeelResult r2 = peel_construct(op, bt, tight);
    CHECK(rel_err(r2.matrix.to_dense(), a) < 1e-11);
}
TEST_CASE("construction: rank-5-plus-noise keeps local ranks at 5") {
    std::mt19937_64 op_rng(56);
    Matrix b5 = random_matrix(256, 5, op_rng);
    Matrix noise = random_matrix(256, 256, op_rng);
    Matrix a = gemm(b5, false, b5, true) + 1e-8 * (noise + noise.transpose());
    DenseOperator op(a, true);
    auto bt = tree1d(256, 32, Admissibility::weak);
    PeelConfig cfg;
    cfg.eps = 1e-6;
    PeelResult r = peel_construct(op, bt, cfg);
    for (Index k : r.matrix.rank_profile()) CHECK(k <= 5);
    CHECK(dense_2norm(r.matrix.to_dense() - a) <= 3e-6 * dense_2norm(a));
}
TEST_CASE("construction: peel is deterministic for a fixed seed") {
    std::mt19937_64 op_rng(57);
    Matrix g = random_matrix(96, 96, op_rng);
    Matrix a = gemm(g, false, g, true);
    auto bt = tree1d(96, 12, Admissibility::weak);
    PeelConfig cfg;
    cfg.eps = 1e-5;
    cfg.seed = 1234;
    DenseOperator op1(a, true), op2(a, true);
    PeelResult r1 = peel_construct(op1, bt, cfg), r2 = peel_construct(op2, bt, cfg);
    CHECK(same_payload(r1.matrix, r2.matrix));
    CHECK(r1.stats.total == r2.stats.total);
}
TEST_CASE("construction: nonsymmetric operator peels both orientations") {
    std::mt19937_64 op_rng(61);
    Matrix g = random_matrix(64, 64, op_rng);
    Matrix a = g + 32.0 * Matrix::Identity(64, 64);
    DenseOperator op(a, false);
    auto bt = tree1d(64, 8, Admissibility::weak);
    PeelConfig cfg;
    cfg.eps = 1e-8;
    PeelResult r = peel_construct(op, bt, cfg);
    CHECK_FALSE(r.matrix.symmetric);
    CHECK(dense_2norm(r.matrix.to_dense() - a) <= 3e-8 * dense_2norm(a));
}
TEST_CASE("construction: estimate_relative_error of a peel result is below its eps") {
    std::mt19937_64 op_rng(60);
    Matrix g = random_matrix(96, 96, op_rng);
    Matrix a = gemm(g, false, g, true);
    DenseOperator op(a, true);
    auto bt = tree1d(96, 12, Admissibility::weak);
    PeelConfig cfg;
    cfg.eps = 1e-4;
    PeelResult r = peel_construct(op, bt, cfg);
    CHECK(estimate_relative_error(op, r.matrix) <= 1e-4);
}

MINI_MAIN
