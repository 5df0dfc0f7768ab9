// h2b200.hpp — C++ host API of the B200 H^2 hot path, mirroring the reference's
// header API (proj/include/h2/*.hpp) over the C ABI in h2c.h. Header-only; link
// with paper_2003_10173_b200/lib/libh2b200.so.
//
// Names, argument meaning and exception types follow the reference:
//   build_cluster_tree / build_block_tree   cluster_tree.hpp:186-188, block_tree.hpp:120-124
//   H2Matrix::matvec / matvec_transpose     h2_matrix.hpp:108-124 (user and internal ordering)
//   LinearOperator, DenseOperator,          linear_operator.hpp:20-115
//   H2Operator, make_operator
//   pnorm_estimate(op, 2)                   linear_operator.hpp:127-153
//   orthogonalize / recompress              algebra.hpp:72-226
//   PeelConfig / peel_construct /           construction.hpp:23-382, 537-546
//   estimate_relative_error, max_rank_error
// Matrices are any column-major type with rows(), cols() and data() (e.g.
// Eigen::MatrixXd, or h2::Matrix below); results come back as the same type.
// Everything numeric runs on the current CUDA device; nothing falls back to
// the CPU.
#ifndef H2B200_HPP
#define H2B200_HPP

#include <cstdint>
#include <functional>
#include <map>
#include <sstream>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "h2c.h"

namespace h2 {
inline namespace b200 {

using Index = std::int64_t;

enum class Ordering { user, internal };      // types.hpp:19
enum class Admissibility { strong, weak };   // block_tree.hpp:18-27

// construction.hpp:61-66
class max_rank_error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

namespace detail {
inline void check(int rc) {
    if (rc == H2C_OK) return;
    const std::string msg = h2c_last_error();
    switch (rc) {
        case H2C_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case H2C_LOGIC_ERROR: throw std::logic_error(msg);
        case H2C_MAX_RANK_ERROR: throw max_rank_error(msg);
        default: throw std::runtime_error(msg);
    }
}
}  // namespace detail

// minimal column-major matrix (stands in for Eigen::MatrixXd when Eigen is absent)
class Matrix {
public:
    Matrix() = default;
    Matrix(Index r, Index c) : r_(r), c_(c), d_(static_cast<size_t>(r * c), 0.0) {}
    static Matrix Identity(Index n, Index m) {
        Matrix a(n, m);
        for (Index i = 0; i < std::min(n, m); ++i) a(i, i) = 1.0;
        return a;
    }
    Index rows() const { return r_; }
    Index cols() const { return c_; }
    double* data() { return d_.data(); }
    const double* data() const { return d_.data(); }
    double& operator()(Index i, Index j) { return d_[static_cast<size_t>(i + j * r_)]; }
    double operator()(Index i, Index j) const { return d_[static_cast<size_t>(i + j * r_)]; }

private:
    Index r_ = 0, c_ = 0;
    std::vector<double> d_;
};

// PointSet (point_set.hpp:18-63): n points of dimension d <= 3, column-major n x d
struct PointSet {
    Index n = 0;
    int dim = 0;
    std::vector<double> coords;
    PointSet(Index n_, int d, std::vector<double> c) : n(n_), dim(d), coords(std::move(c)) {}
};

class ClusterTree {
public:
    ClusterTree(const PointSet& p, Index leaf) {
        detail::check(h2c_cluster_tree_create(p.coords.data(), p.n, p.dim, leaf, &h_));
        int dim = 0, nn = 0, nl = 0;
        detail::check(h2c_cluster_tree_info(h_, &n_, &dim, &depth_, &nn, &nl));
        nodes_ = nn;
    }
    ~ClusterTree() { h2c_cluster_tree_destroy(h_); }
    ClusterTree(const ClusterTree&) = delete;
    ClusterTree& operator=(const ClusterTree&) = delete;
    Index n() const { return n_; }
    int depth() const { return depth_; }
    int num_nodes() const { return nodes_; }
    h2c_cluster_tree handle() const { return h_; }

private:
    h2c_cluster_tree h_ = nullptr;
    int64_t n_ = 0;
    int depth_ = 0, nodes_ = 0;
};

inline std::shared_ptr<const ClusterTree> build_cluster_tree(const PointSet& p, Index leaf) {
    return std::make_shared<const ClusterTree>(p, leaf);
}

class BlockTree {
public:
    BlockTree(std::shared_ptr<const ClusterTree> t, double eta, Admissibility mode) : tree_(std::move(t)) {
        detail::check(h2c_block_tree_create(tree_->handle(), eta, mode == Admissibility::weak ? 1 : 0, &h_));
    }
    ~BlockTree() { h2c_block_tree_destroy(h_); }
    BlockTree(const BlockTree&) = delete;
    BlockTree& operator=(const BlockTree&) = delete;
    Index n() const { return tree_->n(); }
    const ClusterTree& row_tree() const { return *tree_; }
    h2c_block_tree handle() const { return h_; }

private:
    std::shared_ptr<const ClusterTree> tree_;
    h2c_block_tree h_ = nullptr;
};

inline std::shared_ptr<const BlockTree> build_block_tree(std::shared_ptr<const ClusterTree> rows,
                                                         std::shared_ptr<const ClusterTree> cols, double eta,
                                                         Admissibility mode = Admissibility::strong) {
    if (rows != cols) throw std::invalid_argument("block tree: the B200 path requires identical row and column trees");
    return std::make_shared<const BlockTree>(std::move(rows), eta, mode);
}

// device-resident H^2 matrix (h2_matrix.hpp:40-306); value semantics via shared ownership
struct StorageReport {   // h2_matrix.hpp:25-31
    Index dense_reals = 0;
    Index leaf_basis_reals = 0;
    Index transfer_reals = 0;
    Index coupling_reals = 0;
    Index total() const { return dense_reals + leaf_basis_reals + transfer_reals + coupling_reals; }
};
struct ValidationReport {   // h2_matrix.hpp:33-38
    std::vector<std::string> violations;
    std::vector<Index> level_max_rank;
    StorageReport storage;
    bool ok() const { return violations.empty(); }
};

class H2Matrix {
public:
    H2Matrix() = default;
    H2Matrix(h2c_matrix h, std::shared_ptr<const BlockTree> bt)
        : blocks(std::move(bt)), h_(h, [](h2c_matrix p) { h2c_matrix_destroy(p); }) {}
    static H2Matrix zero(std::shared_ptr<const BlockTree> bt, bool symmetric) {   // :53-75
        h2c_matrix h = nullptr;
        detail::check(h2c_matrix_create(bt->handle(), symmetric ? 1 : 0, nullptr, nullptr, &h));
        return H2Matrix(h, std::move(bt));
    }
    Index n() const { return blocks->n(); }
    bool symmetric() const {
        int64_t n = 0;
        int s = 0, o = 0;
        detail::check(h2c_matrix_info(h_.get(), &n, &s, &o));
        return s != 0;
    }
    // y = op(H) x by value (:112-124); M: rows()/cols()/data() column-major
    template <class M>
    M matvec(const M& x) const { return apply(x, false, Ordering::user); }
    template <class M>
    M matvec_transpose(const M& x) const { return apply(x, true, Ordering::user); }
    template <class M>
    M matvec_internal(const M& x) const { return apply(x, false, Ordering::internal); }
    template <class M>
    M matvec_transpose_internal(const M& x) const { return apply(x, true, Ordering::internal); }
    // device buffers: y = alpha op(H) x + beta y (the hot path, no host copies)
    void hgemv(bool transpose, Ordering ord, Index b, const double* x_dev, Index ldx, double* y_dev, Index ldy,
               double alpha = 1.0, double beta = 0.0, void* stream = nullptr) const {
        detail::check(h2c_hgemv(h_.get(), transpose ? 1 : 0, ord == Ordering::internal ? 1 : 0, n(), b, x_dev, ldx,
                                y_dev, ldy, alpha, beta, stream));
    }
    std::vector<int> row_ranks() const {
        std::vector<int> r(static_cast<size_t>(blocks->row_tree().num_nodes()));
        detail::check(h2c_matrix_ranks(h_.get(), r.data(), nullptr));
        return r;
    }
    bool orthonormal() const {
        int64_t n = 0;
        int s = 0, o = 0;
        detail::check(h2c_matrix_info(h_.get(), &n, &s, &o));
        return o != 0;
    }
    // dense expansion in user ordering (:128-163); M: (rows, cols) constructible, data() column-major
    template <class M = Matrix>
    M to_dense(Index cap = 8192) const {
        if (n() > cap) throw std::invalid_argument("to_dense: matrix size exceeds cap");
        M a(n(), n());
        detail::check(h2c_to_dense(h_.get(), cap, a.data()));
        return a;
    }
    ValidationReport validate(Index ortho_cap = 4096) const {   // :308-404
        int nv = 0, nl = 0;
        std::vector<char> msg(1 << 14);
        std::vector<int64_t> prof(128);
        int64_t st[4] = {0, 0, 0, 0};
        detail::check(h2c_validate(h_.get(), ortho_cap, &nv, msg.data(), int64_t(msg.size()), prof.data(),
                                   int(prof.size()), &nl, st));
        ValidationReport r;
        std::string all(msg.data());
        for (size_t a = 0; nv > 0 && a <= all.size();) {
            const size_t e = all.find('\n', a);
            const std::string line = all.substr(a, e == std::string::npos ? std::string::npos : e - a);
            if (!line.empty()) r.violations.push_back(line);
            if (e == std::string::npos) break;
            a = e + 1;
        }
        r.level_max_rank.assign(prof.begin(), prof.begin() + std::min<int>(nl, int(prof.size())));
        r.storage = StorageReport{st[0], st[1], st[2], st[3]};
        return r;
    }
    std::vector<Index> rank_profile() const { return validate(0).level_max_rank; }   // :190-195
    StorageReport storage() const { return validate(0).storage; }                    // :167-188
    h2c_matrix handle() const { return h_.get(); }

    std::shared_ptr<const BlockTree> blocks;

private:
    template <class M>
    M apply(const M& x, bool t, Ordering ord) const {
        if (x.rows() != n() || x.cols() < 1) throw std::invalid_argument("matvec: dimension mismatch");
        M y(x.rows(), x.cols());
        detail::check(h2c_matvec_host(h_.get(), t ? 1 : 0, ord == Ordering::internal ? 1 : 0, x.rows(), x.cols(),
                                      x.data(), y.data()));
        return y;
    }
    std::shared_ptr<h2c_matrix_s> h_;
};

// ---- row-subtree sharded hgemv (the reference is single-process) ----
// One plan per rank (one process per GPU). begin() (owned upsweep + pack) ->
// the exchange -> local() (near field of owned source rows, optional, while the
// exchange is in flight) -> end() (unpack, couplings, downsweep, remaining near
// field, owned rows of y). The exchange is either the caller's collective on
// send / receive buffers (sizes send_rows() / recv_rows() times b doubles,
// peers in rank order) or, after the peer setup below, device-side P2P writes
// and signals: begin(..., nullptr) / end(nullptr, ...).
class ShardedPlan {
public:
    ShardedPlan(const H2Matrix& h, int nranks, int rank, bool transpose = false) : nranks_(nranks), rank_(rank) {
        h2c_dist_plan p = nullptr;
        detail::check(h2c_dist_plan_create(h.handle(), transpose ? 1 : 0, nranks, rank, &p));
        h_.reset(p, [](h2c_dist_plan q) { h2c_dist_plan_destroy(q); });
        send_.assign(size_t(nranks), 0);
        recv_.assign(size_t(nranks), 0);
        int64_t ob = 0, orows = 0;
        detail::check(h2c_dist_plan_counts(p, send_.data(), recv_.data(), &ob, &orows));
        owned_begin_ = ob;
        owned_rows_ = orows;
    }
    int nranks() const { return nranks_; }
    int rank() const { return rank_; }
    const std::vector<int64_t>& send_rows() const { return send_; }
    const std::vector<int64_t>& recv_rows() const { return recv_; }
    Index owned_begin() const { return owned_begin_; }   // internal (cluster) row range of this rank
    Index owned_rows() const { return owned_rows_; }
    // x_dev / y_dev: full n x b user-order device matrices (owned = false) or this rank's
    // owned_rows() rows in cluster order (owned = true)
    void begin(Index b, const double* x_dev, Index ldx, double* sendbuf, void* stream = nullptr, bool owned = false) {
        detail::check(owned ? h2c_dist_hgemv_begin_owned(h_.get(), b, x_dev, ldx, sendbuf, stream)
                            : h2c_dist_hgemv_begin(h_.get(), b, x_dev, ldx, sendbuf, stream));
    }
    void local(Index b, void* stream = nullptr) { detail::check(h2c_dist_hgemv_local(h_.get(), b, stream)); }
    void end(Index b, const double* recvbuf, double* y_dev, Index ldy, double alpha = 1.0, double beta = 0.0,
             void* stream = nullptr, bool owned = false) {
        detail::check(owned ? h2c_dist_hgemv_end_owned(h_.get(), b, recvbuf, y_dev, ldy, alpha, beta, stream)
                            : h2c_dist_hgemv_end(h_.get(), b, recvbuf, y_dev, ldy, alpha, beta, stream));
    }
    // the whole sharded hgemv with the exchange on the caller's ncclComm_t (passed as void*)
    void hgemv_nccl(void* nccl_comm, Index b, const double* x_dev, Index ldx, double* y_dev, Index ldy,
                    double alpha = 1.0, double beta = 0.0, void* stream = nullptr, bool owned = false) {
        detail::check(owned ? h2c_dist_hgemv_nccl_owned(h_.get(), nccl_comm, b, x_dev, ldx, y_dev, ldy, alpha, beta,
                                                        stream)
                            : h2c_dist_hgemv_nccl(h_.get(), nccl_comm, b, x_dev, ldx, y_dev, ldy, alpha, beta, stream));
    }
    // peer transport: alloc on every rank (same max_b), export, allgather the exports,
    // import all of them (or link the plans of every rank held by one process)
    struct PeerInfo {
        std::vector<unsigned char> handles;   // 128 bytes (CUDA IPC)
        std::vector<int64_t> recv_off;        // nranks entries (rows)
    };
    void peer_alloc(Index max_b) { detail::check(h2c_dist_peer_alloc(h_.get(), max_b)); }
    PeerInfo peer_export() const {
        PeerInfo i{std::vector<unsigned char>(128), std::vector<int64_t>(size_t(nranks_))};
        detail::check(h2c_dist_peer_export(h_.get(), i.handles.data(), i.recv_off.data()));
        return i;
    }
    void peer_import(const std::vector<PeerInfo>& all) {
        std::vector<unsigned char> hb;
        std::vector<int64_t> off;
        for (const PeerInfo& i : all) {
            hb.insert(hb.end(), i.handles.begin(), i.handles.end());
            off.insert(off.end(), i.recv_off.begin(), i.recv_off.end());
        }
        detail::check(h2c_dist_peer_import(h_.get(), hb.data(), off.data()));
    }
    static void peer_link(const std::vector<ShardedPlan*>& plans) {
        std::vector<h2c_dist_plan> hs;
        for (ShardedPlan* p : plans) hs.push_back(p->h_.get());
        detail::check(h2c_dist_peer_link(hs.data(), int(hs.size())));
    }
    h2c_dist_plan handle() const { return h_.get(); }

private:
    int nranks_ = 1, rank_ = 0;
    std::vector<int64_t> send_, recv_;
    Index owned_begin_ = 0, owned_rows_ = 0;
    std::shared_ptr<h2c_dist_plan_s> h_;
};

inline H2Matrix orthogonalize(const H2Matrix& h) {   // algebra.hpp:72-113
    h2c_matrix o = nullptr;
    detail::check(h2c_orthogonalize(h.handle(), &o));
    return H2Matrix(o, h.blocks);
}
inline H2Matrix recompress(const H2Matrix& h, double eps) {   // algebra.hpp:144-226
    h2c_matrix o = nullptr;
    detail::check(h2c_recompress(h.handle(), eps, &o));
    return H2Matrix(o, h.blocks);
}

inline double frobenius_norm(const H2Matrix& h) {   // algebra.hpp:119-137 (needs orthonormal bases)
    double v = 0;
    detail::check(h2c_frobenius_norm(h.handle(), &v));
    return v;
}
struct LowRankFactor {   // algebra.hpp:18-21: X Y^T, n x k each, user ordering
    Matrix X, Y;
    Index rank() const { return X.cols(); }
};
inline H2Matrix low_rank_update(const H2Matrix& h, const LowRankFactor& f, double eps) {   // algebra.hpp:334-346
    if (f.X.rows() != h.n() || f.Y.rows() != h.n() || f.X.cols() != f.Y.cols())
        throw std::invalid_argument("low_rank_update: factor dimensions do not match");
    h2c_matrix o = nullptr;
    detail::check(h2c_low_rank_update_host(h.handle(), f.rank(), f.X.data(), f.Y.data(), eps, &o));
    return H2Matrix(o, h.blocks);
}
// local_low_rank_update(h, t, s, U_blk, V_blk, eps) (algebra.hpp:323-332): cluster-order factors
template <class M>
H2Matrix local_low_rank_update(const H2Matrix& h, int t, int s, const M& u_blk, const M& v_blk, double eps) {
    if (u_blk.cols() != v_blk.cols()) throw std::invalid_argument("local update: factor dimensions do not match clusters");
    h2c_matrix o = nullptr;
    detail::check(h2c_local_low_rank_update_host(h.handle(), t, s, u_blk.cols(), u_blk.data(), v_blk.data(), eps, &o));
    return H2Matrix(o, h.blocks);
}

// LinearOperator (linear_operator.hpp:20-55): apply on host matrices (user order)
class LinearOperator {
public:
    explicit LinearOperator(h2c_operator h, Index n, bool sym, std::shared_ptr<void> keep = {})
        : h_(h, [](h2c_operator p) { h2c_operator_destroy(p); }), n_(n), sym_(sym), keep_(std::move(keep)) {}
    Index dim() const { return n_; }
    bool symmetric() const { return sym_; }
    long columns_applied() const {
        int64_t c = 0;
        detail::check(h2c_operator_columns_applied(h_.get(), &c));
        return long(c);
    }
    void reset_counter() const { detail::check(h2c_operator_reset_counter(h_.get())); }
    h2c_operator handle() const { return h_.get(); }
    // apply / apply_transpose (linear_operator.hpp:28-39): n x b host matrix in user ordering
    template <class M>
    Matrix apply(const M& x) const { return run(x, 0); }
    template <class M>
    Matrix apply_transpose(const M& x) const { return run(x, 1); }

private:
    template <class M>
    Matrix run(const M& x, int t) const {
        if (Index(x.rows()) != n_) throw std::invalid_argument("operator apply: dimension mismatch");
        Matrix y(n_, x.cols());
        if (x.cols() > 0) detail::check(h2c_operator_apply_host(h_.get(), t, x.cols(), x.data(), y.data()));
        return y;
    }
    std::shared_ptr<h2c_operator_s> h_;
    Index n_;
    bool sym_;
    std::shared_ptr<void> keep_;
};

// DenseOperator (linear_operator.hpp:86-101)
template <class M>
LinearOperator DenseOperator(const M& a, bool sym = false) {
    if (a.rows() != a.cols()) throw std::invalid_argument("dense operator: square only");
    h2c_operator h = nullptr;
    detail::check(h2c_operator_dense(a.data(), a.rows(), sym ? 1 : 0, &h));
    return LinearOperator(h, a.rows(), sym);
}
// H2Operator (linear_operator.hpp:104-115)
inline LinearOperator H2Operator(const H2Matrix& m) {
    h2c_operator h = nullptr;
    detail::check(h2c_operator_h2(m.handle(), &h));
    return LinearOperator(h, m.n(), m.symmetric(), std::make_shared<H2Matrix>(m));
}
// make_operator (linear_operator.hpp:80-84): host functions on h2::Matrix (n x b, user order)
using HostFn = std::function<Matrix(const Matrix&)>;
inline LinearOperator make_operator(Index n, bool sym, HostFn f, HostFn t = nullptr) {
    struct Ctx {
        Index n;
        HostFn f, t;
    };
    auto ctx = std::make_shared<Ctx>(Ctx{n, std::move(f), std::move(t)});
    auto cb = [](void* c, int transpose, int64_t b, const double* x, double* y, void*) -> int {
        try {
            auto* cx = static_cast<Ctx*>(c);
            Matrix xm(cx->n, b);
            std::copy(x, x + cx->n * b, xm.data());
            const Matrix ym = transpose ? cx->t(xm) : cx->f(xm);
            if (ym.rows() != cx->n || ym.cols() != b) return 1;
            std::copy(ym.data(), ym.data() + cx->n * b, y);
            return 0;
        } catch (...) {
            return 1;
        }
    };
    h2c_operator h = nullptr;
    detail::check(h2c_operator_host_callback(n, sym ? 1 : 0, ctx->t ? 1 : 0, cb, ctx.get(), &h));
    return LinearOperator(h, n, sym, ctx);
}

struct NormEstimate {
    double value = 0;
    int iterations = 0;
};
inline NormEstimate pnorm_estimate(const LinearOperator& op, double p) {   // linear_operator.hpp:127-153
    if (p != 2.0) throw std::invalid_argument("pnorm_estimate: the B200 path implements p = 2");
    NormEstimate e;
    detail::check(h2c_pnorm2_estimate(op.handle(), &e.value, &e.iterations));
    return e;
}

struct PeelConfig {   // construction.hpp:23-31
    double eps = 1e-4;
    Index sample_block_size = 16;
    Index oversampling = 10;
    Index max_rank = 0;
    std::uint64_t seed = 42;
    double norm_scale = 0;
    Index crossover_rank_cap = 128;
    int rng = 0;   // B200 extension: 0 reference host stream, 1 device Philox
};
struct LevelStats {
    int level = 0;
    Index blocks = 0, max_rank = 0;
    long samples = 0;
};
struct SampleStats {   // construction.hpp:40-59
    long total = 0;
    std::vector<LevelStats> levels;
    bool consistent() const {
        long s = 0;
        for (const auto& l : levels) s += l.samples;
        return s == total;
    }
};
struct PeelResult {   // construction.hpp:295-298
    H2Matrix matrix;
    SampleStats stats;
};

inline PeelResult peel_construct(const LinearOperator& op, std::shared_ptr<const BlockTree> bt,
                                 const PeelConfig& cfg) {   // construction.hpp:300-382
    h2c_peel_config c;
    c.eps = cfg.eps;
    c.sample_block_size = cfg.sample_block_size;
    c.oversampling = cfg.oversampling;
    c.max_rank = cfg.max_rank;
    c.seed = cfg.seed;
    c.norm_scale = cfg.norm_scale;
    c.crossover_rank_cap = cfg.crossover_rank_cap;
    c.rng = cfg.rng;
    h2c_matrix h = nullptr;
    int64_t total = 0;
    std::vector<h2c_level_stats> lv(128);
    int nl = 0;
    detail::check(h2c_peel_construct(op.handle(), bt->handle(), &c, &h, &total, lv.data(), int(lv.size()), &nl,
                                     nullptr, nullptr));
    PeelResult r{H2Matrix(h, bt), {}};
    r.stats.total = long(total);
    for (int i = 0; i < nl; ++i) r.stats.levels.push_back({lv[size_t(i)].level, lv[size_t(i)].blocks,
                                                           lv[size_t(i)].max_rank, long(lv[size_t(i)].samples)});
    return r;
}

namespace detail {
// lend a caller's std::mt19937_64 to the library and take it back advanced
// (h2c_rng_set_state / get_state: libstdc++'s textual engine state)
template <class Engine>
struct LentRng {
    Engine& eng;
    h2c_rng r = nullptr;
    explicit LentRng(Engine& e) : eng(e) {
        std::ostringstream out;
        out << eng;
        check(h2c_rng_create(0, &r));
        check(h2c_rng_set_state(r, out.str().c_str()));
    }
    ~LentRng() {
        int64_t need = 0;
        if (h2c_rng_get_state(r, nullptr, &need) == H2C_OK) {
            std::string buf(static_cast<size_t>(need), '\0');
            if (h2c_rng_get_state(r, &buf[0], &need) == H2C_OK) {
                std::istringstream in(buf);
                in >> eng;
            }
        }
        h2c_rng_destroy(r);
    }
};
}  // namespace detail

// sample_block_column(op, ct, t, s, count, rng) (construction.hpp:137-148):
// (Omega restricted to s, op(Omega) restricted to t); rng advances exactly as
// the reference's fill_gaussian would advance it
template <class Engine>
std::pair<Matrix, Matrix> sample_block_column(const LinearOperator& op, const ClusterTree& ct, int t, int s,
                                              Index count, Engine& rng) {
    if (count < 1) throw std::invalid_argument("sample_block_column: count must be >= 1");
    detail::LentRng<Engine> lent(rng);
    Index mt = 0, ms = 0;
    {
        std::vector<int64_t> b(static_cast<size_t>(ct.num_nodes())), e(b.size());
        std::vector<int> lv(b.size()), par(b.size()), c0(b.size()), c1(b.size());
        detail::check(h2c_cluster_tree_nodes(ct.handle(), b.data(), e.data(), lv.data(), par.data(), c0.data(),
                                             c1.data(), nullptr, nullptr));
        if (t < 0 || s < 0 || t >= ct.num_nodes() || s >= ct.num_nodes())
            throw std::invalid_argument("sample_block_column: cluster id out of range");
        mt = e[size_t(t)] - b[size_t(t)];
        ms = e[size_t(s)] - b[size_t(s)];
    }
    Matrix om(ms, count), y(mt, count);
    detail::check(h2c_sample_block_column_host(op.handle(), ct.handle(), t, s, count, lent.r, om.data(), y.data()));
    return {std::move(om), std::move(y)};
}

struct BlockFactor {   // construction.hpp:150-154
    Matrix u, v;
    Index rank = 0;
    double err_est = 0;
};
// adaptive_block_factorization(op, ct, t, s, eps_block, cfg) (construction.hpp:156-198)
inline BlockFactor adaptive_block_factorization(const LinearOperator& op, const ClusterTree& ct, int t, int s,
                                                double eps_block, const PeelConfig& cfg) {
    h2c_peel_config c;
    c.eps = cfg.eps;
    c.sample_block_size = cfg.sample_block_size;
    c.oversampling = cfg.oversampling;
    c.max_rank = cfg.max_rank;
    c.seed = cfg.seed;
    c.norm_scale = cfg.norm_scale;
    c.crossover_rank_cap = cfg.crossover_rank_cap;
    c.rng = cfg.rng;
    h2c_block_factor f = nullptr;
    detail::check(h2c_adaptive_block_factorization(op.handle(), ct.handle(), t, s, eps_block, &c, &f));
    std::unique_ptr<h2c_block_factor_s, void (*)(h2c_block_factor)> guard(f, h2c_block_factor_destroy);
    int64_t ru = 0, rv = 0, k = 0;
    double e = 0;
    detail::check(h2c_block_factor_info(f, &ru, &rv, &k, &e));
    BlockFactor out{Matrix(ru, k), Matrix(rv, k), Index(k), e};
    detail::check(h2c_block_factor_download(f, out.u.data(), out.v.data()));
    return out;
}

inline double estimate_relative_error(const LinearOperator& op, const H2Matrix& h, double op_norm = 0) {
    double v = 0;   // construction.hpp:537-546
    detail::check(h2c_estimate_relative_error(op.handle(), h.handle(), op_norm, &v));
    return v;
}

// ---- h2::oracles (oracles/diffusion1d.hpp, minimal_surface.hpp, registry.hpp): device black boxes ----
namespace oracles {

struct Diffusion1DConfig {   // diffusion1d.hpp:62-73
    Index n = 512;
    double pad = 0.5;
    double final_time = 30.0;
    Index steps = 512;
    double t_p = 1.0;
    double t_0 = 0.0;
    double source_amplitude = 1000.0;
    double alpha = 3e-5, beta = 1e-3;
    std::vector<double> source_positions{-0.5, 0.0, 0.5};
    Index num_receivers = 8;
};

class Diffusion1D {   // diffusion1d.hpp:75-123, Hessian at the target only (:173-181)
public:
    explicit Diffusion1D(Diffusion1DConfig cfg = {}) : cfg_(std::move(cfg)) {
        h2c_diff1d_config c;
        h2c_diff1d_config_default(&c);
        c.n = cfg_.n;
        c.steps = cfg_.steps;
        c.final_time = cfg_.final_time;
        c.t_p = cfg_.t_p;
        c.t_0 = cfg_.t_0;
        c.source_amplitude = cfg_.source_amplitude;
        c.alpha = cfg_.alpha;
        c.beta = cfg_.beta;
        c.pad = cfg_.pad;
        c.num_sources = int(cfg_.source_positions.size());
        c.source_positions = cfg_.source_positions.data();
        c.num_receivers = cfg_.num_receivers;
        h2c_diff1d d = nullptr;
        detail::check(h2c_diff1d_create(&c, nullptr, &d));
        h_ = std::shared_ptr<h2c_diff1d_s>(d, [](h2c_diff1d p) { h2c_diff1d_destroy(p); });
    }
    Index n() const { return cfg_.n; }
    const Diffusion1DConfig& config() const { return cfg_; }
    double spacing() const { return info().h; }
    double dt() const { return info().dt; }
    long pde_solves() const { return long(info().solves); }
    PointSet points() const {   // Grid1D(-1, 1, n).points() (grid.hpp:10-24)
        std::vector<double> c(static_cast<size_t>(cfg_.n));
        const double h = 2.0 / double(cfg_.n - 1);
        for (Index i = 0; i < cfg_.n; ++i) c[size_t(i)] = -1.0 + h * double(i);
        return PointSet(cfg_.n, 1, c);
    }
    // hessian_operator(include_tv) (:177-181): the operator keeps the problem alive
    LinearOperator hessian_operator(bool include_tv = true) const {
        h2c_operator o = nullptr;
        detail::check(h2c_diff1d_operator(h_.get(), include_tv ? 1 : 0, &o));
        return LinearOperator(o, cfg_.n, true, h_);
    }

private:
    struct Info {
        int64_t ns, npad, solves;
        double h, dt;
    };
    Info info() const {
        Info i{};
        detail::check(h2c_diff1d_info(h_.get(), &i.ns, &i.npad, &i.h, &i.dt, &i.solves));
        return i;
    }
    Diffusion1DConfig cfg_;
    std::shared_ptr<h2c_diff1d_s> h_;
};

class MinimalSurface {   // minimal_surface.hpp:22-175, Hessian at newton_state(steps) (registry.hpp:89-101)
public:
    explicit MinimalSurface(Index interior, double rim_amplitude = 0.5, int newton_steps = 0) : g_(interior) {
        h2c_surface s = nullptr;
        detail::check(h2c_surface_create(interior, rim_amplitude, newton_steps, &s));
        h_ = std::shared_ptr<h2c_surface_s>(s, [](h2c_surface p) { h2c_surface_destroy(p); });
    }
    Index n() const { return g_ * g_; }
    double spacing() const { return 1.0 / double(g_ + 1); }
    PointSet points() const {   // Grid2D(interior).points() (grid.hpp:38-48), n x 2 column-major
        std::vector<double> c(static_cast<size_t>(2 * n()));
        for (Index j = 1; j <= g_; ++j)
            for (Index i = 1; i <= g_; ++i) {
                const Index r = (j - 1) * g_ + (i - 1);
                c[size_t(r)] = spacing() * double(i);
                c[size_t(r + n())] = spacing() * double(j);
            }
        return PointSet(n(), 2, c);
    }
    std::vector<double> state() const {   // the interior surface the Hessian is taken at
        std::vector<double> m(static_cast<size_t>(n()));
        detail::check(h2c_surface_state(h_.get(), m.data()));
        return m;
    }
    // hessian_operator (:163-167): the operator keeps the problem alive
    LinearOperator hessian_operator() const {
        h2c_operator o = nullptr;
        detail::check(h2c_surface_operator(h_.get(), &o));
        return LinearOperator(o, n(), true, h_);
    }

private:
    Index g_;
    std::shared_ptr<h2c_surface_s> h_;
};

struct AdvDiff2DConfig {   // advdiff2d.hpp:21-28
    Index grid = 32;
    double kappa = 1e-3;
    double reaction = 0.5;
    Index num_observations = 100;
    double noise_rel = 0.01;
    uint64_t obs_seed = 7;
};

class AdvDiff2D {   // advdiff2d.hpp:30-146: misfit Hessian of the stationary source inversion
public:
    explicit AdvDiff2D(AdvDiff2DConfig cfg = {}) : cfg_(cfg) {
        h2c_advdiff_config c;
        h2c_advdiff_config_default(&c);
        c.grid = cfg_.grid;
        c.kappa = cfg_.kappa;
        c.reaction = cfg_.reaction;
        c.num_observations = cfg_.num_observations;
        c.noise_rel = cfg_.noise_rel;
        c.obs_seed = cfg_.obs_seed;
        h2c_advdiff a = nullptr;
        detail::check(h2c_advdiff_create(&c, &a));
        h_ = std::shared_ptr<h2c_advdiff_s>(a, [](h2c_advdiff p) { h2c_advdiff_destroy(p); });
    }
    Index n() const { return cfg_.grid * cfg_.grid; }
    const AdvDiff2DConfig& config() const { return cfg_; }
    double sigma() const {
        double s = 0;
        detail::check(h2c_advdiff_info(h_.get(), nullptr, &s, nullptr, nullptr));
        return s;
    }
    long solves() const {
        int64_t v = 0;
        detail::check(h2c_advdiff_info(h_.get(), nullptr, nullptr, nullptr, &v));
        return long(v);
    }
    PointSet points() const {   // Grid2D(grid).points() (grid.hpp:38-48), n x 2 column-major
        const Index g = cfg_.grid;
        const double h = 1.0 / double(g + 1);
        std::vector<double> c(static_cast<size_t>(2 * n()));
        for (Index j = 1; j <= g; ++j)
            for (Index i = 1; i <= g; ++i) {
                const Index r = (j - 1) * g + (i - 1);
                c[size_t(r)] = h * double(i);
                c[size_t(r + n())] = h * double(j);
            }
        return PointSet(n(), 2, c);
    }
    // hessian_operator (:66-68): the operator keeps the problem alive
    LinearOperator hessian_operator() const {
        h2c_operator o = nullptr;
        detail::check(h2c_advdiff_operator(h_.get(), &o));
        return LinearOperator(o, n(), true, h_);
    }

private:
    AdvDiff2DConfig cfg_;
    std::shared_ptr<h2c_advdiff_s> h_;
};

struct Oracle {   // registry.hpp:58-81
    std::string name;
    std::shared_ptr<LinearOperator> op;
    PointSet points{0, 1, {}};
    Index leaf = 32;
    Admissibility mode = Admissibility::weak;
    double eta = 1.0;
    std::shared_ptr<MinimalSurface> surface;
    std::shared_ptr<Diffusion1D> diffusion;
    std::shared_ptr<AdvDiff2D> advdiff;
    std::shared_ptr<const BlockTree> default_block_tree() const {
        auto ct = build_cluster_tree(points, leaf);
        return build_block_tree(ct, ct, eta, mode);
    }
};

using Config = std::map<std::string, std::string>;
// make_oracle("surface<N>" | "diff1d-<n>" | "advdiff-<G>[-k..][-obs..]", config) (registry.hpp:83-154)
inline Oracle make_oracle(const std::string& name, const Config& config = {}) {
    auto num = [&](const char* k, double d) {
        auto it = config.find(k);
        return it == config.end() ? d : std::stod(it->second);
    };
    if (name.rfind("surface", 0) == 0) {   // registry.hpp:89-101
        Oracle o;
        o.name = name;
        o.surface = std::make_shared<MinimalSurface>(Index(std::stoll(name.substr(7))), num("rim", 0.5),
                                                     int(num("newton_steps", 0)));
        o.op = std::make_shared<LinearOperator>(o.surface->hessian_operator());
        o.points = o.surface->points();
        o.leaf = Index(num("leaf", 64));
        o.mode = Admissibility::strong;
        o.eta = num("eta", 1.0);
        return o;
    }
    if (name.rfind("advdiff-", 0) == 0) {   // registry.hpp:125-150
        AdvDiff2DConfig ac;
        std::string rest = name.substr(8);
        const auto dash = rest.find('-');
        ac.grid = Index(std::stoll(rest.substr(0, dash)));
        std::string tail = dash == std::string::npos ? "" : rest.substr(dash);
        if (const auto at = tail.find("-obs"); at != std::string::npos) {
            ac.num_observations = Index(std::stoll(tail.substr(at + 4)));
            tail = tail.substr(0, at);
        }
        if (tail.rfind("-k", 0) == 0) ac.kappa = std::stod(tail.substr(2));
        ac.kappa = num("kappa", ac.kappa);
        ac.num_observations = Index(num("obs", double(ac.num_observations)));
        ac.noise_rel = num("noise", ac.noise_rel);
        ac.obs_seed = uint64_t(num("obs_seed", double(ac.obs_seed)));
        ac.reaction = num("c", ac.reaction);
        Oracle o;
        o.name = name;
        o.advdiff = std::make_shared<AdvDiff2D>(ac);
        o.op = std::make_shared<LinearOperator>(o.advdiff->hessian_operator());
        o.points = o.advdiff->points();
        o.leaf = Index(num("leaf", 64));
        o.mode = Admissibility::strong;
        o.eta = num("eta", 1.0);
        return o;
    }
    if (name.rfind("diff1d-", 0) != 0) throw std::invalid_argument("unknown oracle " + name);
    Diffusion1DConfig dc;
    dc.n = Index(std::stoll(name.substr(7)));
    dc.steps = Index(num("steps", double(dc.steps)));
    dc.final_time = num("T", dc.final_time);
    dc.t_p = num("tp", dc.t_p);
    dc.t_0 = num("t0", dc.t_0);
    dc.alpha = num("alpha", dc.alpha);
    dc.source_amplitude = num("amp", dc.source_amplitude);
    dc.beta = num("beta", dc.beta);
    dc.pad = num("pad", dc.pad);
    Oracle o;
    o.name = name;
    o.diffusion = std::make_shared<Diffusion1D>(dc);
    o.op = std::make_shared<LinearOperator>(o.diffusion->hessian_operator(num("tv", 1) != 0));
    o.points = o.diffusion->points();
    o.leaf = Index(num("leaf", 32));
    o.eta = num("eta", 1.0);
    return o;
}

}  // namespace oracles

}  // namespace b200
}  // namespace h2

#endif  // H2B200_HPP
