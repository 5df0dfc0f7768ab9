// extern "C" boundary (include/h2c.h) over the C++ host layer and CUDA kernels.
#include "../../include/h2c.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <sstream>
#include <string>

#include "h2dev.hpp"
#include "hara.hpp"
#include "inversion.hpp"
#include "diffusion1d.hpp"
#include "surface.hpp"
#include "advdiff.hpp"
#include "serialize.hpp"
#include "matrix.hpp"
#include "blockops.hpp"
#include "refstream.hpp"

struct h2c_cluster_tree_s {
    std::shared_ptr<h2b::ClusterTree> t;
};
struct h2c_block_tree_s {
    std::shared_ptr<h2b::BlockTree> b;
};
struct h2c_matrix_s {
    std::unique_ptr<h2b::H2Dev> h;
    h2b::Workspace ws;   // legacy-stream calls and timing
    // hgemv workspace per stream: the matrix and its plans are immutable and
    // shared, scratch (x blocked, x-hat, y-hat, host staging) is per stream
    std::mutex mu;
    std::map<cudaStream_t, std::unique_ptr<h2b::Workspace>> per_stream;
    h2b::Workspace& ws_for(cudaStream_t s) {
        if (s == nullptr) return ws;
        std::lock_guard<std::mutex> g(mu);
        auto& w = per_stream[s];
        if (!w) w = std::make_unique<h2b::Workspace>();
        return *w;
    }
};
struct h2c_dist_plan_s {
    std::shared_ptr<h2b::DistPlan> p;
};
struct h2c_lowrank_s {
    h2b::LowRankResultDev r;
    int64_t n = 0;
};
struct h2c_operator_s {
    std::unique_ptr<h2b::DevOperator> op;
};
struct h2c_rng_s {
    std::mt19937_64 g;
};
struct h2c_block_factor_s {
    h2b::BlockFactorDev f;
    int64_t rows_u = 0, rows_v = 0;
};

namespace {
thread_local std::string g_err;
thread_local int g_io_kind = -1;

template <class F>
int guard(F&& f) {
    try {
        f();
        return H2C_OK;
    } catch (const h2b::cuda_error& e) {
        g_err = e.what();
        return H2C_CUDA_ERROR;
    } catch (const h2b::io_error& e) {
        g_err = e.what();
        g_io_kind = int(e.kind);
        return H2C_IO_ERROR;
    } catch (const h2b::divergence_error& e) {
        g_err = e.what();
        return H2C_DIVERGENCE_ERROR;
    } catch (const h2b::max_rank_error& e) {
        g_err = e.what();
        return H2C_MAX_RANK_ERROR;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return H2C_INVALID_ARGUMENT;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return H2C_LOGIC_ERROR;
    } catch (const std::exception& e) {
        g_err = e.what();
        return H2C_RUNTIME_ERROR;
    }
}
void need(bool ok, const char* msg) {
    if (!ok) throw std::invalid_argument(msg);
}
}  // namespace

extern "C" {

const char* h2c_last_error(void) { return g_err.c_str(); }
const char* h2c_version(void) { return "h2b200 0.1 (sm_100a)"; }

int h2c_cluster_tree_create(const double* coords, int64_t n, int dim, int64_t leaf_size, h2c_cluster_tree* out) {
    return guard([&] {
        need(out != nullptr, "null output handle");
        need(coords != nullptr || n == 0, "null coordinates");
        auto t = h2b::build_cluster_tree(coords, n, dim, leaf_size);
        *out = new h2c_cluster_tree_s{std::move(t)};
    });
}
int h2c_cluster_tree_create_device(const double* coords, int64_t n, int dim, int64_t leaf_size, void* stream,
                                   h2c_cluster_tree* out) {
    return guard([&] {
        need(out != nullptr, "null output handle");
        need(coords != nullptr || n == 0, "null coordinates");
        auto t = h2b::build_cluster_tree_device(coords, n, dim, leaf_size, static_cast<cudaStream_t>(stream));
        *out = new h2c_cluster_tree_s{std::move(t)};
    });
}
void h2c_cluster_tree_destroy(h2c_cluster_tree t) { delete t; }

int h2c_cluster_tree_info(h2c_cluster_tree t, int64_t* n, int* dim, int* depth, int* num_nodes, int* num_leaves) {
    return guard([&] {
        need(t != nullptr, "null tree");
        if (n) *n = t->t->n;
        if (dim) *dim = t->t->dim;
        if (depth) *depth = t->t->depth;
        if (num_nodes) *num_nodes = t->t->num_nodes();
        if (num_leaves) *num_leaves = int(t->t->leaves.size());
    });
}

int h2c_cluster_tree_nodes(h2c_cluster_tree t, int64_t* begin, int64_t* end, int* level, int* parent, int* child0,
                           int* child1, double* lo, double* hi) {
    return guard([&] {
        need(t != nullptr, "null tree");
        const auto& c = *t->t;
        const size_t nn = size_t(c.num_nodes());
        if (begin) std::memcpy(begin, c.begin.data(), nn * sizeof(int64_t));
        if (end) std::memcpy(end, c.end.data(), nn * sizeof(int64_t));
        if (level) std::memcpy(level, c.level.data(), nn * sizeof(int));
        if (parent) std::memcpy(parent, c.parent.data(), nn * sizeof(int));
        if (child0) std::memcpy(child0, c.child0.data(), nn * sizeof(int));
        if (child1) std::memcpy(child1, c.child1.data(), nn * sizeof(int));
        if (lo) std::memcpy(lo, c.lo.data(), 3 * nn * sizeof(double));
        if (hi) std::memcpy(hi, c.hi.data(), 3 * nn * sizeof(double));
    });
}

int h2c_cluster_tree_perm(h2c_cluster_tree t, int64_t* perm) {
    return guard([&] {
        need(t != nullptr && perm != nullptr, "null argument");
        std::memcpy(perm, t->t->perm.data(), t->t->perm.size() * sizeof(int64_t));
    });
}

int h2c_block_tree_create(h2c_cluster_tree t, double eta, int weak, h2c_block_tree* out) {
    return guard([&] {
        need(t != nullptr && out != nullptr, "null argument");
        *out = new h2c_block_tree_s{h2b::build_block_tree(t->t, eta, weak != 0)};
    });
}
void h2c_block_tree_destroy(h2c_block_tree b) { delete b; }

int h2c_block_tree_info(h2c_block_tree b, int* num_nodes, int* num_adm, int* num_dense, int* max_level) {
    return guard([&] {
        need(b != nullptr, "null block tree");
        if (num_nodes) *num_nodes = b->b->num_nodes();
        if (num_adm) *num_adm = int(b->b->adm.size());
        if (num_dense) *num_dense = int(b->b->dense.size());
        if (max_level) *max_level = b->b->max_level;
    });
}

int h2c_block_tree_nodes(h2c_block_tree b, int* row, int* col, int* level, int* parent, int* tag) {
    return guard([&] {
        need(b != nullptr, "null block tree");
        const auto& t = *b->b;
        const size_t nn = size_t(t.num_nodes());
        if (row) std::memcpy(row, t.row.data(), nn * sizeof(int));
        if (col) std::memcpy(col, t.col.data(), nn * sizeof(int));
        if (level) std::memcpy(level, t.level.data(), nn * sizeof(int));
        if (parent) std::memcpy(parent, t.parent.data(), nn * sizeof(int));
        if (tag) std::memcpy(tag, t.tag.data(), nn * sizeof(int));
    });
}

int h2c_block_tree_params(h2c_block_tree b, double* eta, int* weak) {
    return guard([&] {
        need(b != nullptr, "null block tree");
        if (eta) *eta = b->b->eta;
        if (weak) *weak = b->b->weak ? 1 : 0;
    });
}

int h2c_block_tree_cluster_tree(h2c_block_tree b, h2c_cluster_tree* out) {
    return guard([&] {
        need(b != nullptr && out != nullptr, "null argument");
        *out = new h2c_cluster_tree_s{std::const_pointer_cast<h2b::ClusterTree>(b->b->tree)};
    });
}

int h2c_block_tree_leaves(h2c_block_tree b, int* adm, int* dense) {
    return guard([&] {
        need(b != nullptr, "null block tree");
        if (adm) std::memcpy(adm, b->b->adm.data(), b->b->adm.size() * sizeof(int));
        if (dense) std::memcpy(dense, b->b->dense.data(), b->b->dense.size() * sizeof(int));
    });
}

int h2c_matrix_create(h2c_block_tree b, int symmetric, const int* row_ranks, const int* col_ranks, h2c_matrix* out) {
    return guard([&] {
        need(b != nullptr && out != nullptr, "null argument");
        auto m = new h2c_matrix_s;
        try {
            m->h = h2b::make_h2(b->b, symmetric != 0, row_ranks, col_ranks);
            m->h->orthonormal = row_ranks == nullptr;   // zero(): orthonormal (h2_matrix.hpp:74)
        } catch (...) {
            delete m;
            throw;
        }
        *out = m;
    });
}
void h2c_matrix_destroy(h2c_matrix h) {
    if (h) cudaDeviceSynchronize();   // device work on any stream may still read it
    if (h) {
        // per-stream scratch is freed on its own stream; drop it while those streams still exist
        for (auto& kv : h->per_stream) kv.second.reset();
    }
    delete h;
}

int h2c_matrix_info(h2c_matrix h, int64_t* n, int* symmetric, int* orthonormal) {
    return guard([&] {
        need(h != nullptr, "null matrix");
        if (n) *n = h->h->tree().n;
        if (symmetric) *symmetric = h->h->symmetric;
        if (orthonormal) *orthonormal = h->h->orthonormal;
    });
}

int h2c_matrix_set_orthonormal(h2c_matrix h, int orthonormal) {
    return guard([&] {
        need(h != nullptr, "null matrix");
        h->h->orthonormal = orthonormal != 0;
    });
}

int h2c_matrix_sizes(h2c_matrix h, int64_t* sizes) {
    return guard([&] {
        need(h != nullptr && sizes != nullptr, "null argument");
        h2b::packed_sizes(*h->h, sizes);
    });
}

int h2c_matrix_ranks(h2c_matrix h, int* row_ranks, int* col_ranks) {
    return guard([&] {
        need(h != nullptr, "null matrix");
        const auto& m = *h->h;
        if (row_ranks) std::memcpy(row_ranks, m.row.rank.data(), m.row.rank.size() * sizeof(int));
        if (col_ranks) {
            const auto& r = m.vbasis().rank;
            std::memcpy(col_ranks, r.data(), r.size() * sizeof(int));
        }
    });
}

int h2c_matrix_upload(h2c_matrix h, const double* U, const double* E, const double* V, const double* F,
                      const double* S, const double* D) {
    return guard([&] {
        need(h != nullptr, "null matrix");
        const double* parts[6] = {U, E, V, F, S, D};
        h2b::upload_packed(*h->h, parts);
    });
}

int h2c_matrix_download(h2c_matrix h, double* U, double* E, double* V, double* F, double* S, double* D) {
    return guard([&] {
        need(h != nullptr, "null matrix");
        double* parts[6] = {U, E, V, F, S, D};
        h2b::download_packed(*h->h, parts);
    });
}

int h2c_matrix_kernel(h2c_block_tree b, const double* coords, int kind, double ell, int rank, h2c_matrix* out) {
    return guard([&] {
        need(b != nullptr && coords != nullptr && out != nullptr, "null argument");
        need(kind >= 0 && kind <= 2, "kernel kind must be 0, 1 or 2");
        need(rank >= 1, "rank must be >= 1");
        auto m = new h2c_matrix_s;
        try {
            m->h = h2b::make_kernel_h2(b->b, coords, kind, ell, rank);
        } catch (...) {
            delete m;
            throw;
        }
        *out = m;
    });
}

int h2c_matrix_kernel_sharded(h2c_block_tree b, const double* coords, int kind, double ell, int rank, int nranks,
                              int shard, h2c_matrix* out) {
    return guard([&] {
        need(b != nullptr && coords != nullptr && out != nullptr, "null argument");
        need(kind >= 0 && kind <= 2 && rank >= 1, "kernel: bad kind or rank");
        auto m = new h2c_matrix_s;
        try {
            m->h = h2b::make_kernel_h2(b->b, coords, kind, ell, rank, nranks, shard);
        } catch (...) {
            delete m;
            throw;
        }
        *out = m;
    });
}

int h2c_hgemv(h2c_matrix h, int transpose, int ordering, int64_t n, int64_t b, const double* x, int64_t ldx,
              double* y, int64_t ldy, double alpha, double beta, void* stream) {
    return guard([&] {
        need(h != nullptr, "null matrix");
        need(ordering == 0 || ordering == 1, "ordering must be 0 (user) or 1 (internal)");
        need(x != nullptr && y != nullptr, "null vector pointer");
        h2b::hgemv(*h->h, transpose != 0, ordering == 0, n, b, x, ldx, y, ldy, alpha, beta,
                   static_cast<cudaStream_t>(stream), h->ws_for(static_cast<cudaStream_t>(stream)));
    });
}

int h2c_matvec_host(h2c_matrix h, int transpose, int ordering, int64_t n, int64_t b, const double* x, double* y) {
    return guard([&] {
        need(h != nullptr, "null matrix");
        need(x != nullptr && y != nullptr, "null vector pointer");
        if (n != h->h->tree().n) throw std::invalid_argument("matvec: dimension mismatch");
        if (b < 1) throw std::invalid_argument("matvec: need at least one column");
        const size_t cnt = size_t(n * b);
        if (h->ws.hx.size() < cnt) h->ws.hx.resize(cnt);
        if (h->ws.hy.size() < cnt) h->ws.hy.resize(cnt);
        H2B_CUDA(cudaMemcpyAsync(h->ws.hx.data(), x, cnt * sizeof(double), cudaMemcpyHostToDevice, nullptr));
        h2b::hgemv(*h->h, transpose != 0, ordering == 0, n, b, h->ws.hx.data(), n, h->ws.hy.data(), n, 1.0, 0.0,
                   nullptr, h->ws);
        H2B_CUDA(cudaMemcpyAsync(y, h->ws.hy.data(), cnt * sizeof(double), cudaMemcpyDeviceToHost, nullptr));
        H2B_CUDA(cudaStreamSynchronize(nullptr));
    });
}

int h2c_matvec_host_async(h2c_matrix h, int transpose, int ordering, int64_t n, int64_t b, const double* x, double* y,
                          void* stream) {
    return guard([&] {
        need(h != nullptr, "null matrix");
        need(x != nullptr && y != nullptr, "null vector pointer");
        if (n != h->h->tree().n) throw std::invalid_argument("matvec: dimension mismatch");
        if (b < 1) throw std::invalid_argument("matvec: need at least one column");
        auto s = static_cast<cudaStream_t>(stream);
        h2b::Workspace& w = h->ws_for(s);
        const size_t cnt = size_t(n * b);
        if (w.hx.size() < cnt) w.hx.resize(cnt, s);
        if (w.hy.size() < cnt) w.hy.resize(cnt, s);
        H2B_CUDA(cudaMemcpyAsync(w.hx.data(), x, cnt * sizeof(double), cudaMemcpyHostToDevice, s));
        h2b::hgemv(*h->h, transpose != 0, ordering == 0, n, b, w.hx.data(), n, w.hy.data(), n, 1.0, 0.0, s, w);
        H2B_CUDA(cudaMemcpyAsync(y, w.hy.data(), cnt * sizeof(double), cudaMemcpyDeviceToHost, s));
    });
}

int h2c_hgemv_stage_times(h2c_matrix h, int transpose, int ordering, int64_t n, int64_t b, const double* x,
                          int64_t ldx, double* y, int64_t ldy, void* stream, int max_records, int* count,
                          int* stage, double* ms, double* flops, double* bytes) {
    return guard([&] {
        need(h != nullptr && count != nullptr, "null argument");
        std::vector<h2b::StageRecord> rec;
        h2b::hgemv_timed(*h->h, transpose != 0, ordering == 0, n, b, x, ldx, y, ldy, 1.0, 0.0,
                         static_cast<cudaStream_t>(stream), h->ws_for(static_cast<cudaStream_t>(stream)), rec);
        *count = int(rec.size());
        for (int i = 0; i < int(rec.size()) && i < max_records; ++i) {
            if (stage) stage[i] = rec[size_t(i)].stage;
            if (ms) ms[i] = rec[size_t(i)].ms;
            if (flops) flops[i] = rec[size_t(i)].flops;
            if (bytes) bytes[i] = rec[size_t(i)].bytes;
        }
    });
}

int h2c_hgemv_launches(h2c_matrix h, int transpose, int64_t b, int* launches) {
    return guard([&] {
        need(h != nullptr && launches != nullptr, "null argument");
        *launches = h2b::hgemv_launch_count(*h->h, transpose != 0, b);
    });
}

// ---- operators -------------------------------------------------------------
namespace {
struct CallbackError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
h2c_matrix wrap_matrix(std::unique_ptr<h2b::H2Dev> h) {
    auto m = new h2c_matrix_s;
    m->h = std::move(h);
    return m;
}
}  // namespace

int h2c_operator_dense(const double* a, int64_t n, int symmetric, h2c_operator* out) {
    return guard([&] {
        need(a != nullptr && out != nullptr && n > 0, "dense operator: null matrix or n < 1");
        *out = new h2c_operator_s{std::make_unique<h2b::DenseDevOperator>(a, n, symmetric != 0)};
    });
}

int h2c_operator_h2(h2c_matrix h, h2c_operator* out) {
    return guard([&] {
        need(h != nullptr && out != nullptr, "null argument");
        *out = new h2c_operator_s{std::make_unique<h2b::H2DevOperator>(*h->h)};
    });
}

int h2c_operator_device_callback(int64_t n, int symmetric, int has_transpose, h2c_apply_fn fn, void* ctx,
                                 h2c_operator* out) {
    return guard([&] {
        need(fn != nullptr && out != nullptr && n > 0, "callback operator: null function or n < 1");
        auto f = [fn, ctx](bool t, int64_t b, const double* x, double* y, cudaStream_t s) {
            if (fn(ctx, t ? 1 : 0, b, x, y, s) != 0) throw CallbackError("operator callback failed");
        };
        *out = new h2c_operator_s{std::make_unique<h2b::FunctionDevOperator>(n, symmetric != 0, f, has_transpose != 0)};
    });
}

int h2c_operator_host_callback(int64_t n, int symmetric, int has_transpose, h2c_apply_fn fn, void* ctx,
                               h2c_operator* out) {
    return guard([&] {
        need(fn != nullptr && out != nullptr && n > 0, "callback operator: null function or n < 1");
        auto f = [fn, ctx, n](bool t, int64_t b, const double* x, double* y, cudaStream_t s) {
            std::vector<double> hx(size_t(n * b)), hy(size_t(n * b));
            H2B_CUDA(cudaMemcpyAsync(hx.data(), x, hx.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
            H2B_CUDA(cudaStreamSynchronize(s));
            if (fn(ctx, t ? 1 : 0, b, hx.data(), hy.data(), nullptr) != 0) throw CallbackError("operator callback failed");
            H2B_CUDA(cudaMemcpyAsync(y, hy.data(), hy.size() * sizeof(double), cudaMemcpyHostToDevice, s));
            H2B_CUDA(cudaStreamSynchronize(s));
        };
        *out = new h2c_operator_s{std::make_unique<h2b::FunctionDevOperator>(n, symmetric != 0, f, has_transpose != 0)};
    });
}

void h2c_operator_destroy(h2c_operator op) { delete op; }

int h2c_operator_apply(h2c_operator op, int transpose, int64_t b, const double* x, double* y, void* stream) {
    return guard([&] {
        need(op != nullptr && x != nullptr && y != nullptr, "null argument");
        need(b >= 1, "operator apply: need at least one column");
        auto s = static_cast<cudaStream_t>(stream);
        if (transpose) op->op->apply_transpose(b, x, y, s);
        else op->op->apply(b, x, y, s);
    });
}

int h2c_operator_apply_host(h2c_operator op, int transpose, int64_t b, const double* x, double* y) {
    return guard([&] {
        need(op != nullptr && x != nullptr && y != nullptr, "null argument");
        need(b >= 1, "operator apply: need at least one column");
        const size_t nb = size_t(op->op->dim()) * size_t(b);
        h2b::DeviceArray<double> dx(nb, nullptr), dy(nb, nullptr);
        H2B_CUDA(cudaMemcpy(dx.data(), x, nb * sizeof(double), cudaMemcpyHostToDevice));
        if (transpose) op->op->apply_transpose(b, dx.data(), dy.data(), nullptr);
        else op->op->apply(b, dx.data(), dy.data(), nullptr);
        H2B_CUDA(cudaMemcpy(y, dy.data(), nb * sizeof(double), cudaMemcpyDeviceToHost));
    });
}

int h2c_operator_columns_applied(h2c_operator op, int64_t* cols) {
    return guard([&] {
        need(op != nullptr && cols != nullptr, "null argument");
        *cols = op->op->columns_applied();
    });
}

int h2c_operator_reset_counter(h2c_operator op) {
    return guard([&] {
        need(op != nullptr, "null argument");
        op->op->reset_counter();
    });
}

int h2c_pnorm2_estimate(h2c_operator op, double* value, int* iterations) {
    return guard([&] {
        need(op != nullptr && value != nullptr, "null argument");
        const h2b::NormEstimate e = h2b::pnorm2_estimate(*op->op, nullptr);
        *value = e.value;
        if (iterations) *iterations = e.iterations;
    });
}

int h2c_orthogonalize(h2c_matrix in, h2c_matrix* out) {
    return guard([&] {
        need(in != nullptr && out != nullptr, "null argument");
        *out = wrap_matrix(h2b::orthogonalize(*in->h, nullptr));
    });
}

int h2c_recompress(h2c_matrix in, double eps, h2c_matrix* out) {
    return guard([&] {
        need(in != nullptr && out != nullptr, "null argument");
        *out = wrap_matrix(h2b::recompress(*in->h, eps, nullptr));
    });
}

void h2c_peel_config_default(h2c_peel_config* cfg) {
    if (!cfg) return;
    const h2b::PeelConfig d;
    cfg->eps = d.eps;
    cfg->sample_block_size = d.sample_block_size;
    cfg->oversampling = d.oversampling;
    cfg->max_rank = d.max_rank;
    cfg->seed = d.seed;
    cfg->norm_scale = d.norm_scale;
    cfg->crossover_rank_cap = d.crossover_rank_cap;
    cfg->rng = d.rng;
}

int h2c_peel_construct(h2c_operator op, h2c_block_tree bt, const h2c_peel_config* cfg, h2c_matrix* out,
                       int64_t* total_samples, h2c_level_stats* levels, int max_levels, int* num_levels,
                       double* op_ms, double* total_ms) {
    return guard([&] {
        need(op != nullptr && bt != nullptr && out != nullptr, "null argument");
        h2b::PeelConfig c;
        if (cfg) {
            c.eps = cfg->eps;
            c.sample_block_size = cfg->sample_block_size;
            c.oversampling = cfg->oversampling;
            c.max_rank = cfg->max_rank;
            c.seed = cfg->seed;
            c.norm_scale = cfg->norm_scale;
            c.crossover_rank_cap = cfg->crossover_rank_cap;
            c.rng = cfg->rng;
        }
        h2b::PeelResult r = h2b::peel_construct(*op->op, bt->b, c, nullptr);
        if (total_samples) *total_samples = r.stats.total;
        if (num_levels) *num_levels = int(r.stats.levels.size());
        if (levels)
            for (int i = 0; i < int(r.stats.levels.size()) && i < max_levels; ++i) {
                const h2b::LevelStats& l = r.stats.levels[size_t(i)];
                levels[i] = h2c_level_stats{l.level, l.blocks, l.max_rank, l.samples};
            }
        if (op_ms) *op_ms = r.times.op_ms;
        if (total_ms) *total_ms = r.times.total_ms;
        *out = wrap_matrix(std::move(r.matrix));
    });
}

int h2c_estimate_relative_error(h2c_operator op, h2c_matrix h, double op_norm, double* out) {
    return guard([&] {
        need(op != nullptr && h != nullptr && out != nullptr, "null argument");
        *out = h2b::estimate_relative_error(*op->op, *h->h, op_norm, nullptr);
    });
}

// ---- sharded hgemv ----------------------------------------------------------
int h2c_dist_plan_create(h2c_matrix h, int transpose, int nranks, int rank, h2c_dist_plan* out) {
    return guard([&] {
        need(h != nullptr && out != nullptr, "null argument");
        *out = new h2c_dist_plan_s{h2b::make_dist_plan(*h->h, transpose != 0, nranks, rank)};
    });
}

void h2c_dist_plan_destroy(h2c_dist_plan p) {
    if (p) cudaDeviceSynchronize();
    delete p;
}

int h2c_dist_plan_counts(h2c_dist_plan p, int64_t* send_rows, int64_t* recv_rows, int64_t* owned_begin,
                         int64_t* owned_rows) {
    return guard([&] {
        need(p != nullptr, "null argument");
        std::vector<int64_t> s, r;
        h2b::dist_counts(*p->p, s, r);
        for (size_t i = 0; i < s.size(); ++i) {
            if (send_rows) send_rows[i] = s[i];
            if (recv_rows) recv_rows[i] = r[i];
        }
        int64_t beg = 0;
        const int64_t rows = h2b::dist_owned_rows(*p->p, &beg);
        if (owned_begin) *owned_begin = beg;
        if (owned_rows) *owned_rows = rows;
    });
}

int h2c_dist_plan_launches(h2c_dist_plan p, int* launches) {
    return guard([&] {
        need(p != nullptr && launches != nullptr, "null argument");
        *launches = h2b::dist_launch_count(*p->p);
    });
}

int h2c_dist_hgemv_begin(h2c_dist_plan p, int64_t b, const double* x, int64_t ldx, double* sendbuf, void* stream) {
    return guard([&] {
        need(p != nullptr && x != nullptr, "null argument");
        need(b >= 1, "matvec: need at least one column");
        h2b::dist_hgemv_begin(*p->p, b, x, ldx, sendbuf, static_cast<cudaStream_t>(stream));
    });
}

int h2c_dist_hgemv_local(h2c_dist_plan p, int64_t b, void* stream) {
    return guard([&] {
        need(p != nullptr, "null plan");
        need(b >= 1, "dist hgemv: need at least one column");
        h2b::dist_hgemv_local(*p->p, b, static_cast<cudaStream_t>(stream));
    });
}
int h2c_dist_hgemv_end(h2c_dist_plan p, int64_t b, const double* recvbuf, double* y, int64_t ldy, double alpha,
                       double beta, void* stream) {
    return guard([&] {
        need(p != nullptr && y != nullptr, "null argument");
        need(b >= 1, "matvec: need at least one column");
        h2b::dist_hgemv_end(*p->p, b, recvbuf, y, ldy, alpha, beta, static_cast<cudaStream_t>(stream));
    });
}

int h2c_dist_hgemv_nccl(h2c_dist_plan p, void* nccl_comm, int64_t b, const double* x, int64_t ldx, double* y,
                        int64_t ldy, double alpha, double beta, void* stream) {
    return guard([&] {
        need(p != nullptr && x != nullptr && y != nullptr, "null argument");
        need(b >= 1, "matvec: need at least one column");
        h2b::dist_hgemv_nccl(*p->p, nccl_comm, b, x, ldx, y, ldy, alpha, beta, static_cast<cudaStream_t>(stream));
    });
}
int h2c_dist_hgemv_nccl_owned(h2c_dist_plan p, void* nccl_comm, int64_t b, const double* x_owned, int64_t ldx,
                              double* y_owned, int64_t ldy, double alpha, double beta, void* stream) {
    return guard([&] {
        need(p != nullptr && x_owned != nullptr && y_owned != nullptr, "null argument");
        need(b >= 1, "matvec: need at least one column");
        h2b::dist_hgemv_nccl(*p->p, nccl_comm, b, x_owned, ldx, y_owned, ldy, alpha, beta,
                             static_cast<cudaStream_t>(stream), true);
    });
}

int h2c_dist_peer_alloc(h2c_dist_plan p, int64_t max_b) {
    return guard([&] {
        need(p != nullptr, "null plan");
        h2b::dist_peer_alloc(*p->p, max_b);
    });
}
int h2c_dist_peer_export(h2c_dist_plan p, void* handles, int64_t* recv_off) {
    return guard([&] {
        need(p != nullptr && handles != nullptr && recv_off != nullptr, "null argument");
        static_assert(sizeof(h2b::PeerHandles) == 128, "two CUDA IPC handles");
        std::vector<int64_t> off;
        const h2b::PeerHandles h = h2b::dist_peer_export(*p->p, off);
        std::memcpy(handles, &h, sizeof(h));
        std::copy(off.begin(), off.end(), recv_off);
    });
}
int h2c_dist_peer_import(h2c_dist_plan p, const void* handles, const int64_t* recv_offs) {
    return guard([&] {
        need(p != nullptr && handles != nullptr && recv_offs != nullptr, "null argument");
        int64_t P = 0;
        std::vector<int64_t> s, r;
        h2b::dist_counts(*p->p, s, r);
        P = int64_t(s.size());
        std::vector<h2b::PeerHandles> all(static_cast<size_t>(P));
        std::memcpy(all.data(), handles, size_t(P) * sizeof(h2b::PeerHandles));
        h2b::dist_peer_import(*p->p, all, std::vector<int64_t>(recv_offs, recv_offs + P * P));
    });
}
int h2c_dist_peer_link(h2c_dist_plan* plans, int n) {
    return guard([&] {
        need(plans != nullptr && n >= 1, "null argument");
        std::vector<h2b::DistPlan*> v;
        for (int i = 0; i < n; ++i) {
            need(plans[i] != nullptr, "null plan");
            v.push_back(plans[i]->p.get());
        }
        h2b::dist_peer_link(v);
    });
}

int h2c_dist_hgemv_begin_owned(h2c_dist_plan p, int64_t b, const double* x_owned, int64_t ldx, double* sendbuf,
                               void* stream) {
    return guard([&] {
        need(p != nullptr && x_owned != nullptr, "null argument");
        need(b >= 1, "matvec: need at least one column");
        h2b::dist_hgemv_begin(*p->p, b, x_owned, ldx, sendbuf, static_cast<cudaStream_t>(stream), true);
    });
}
int h2c_dist_hgemv_end_owned(h2c_dist_plan p, int64_t b, const double* recvbuf, double* y_owned, int64_t ldy,
                             double alpha, double beta, void* stream) {
    return guard([&] {
        need(p != nullptr && y_owned != nullptr, "null argument");
        need(b >= 1, "matvec: need at least one column");
        h2b::dist_hgemv_end(*p->p, b, recvbuf, y_owned, ldy, alpha, beta, static_cast<cudaStream_t>(stream), true);
    });
}

int h2c_partition_owner(h2c_block_tree b, int nranks, int* owner) {
    return guard([&] {
        need(b != nullptr && owner != nullptr, "null argument");
        const h2b::DistSpec d = h2b::make_dist_spec(*b->b->tree, nranks, 0);
        std::copy(d.owner.begin(), d.owner.end(), owner);
    });
}

int h2c_partition_exchange(h2c_block_tree b, int symmetric, int transpose, const int* up_ranks, int nranks, int src,
                           int dst, int64_t* count, int* arr, int* node, int64_t* rows) {
    return guard([&] {
        need(b != nullptr && up_ranks != nullptr && count != nullptr, "null argument");
        need(src >= 0 && src < nranks && dst >= 0 && dst < nranks, "rank out of range");
        const h2b::ClusterTree& ct = *b->b->tree;
        const h2b::DistSpec d = h2b::make_dist_spec(ct, nranks, dst);
        std::vector<int> ur(up_ranks, up_ranks + ct.num_nodes());
        std::vector<int64_t> cu(size_t(ct.num_nodes()));
        int64_t o = 0;
        for (int v = 0; v < ct.num_nodes(); ++v) {
            cu[size_t(v)] = o;
            o += ur[size_t(v)];
        }
        const auto items = h2b::exchange_items(*b->b, symmetric != 0, transpose != 0, ur, d, src, dst, cu);
        *count = int64_t(items.size());
        if (arr)
            for (size_t i = 0; i < items.size(); ++i) {
                arr[i] = items[i].arr;
                if (node) node[i] = items[i].node;
                if (rows) rows[i] = items[i].rows;
            }
    });
}

// ---- inversion ------------------------------------------------------------------
int h2c_scaled_identity(h2c_block_tree b, double value, h2c_matrix* out) {
    return guard([&] {
        need(b != nullptr && out != nullptr, "null argument");
        *out = wrap_matrix(h2b::scaled_identity(b->b, value, nullptr));
    });
}

int h2c_matrix_add_diagonal(h2c_matrix h, double value) {
    return guard([&] {
        need(h != nullptr, "null argument");
        h2b::add_diagonal(*h->h, value, nullptr);
    });
}

int h2c_scaled_identity_start(h2c_matrix a, h2c_matrix* out) {
    return guard([&] {
        need(a != nullptr && out != nullptr, "null argument");
        *out = wrap_matrix(h2b::scaled_identity_start(*a->h, nullptr));
    });
}

int h2c_pnorm_estimate(h2c_operator op, double p, double* value, int* iterations) {
    return guard([&] {
        need(op != nullptr && value != nullptr, "null argument");
        h2b::NormEstimate e;
        if (p == 2.0) e = h2b::pnorm2_estimate(*op->op, nullptr);
        else if (p == 1.0) e = h2b::pnorm_1inf_estimate(*op->op, false, nullptr);
        else if (std::isinf(p)) e = h2b::pnorm_1inf_estimate(*op->op, true, nullptr);
        else throw std::invalid_argument("pnorm_estimate: p must be 1, 2 or inf");
        *value = e.value;
        if (iterations) *iterations = e.iterations;
    });
}

int h2c_sampler_operator(h2c_matrix xk, h2c_matrix a, int kind, int arg, h2c_operator* out) {
    return guard([&] {
        need(xk != nullptr && a != nullptr && out != nullptr, "null argument");
        std::unique_ptr<h2b::DevOperator> op;
        if (kind == 0) op = h2b::ns_sampler(*xk->h, *a->h);
        else if (kind == 1) op = h2b::hyperpower_sampler(*xk->h, *a->h, arg);
        else if (kind == 2) op = h2b::unrolled_sampler(*xk->h, *a->h, arg);
        else throw std::invalid_argument("sampler kind must be 0, 1 or 2");
        *out = new h2c_operator_s{std::move(op)};
    });
}

int h2c_residual_norm(h2c_matrix a, h2c_matrix x, double* out) {
    return guard([&] {
        need(a != nullptr && x != nullptr && out != nullptr, "null argument");
        *out = h2b::residual_norm(*a->h, *x->h, nullptr);
    });
}

int h2c_residual_norm_op(h2c_operator a, h2c_operator x, double* out) {
    return guard([&] {
        need(a != nullptr && x != nullptr && out != nullptr, "null argument");
        *out = h2b::residual_norm(*a->op, *x->op, nullptr);
    });
}

namespace {
void export_trace(const h2b::ConvergenceTrace& t, h2c_trace_row* rows, int max_rows, int* num_rows,
                  double* final_residual, int* converged) {
    if (num_rows) *num_rows = int(t.rows.size());
    if (rows)
        for (int i = 0; i < int(t.rows.size()) && i < max_rows; ++i) {
            const h2b::TraceRow& r = t.rows[size_t(i)];
            rows[i] = h2c_trace_row{r.iter, r.residual, r.eps_k, r.samples, r.wall_seconds};
        }
    if (final_residual) *final_residual = t.final_residual;
    if (converged) *converged = t.converged ? 1 : 0;
}
}  // namespace

int h2c_h_inverse(h2c_matrix a, h2c_matrix x0, int method, int arg, int dynamic_schedule, double eps_initial,
                  double eps, const h2c_peel_config* cfg, int max_iter, h2c_matrix* out, h2c_trace_row* rows,
                  int max_rows, int* num_rows, double* final_residual, int* converged) {
    return guard([&] {
        need(a != nullptr && x0 != nullptr && out != nullptr, "null argument");
        h2b::PeelConfig c;
        if (cfg) {
            c.eps = cfg->eps;
            c.sample_block_size = cfg->sample_block_size;
            c.oversampling = cfg->oversampling;
            c.max_rank = cfg->max_rank;
            c.seed = cfg->seed;
            c.norm_scale = cfg->norm_scale;
            c.crossover_rank_cap = cfg->crossover_rank_cap;
            c.rng = cfg->rng;
        }
        h2b::ThresholdSchedule sched;
        sched.dynamic = dynamic_schedule != 0;
        sched.eps_initial = eps_initial;
        try {
            h2b::InverseResult r = method == 2 ? h2b::h_unrolled(*a->h, *x0->h, arg, eps, c, nullptr)
                                               : h2b::h_iterative_inverse(*a->h, *x0->h, sched, eps, c, method, arg,
                                                                          max_iter, nullptr);
            export_trace(r.trace, rows, max_rows, num_rows, final_residual, converged);
            *out = wrap_matrix(std::move(r.X));
        } catch (const h2b::divergence_error& e) {
            export_trace(e.trace, rows, max_rows, num_rows, final_residual, converged);
            throw;
        }
    });
}

int h2c_low_rank_update(h2c_matrix h, int64_t k, const double* X, const double* Y, double eps, h2c_matrix* out) {
    return guard([&] {
        need(h != nullptr && out != nullptr, "null argument");
        need(k == 0 || (X != nullptr && Y != nullptr), "null factor");
        *out = wrap_matrix(h2b::low_rank_update(*h->h, X, Y, int(k), eps, nullptr));
    });
}

int h2c_desymmetrized(h2c_matrix h, h2c_matrix* out) {
    return guard([&] {
        need(h != nullptr && out != nullptr, "null argument");
        *out = wrap_matrix(h2b::desymmetrized(*h->h, nullptr));
    });
}

// ---- randomized low-rank / hybrid ---------------------------------------------------
namespace {
h2b::PeelConfig to_cfg(const h2c_peel_config* cfg) {
    h2b::PeelConfig c;
    if (cfg) {
        c.eps = cfg->eps;
        c.sample_block_size = cfg->sample_block_size;
        c.oversampling = cfg->oversampling;
        c.max_rank = cfg->max_rank;
        c.seed = cfg->seed;
        c.norm_scale = cfg->norm_scale;
        c.crossover_rank_cap = cfg->crossover_rank_cap;
        c.rng = cfg->rng;
    }
    return c;
}
}  // namespace

int h2c_randomized_lowrank(h2c_operator op, double eps, int64_t max_rank, const h2c_peel_config* cfg,
                           h2c_lowrank* out) {
    return guard([&] {
        need(op != nullptr && out != nullptr, "null argument");
        auto f = new h2c_lowrank_s;
        try {
            f->r = h2b::randomized_lowrank(*op->op, eps, max_rank, to_cfg(cfg), 0, nullptr);
            f->n = op->op->dim();
        } catch (...) {
            delete f;
            throw;
        }
        *out = f;
    });
}

int h2c_lowrank_info(h2c_lowrank f, int64_t* n, int64_t* rank, int* symmetric_form, double* residual_estimate,
                     int* max_rank_reached, int64_t* total_samples) {
    return guard([&] {
        need(f != nullptr, "null argument");
        if (n) *n = f->n;
        if (rank) *rank = f->r.rank;
        if (symmetric_form) *symmetric_form = f->r.X == f->r.Y ? 1 : 0;
        if (residual_estimate) *residual_estimate = f->r.residual_estimate;
        if (max_rank_reached) *max_rank_reached = f->r.max_rank_reached ? 1 : 0;
        if (total_samples) *total_samples = f->r.stats.total;
    });
}

int h2c_lowrank_download(h2c_lowrank f, double* X, double* Y) {
    return guard([&] {
        need(f != nullptr, "null argument");
        const size_t cnt = size_t(f->n * f->r.rank);
        if (cnt == 0) return;
        if (X) H2B_CUDA(cudaMemcpy(X, f->r.X->data(), cnt * sizeof(double), cudaMemcpyDeviceToHost));
        if (Y) H2B_CUDA(cudaMemcpy(Y, f->r.Y->data(), cnt * sizeof(double), cudaMemcpyDeviceToHost));
    });
}

void h2c_lowrank_destroy(h2c_lowrank f) {
    if (f) cudaDeviceSynchronize();
    delete f;
}

int h2c_hybrid_construct(h2c_operator op, h2c_block_tree bt, const h2c_peel_config* cfg, h2c_matrix* out,
                         int64_t* global_rank, int64_t* total_samples, h2c_level_stats* levels, int max_levels,
                         int* num_levels) {
    return guard([&] {
        need(op != nullptr && bt != nullptr && out != nullptr, "null argument");
        h2b::HybridResultDev r = h2b::hybrid_construct(*op->op, bt->b, to_cfg(cfg), nullptr);
        if (global_rank) *global_rank = r.global_rank;
        if (total_samples) *total_samples = r.stats.total;
        if (num_levels) *num_levels = int(r.stats.levels.size());
        if (levels)
            for (int i = 0; i < int(r.stats.levels.size()) && i < max_levels; ++i) {
                const h2b::LevelStats& l = r.stats.levels[size_t(i)];
                levels[i] = h2c_level_stats{l.level, l.blocks, l.max_rank, l.samples};
            }
        *out = wrap_matrix(std::move(r.matrix));
    });
}

// ---- H2M1 --------------------------------------------------------------------------
int h2c_serialize_size(h2c_matrix h, int64_t* bytes) {
    return guard([&] {
        need(h != nullptr && bytes != nullptr, "null argument");
        *bytes = int64_t(h2b::serialize(*h->h).size());
    });
}

int h2c_serialize(h2c_matrix h, void* buf, int64_t bytes) {
    return guard([&] {
        need(h != nullptr && buf != nullptr, "null argument");
        const std::string s = h2b::serialize(*h->h);
        need(int64_t(s.size()) <= bytes, "serialize: buffer too small");
        std::memcpy(buf, s.data(), s.size());
    });
}

namespace {
void wrap_deserialized(h2b::Deserialized d, h2c_block_tree* bt_out, h2c_matrix* out) {
    auto bt = new h2c_block_tree_s{std::const_pointer_cast<h2b::BlockTree>(d.bt)};
    *out = wrap_matrix(std::move(d.h));
    *bt_out = bt;
}
}  // namespace

int h2c_deserialize(const void* buf, int64_t bytes, h2c_block_tree* bt_out, h2c_matrix* out) {
    return guard([&] {
        need(buf != nullptr && bt_out != nullptr && out != nullptr && bytes >= 0, "null argument");
        wrap_deserialized(h2b::deserialize(static_cast<const char*>(buf), size_t(bytes)), bt_out, out);
    });
}

int h2c_write_h2_file(h2c_matrix h, const char* path) {
    return guard([&] {
        need(h != nullptr && path != nullptr, "null argument");
        const std::string s = h2b::serialize(*h->h);
        FILE* f = std::fopen(path, "wb");
        if (!f) throw h2b::io_error(h2b::io_error::malformed, std::string("cannot open ") + path + " for writing");
        const size_t w = std::fwrite(s.data(), 1, s.size(), f);
        std::fclose(f);
        if (w != s.size()) throw h2b::io_error(h2b::io_error::malformed, std::string("short write to ") + path);
    });
}

int h2c_read_h2_file(const char* path, h2c_block_tree* bt_out, h2c_matrix* out) {
    return guard([&] {
        need(path != nullptr && bt_out != nullptr && out != nullptr, "null argument");
        FILE* f = std::fopen(path, "rb");
        if (!f) throw h2b::io_error(h2b::io_error::malformed, std::string("cannot open ") + path);
        std::string s;
        char tmp[1 << 16];
        size_t r;
        while ((r = std::fread(tmp, 1, sizeof tmp, f)) > 0) s.append(tmp, r);
        std::fclose(f);
        wrap_deserialized(h2b::deserialize(s.data(), s.size()), bt_out, out);
    });
}

int h2c_last_io_error_kind(void) { return g_io_kind; }

// ---- diffusion1d device operator ----
struct h2c_diff1d_s {
    std::shared_ptr<h2b::Diffusion1DDev> d;
};

void h2c_diff1d_config_default(h2c_diff1d_config* cfg) {
    if (!cfg) return;
    const h2b::Diff1DConfig d;
    cfg->n = d.n;
    cfg->steps = d.steps;
    cfg->final_time = d.final_time;
    cfg->t_p = d.t_p;
    cfg->t_0 = d.t_0;
    cfg->source_amplitude = d.source_amplitude;
    cfg->alpha = d.alpha;
    cfg->beta = d.beta;
    cfg->pad = d.pad;
    cfg->num_sources = int(d.source_positions.size());
    cfg->source_positions = nullptr;
    cfg->num_receivers = d.num_receivers;
}

int h2c_diff1d_create(const h2c_diff1d_config* cfg, void* stream, h2c_diff1d* out) {
    return guard([&] {
        need(cfg != nullptr && out != nullptr, "null argument");
        h2b::Diff1DConfig c;
        c.n = cfg->n;
        c.steps = cfg->steps;
        c.final_time = cfg->final_time;
        c.t_p = cfg->t_p;
        c.t_0 = cfg->t_0;
        c.source_amplitude = cfg->source_amplitude;
        c.alpha = cfg->alpha;
        c.beta = cfg->beta;
        c.pad = cfg->pad;
        if (cfg->source_positions) {
            need(cfg->num_sources > 0, "diffusion1d: num_sources < 1");
            c.source_positions.assign(cfg->source_positions, cfg->source_positions + cfg->num_sources);
        }
        c.num_receivers = cfg->num_receivers;
        auto s = static_cast<cudaStream_t>(stream);
        auto d = std::make_shared<h2b::Diffusion1DDev>(c, s);
        H2B_CUDA(cudaStreamSynchronize(s));
        *out = new h2c_diff1d_s{std::move(d)};
    });
}

void h2c_diff1d_destroy(h2c_diff1d d) { delete d; }

int h2c_diff1d_info(h2c_diff1d d, int64_t* nstate, int64_t* npad, double* spacing, double* dt, int64_t* pde_solves) {
    return guard([&] {
        need(d != nullptr, "null argument");
        if (nstate) *nstate = d->d->nstate();
        if (npad) *npad = d->d->npad();
        if (spacing) *spacing = d->d->spacing();
        if (dt) *dt = d->d->dt();
        if (pde_solves) *pde_solves = d->d->pde_solves();
    });
}

int h2c_diff1d_hessvec(h2c_diff1d d, int include_tv, int64_t b, const double* x, double* y, void* stream) {
    return guard([&] {
        need(d != nullptr && x != nullptr && y != nullptr, "null argument");
        d->d->hessvec(include_tv != 0, b, x, y, static_cast<cudaStream_t>(stream));
    });
}

int h2c_diff1d_state_field(h2c_diff1d d, int source, double* out) {
    return guard([&] {
        need(d != nullptr && out != nullptr, "null argument");
        auto v = d->d->state_field(source, nullptr);
        std::memcpy(out, v.data(), v.size() * sizeof(double));
    });
}

int h2c_diff1d_operator(h2c_diff1d d, int include_tv, h2c_operator* out) {
    return guard([&] {
        need(d != nullptr && out != nullptr, "null argument");
        *out = new h2c_operator_s{h2b::diffusion_hessian_operator(d->d, include_tv != 0)};
    });
}

struct h2c_surface_s {
    std::shared_ptr<h2b::MinimalSurfaceDev> s;
};

int h2c_surface_create(int64_t interior, double rim, int newton_steps, h2c_surface* out) {
    return guard([&] {
        need(out != nullptr, "null argument");
        auto s = std::make_shared<h2b::MinimalSurfaceDev>(interior, rim, newton_steps);
        H2B_CUDA(cudaDeviceSynchronize());   // CSR uploads complete before any stream uses them
        *out = new h2c_surface_s{std::move(s)};
    });
}

void h2c_surface_destroy(h2c_surface s) { delete s; }

int h2c_surface_info(h2c_surface s, int64_t* n, int64_t* nnz, double* spacing) {
    return guard([&] {
        need(s != nullptr, "null argument");
        if (n) *n = s->s->n();
        if (nnz) *nnz = s->s->nnz();
        if (spacing) *spacing = s->s->spacing();
    });
}

int h2c_surface_state(h2c_surface s, double* out) {
    return guard([&] {
        need(s != nullptr && out != nullptr, "null argument");
        std::memcpy(out, s->s->state().data(), s->s->state().size() * sizeof(double));
    });
}

int h2c_surface_hessvec(h2c_surface s, int64_t b, const double* x, double* y, void* stream) {
    return guard([&] {
        need(s != nullptr && x != nullptr && y != nullptr, "null argument");
        s->s->hessvec(b, x, y, static_cast<cudaStream_t>(stream));
    });
}

int h2c_surface_operator(h2c_surface s, h2c_operator* out) {
    return guard([&] {
        need(s != nullptr && out != nullptr, "null argument");
        *out = new h2c_operator_s{h2b::surface_hessian_operator(s->s)};
    });
}

struct h2c_advdiff_s {
    std::shared_ptr<h2b::AdvDiff2DDev> a;
};

void h2c_advdiff_config_default(h2c_advdiff_config* cfg) {
    if (!cfg) return;
    const h2b::AdvDiffConfig d;
    cfg->grid = d.grid;
    cfg->kappa = d.kappa;
    cfg->reaction = d.reaction;
    cfg->num_observations = d.num_observations;
    cfg->noise_rel = d.noise_rel;
    cfg->obs_seed = d.obs_seed;
}

int h2c_advdiff_create(const h2c_advdiff_config* cfg, h2c_advdiff* out) {
    return guard([&] {
        need(cfg != nullptr && out != nullptr, "null argument");
        h2b::AdvDiffConfig c;
        c.grid = cfg->grid;
        c.kappa = cfg->kappa;
        c.reaction = cfg->reaction;
        c.num_observations = cfg->num_observations;
        c.noise_rel = cfg->noise_rel;
        c.obs_seed = cfg->obs_seed;
        *out = new h2c_advdiff_s{std::make_shared<h2b::AdvDiff2DDev>(c)};
    });
}

void h2c_advdiff_destroy(h2c_advdiff a) { delete a; }

int h2c_advdiff_info(h2c_advdiff a, int64_t* n, double* sigma, int64_t* num_observations, int64_t* solves) {
    return guard([&] {
        need(a != nullptr, "null argument");
        if (n) *n = a->a->n();
        if (sigma) *sigma = a->a->sigma();
        if (num_observations) *num_observations = int64_t(a->a->observation_nodes().size());
        if (solves) *solves = a->a->solves();
    });
}

int h2c_advdiff_observations(h2c_advdiff a, int64_t* out) {
    return guard([&] {
        need(a != nullptr && out != nullptr, "null argument");
        const auto& o = a->a->observation_nodes();
        std::memcpy(out, o.data(), o.size() * sizeof(int64_t));
    });
}

int h2c_advdiff_hessvec(h2c_advdiff a, int64_t b, const double* x, double* y, void* stream) {
    return guard([&] {
        need(a != nullptr && x != nullptr && y != nullptr, "null argument");
        a->a->misfit_hessvec(b, x, y, static_cast<cudaStream_t>(stream));
    });
}

int h2c_advdiff_operator(h2c_advdiff a, h2c_operator* out) {
    return guard([&] {
        need(a != nullptr && out != nullptr, "null argument");
        *out = new h2c_operator_s{h2b::advdiff_hessian_operator(a->a)};
    });
}


// ---- block-level construction primitives (construction.hpp:137-198) -------------
int h2c_rng_create(uint64_t seed, h2c_rng* out) {
    return guard([&] {
        need(out != nullptr, "null output handle");
        *out = new h2c_rng_s{std::mt19937_64(seed)};
    });
}
void h2c_rng_destroy(h2c_rng r) { delete r; }
int h2c_rng_set_state(h2c_rng r, const char* state) {
    return guard([&] {
        need(r != nullptr && state != nullptr, "null argument");
        std::istringstream in(state);
        in >> r->g;
        need(!in.fail(), "h2c_rng_set_state: malformed engine state");
    });
}
int h2c_rng_get_state(h2c_rng r, char* buf, int64_t* bytes) {
    return guard([&] {
        need(r != nullptr && bytes != nullptr, "null argument");
        std::ostringstream out;
        out << r->g;
        const std::string st = out.str();
        const int64_t cap = *bytes;
        *bytes = int64_t(st.size()) + 1;
        if (buf && cap >= *bytes) std::memcpy(buf, st.c_str(), st.size() + 1);
    });
}
int h2c_rng_fill_gaussian(h2c_rng r, int64_t rows, int64_t cols, double* out) {
    return guard([&] {
        need(r != nullptr && (out != nullptr || rows * cols == 0), "null argument");
        need(rows >= 0 && cols >= 0, "negative size");
        h2b::ref_fill_gaussian(out, rows, cols, rows, r->g);
    });
}

int h2c_sample_block_column(h2c_operator op, h2c_cluster_tree ct, int t, int s, int64_t count, h2c_rng rng,
                            double* omega_s, double* y_t, void* stream) {
    return guard([&] {
        need(op != nullptr && ct != nullptr && rng != nullptr, "null argument");
        need(omega_s != nullptr && y_t != nullptr, "null output buffer");
        need(op->op->dim() == ct->t->n, "sample_block_column: operator and tree sizes differ");
        h2b::sample_block_column(*op->op, *ct->t, t, s, count, rng->g, omega_s, y_t,
                                 static_cast<cudaStream_t>(stream));
    });
}

int h2c_sample_block_column_host(h2c_operator op, h2c_cluster_tree ct, int t, int s, int64_t count, h2c_rng rng,
                                 double* omega_s, double* y_t) {
    return guard([&] {
        need(op != nullptr && ct != nullptr && rng != nullptr, "null argument");
        need(omega_s != nullptr && y_t != nullptr, "null output buffer");
        need(op->op->dim() == ct->t->n, "sample_block_column: operator and tree sizes differ");
        need(t >= 0 && t < ct->t->num_nodes() && s >= 0 && s < ct->t->num_nodes(),
             "sample_block_column: cluster id out of range");
        const size_t no = size_t(std::max<int64_t>(count, 0) * ct->t->size(s));
        const size_t ny = size_t(std::max<int64_t>(count, 0) * ct->t->size(t));
        h2b::DeviceArray<double> om(std::max<size_t>(no, 1)), y(std::max<size_t>(ny, 1));
        h2b::sample_block_column(*op->op, *ct->t, t, s, count, rng->g, om.data(), y.data(), nullptr);
        H2B_CUDA(cudaMemcpy(omega_s, om.data(), no * sizeof(double), cudaMemcpyDeviceToHost));
        H2B_CUDA(cudaMemcpy(y_t, y.data(), ny * sizeof(double), cudaMemcpyDeviceToHost));
    });
}

int h2c_adaptive_block_factorization(h2c_operator op, h2c_cluster_tree ct, int t, int s, double eps_block,
                                     const h2c_peel_config* cfg, h2c_block_factor* out) {
    return guard([&] {
        need(op != nullptr && ct != nullptr && out != nullptr, "null argument");
        need(op->op->dim() == ct->t->n, "adaptive_block_factorization: operator and tree sizes differ");
        auto f = std::make_unique<h2c_block_factor_s>();
        f->f = h2b::adaptive_block_factorization(*op->op, *ct->t, t, s, eps_block, to_cfg(cfg), nullptr);
        f->rows_u = ct->t->size(t);
        f->rows_v = ct->t->size(s);
        *out = f.release();
    });
}
int h2c_block_factor_info(h2c_block_factor f, int64_t* rows_u, int64_t* rows_v, int64_t* rank, double* err_est) {
    return guard([&] {
        need(f != nullptr, "null block factor");
        if (rows_u) *rows_u = f->rows_u;
        if (rows_v) *rows_v = f->rows_v;
        if (rank) *rank = f->f.rank;
        if (err_est) *err_est = f->f.err_est;
    });
}
int h2c_block_factor_download(h2c_block_factor f, double* u, double* v) {
    return guard([&] {
        need(f != nullptr, "null block factor");
        const size_t nu = size_t(f->rows_u * f->f.rank), nv = size_t(f->rows_v * f->f.rank);
        if (u && nu) H2B_CUDA(cudaMemcpy(u, f->f.u.data(), nu * sizeof(double), cudaMemcpyDeviceToHost));
        if (v && nv) H2B_CUDA(cudaMemcpy(v, f->f.v.data(), nv * sizeof(double), cudaMemcpyDeviceToHost));
    });
}
void h2c_block_factor_destroy(h2c_block_factor f) { delete f; }

// ---- algebra and diagnostics -------------------------------------------------------
int h2c_local_low_rank_update(h2c_matrix h, int t, int s, int64_t k, const double* U, int64_t ldu, const double* V,
                              int64_t ldv, double eps, h2c_matrix* out) {
    return guard([&] {
        need(h != nullptr && out != nullptr, "null argument");
        *out = wrap_matrix(h2b::local_low_rank_update(*h->h, t, s, k, U, ldu, V, ldv, eps, nullptr));
    });
}
int h2c_low_rank_update_host(h2c_matrix h, int64_t k, const double* X, const double* Y, double eps, h2c_matrix* out) {
    return guard([&] {
        need(h != nullptr && out != nullptr, "null argument");
        need(k >= 0 && (k == 0 || (X != nullptr && Y != nullptr)), "null factor");
        const size_t sz = size_t(h->h->tree().n * k);
        h2b::DeviceArray<double> xd, yd;
        xd.upload(X, sz);
        // a bitwise-equal pair stays one buffer: the symmetric update keeps symmetric storage
        const bool same = X == Y || (sz && std::memcmp(X, Y, sz * sizeof(double)) == 0);
        if (!same) yd.upload(Y, sz);
        *out = wrap_matrix(h2b::low_rank_update(*h->h, xd.data(), same ? xd.data() : yd.data(), int(k), eps, nullptr));
    });
}
int h2c_local_low_rank_update_host(h2c_matrix h, int t, int s, int64_t k, const double* U, const double* V, double eps,
                                   h2c_matrix* out) {
    return guard([&] {
        need(h != nullptr && out != nullptr, "null argument");
        const h2b::ClusterTree& ct = h->h->tree();
        need(t >= 0 && t < ct.num_nodes() && s >= 0 && s < ct.num_nodes(), "local update: cluster id out of range");
        need(k >= 0 && (k == 0 || (U != nullptr && V != nullptr)), "null factor");
        const int64_t mt = ct.size(t), ms = ct.size(s);
        h2b::DeviceArray<double> ud, vd;
        ud.upload(U, size_t(mt * k));
        const bool same = mt == ms && (U == V || (k && std::memcmp(U, V, size_t(mt * k) * sizeof(double)) == 0));
        if (!same) vd.upload(V, size_t(ms * k));
        *out = wrap_matrix(h2b::local_low_rank_update(*h->h, t, s, k, ud.data(), std::max<int64_t>(mt, 1),
                                                      same ? ud.data() : vd.data(), std::max<int64_t>(ms, 1), eps,
                                                      nullptr));
    });
}
int h2c_frobenius_norm(h2c_matrix h, double* out) {
    return guard([&] {
        need(h != nullptr && out != nullptr, "null argument");
        *out = h2b::frobenius_norm(*h->h, nullptr);
    });
}
int h2c_to_dense(h2c_matrix h, int64_t cap, double* a) {
    return guard([&] {
        need(h != nullptr && a != nullptr, "null argument");
        h2b::to_dense(*h->h, cap, a, nullptr);
    });
}
int h2c_validate(h2c_matrix h, int64_t ortho_cap, int* num_violations, char* messages, int64_t message_bytes,
                 int64_t* level_max_rank, int max_levels, int* num_levels, int64_t* storage) {
    return guard([&] {
        need(h != nullptr, "null matrix");
        const h2b::ValidationReportDev r = h2b::validate(*h->h, ortho_cap, nullptr);
        if (num_violations) *num_violations = int(r.violations.size());
        if (messages && message_bytes > 0) {
            std::string all;
            for (size_t i = 0; i < r.violations.size(); ++i) all += (i ? "\n" : "") + r.violations[i];
            const size_t nb = std::min<size_t>(all.size(), size_t(message_bytes - 1));
            std::memcpy(messages, all.data(), nb);
            messages[nb] = 0;
        }
        if (num_levels) *num_levels = int(r.level_max_rank.size());
        if (level_max_rank)
            for (int i = 0; i < max_levels && i < int(r.level_max_rank.size()); ++i)
                level_max_rank[i] = r.level_max_rank[size_t(i)];
        if (storage) {
            storage[0] = r.storage.dense_reals;
            storage[1] = r.storage.leaf_basis_reals;
            storage[2] = r.storage.transfer_reals;
            storage[3] = r.storage.coupling_reals;
        }
    });
}

}  // extern "C"
