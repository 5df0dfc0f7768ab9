// H2M1 binary container for device H^2 matrices, byte-compatible with the
// reference's serialize.hpp:1-322 (magic "H2M1", u32 version 1, sections
// <u32 tag, u64 length, payload>, little-endian, raw IEEE doubles): a file
// written here is readable by the reference and vice versa. The payload moves
// straight between the packed HBM arrays and the stream; the block tree is
// rebuilt from the stored cluster tree and (eta, mode) and checked by counts
// (serialize.hpp:283-287).
#include "serialize.hpp"

#include <cstring>
#include <string>

#include "matrix.hpp"

namespace h2b {

namespace {

constexpr char kMagic[4] = {'H', '2', 'M', '1'};
constexpr uint32_t kVersion = 1;
enum Section : uint32_t {   // serialize.hpp:30-38
    kSecClusterTree = 1,
    kSecBlockParams = 2,
    kSecFlags = 3,
    kSecRowBasis = 4,
    kSecColBasis = 5,
    kSecCouplings = 6,
    kSecDense = 7,
};

struct Buf {
    std::string s;
    template <class T>
    void put(T v) {
        s.append(reinterpret_cast<const char*>(&v), sizeof(T));
    }
    void put_matrix(int64_t r, int64_t c, const double* d) {
        put<int64_t>(r);
        put<int64_t>(c);
        if (r * c > 0) s.append(reinterpret_cast<const char*>(d), size_t(r * c) * sizeof(double));
    }
};

struct In {
    const char* p;
    size_t n, at = 0;
    template <class T>
    T get() {
        if (at + sizeof(T) > n) throw io_error(io_error::truncated, "H2M1: truncated stream");
        T v;
        std::memcpy(&v, p + at, sizeof(T));
        at += sizeof(T);
        return v;
    }
    // returns (rows, cols, pointer to the raw doubles)
    std::tuple<int64_t, int64_t, const char*> get_matrix() {
        const int64_t r = get<int64_t>(), c = get<int64_t>();
        if (r < 0 || c < 0 || r > (int64_t(1) << 32) || c > (int64_t(1) << 32))
            throw io_error(io_error::malformed, "H2M1: bad matrix header");
        const size_t bytes = size_t(r * c) * sizeof(double);
        if (at + bytes > n) throw io_error(io_error::truncated, "H2M1: truncated matrix payload");
        const char* d = p + at;
        at += bytes;
        return {r, c, d};
    }
};

void section(Buf& out, uint32_t tag, const Buf& body) {
    out.put<uint32_t>(tag);
    out.put<uint64_t>(body.s.size());
    out.s += body.s;
}

void write_basis(Buf& w, const ClusterTree& ct, const BasisDev& b, const std::vector<double>& leaf,
                 const std::vector<double>& xfer) {   // serialize.hpp:88-95
    for (int v = 0; v < ct.num_nodes(); ++v) w.put<int64_t>(b.rank[size_t(v)]);
    for (int v = 0; v < ct.num_nodes(); ++v) {
        const int k = b.rank[size_t(v)];
        if (ct.is_leaf(v)) w.put_matrix(ct.size(v), k, leaf.data() + b.leaf_off[size_t(v)]);
        const int par = ct.parent[size_t(v)];
        if (par >= 0) w.put_matrix(k, b.rank[size_t(par)], xfer.data() + b.xfer_off[size_t(v)]);
    }
}

}  // namespace

std::string serialize(const H2Dev& h) {
    if (h.shard_nranks > 0) throw std::invalid_argument("serialize: a row-subtree shard is not a whole matrix");
    const ClusterTree& ct = h.tree();
    const BlockTree& bt = *h.bt;
    auto U = h.row.leaf.download(), E = h.row.xfer.download(), S = h.S.download(), D = h.D.download();
    std::vector<double> V, F;
    if (!h.symmetric) {
        V = h.col.leaf.download();
        F = h.col.xfer.download();
    }
    Buf out;
    out.s.append(kMagic, 4);
    out.put<uint32_t>(kVersion);
    {   // serialize.hpp:123-141
        Buf b;
        b.put<int64_t>(ct.n);
        b.put<int32_t>(ct.dim);
        b.put<int64_t>(ct.leaf_size);
        b.put<int32_t>(ct.num_nodes());
        for (int v = 0; v < ct.num_nodes(); ++v) {
            b.put<int64_t>(ct.begin[size_t(v)]);
            b.put<int64_t>(ct.end[size_t(v)]);
            b.put<int32_t>(ct.level[size_t(v)]);
            b.put<int32_t>(ct.parent[size_t(v)]);
            b.put<int32_t>(ct.child0[size_t(v)]);
            b.put<int32_t>(ct.child1[size_t(v)]);
            for (int a = 0; a < ct.dim; ++a) b.put<double>(ct.lo[size_t(3 * v + a)]);
            for (int a = 0; a < ct.dim; ++a) b.put<double>(ct.hi[size_t(3 * v + a)]);
        }
        for (int64_t i = 0; i < ct.n; ++i) b.put<int64_t>(ct.perm[size_t(i)]);
        section(out, kSecClusterTree, b);
    }
    {   // :142-148
        Buf b;
        b.put<double>(bt.eta);
        b.put<uint8_t>(bt.weak ? 1 : 0);
        b.put<int64_t>(bt.num_nodes());
        b.put<int64_t>(int64_t(bt.adm.size()));
        b.put<int64_t>(int64_t(bt.dense.size()));
        section(out, kSecBlockParams, b);
    }
    {
        Buf b;
        b.put<uint8_t>(h.symmetric ? 1 : 0);
        b.put<uint8_t>(h.orthonormal ? 1 : 0);
        section(out, kSecFlags, b);
    }
    {
        Buf b;
        write_basis(b, ct, h.row, U, E);
        section(out, kSecRowBasis, b);
    }
    if (!h.symmetric) {
        Buf b;
        write_basis(b, ct, h.col, V, F);
        section(out, kSecColBasis, b);
    }
    const BasisDev& cb = h.symmetric ? h.row : h.col;
    {   // :158-168
        Buf b;
        int64_t count = 0;
        for (size_t i = 0; i < bt.adm.size(); ++i)
            if (h.s_off[i] >= 0) ++count;
        b.put<int64_t>(count);
        for (size_t i = 0; i < bt.adm.size(); ++i) {
            if (h.s_off[i] < 0) continue;
            const int blk = bt.adm[i];
            b.put<int32_t>(blk);
            b.put_matrix(h.row.rank[size_t(bt.row[size_t(blk)])], cb.rank[size_t(bt.col[size_t(blk)])],
                         S.data() + h.s_off[i]);
        }
        section(out, kSecCouplings, b);
    }
    {   // :169-179
        Buf b;
        int64_t count = 0;
        for (size_t i = 0; i < bt.dense.size(); ++i)
            if (h.d_off[i] >= 0) ++count;
        b.put<int64_t>(count);
        for (size_t i = 0; i < bt.dense.size(); ++i) {
            if (h.d_off[i] < 0) continue;
            const int blk = bt.dense[i];
            b.put<int32_t>(blk);
            b.put_matrix(ct.size(bt.row[size_t(blk)]), ct.size(bt.col[size_t(blk)]), D.data() + h.d_off[i]);
        }
        section(out, kSecDense, b);
    }
    return out.s;
}

Deserialized deserialize(const char* data, size_t size) {   // serialize.hpp:184-308
    if (size < 4 || std::memcmp(data, kMagic, 4) != 0) throw io_error(io_error::bad_magic, "H2M1: bad magic");
    In r{data, size, 4};
    const uint32_t version = r.get<uint32_t>();
    if (version != kVersion)
        throw io_error(io_error::version_mismatch, "H2M1: unsupported version " + std::to_string(version));
    std::shared_ptr<ClusterTree> ct;
    bool have_flags = false, have_row = false, sym = false, ortho = false;
    double eta = 1.0;
    bool weak = false;
    int64_t check_nodes = -1, check_adm = -1, check_dense = -1;
    struct Mat {
        int64_t r, c;
        const char* d;
    };
    struct BasisIn {
        std::vector<int> rank;
        std::vector<Mat> leaf, xfer;   // per node (leaf / non-root)
    };
    BasisIn rowb, colb;
    bool have_col = false;
    std::vector<std::pair<int32_t, Mat>> coup, dens;
    auto read_basis = [&](BasisIn& b) {
        if (!ct) throw io_error(io_error::malformed, "H2M1: basis before cluster tree");
        const int nn = ct->num_nodes();
        b.rank.assign(size_t(nn), 0);
        b.leaf.assign(size_t(nn), Mat{0, 0, nullptr});
        b.xfer.assign(size_t(nn), Mat{0, 0, nullptr});
        for (int v = 0; v < nn; ++v) b.rank[size_t(v)] = int(r.get<int64_t>());
        for (int v = 0; v < nn; ++v) {
            if (ct->is_leaf(v)) {
                auto [mr, mc, d] = r.get_matrix();
                b.leaf[size_t(v)] = Mat{mr, mc, d};
            }
            if (ct->parent[size_t(v)] >= 0) {
                auto [mr, mc, d] = r.get_matrix();
                b.xfer[size_t(v)] = Mat{mr, mc, d};
            }
        }
    };
    while (r.at < size) {
        const uint32_t tag = r.get<uint32_t>();
        const uint64_t len = r.get<uint64_t>();
        (void)len;
        switch (tag) {
            case kSecClusterTree: {
                const int64_t n = r.get<int64_t>();
                const int32_t dim = r.get<int32_t>();
                const int64_t lsz = r.get<int64_t>();
                const int32_t nv = r.get<int32_t>();
                if (n < 1 || dim < 1 || dim > 3 || nv < 1)
                    throw io_error(io_error::malformed, "H2M1: bad cluster tree header");
                std::vector<int64_t> begin(static_cast<size_t>(nv)), end(static_cast<size_t>(nv));
                std::vector<int> level(static_cast<size_t>(nv)), parent(static_cast<size_t>(nv)), c0(static_cast<size_t>(nv)),
                    c1(static_cast<size_t>(nv));
                std::vector<double> lo(size_t(3 * nv), 0.0), hi(size_t(3 * nv), 0.0);
                for (int v = 0; v < nv; ++v) {
                    begin[size_t(v)] = r.get<int64_t>();
                    end[size_t(v)] = r.get<int64_t>();
                    level[size_t(v)] = r.get<int32_t>();
                    parent[size_t(v)] = r.get<int32_t>();
                    c0[size_t(v)] = r.get<int32_t>();
                    c1[size_t(v)] = r.get<int32_t>();
                    for (int a = 0; a < dim; ++a) lo[size_t(3 * v + a)] = r.get<double>();
                    for (int a = 0; a < dim; ++a) hi[size_t(3 * v + a)] = r.get<double>();
                }
                std::vector<int64_t> perm(static_cast<size_t>(n));
                for (auto& p : perm) p = r.get<int64_t>();
                ct = restore_cluster_tree(n, dim, lsz, std::move(begin), std::move(end), std::move(level),
                                          std::move(parent), std::move(c0), std::move(c1), std::move(lo),
                                          std::move(hi), std::move(perm));
                break;
            }
            case kSecBlockParams:
                eta = r.get<double>();
                weak = r.get<uint8_t>() != 0;
                check_nodes = r.get<int64_t>();
                check_adm = r.get<int64_t>();
                check_dense = r.get<int64_t>();
                break;
            case kSecFlags:
                sym = r.get<uint8_t>() != 0;
                ortho = r.get<uint8_t>() != 0;
                have_flags = true;
                break;
            case kSecRowBasis:
                read_basis(rowb);
                have_row = true;
                break;
            case kSecColBasis:
                read_basis(colb);
                have_col = true;
                break;
            case kSecCouplings:
            case kSecDense: {
                const int64_t count = r.get<int64_t>();
                for (int64_t i = 0; i < count; ++i) {
                    const int32_t b = r.get<int32_t>();
                    auto [mr, mc, d] = r.get_matrix();
                    (tag == kSecCouplings ? coup : dens).emplace_back(b, Mat{mr, mc, d});
                }
                break;
            }
            default:
                throw io_error(io_error::malformed, "H2M1: unknown section " + std::to_string(tag));
        }
    }
    if (!ct || !have_flags || !have_row) throw io_error(io_error::truncated, "H2M1: missing sections");
    if (!sym && !have_col) throw io_error(io_error::truncated, "H2M1: missing column basis");
    auto bt = build_block_tree(ct, eta, weak);
    if ((check_nodes >= 0 && check_nodes != bt->num_nodes()) ||
        (check_adm >= 0 && check_adm != int64_t(bt->adm.size())) ||
        (check_dense >= 0 && check_dense != int64_t(bt->dense.size())))
        throw io_error(io_error::malformed, "H2M1: block structure mismatch after rebuild");
    auto h = make_h2(bt, sym, rowb.rank.data(), sym ? nullptr : colb.rank.data());
    h->orthonormal = ortho;
    const ClusterTree& t = *ct;
    // host staging in the packed layout, then one upload per part
    auto pack_basis = [&](const BasisIn& in, const BasisDev& lay, std::vector<double>& leaf, std::vector<double>& xf) {
        leaf.assign(lay.leaf.size(), 0.0);
        xf.assign(lay.xfer.size(), 0.0);
        for (int v = 0; v < t.num_nodes(); ++v) {
            const int k = lay.rank[size_t(v)];
            if (t.is_leaf(v)) {
                const Mat& m = in.leaf[size_t(v)];
                if (m.r != t.size(v) || m.c != k) throw io_error(io_error::malformed, "H2M1: leaf basis shape");
                if (m.r > 0 && m.c > 0) std::memcpy(leaf.data() + lay.leaf_off[size_t(v)], m.d, size_t(m.r * m.c) * 8);
            }
            const int par = t.parent[size_t(v)];
            if (par >= 0) {
                const Mat& m = in.xfer[size_t(v)];
                if (m.r != k || m.c != lay.rank[size_t(par)])
                    throw io_error(io_error::malformed, "H2M1: transfer shape");
                if (m.r > 0 && m.c > 0) std::memcpy(xf.data() + lay.xfer_off[size_t(v)], m.d, size_t(m.r * m.c) * 8);
            }
        }
    };
    std::vector<double> U, E, V, F, S(h->S.size(), 0.0), Dd(h->D.size(), 0.0);
    pack_basis(rowb, h->row, U, E);
    if (!sym) pack_basis(colb, h->col, V, F);
    const BasisDev& cb = sym ? h->row : h->col;
    for (auto& [b, m] : coup) {
        if (b < 0 || b >= bt->num_nodes() || bt->adm_ord[size_t(b)] < 0)
            throw io_error(io_error::malformed, "H2M1: coupling at non-admissible block");
        const int64_t i = bt->adm_ord[size_t(b)];
        if (h->s_off[size_t(i)] < 0) continue;   // non-canonical slot of a symmetric matrix stays empty
        if (m.r != h->row.rank[size_t(bt->row[size_t(b)])] || m.c != cb.rank[size_t(bt->col[size_t(b)])])
            throw io_error(io_error::malformed, "H2M1: coupling shape");
        if (m.r > 0 && m.c > 0) std::memcpy(S.data() + h->s_off[size_t(i)], m.d, size_t(m.r * m.c) * 8);
    }
    for (auto& [b, m] : dens) {
        if (b < 0 || b >= bt->num_nodes() || bt->dense_ord[size_t(b)] < 0)
            throw io_error(io_error::malformed, "H2M1: dense payload at non-dense block");
        const int64_t i = bt->dense_ord[size_t(b)];
        if (h->d_off[size_t(i)] < 0) continue;
        if (m.r != t.size(bt->row[size_t(b)]) || m.c != t.size(bt->col[size_t(b)]))
            throw io_error(io_error::malformed, "H2M1: dense shape");
        if (m.r > 0 && m.c > 0) std::memcpy(Dd.data() + h->d_off[size_t(i)], m.d, size_t(m.r * m.c) * 8);
    }
    const double* parts[6] = {U.data(), E.data(), sym ? nullptr : V.data(), sym ? nullptr : F.data(), S.data(),
                              Dd.data()};
    upload_packed(*h, parts);
    return {bt, std::move(h)};
}

}  // namespace h2b
