#pragma once
// ============================================================================
// ORACLE — TEST INFRASTRUCTURE ONLY.
// CPU restatement of the reference's dense-matrix layer. The reference types
// everything in Eigen (types.hpp:13-15) and calls Eigen's GEMM, HouseholderQR,
// BDCSVD and JacobiSVD; Eigen is absent from this image, so this
// file supplies a small column-major Matrix plus:
//   * Householder QR with Eigen's reflector convention  (algebra.hpp:31-38)
//   * thin-U SVD via QR/LQ + one-sided (Hestenes) Jacobi (algebra.hpp:186,
//     construction.hpp:112, linear_operator.hpp:145)
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
// anything under oracle/. The product (paper_2003_10173_b200/) never links it.
// ============================================================================
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <utility>
#include <vector>

namespace h2 {
inline namespace oracle {

using Index = std::int64_t;

class Matrix {
public:
    Matrix() = default;
    Matrix(Index r, Index c) : r_(r), c_(c), d_(size_t(r * c), 0.0) {
        if (r < 0 || c < 0) throw std::invalid_argument("Matrix: negative size");
    }
    static Matrix Zero(Index r, Index c) { return Matrix(r, c); }
    static Matrix Identity(Index r, Index c) {
        Matrix m(r, c);
        for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = 1.0;
        return m;
    }
    static Matrix Constant(Index r, Index c, double v) {
        Matrix m(r, c);
        std::fill(m.d_.begin(), m.d_.end(), v);
        return m;
    }

    Index rows() const { return r_; }
    Index cols() const { return c_; }
    Index size() const { return r_ * c_; }
    double* data() { return d_.data(); }
    const double* data() const { return d_.data(); }
    double* col(Index j) { return d_.data() + j * r_; }
    const double* col(Index j) const { return d_.data() + j * r_; }

    double& operator()(Index i, Index j) { return d_[size_t(i + j * r_)]; }
    double operator()(Index i, Index j) const { return d_[size_t(i + j * r_)]; }
    double& operator[](Index i) { return d_[size_t(i)]; }
    double operator[](Index i) const { return d_[size_t(i)]; }

    void resize(Index r, Index c) { *this = Matrix(r, c); }
    void setZero(Index r, Index c) { *this = Matrix(r, c); }
    void setZero() { std::fill(d_.begin(), d_.end(), 0.0); }

    Matrix block(Index i0, Index j0, Index nr, Index nc) const {
        Matrix b(nr, nc);
        for (Index j = 0; j < nc; ++j)
            std::memcpy(b.col(j), col(j0 + j) + i0, sizeof(double) * size_t(nr));
        return b;
    }
    void set_block(Index i0, Index j0, const Matrix& b) {
        for (Index j = 0; j < b.cols(); ++j)
            std::memcpy(col(j0 + j) + i0, b.col(j), sizeof(double) * size_t(b.rows()));
    }
    void add_block(Index i0, Index j0, const Matrix& b, double s = 1.0) {
        for (Index j = 0; j < b.cols(); ++j) {
            double* dst = col(j0 + j) + i0;
            const double* src = b.col(j);
            for (Index i = 0; i < b.rows(); ++i) dst[i] += s * src[i];
        }
    }
    Matrix middleRows(Index i0, Index n) const { return block(i0, 0, n, c_); }
    Matrix topRows(Index n) const { return block(0, 0, n, c_); }
    Matrix bottomRows(Index n) const { return block(r_ - n, 0, n, c_); }
    Matrix leftCols(Index n) const { return block(0, 0, r_, n); }
    Matrix rightCols(Index n) const { return block(0, c_ - n, r_, n); }
    Matrix middleCols(Index j0, Index n) const { return block(0, j0, r_, n); }

    Matrix transpose() const {
        Matrix t(c_, r_);
        for (Index j = 0; j < c_; ++j)
            for (Index i = 0; i < r_; ++i) t(j, i) = (*this)(i, j);
        return t;
    }
    double squaredNorm() const {
        double s = 0;
        for (double v : d_) s += v * v;
        return s;
    }
    double norm() const { return std::sqrt(squaredNorm()); }

    Matrix& operator+=(const Matrix& o) {
        check_same(o);
        for (size_t i = 0; i < d_.size(); ++i) d_[i] += o.d_[i];
        return *this;
    }
    Matrix& operator-=(const Matrix& o) {
        check_same(o);
        for (size_t i = 0; i < d_.size(); ++i) d_[i] -= o.d_[i];
        return *this;
    }
    Matrix& operator*=(double s) {
        for (double& v : d_) v *= s;
        return *this;
    }
    friend Matrix operator+(Matrix a, const Matrix& b) { return a += b; }
    friend Matrix operator-(Matrix a, const Matrix& b) { return a -= b; }
    friend Matrix operator*(double s, Matrix a) { return a *= s; }
    friend Matrix operator*(Matrix a, double s) { return a *= s; }
    friend Matrix operator/(Matrix a, double s) { return a *= (1.0 / s); }
    friend Matrix operator-(Matrix a) { return a *= -1.0; }

    bool bitwise_equal(const Matrix& o) const {
        return r_ == o.r_ && c_ == o.c_ &&
               (d_.empty() || std::memcmp(d_.data(), o.d_.data(), sizeof(double) * d_.size()) == 0);
    }

private:
    void check_same(const Matrix& o) const {
        if (r_ != o.r_ || c_ != o.c_) throw std::invalid_argument("Matrix: shape mismatch");
    }
    Index r_ = 0, c_ = 0;
    std::vector<double> d_;
};

using Vector = Matrix;   // n x 1

// C = op(A) * op(B), column-major, plain loops that the compiler vectorises
inline Matrix gemm(const Matrix& a, bool ta, const Matrix& b, bool tb) {
    const Index m = ta ? a.cols() : a.rows(), k = ta ? a.rows() : a.cols();
    const Index kb = tb ? b.cols() : b.rows(), n = tb ? b.rows() : b.cols();
    if (k != kb) throw std::invalid_argument("gemm: inner dimension mismatch");
    Matrix c(m, n);
    if (m == 0 || n == 0 || k == 0) return c;
    if (!ta) {
        for (Index j = 0; j < n; ++j) {
            double* cj = c.col(j);
            for (Index p = 0; p < k; ++p) {
                const double bpj = tb ? b(j, p) : b(p, j);
                if (bpj == 0.0) continue;
                const double* ap = a.col(p);
                for (Index i = 0; i < m; ++i) cj[i] += ap[i] * bpj;
            }
        }
    } else {
        // c(i,j) = dot(a.col(i), op(b).col(j))
        std::vector<double> bj(size_t(k), 0.0);
        for (Index j = 0; j < n; ++j) {
            const double* bcol;
            if (!tb) bcol = b.col(j);
            else {
                for (Index p = 0; p < k; ++p) bj[size_t(p)] = b(j, p);
                bcol = bj.data();
            }
            for (Index i = 0; i < m; ++i) {
                const double* ai = a.col(i);
                double s = 0;
                for (Index p = 0; p < k; ++p) s += ai[p] * bcol[p];
                c(i, j) = s;
            }
        }
    }
    return c;
}
inline Matrix operator*(const Matrix& a, const Matrix& b) { return gemm(a, false, b, false); }

// y += op(A) * x  into a strided destination (used by the hgemv stages)
inline void gemm_acc(const Matrix& a, bool ta, const double* x, Index ldx, Index nb, double* y,
                     Index ldy, double alpha = 1.0) {
    const Index m = ta ? a.cols() : a.rows(), k = ta ? a.rows() : a.cols();
    if (m == 0 || k == 0) return;
    for (Index j = 0; j < nb; ++j) {
        const double* xj = x + j * ldx;
        double* yj = y + j * ldy;
        if (!ta) {
            for (Index p = 0; p < k; ++p) {
                const double s = alpha * xj[p];
                const double* ap = a.col(p);
                for (Index i = 0; i < m; ++i) yj[i] += ap[i] * s;
            }
        } else {
            for (Index i = 0; i < m; ++i) {
                const double* ai = a.col(i);
                double s = 0;
                for (Index p = 0; p < k; ++p) s += ai[p] * xj[p];
                yj[i] += alpha * s;
            }
        }
    }
}

// ---- Householder QR (Eigen HouseholderQR convention) -----------------------
// Reflector H = I - tau v v^T with v(0) = 1, chosen so H x = beta e0 with
// beta = -sign(x0) |x|; a column whose tail is already zero gets tau = 0.
struct HouseholderQR {
    Matrix qr;                 // R on/above the diagonal, essential parts below
    std::vector<double> tau;
    explicit HouseholderQR(Matrix a) : qr(std::move(a)) {
        const Index m = qr.rows(), n = qr.cols(), p = std::min(m, n);
        tau.assign(size_t(p), 0.0);
        for (Index j = 0; j < p; ++j) {
            double* cj = qr.col(j);
            double tail = 0;
            for (Index i = j + 1; i < m; ++i) tail += cj[i] * cj[i];
            const double c0 = cj[j];
            const double tiny = std::numeric_limits<double>::min();
            if (tail <= tiny) {
                tau[size_t(j)] = 0;
                for (Index i = j + 1; i < m; ++i) cj[i] = 0;
                continue;
            }
            double beta = std::sqrt(c0 * c0 + tail);
            if (c0 >= 0) beta = -beta;
            const double inv = 1.0 / (c0 - beta);
            for (Index i = j + 1; i < m; ++i) cj[i] *= inv;
            tau[size_t(j)] = (beta - c0) / beta;
            cj[j] = beta;
            // apply H to the trailing columns
            for (Index c = j + 1; c < n; ++c) {
                double* cc = qr.col(c);
                double s = cc[j];
                for (Index i = j + 1; i < m; ++i) s += cj[i] * cc[i];
                s *= tau[size_t(j)];
                cc[j] -= s;
                for (Index i = j + 1; i < m; ++i) cc[i] -= s * cj[i];
            }
        }
    }
    // Q * I(m, ncols)
    Matrix thinQ(Index ncols) const {
        const Index m = qr.rows(), p = Index(tau.size());
        Matrix q = Matrix::Identity(m, ncols);
        for (Index j = p - 1; j >= 0; --j) {
            const double t = tau[size_t(j)];
            if (t == 0) continue;
            const double* v = qr.col(j);
            for (Index c = 0; c < ncols; ++c) {
                double* qc = q.col(c);
                double s = qc[j];
                for (Index i = j + 1; i < m; ++i) s += v[i] * qc[i];
                s *= t;
                qc[j] -= s;
                for (Index i = j + 1; i < m; ++i) qc[i] -= s * v[i];
            }
        }
        return q;
    }
    Matrix R(Index nrows) const {
        Matrix r(nrows, qr.cols());
        for (Index j = 0; j < qr.cols(); ++j)
            for (Index i = 0; i <= std::min(j, nrows - 1); ++i) r(i, j) = qr(i, j);
        return r;
    }
};

// ---- one-sided Jacobi on a square matrix: B V = U diag(s) -------------------
// returns left singular vectors (columns) and singular values, sorted
// descending. Columns for exactly-zero singular values are left zero (callers
// only ever keep columns with s > tol >= 0).
inline void jacobi_left(Matrix b, Matrix& u, std::vector<double>& s) {
    const Index m = b.rows(), n = b.cols();
    const double tol = 1e-15;
    for (int sweep = 0; sweep < 60; ++sweep) {
        bool rotated = false;
        for (Index i = 0; i < n - 1; ++i)
            for (Index j = i + 1; j < n; ++j) {
                double* bi = b.col(i);
                double* bj = b.col(j);
                double alpha = 0, beta = 0, gamma = 0;
                for (Index k = 0; k < m; ++k) {
                    alpha += bi[k] * bi[k];
                    beta += bj[k] * bj[k];
                    gamma += bi[k] * bj[k];
                }
                if (gamma == 0.0 || std::abs(gamma) <= tol * std::sqrt(alpha * beta)) continue;
                rotated = true;
                const double zeta = (beta - alpha) / (2.0 * gamma);
                const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / std::sqrt(1.0 + t * t), sn = c * t;
                for (Index k = 0; k < m; ++k) {
                    const double x = bi[k], y = bj[k];
                    bi[k] = c * x - sn * y;
                    bj[k] = sn * x + c * y;
                }
            }
        if (!rotated) break;
    }
    std::vector<double> nrm(static_cast<size_t>(n));
    for (Index j = 0; j < n; ++j) {
        double a = 0;
        for (Index k = 0; k < m; ++k) a += b(k, j) * b(k, j);
        nrm[size_t(j)] = std::sqrt(a);
    }
    std::vector<Index> order(static_cast<size_t>(n));
    std::iota(order.begin(), order.end(), Index(0));
    std::stable_sort(order.begin(), order.end(),
                     [&](Index x, Index y) { return nrm[size_t(x)] > nrm[size_t(y)]; });
    u = Matrix(m, n);
    s.assign(size_t(n), 0.0);
    for (Index j = 0; j < n; ++j) {
        const Index src = order[size_t(j)];
        s[size_t(j)] = nrm[size_t(src)];
        if (nrm[size_t(src)] > 0)
            for (Index k = 0; k < m; ++k) u(k, j) = b(k, src) / nrm[size_t(src)];
    }
}

// thin SVD: singular values (descending) and thin U (m x min(m,n)); stands in
// for Eigen::BDCSVD(a, ComputeThinU) and JacobiSVD singular values
struct ThinSVD {
    Matrix U;
    std::vector<double> S;
    explicit ThinSVD(const Matrix& a, bool want_u = true) {
        const Index m = a.rows(), n = a.cols(), p = std::min(m, n);
        if (p == 0) {
            U = Matrix(m, 0);
            return;
        }
        if (m >= n) {
            HouseholderQR qr(a);
            Matrix ur;
            jacobi_left(qr.R(n), ur, S);
            if (want_u) U = qr.thinQ(n) * ur;
        } else {
            HouseholderQR qr(a.transpose());   // a^T = Q R  =>  a = R^T Q^T
            jacobi_left(qr.R(m).transpose(), U, S);
        }
        if (want_u) canonical_signs(U);
    }
    // each column's largest-magnitude entry (lowest row on ties) positive: the
    // sign convention the device SVD uses (la.cu canon_sign_kernel), so HARA's
    // O(eps) cross terms -- and its later decisions -- agree with the device path
    static void canonical_signs(Matrix& u) {
        for (Index j = 0; j < u.cols(); ++j) {
            Index bi = 0;
            double best = -1.0;
            for (Index i = 0; i < u.rows(); ++i)
                if (std::abs(u(i, j)) > best) {
                    best = std::abs(u(i, j));
                    bi = i;
                }
            if (u.rows() > 0 && u(bi, j) < 0)
                for (Index i = 0; i < u.rows(); ++i) u(i, j) = -u(i, j);
        }
    }
};

inline double spectral_norm(const Matrix& a) {
    if (a.size() == 0) return 0.0;
    ThinSVD s(a, false);
    return s.S[0];
}

}  // namespace oracle
}  // namespace h2
