#pragma once
// Batched small dense linear algebra on the B200 for the HARA construction and
// recompression (reference: Eigen's GEMM, HouseholderQR, BDCSVD/JacobiSVD at
// algebra.hpp:31-46, 186 and construction.hpp:108-112, linear_operator.hpp:139-150).
// Every routine takes a list of independent problems (one per cluster node /
// block / sampled pair) and runs them as one or a few launches; each problem
// lives in HBM at caller-provided pointers (column-major, FP64).
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "common.hpp"

namespace h2b {
namespace la {

// stream-ordered device buffer (cudaMallocAsync / cudaFreeAsync)
class DBuf {
public:
    DBuf() = default;
    DBuf(size_t n, cudaStream_t s) { alloc(n, s); }
    ~DBuf() { release(); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p_(o.p_), n_(o.n_), s_(o.s_) { o.p_ = nullptr; o.n_ = 0; }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) {
            release();
            p_ = o.p_; n_ = o.n_; s_ = o.s_;
            o.p_ = nullptr; o.n_ = 0;
        }
        return *this;
    }
    void alloc(size_t n, cudaStream_t s) {
        release();
        s_ = s;
        n_ = n;
        if (n) {
            ensure_mem_pool();
            H2B_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p_), n * sizeof(double), s));
        }
    }
    void zero() {
        if (n_) H2B_CUDA(cudaMemsetAsync(p_, 0, n_ * sizeof(double), s_));
    }
    double* data() const { return p_; }
    size_t size() const { return n_; }
    void release() {
        if (p_) cudaFreeAsync(p_, s_);
        p_ = nullptr;
        n_ = 0;
    }

private:
    double* p_ = nullptr;
    size_t n_ = 0;
    cudaStream_t s_ = nullptr;
};

// C = alpha op(A) op(B) + beta C ; op(A) m x k, op(B) k x n
struct GemmDesc {
    const double* A;
    const double* B;
    double* C;
    int m, n, k;
    int lda, ldb, ldc;
    int ta, tb;
    double alpha, beta;
};
void bgemm(const std::vector<GemmDesc>& d, cudaStream_t s);

// block copy: mode 0 dst = src (rows x cols), 1 dst = src^T (dst rows x cols,
// src is cols x rows), 2 dst = identity (src unused), 3 dst += src,
// 4 dst = 0.5 (src + src^T) added to dst (square; symmetrised add)
struct CopyDesc {
    const double* src;
    double* dst;
    int rows, cols;
    int lds, ldd;
    int mode;
};
void bcopy(const std::vector<CopyDesc>& d, cudaStream_t s);

// thin Householder QR (Eigen/LAPACK reflector convention, algebra.hpp:31-38):
// A (m x n) -> R (kp x n, upper trapezoidal), optional explicit Q (m x kp),
// kp = min(m, n). Tall problems run as TSQR (chunk QR, stacked R factors).
// R or Q may be null (not wanted). A is read only.
struct QrDesc {
    const double* A;
    int m, n, lda;
    double* R;
    int ldr;
    double* Q;
    int ldq;
};
void bqr(const std::vector<QrDesc>& d, cudaStream_t s);

// one-sided (Hestenes) Jacobi SVD of a small matrix M = op(A) (rows x cols,
// trans: M = A^T): sigma (cols values, descending) and the right singular
// vectors V (cols x cols, columns in the same order).
struct SvdDesc {
    const double* A;
    int rows, cols, lda;
    int trans;
    double* sigma;
    double* V;      // optional: right singular vectors (cols x cols)
    int ldv;
    double* U = nullptr;   // optional: left singular vectors, the normalised rotated columns (rows x cols)
    int ldu = 0;
    // convergence is judged only on pairs with a column above skip_rel * ||A||_F (the caller
    // discards everything below it); pairs below are still rotated while sweeps run. 0 = all pairs
    double skip_rel = 0;
};
void bjacobi(const std::vector<SvdDesc>& d, cudaStream_t s);

// thin SVD, left factor: A (m x c) -> U (m x min(m,c)) and sigma (descending),
// via QR + Jacobi (no Gram matrix). If P is given and c > m, also
// P = lq_reduce(A) = R^T of thin_qr(A^T) (m x m, algebra.hpp:42-46).
struct LeftSvdDesc {
    const double* A;
    int m, c, lda;
    double* U;
    int ldu;
    double* sigma;
    double* P;    // optional (only written when c > m)
    int ldp;
    double skip_rel = 0;   // see SvdDesc::skip_rel
};
void bleft_svd(const std::vector<LeftSvdDesc>& d, cudaStream_t s);

// rows of an n x c column-major matrix between orderings:
// gather: out[i, j] = in[perm[i], j]   scatter: out[perm[i], j] = in[i, j]
void permute_rows(const double* in, int64_t ldi, double* out, int64_t ldo, const int* perm, int64_t n, int64_t c,
                  bool scatter, cudaStream_t s);

}  // namespace la
}  // namespace h2b
