#pragma once
// FP64 tensor-core tile building blocks for sm_100a, shared by the hgemv
// segmented GEMM (hgemv.cu) and the batched GEMM of the HARA algebra (la.cu):
// cp.async staging of FP64 tiles into bank-conflict-free shared-memory
// layouts and the DMMA (mma.sync m8n8k4 f64 -- the FP64 tensor path; tcgen05
// has no f64 kind) inner loop over one K chunk.
#include <cstdint>

namespace h2b {
namespace tile {

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, int src_bytes) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async16(double* smem, const double* gmem, int src_bytes) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// Shared-memory tile formats (FP64, one 32-wide K chunk):
//  * "mc" (m-contiguous, for A = stored block used as is): element (m, k) at
//    k*MT + (m ^ ((k & 3) << 2)). The XOR on m bits 2..3 makes the DMMA A
//    fragment (lane (g, t4) reads (m0 + g, 4 k4 + t4)) bank-conflict free and
//    keeps the per-lane address linear in k4.
//  * "kc" (k-contiguous, for A^T and for every B operand): element (k, c) at
//    c*KP + k with KP = 32 + 4 doubles of padding: conflict free for the
//    fragments (c0 + g, 4 k4 + t4), again linear in k4.
// KC = K chunk per pipeline stage (32 or 16); KP = KC + 4 (padded leading dim)

template <int MT>
__device__ __forceinline__ int mc_pos(int m, int k) {
    return k * MT + (m ^ ((k & 3) << 2));
}

// stage an MT x KC block (m-contiguous in global, column stride lda): rows >= rv
// or k >= kv are zero-filled
template <int MT, int KC, int NT, bool VEC>
__device__ __forceinline__ void load_mc(double* tile, const double* base, int64_t lda, int rv, int kv, int tid) {
    if constexpr (VEC) {
        constexpr int NP = MT * KC / 2;
#pragma unroll
        for (int p0 = 0; p0 < NP; p0 += NT) {
            const int p = p0 + tid;
            if (NP % NT == 0 || p < NP) {
                const int m = (p % (MT / 2)) * 2, k = p / (MT / 2);
                const int nb = k < kv ? max(0, min(2, rv - m)) * 8 : 0;
                cp_async16(tile + mc_pos<MT>(m, k), nb ? base + m + k * lda : base, nb);
            }
        }
    } else {
        constexpr int NE = MT * KC;
#pragma unroll
        for (int p0 = 0; p0 < NE; p0 += NT) {
            const int p = p0 + tid;
            if (NE % NT == 0 || p < NE) {
                const int m = p % MT, k = p / MT;
                const bool ok = m < rv && k < kv;
                cp_async8(tile + mc_pos<MT>(m, k), ok ? base + m + k * lda : base, ok ? 8 : 0);
            }
        }
    }
}

// stage a KC x C block whose K index is contiguous in global (element (k, c) at
// base[k + c*ld]) into the padded "kc" format; k >= kv or c >= cv zero-filled
template <int C, int KC, int NT, bool VEC>
__device__ __forceinline__ void load_kc(double* tile, const double* base, int64_t ld, int kv, int cv, int tid) {
    constexpr int KP = KC + 4;
    if constexpr (VEC) {
        constexpr int NP = C * KC / 2;
#pragma unroll
        for (int p0 = 0; p0 < NP; p0 += NT) {
            const int p = p0 + tid;
            if (NP % NT == 0 || p < NP) {
                const int k = (p % (KC / 2)) * 2, c = p / (KC / 2);
                const int nb = c < cv ? max(0, min(2, kv - k)) * 8 : 0;
                cp_async16(tile + c * KP + k, nb ? base + k + c * ld : base, nb);
            }
        }
    } else {
        constexpr int NE = C * KC;
#pragma unroll
        for (int p0 = 0; p0 < NE; p0 += NT) {
            const int p = p0 + tid;
            if (NE % NT == 0 || p < NE) {
                const int k = p % KC, c = p / KC;
                const bool ok = k < kv && c < cv;
                cp_async8(tile + c * KP + k, ok ? base + k + c * ld : base, ok ? 8 : 0);
            }
        }
    }
}

// one K chunk of DMMA work for one warp: acc[TM][TN] += op(A) B over ksteps*4
// K values; fragments are double buffered in registers so the shared-memory
// loads of step k4+1 overlap the DMMAs of step k4
template <int MT, int KC, int TM, int TN, bool TRANS>
__device__ __forceinline__ void chunk_mma(const double* __restrict__ at, const double* __restrict__ bt,
                                          double (&acc)[TM][TN][2], const int (&offa)[TM], const int (&offb)[TN],
                                          int ksteps) {
    constexpr int ASTEP = TRANS ? 4 : 4 * MT;
    double a[2][TM], b[2][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i) a[0][i] = at[offa[i]];
#pragma unroll
    for (int j = 0; j < TN; ++j) b[0][j] = bt[offb[j]];
    if (ksteps == KC / 4) {
#pragma unroll
        for (int k4 = 0; k4 < KC / 4; ++k4) {
            const int cur = k4 & 1, nxt = cur ^ 1;
            if (k4 + 1 < KC / 4) {
#pragma unroll
                for (int i = 0; i < TM; ++i) a[nxt][i] = at[offa[i] + (k4 + 1) * ASTEP];
#pragma unroll
                for (int j = 0; j < TN; ++j) b[nxt][j] = bt[offb[j] + (k4 + 1) * 4];
            }
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) dmma(acc[i][j][0], acc[i][j][1], a[cur][i], b[cur][j]);
        }
    } else {
        for (int k4 = 0; k4 < ksteps; ++k4) {
            double aa[TM], bb[TN];
#pragma unroll
            for (int i = 0; i < TM; ++i) aa[i] = at[offa[i] + k4 * ASTEP];
#pragma unroll
            for (int j = 0; j < TN; ++j) bb[j] = bt[offb[j] + k4 * 4];
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) dmma(acc[i][j][0], acc[i][j][1], aa[i], bb[j]);
        }
    }
}

}  // namespace tile
}  // namespace h2b
