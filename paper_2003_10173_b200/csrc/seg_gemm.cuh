#pragma once
// Segmented batched FP64 GEMM on the DMMA tensor path (mma.sync m8n8k4 f64,
// SASS DMMA.8x8x4; tcgen05 has no f64 kind, so this is sm_100a's FP64 tensor
// instruction). One CTA computes one output block  C(rows x b-tile) =
// sum_e op(A_e) B_e  over a task's entry list and applies a stage-specific
// epilogue. Every hgemv stage is an instance:
//   leaf upsweep   xhat_t  = U_t^T X_t
//   transfer up    xhat_v  = E_c0^T xhat_c0 + E_c1^T xhat_c1
//   coupling       yhat_t  = sum_s op(S_ts) xhat_s
//   downsweep      yhat_c += E_c yhat_v
//   leaf + dense   y[perm(t)] = alpha (U_t yhat_t + sum_s op(D_ts) X_s) + beta y
// Operands are staged HBM -> shared memory with cp.async (zero-filled ragged
// edges, XOR-swizzled so every fragment load is bank-conflict free) in a
// STAGES-deep pipeline; K is consumed in chunks of 32.
#include <cstdint>

namespace h2b {

struct SegTask {
    int e_begin, e_end;   // entry range
    int nsteps;           // sum over entries of ceil(k / 32)
    int nsteps16;         // sum over entries of ceil(k / 16)
    int rows;             // total output rows of this output block
    int row0;             // first output row handled by this task (row tiling)
    int out_ld;           // leading dimension of the output block (coefficient outputs)
    int64_t out_unit;     // output offset: out + out_unit * b (coefficients) / leaf begin (MODE_Y)
};

struct SegEntry {
    const double* A;      // stored block, column-major
    int64_t b_unit;       // B = src[src] + b_unit * b
    int lda, ldb;
    int k;                // inner dimension
    int trans;            // op(A) = A^T
    int src;              // 0 = X (internal blocked), 1 = xhat, 2 = yhat
    int pad;
};

enum SegMode : int { kModeSet = 0, kModeAdd = 1, kModeY = 2 };

struct SegArgs {
    const SegTask* tasks;
    const SegEntry* entries;
    const double* src0;
    const double* src1;
    const double* src2;
    double* out;
    const double* yadd;   // MODE_Y: blocked internal-order partial sums added before alpha (nullptr = none)
    const int* perm;      // MODE_Y: user row of internal row (nullptr = identity)
    int64_t b;
    int64_t ldy;
    double alpha, beta;
};

}  // namespace h2b
