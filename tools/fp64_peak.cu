// FP64 peak microbenchmark for B200 (sm_100a): DFMA vs DMMA (mma.sync m8n8k4 f64)
// and a plain fp64 copy stream. Used once to pick the hgemv inner-loop design
// and to record the FP64 roofline denominator (MEASURED_PEAKS.json has none).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
    double r[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) r[i] = fma(r[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += r[i];
    if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
    for (; i < n; i += st) b[i] = a[i];
}

int main() {
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out; CK(cudaMalloc(&out, 1024 * sizeof(double)));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms;
    // iteration count sized so each timed kernel runs ~1 s: the SM clock the
    // peak is quoted at is the steady one under load (sampled by the caller)
    for (int threads : {256, 512, 1024}) {
        int blocks = sms * (2048 / threads), iters = 4096 * 160;
        dfma_kernel<<<blocks, threads>>>(out, 64, 1.0000001, 1e-9);
        cudaEventRecord(e0);
        dfma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 16 * iters * (double)blocks * threads;
        printf("DFMA threads=%d: %.2f TFLOP/s\n", threads, fl / ms / 1e9);
        dmma_kernel<<<blocks, threads>>>(out, 64);
        cudaEventRecord(e0);
        dmma_kernel<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
        fl = 2.0 * 8 * 256 * iters * (double)blocks * (threads / 32);
        printf("DMMA threads=%d: %.2f TFLOP/s\n", threads, fl / ms / 1e9);
    }
    // DMMA throughput vs resident warps per SM (8 independent accumulators per warp)
    for (int w : {1, 2, 4, 8, 12, 16, 24, 32}) {
        const int blocks = sms * w, iters = 4096;
        dmma_kernel<<<blocks, 32>>>(out, 64);
        cudaEventRecord(e0);
        dmma_kernel<<<blocks, 32>>>(out, iters);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
        const double fl = 2.0 * 8 * 256 * iters * (double)blocks;
        printf("DMMA warps/SM=%d: %.2f TFLOP/s\n", w, fl / ms / 1e9);
    }
    size_t n = (size_t)1 << 28;  // 2 GiB of doubles per buffer
    double2 *a, *b; CK(cudaMalloc(&a, n * 8)); CK(cudaMalloc(&b, n * 8));
    cudaMemset(a, 0, n * 8);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        copy_kernel<<<sms * 8, 256>>>(a, b, n / 2);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
        printf("copy: %.1f GB/s\n", 2.0 * n * 8 / ms / 1e6);
    }
    CK(cudaGetLastError());
    return 0;
}
