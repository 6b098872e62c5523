// FP64 peak microbenchmarks for the roofline denominators: the DMMA pipe
// (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4) and the FP64 FMA pipe (DFMA), each with independent
// accumulator chains on every SM.  Built and run by tools/fp64_peak.py (which also times cuBLAS
// DGEMM burst and sustained); results -> profiles/fp64_peak_measured.json.
#include <cuda_runtime.h>
#include <cstdint>

__global__ void __launch_bounds__(256) k_dmma(double* out, int iters) {
    double c[8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j][0] = c[j][1] = 0.0;
    const double a = 1e-3 * (threadIdx.x + 1), b = 1.0 - 1e-4 * threadIdx.x;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[j][0]), "+d"(c[j][1])
                         : "d"(a), "d"(b));
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
    if (s == 12345.678) out[0] = s;  // keep the chains alive
}

__global__ void __launch_bounds__(256) k_dfma(double* out, int iters) {
    double c[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j] = 1e-3 * (j + threadIdx.x);
    const double a = 0.999999, b = 1e-7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) c[j] = fma(c[j], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += c[j];
    if (s == 12345.678) out[0] = s;
}

extern "C" {
// Returns milliseconds of one launch (CUDA events), or -1.  kind 0: DMMA, 1: DFMA.
float fp64_peak_run(int kind, int blocks, int threads, int iters) {
    double* out = nullptr;
    if (cudaMalloc(&out, 8) != cudaSuccess) return -1.f;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    if (kind == 0) k_dmma<<<blocks, threads>>>(out, iters);
    else k_dfma<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = -1.f;
    if (cudaGetLastError() == cudaSuccess) cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    return ms;
}
}
