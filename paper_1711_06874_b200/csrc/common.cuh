// common.cuh — sm_100a building blocks shared by the Tucker kernels: FP64 tensor-core MMA
// (DMMA via mma.sync m8n8k4 f64 — tcgen05 has no f64 kind), mbarrier / TMA (cp.async.bulk.tensor)
// wrappers, the 128-byte swizzle used by both TMA and the cp.async fallback, reductions, and the
// host-side launch bookkeeping.  Nothing here is shared with oracle/.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/tucker.h"

namespace tk {

// ------------------------------------------------------------------------------------------
// host bookkeeping
int64_t& launch_counter();  // per-thread count of kernel launches of the current ABI call
#define TK_LAUNCHED() (++::tk::launch_counter())

// TUCKER_DEBUG=1 in the environment: a failing CUDA call is reported on stderr (file:line, error)
int report_cuda(cudaError_t e, const char* file, int line);

#define TK_CUDA(call)                                                              \
    do {                                                                           \
        cudaError_t e_ = (call);                                                   \
        if (e_ != cudaSuccess) return ::tk::report_cuda(e_, __FILE__, __LINE__);   \
    } while (0)

#define TK_CHECK_LAUNCH()                                                          \
    do {                                                                           \
        TK_LAUNCHED();                                                             \
        cudaError_t e_ = cudaGetLastError();                                       \
        if (e_ != cudaSuccess) return ::tk::report_cuda(e_, __FILE__, __LINE__);   \
    } while (0)

#define TK_RC(call)                   \
    do {                              \
        int rc_ = (call);             \
        if (rc_ != TUCKER_OK) return rc_; \
    } while (0)

constexpr int kNumSMs = 148;

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda link dependency).
typedef CUresult (*PFN_tmapEncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                        const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                        const cuuint32_t*, CUtensorMapInterleave,
                                        CUtensorMapSwizzle, CUtensorMapL2promotion,
                                        CUtensorMapFloatOOBfill);
PFN_tmapEncodeTiled tmap_encoder();

// FP64 tensor map with 128-byte swizzle; dims[0] innermost (elements), strides in bytes for
// dims 1..rank-1, box in elements.  Returns false if the driver rejects the request.
bool make_tmap_f64(CUtensorMap* map, const void* base, int rank, const uint64_t* dims,
                   const uint64_t* strides_bytes, const uint32_t* box);

// ------------------------------------------------------------------------------------------
// device helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// D(8x8) += A(8x4, row) * B(4x8, col), FP64.  Fragment ownership (lane = 4*r + q):
//   a = A[r][q], b = B[q][r], d = {D[r][2q], D[r][2q+1]}.   SASS: DMMA.8x8x4.
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(d[0]), "+d"(d[1])
        : "d"(a), "d"(b));
}

__device__ __forceinline__ void lds128(double& x, double& y, const double* p) {
    asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];\n" : "=d"(x), "=d"(y) : "r"(smem_u32(p)));
}

__device__ __forceinline__ void lds128_u32(double& x, double& y, uint32_t addr) {
    asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];\n" : "=d"(x), "=d"(y) : "r"(addr));
}

// 128-byte swizzle (CU_TENSOR_MAP_SWIZZLE_128B): inside every 1024-byte-aligned group of eight
// 128-byte lines, the 16-byte chunk index of line L is XOR-ed with (L & 7).  Tiles are stored as
// lines of 16 doubles; element (line, col) lives at double offset swz(line, col).
__device__ __forceinline__ int swz(int line, int col) {
    return line * 16 + ((((col >> 1) ^ (line & 7)) << 1) | (col & 1));
}
__device__ __forceinline__ int swz_chunk(int line, int chunk) {  // first double of a 16-B chunk
    return line * 16 + ((chunk ^ (line & 7)) << 1);
}

// mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE;\n"
        "bra LAB_WAIT;\n"
        "DONE:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// TMA tile loads (global -> shared), completion signalled on an mbarrier (complete_tx::bytes).
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];\n" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];\n" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// cp.async 8-byte copy with zero fill when !valid (LDGSTS).
__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(valid ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Deterministic block sum (fixed shuffle tree, fixed warp order).  `red` holds >= 33 doubles.
// All threads of the block must call it; returns the total on every thread.
__device__ __forceinline__ double block_sum(double v, double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double t = 0.0;
    if (warp == 0) {
        t = lane < nw ? red[lane] : 0.0;
        t = warp_sum(t);
        if (lane == 0) red[32] = t;
    }
    __syncthreads();
    return red[32];
}

}  // namespace tk
