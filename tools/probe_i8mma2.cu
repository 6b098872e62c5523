// probe_i8mma2.cu — CTA-pair (cta_group::2) check of the tcgen05 kind::i8 encodings used by
// gram_i8.cu: D (256 x N, s32) = A B^T, A (256 x K) split by rows across the pair (128 each),
// B (N x K) split by N across the pair (N/2 rows each), accumulators in both CTAs' TMEM.
//   nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -o probe_i8mma2 tools/probe_i8mma2.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int M = 256, N = 256, K = 512, BK = 128;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa0(uint32_t a) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;\n" : "=r"(r) : "r"(a));
    return r;
}
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) |
           ((uint64_t)2 << 61);
}
__device__ __forceinline__ void wait(uint32_t bar, uint32_t ph) {
    asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(bar), "r"(ph) : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) k_probe(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb,
                                                  int32_t* D, uint32_t idesc, uint32_t* tm_out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* sA = sm;                          // [K/BK][128][128]
    uint8_t* sB = sm + (K / BK) * 128 * BK;    // [K/BK][N/2][128]
    __shared__ __align__(8) uint64_t bar_tma, bar_mma;
    __shared__ uint32_t tmem_base;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(rank));
    const int tid = threadIdx.x, warp = tid >> 5;
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar_tma)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar_mma)));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(su32(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = tmem_base;
    if (tid == 0) tm_out[rank] = tmem;
    const uint32_t bar_leader = mapa0(su32(&bar_tma));
    if (tid == 0) {
        if (rank == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(&bar_tma)),
                         "r"((uint32_t)(2 * (128 + N / 2) * K)) : "memory");
        for (int kb = 0; kb < K / BK; ++kb) {
            asm volatile("cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n"
                         ::"r"(su32(sA + kb * 128 * BK)), "l"((uint64_t)&ma), "r"(bar_leader), "r"(kb * BK), "r"((int)rank * 128) : "memory");
            asm volatile("cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n"
                         ::"r"(su32(sB + kb * (N / 2) * BK)), "l"((uint64_t)&mb), "r"(bar_leader), "r"(kb * BK), "r"((int)rank * (N / 2)) : "memory");
        }
        if (rank == 0) {
            wait(su32(&bar_tma), 0);
            asm volatile("tcgen05.fence::after_thread_sync;\n");
            for (int kb = 0; kb < K / BK; ++kb)
                for (int k = 0; k < BK / 32; ++k) {
                    const uint64_t da = sdesc(su32(sA + kb * 128 * BK) + 32 * k);
                    const uint64_t db = sdesc(su32(sB + kb * (N / 2) * BK) + 32 * k);
                    const uint32_t acc = (kb | k) ? 1u : 0u;
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                                 "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                                 ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
                }
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n"
                         ::"r"(su32(&bar_mma)), "h"((uint16_t)3) : "memory");
        }
    }
    __syncwarp();
    wait(su32(&bar_mma), 0);
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const int row = rank * 128 + warp * 32 + (tid & 31);
    for (int c0 = 0; c0 < N; c0 += 8) {
        uint32_t v[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        for (int j = 0; j < 8; ++j) D[row * N + c0 + j] = (int32_t)v[j];
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;\n" ::"r"(tmem));
}

typedef CUresult (*PFN_enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                            const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                            CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    std::vector<int8_t> A(M * K), B(N * K);
    srand(7);
    for (auto& x : A) x = (int8_t)(rand() & 255);
    for (auto& x : B) x = (int8_t)(rand() & 255);
    int8_t *dA, *dB; int32_t* dD; uint32_t* dT;
    CK(cudaMalloc(&dA, M * K)); CK(cudaMalloc(&dB, N * K)); CK(cudaMalloc(&dD, M * N * 4)); CK(cudaMalloc(&dT, 8));
    CK(cudaMemcpy(dA, A.data(), M * K, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), N * K, cudaMemcpyHostToDevice));
    void* p; cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    PFN_enc enc = (PFN_enc)p;
    CUtensorMap ma, mb;
    cuuint64_t dims[2] = {K, M}, str[1] = {K};
    cuuint32_t boxa[2] = {BK, 128}, boxb[2] = {BK, N / 2}, es[2] = {1, 1};
    if (enc(&ma, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, dA, dims, str, boxa, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("enc A\n"); return 1; }
    dims[1] = N;
    if (enc(&mb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, dB, dims, str, boxb, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("enc B\n"); return 1; }
    std::vector<int32_t> ref(M * N);
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            int32_t s = 0;
            for (int k = 0; k < K; ++k) s += (int32_t)A[m * K + k] * (int32_t)B[n * K + k];
            ref[m * N + n] = s;
        }
    const size_t smem = (size_t)(128 + N / 2) * K;
    CK(cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    CK(cudaMemset(dD, 0, M * N * 4));
    k_probe<<<2, 128, smem>>>(ma, mb, dD, idesc, dT);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("launch: %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<int32_t> got(M * N);
    uint32_t tm[2];
    CK(cudaMemcpy(got.data(), dD, M * N * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(tm, dT, 8, cudaMemcpyDeviceToHost));
    int bad = 0, first = -1;
    for (int i = 0; i < M * N; ++i)
        if (got[i] != ref[i]) { if (first < 0) first = i; ++bad; }
    printf("tmem %u %u  mismatches=%d", tm[0], tm[1], bad);
    if (first >= 0) printf(" first (%d,%d) got %d ref %d", first / N, first % N, got[first], ref[first]);
    printf("\n");
    return 0;
}
