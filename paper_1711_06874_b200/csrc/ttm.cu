// ttm.cu — a-5 core projection beta = F x1 U1^T x2 U2^T x3 U3^T and
// a-6 relative Frobenius error E = ||F - beta x1 U1 x2 U2 x3 U3|| / ||F||.
//
// Core, in the order of SURVEY §8 a-5:
//   TTM1  T1[(i,j),c] = sum_k F[i,j,k] U3[k,c]      (n1 n2) x n3 times n3 x r3 — streams F once;
//         DMMA (mma.sync m8n8k4 f64) with F tiles staged by cp.async in the 128-B swizzled layout.
//   TTM2  T2[i,b,c]   = sum_j U2[j,b] T1[i,j,c]     batched small GEMM (DFMA)
//   TTM3  beta[a,b,c] = sum_i U1[i,a] T2[i,b,c]     small GEMM (DFMA)
// Error, SURVEY §8 a-6:
//   X[i,b,c] = sum_a U1[i,a] beta[a,b,c];  W[i,j,c] = sum_b U2[j,b] X[i,b,c]  (small GEMMs)
//   Ft[(i,j),k] = sum_c W[(i,j),c] U3[k,c] on DMMA tiles, fused with the streaming read of F and
//   the per-CTA sums of (F - Ft)^2 and F^2; a single-CTA pass adds the CTA partials in index order.
//   No float atomics: the result is bitwise reproducible.
#include "common.cuh"
#include "kernels.h"

namespace tk {

// ------------------------------------------------------------------------------ small GEMM
__global__ void __launch_bounds__(256) k_small_gemm(SmallGemm p) {
    __shared__ double sA[16][65];
    __shared__ double sB[16][65];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t m0 = blockIdx.y * 64, n0 = blockIdx.x * 64, b = blockIdx.z;
    const double* A = p.A + b * p.sab;
    const double* B = p.B + b * p.sbb;
    double acc[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
    for (int64_t k0 = 0; k0 < p.K; k0 += 16) {
        for (int t = threadIdx.x; t < 16 * 64; t += 256) {
            const int kk = t & 15, mm = t >> 4;
            const int64_t m = m0 + mm, k = k0 + kk;
            sA[kk][mm] = (m < p.M && k < p.K) ? A[m * p.sam + k * p.sak] : 0.0;
            const int nn = t & 63, kb = t >> 6;
            const int64_t n = n0 + nn, k2 = k0 + kb;
            sB[kb][nn] = (n < p.N && k2 < p.K) ? B[k2 * p.sbk + n * p.sbn] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
            double av[4], bv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) av[u] = sA[kk][ty * 4 + u];
#pragma unroll
            for (int v = 0; v < 4; ++v) bv[v] = sB[kk][tx * 4 + v];
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u][v] = fma(av[u], bv[v], acc[u][v]);
        }
        __syncthreads();
    }
    double* C = p.C + b * p.scb;
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int64_t m = m0 + ty * 4 + u, n = n0 + tx * 4 + v;
            if (m < p.M && n < p.N) C[m * p.scm + n * p.scn] = acc[u][v];
        }
}

int launch_small_gemm(const SmallGemm& p, cudaStream_t st) {
    if (p.M <= 0 || p.N <= 0 || p.batch <= 0) return TUCKER_OK;
    dim3 grid((unsigned)ceil_div(p.N, 64), (unsigned)ceil_div(p.M, 64), (unsigned)p.batch);
    k_small_gemm<<<grid, 256, 0, st>>>(p);
    TK_CHECK_LAUNCH();
    return TUCKER_OK;
}

// ------------------------------------------------------------------------------------ TTM1
// C (M x R) = A (M x K) * B^T, B (R x K) row-major; R <= 64.  CTA: 8 warps x 32 rows = 256 rows,
// warp tile 32 x RP (RP = R rounded up to 8).  Stage = 16 k: A tile [256 lines][16], B tile
// [64 lines][16], swizzled.  K-major fragments with k = 4q + s (see gram.cu).
namespace ttm1 {
constexpr int BMR = 256, BK = 16, STAGES = 4;
constexpr int ATILE = BMR * BK, BTILE = 64 * BK;

template <int NI>
__device__ __forceinline__ void load_stage(const double* __restrict__ A, const double* __restrict__ B,
                                           int64_t M, int64_t K, int R, int64_t m0, int64_t k0,
                                           double* dA, double* dB, bool vec) {
    const int tid = threadIdx.x;
    if (vec) {  // 16-byte copies (row stride and base 16-B aligned)
#pragma unroll
        for (int u = 0; u < ATILE / 2 / 256; ++u) {
            const int e = tid + 256 * u, line = e >> 3, ch = e & 7;
            const int64_t m = m0 + line, k = k0 + 2 * ch;
            const bool ok = (m < M) && (k < K);
            const double* src = ok ? A + m * K + k : A;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dA + swz_chunk(line, ch))),
                         "l"(src), "r"(ok ? 16 : 0)
                         : "memory");
        }
    } else {
#pragma unroll
        for (int u = 0; u < ATILE / 256; ++u) {
            const int e = tid + 256 * u, line = e >> 4, col = e & 15;
            const int64_t m = m0 + line, k = k0 + col;
            const bool ok = (m < M) && (k < K);
            cp_async8(dA + swz(line, col), ok ? A + m * K + k : A, ok);
        }
    }
    for (int e = tid; e < NI * 8 * BK; e += 256) {
        const int line = e >> 4, col = e & 15;
        const int64_t k = k0 + col;
        const bool ok = (line < R) && (k < K);
        cp_async8(dB + swz(line, col), ok ? B + (int64_t)line * K + k : B, ok);
    }
}

template <int NI>
__global__ void __launch_bounds__(256) k_ttm1(const double* __restrict__ A, const double* __restrict__ B,
                                              double* __restrict__ C, int64_t M, int64_t K, int R, bool vec) {
    extern __shared__ uint8_t smem_raw[];
    double* smem = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    double* sA = smem;
    double* sB = smem + STAGES * ATILE;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, r = lane >> 2, q = lane & 3;
    const int64_t m0 = (int64_t)blockIdx.x * BMR;
    const int64_t nkb = ceil_div(K, BK);
    double acc[4][NI][2];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < nkb) load_stage<NI>(A, B, M, K, R, m0, s * BK, sA + s * ATILE, sB + s * BTILE, vec);
        cp_async_commit();
    }
    for (int64_t kb = 0; kb < nkb; ++kb) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        const int stg = (int)(kb % STAGES);
        const double* tA = sA + stg * ATILE;
        const double* tB = sB + stg * BTILE;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            double a[4][2], b[NI][2];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) lds128(a[mi][0], a[mi][1], tA + swz_chunk(warp * 32 + mi * 8 + r, 2 * q + h));
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) lds128(b[ni][0], b[ni][1], tB + swz_chunk(ni * 8 + r, 2 * q + h));
#pragma unroll
            for (int s = 0; s < 2; ++s)
#pragma unroll
                for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                    for (int ni = 0; ni < NI; ++ni) dmma(acc[mi][ni], a[mi][s], b[ni][s]);
        }
        const int64_t nxt = kb + STAGES - 1;
        if (nxt < nkb) {
            const int ns = (int)(nxt % STAGES);
            load_stage<NI>(A, B, M, K, R, m0, nxt * BK, sA + ns * ATILE, sB + ns * BTILE, vec);
        }
        cp_async_commit();
    }
    cp_async_wait<0>();
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
            const int64_t row = m0 + warp * 32 + mi * 8 + r;
            const int col = ni * 8 + 2 * q;
            if (row < M) {
                if (col < R) C[row * R + col] = acc[mi][ni][0];
                if (col + 1 < R) C[row * R + col + 1] = acc[mi][ni][1];
            }
        }
}

static size_t smem_bytes() { return (size_t)STAGES * (ATILE + BTILE) * 8 + 1024; }
}  // namespace ttm1

template <int NI>
static int run_ttm1(const double* A, const double* B, double* C, int64_t M, int64_t K, int R, cudaStream_t st) {
    const size_t sm = ttm1::smem_bytes();
    TK_CUDA(cudaFuncSetAttribute(ttm1::k_ttm1<NI>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    const bool vec = (K % 2 == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
    ttm1::k_ttm1<NI><<<(unsigned)ceil_div(M, ttm1::BMR), 256, sm, st>>>(A, B, C, M, K, R, vec);
    TK_CHECK_LAUNCH();
    return TUCKER_OK;
}

// C (M x R) = A (M x K) * B^T with B = R x K row-major.
static int launch_ttm1(const double* A, const double* B, double* C, int64_t M, int64_t K, int R, cudaStream_t st) {
    switch ((R + 7) / 8) {
        case 1: return run_ttm1<1>(A, B, C, M, K, R, st);
        case 2: return run_ttm1<2>(A, B, C, M, K, R, st);
        case 3: return run_ttm1<3>(A, B, C, M, K, R, st);
        case 4: return run_ttm1<4>(A, B, C, M, K, R, st);
        case 5: return run_ttm1<5>(A, B, C, M, K, R, st);
        case 6: return run_ttm1<6>(A, B, C, M, K, R, st);
        case 7: return run_ttm1<7>(A, B, C, M, K, R, st);
        case 8: return run_ttm1<8>(A, B, C, M, K, R, st);
        default: return TUCKER_ERR_UNSUPPORTED;
    }
}

__global__ void k_transpose(const double* __restrict__ U, double* __restrict__ UT, int64_t n, int r) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * r; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / r;
        const int c = (int)(t % r);
        UT[(int64_t)c * n + i] = U[t];
    }
}

size_t ttm_ws_bytes(const int64_t n[3], const int32_t r[3]) {
    return align_up((size_t)n[0] * n[1] * r[2] * 8, 256) + align_up((size_t)n[0] * r[1] * r[2] * 8, 256) +
           align_up((size_t)n[2] * r[2] * 8, 256);
}

int launch_ttm_core(const int64_t n[3], const int32_t r[3], const double* F, const double* U1, const double* U2,
                    const double* U3, double* core, void* ws, size_t ws_bytes, cudaStream_t st) {
    if (ws_bytes < ttm_ws_bytes(n, r)) return TUCKER_ERR_SIZE;
    char* w = static_cast<char*>(ws);
    double* T1 = reinterpret_cast<double*>(w);
    w += align_up((size_t)n[0] * n[1] * r[2] * 8, 256);
    double* T2 = reinterpret_cast<double*>(w);
    w += align_up((size_t)n[0] * r[1] * r[2] * 8, 256);
    double* UT3 = reinterpret_cast<double*>(w);
    k_transpose<<<64, 256, 0, st>>>(U3, UT3, n[2], r[2]);
    TK_CHECK_LAUNCH();
    TK_RC(launch_ttm1(F, UT3, T1, n[0] * n[1], n[2], r[2], st));
    SmallGemm g2{r[1], r[2], n[1], n[0], U2, 1, r[1], 0, T1, r[2], 1, n[1] * r[2], T2, r[2], 1, (int64_t)r[1] * r[2]};
    TK_RC(launch_small_gemm(g2, st));
    SmallGemm g3{r[0], (int64_t)r[1] * r[2], n[0], 1, U1, 1, r[0], 0, T2, (int64_t)r[1] * r[2], 1, 0, core,
                 (int64_t)r[1] * r[2], 1, 0};
    TK_RC(launch_small_gemm(g3, st));
    return TUCKER_OK;
}

// ---------------------------------------------------------------------------------- error
namespace errk {
constexpr int BM = 128, BN = 128;

// A = W (M x R), B = U3 (N x R); tiles [kb][128 lines][16] with R padded to KB*16.
__global__ void __launch_bounds__(256) k_err(const double* __restrict__ W, const double* __restrict__ U3,
                                             const double* __restrict__ F, int64_t M, int64_t N, int R, int KB,
                                             double* __restrict__ partial) {
    extern __shared__ uint8_t smem_raw[];
    double* smem = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    double* sA = smem;                // KB * 2048
    double* sB = smem + KB * BM * 16;  // KB * 2048
    __shared__ double red[40];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wm = warp >> 2, wn = warp & 3, r = lane >> 2, q = lane & 3;
    const int64_t m0 = (int64_t)blockIdx.x * BM;
    for (int e = tid; e < KB * BM * 16; e += 256) {
        const int kb = e / (BM * 16), rem = e % (BM * 16), line = rem >> 4, col = rem & 15;
        const int k = kb * 16 + col;
        const int64_t m = m0 + line;
        const bool ok = (m < M) && (k < R);
        cp_async8(sA + kb * BM * 16 + swz(line, col), ok ? W + m * R + k : W, ok);
    }
    cp_async_commit();
    double sd = 0.0, sf = 0.0;
    for (int64_t n0 = 0; n0 < N; n0 += BN) {
        __syncthreads();  // previous tile's readers of sB are done
        for (int e = tid; e < KB * BN * 16; e += 256) {
            const int kb = e / (BN * 16), rem = e % (BN * 16), line = rem >> 4, col = rem & 15;
            const int k = kb * 16 + col;
            const int64_t nn = n0 + line;
            const bool ok = (nn < N) && (k < R);
            cp_async8(sB + kb * BN * 16 + swz(line, col), ok ? U3 + nn * R + k : U3, ok);
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
        double acc[8][4][2];
#pragma unroll
        for (int mi = 0; mi < 8; ++mi)
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
        for (int kb = 0; kb < KB; ++kb) {
            const double* tA = sA + kb * BM * 16;
            const double* tB = sB + kb * BN * 16;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                double a[8][2], b[4][2];
#pragma unroll
                for (int mi = 0; mi < 8; ++mi) lds128(a[mi][0], a[mi][1], tA + swz_chunk(wm * 64 + mi * 8 + r, 2 * q + h));
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) lds128(b[ni][0], b[ni][1], tB + swz_chunk(wn * 32 + ni * 8 + r, 2 * q + h));
#pragma unroll
                for (int s = 0; s < 2; ++s)
#pragma unroll
                    for (int mi = 0; mi < 8; ++mi)
#pragma unroll
                        for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], a[mi][s], b[ni][s]);
            }
        }
#pragma unroll
        for (int mi = 0; mi < 8; ++mi)
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) {
                const int64_t row = m0 + wm * 64 + mi * 8 + r;
                const int64_t col = n0 + wn * 32 + ni * 8 + 2 * q;
                if (row < M) {
#pragma unroll
                    for (int u = 0; u < 2; ++u)
                        if (col + u < N) {
                            const double f = __ldcs(F + row * N + col + u);
                            const double d = f - acc[mi][ni][u];
                            sd = fma(d, d, sd);
                            sf = fma(f, f, sf);
                        }
                }
            }
    }
    sd = block_sum(sd, red);
    sf = block_sum(sf, red);
    if (tid == 0) {
        partial[2 * blockIdx.x] = sd;
        partial[2 * blockIdx.x + 1] = sf;
    }
}

__global__ void __launch_bounds__(1024) k_err_final(const double* __restrict__ partial, int64_t nb, double* out3) {
    __shared__ double red[40];
    double sd = 0.0, sf = 0.0;
    // each thread sums a contiguous index range in order; then a fixed tree
    const int64_t per = ceil_div(nb, (int64_t)blockDim.x);
    for (int64_t b = threadIdx.x * per; b < min((int64_t)(threadIdx.x + 1) * per, nb); ++b) {
        sd += partial[2 * b];
        sf += partial[2 * b + 1];
    }
    sd = block_sum(sd, red);
    sf = block_sum(sf, red);
    if (threadIdx.x == 0) {
        const double nf = sqrt(sf), nd = sqrt(sd);
        out3[0] = nd / nf;
        out3[1] = nf;
        out3[2] = nd;
    }
}
}  // namespace errk

size_t err_ws_bytes(const int64_t n[3], const int32_t r[3]) {
    const int64_t M = n[0] * n[1];
    return align_up((size_t)n[0] * r[1] * r[2] * 8, 256) + align_up((size_t)M * r[2] * 8, 256) +
           align_up((size_t)2 * ceil_div(M, errk::BM) * 8, 256);
}

int launch_error(const int64_t n[3], const int32_t r[3], const double* F, const double* U1, const double* U2,
                 const double* U3, const double* core, double* out3, void* ws, size_t ws_bytes, cudaStream_t st) {
    if (ws_bytes < err_ws_bytes(n, r)) return TUCKER_ERR_SIZE;
    if (r[2] > 64) return TUCKER_ERR_UNSUPPORTED;
    const int64_t M = n[0] * n[1];
    char* w = static_cast<char*>(ws);
    double* X = reinterpret_cast<double*>(w);
    w += align_up((size_t)n[0] * r[1] * r[2] * 8, 256);
    double* W = reinterpret_cast<double*>(w);
    w += align_up((size_t)M * r[2] * 8, 256);
    double* partial = reinterpret_cast<double*>(w);
    const int64_t r23 = (int64_t)r[1] * r[2];
    // X (n1 x r2r3) = U1 (n1 x r1) * core (r1 x r2r3)
    SmallGemm gx{n[0], r23, r[0], 1, U1, r[0], 1, 0, core, r23, 1, 0, X, r23, 1, 0};
    TK_RC(launch_small_gemm(gx, st));
    // W[i] (n2 x r3) = U2 (n2 x r2) * X[i] (r2 x r3)
    SmallGemm gw{n[1], r[2], r[1], n[0], U2, r[1], 1, 0, X, r[2], 1, r23, W, r[2], 1, n[1] * r[2]};
    TK_RC(launch_small_gemm(gw, st));
    const int KB = (int)ceil_div(r[2], 16);
    const size_t sm = (size_t)2 * KB * errk::BM * 16 * 8 + 1024;
    TK_CUDA(cudaFuncSetAttribute(errk::k_err, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    const int64_t nb = ceil_div(M, errk::BM);
    errk::k_err<<<(unsigned)nb, 256, sm, st>>>(W, U3, F, M, n[2], r[2], KB, partial);
    TK_CHECK_LAUNCH();
    errk::k_err_final<<<1, 1024, 0, st>>>(partial, nb, out3);
    TK_CHECK_LAUNCH();
    return TUCKER_OK;
}

}  // namespace tk
