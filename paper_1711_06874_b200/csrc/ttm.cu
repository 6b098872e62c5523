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
#include <cstring>

#include "common.cuh"
#include "fill_eval.cuh"
#include "kernels.h"
#include "prof.h"

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
            if (m < p.M && n < p.N) {
                double* c = C + m * p.scm + n * p.scn;
                *c = p.sub ? *c - acc[u][v] : acc[u][v];
            }
        }
}

int launch_small_gemm(const SmallGemm& p, cudaStream_t st) {
    if (p.M <= 0 || p.N <= 0 || p.batch <= 0) return TUCKER_OK;
    dim3 grid((unsigned)ceil_div(p.N, 64), (unsigned)ceil_div(p.M, 64), (unsigned)p.batch);
    k_small_gemm<<<grid, 256, 0, st>>>(p);
    TK_CHECK_LAUNCH();
    return TUCKER_OK;
}

// C = sum_s P[s] in index order (the split-K slices of launch_small_gemm_splitk; deterministic).
__global__ void __launch_bounds__(256) k_splitk_sum(const double* __restrict__ P, int S, int64_t MN,
                                                    double* __restrict__ C) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < MN; e += (int64_t)gridDim.x * blockDim.x) {
        double s = P[e];
        for (int q = 1; q < S; ++q) s += P[(int64_t)q * MN + e];
        C[e] = s;
    }
}

// A single (batch = 1, sub = 0, C contiguous M x N) small GEMM with a long K and few output tiles
// (the core's last product: r1 x r2 r3 over K = n1) split into S K-slices run as a batch into
// `scratch` (S M N doubles), then summed in slice order.  S = the largest of 16, 8, 4, 2 that divides K
// and leaves >= 64 per slice; otherwise the plain kernel.
int launch_small_gemm_splitk(const SmallGemm& p, double* scratch, size_t scratch_bytes, cudaStream_t st) {
    const int64_t tiles = ceil_div(p.N, 64) * ceil_div(p.M, 64);
    int S = 1;
    for (int c = 16; c >= 2 && S == 1; c /= 2)
        if (p.K % c == 0 && p.K / c >= 64) S = c;
    if (p.batch != 1 || p.sub || p.scn != 1 || p.scm != p.N || tiles >= 148 || S == 1 ||
        (size_t)S * p.M * p.N * 8 > scratch_bytes || !scratch)
        return launch_small_gemm(p, st);
    const int64_t kc = p.K / S;
    SmallGemm q = p;
    q.K = kc;
    q.batch = S;
    q.sab = kc * p.sak;
    q.sbb = kc * p.sbk;
    q.C = scratch;
    q.scb = p.M * p.N;
    TK_RC(launch_small_gemm(q, st));
    const int64_t MN = p.M * p.N;
    k_splitk_sum<<<(unsigned)std::min<int64_t>(ceil_div(MN, 256), 1024), 256, 0, st>>>(scratch, S, MN, p.C);
    TK_CHECK_LAUNCH();
    return TUCKER_OK;
}

// ------------------------------------------------------------------------------- TTM1 + TTM2
// Fused first two mode products over one slab F[i,:,:] (n2 x n3) per CTA row-tile:
//   T1 tile (256 rows j x R) = F[i, j0:j0+256, :] U3            DMMA, streams F once
//   P[b][c] = sum_{j in tile} U2[j][b] T1[j][c]                  DMMA epilogue (T1 stays on chip)
// grid = (JT = ceil(n2/256), n1).  With JT = 1 the CTA writes T2[i] directly, otherwise P goes to
// part[i][jt] and k_t2_reduce adds the JT partials in index order (deterministic).
// Mainloop: 8 MMA warps x 32 rows, warp tile 32 x RP (RP = R rounded up to 8); stage = 16 k.
// A tile [256 lines][16] arrives by TMA (3-D map over F, rows past n2 zero-filled, SWIZZLE_128B);
// the B tile [RP lines][16] is a contiguous block of U3 pre-packed once per call in the same
// swizzled layout and arrives by one cp.async.bulk; a 5-stage mbarrier ring, thread 0 producing.
// Odd n3 (no TMA-legal stride) uses a cp.async variant of the same mainloop.
namespace ttm1 {
constexpr int BMR = 256, BK = 16, STAGES = 5, STAGES_C = 4;
constexpr int ATILE = BMR * BK;

struct Args12 {
    const double* F;   // n1 x n2 x n3
    const double* Bp;  // packed U3: [nkb][RP][16] swizzled
    const double* U2;  // n2 x r2
    double* out;       // JT == 1: T2 (n1 x r2 x R); else part (n1 x JT x r2 x R)
    int64_t n2, n3;
    int R, r2, JT;
    int64_t i_off;     // global index of slab 0 of F (fused path: F is a chunk of slabs)
    double* t1_out;    // optional: T1 = F x3 U3^T stored as (n1 n2) x R (Tucker-ALS needs it)
};

// Bp[kb][c][kk] (swizzled) = U3[16 kb + kk][c]   (0 outside c < R, k < n3)
__global__ void k_pack_u3(const double* __restrict__ U3, int64_t n3, int R, int RP, double* __restrict__ Bp) {
    const int64_t nkb = ceil_div(n3, BK), tot = nkb * RP * BK;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t kb = t / (RP * BK);
        const int rem = (int)(t % (RP * BK)), line = rem >> 4, col = rem & 15;
        const int64_t k = kb * BK + col;
        Bp[kb * RP * BK + swz(line, col)] = (line < R && k < n3) ? U3[k * R + line] : 0.0;
    }
}

template <int NI>
__device__ __forceinline__ void mma_stage(const double* tA, const double* tB, double (&acc)[4][NI][2], int warp,
                                          int r, int q) {
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
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

template <int NI, bool TMA>
__global__ void __launch_bounds__(256, 1) k_ttm12(const __grid_constant__ CUtensorMap mapA, const Args12 g) {
    constexpr int RP = NI * 8, BTILE = RP * BK;
    constexpr uint32_t ABYTES = ATILE * 8, BBYTES = BTILE * 8;
    constexpr int NS = TMA ? STAGES : STAGES_C;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    double* sA = reinterpret_cast<double*>(smem_raw);
    double* sB = sA + NS * ATILE;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + NS * BTILE);
    uint64_t* empty = full + NS;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, r = lane >> 2, q = lane & 3;
    const int64_t i = blockIdx.y;
    const int jt = blockIdx.x;
    const int64_t m0 = (int64_t)jt * BMR, M = g.n2, K = g.n3;
    const int R = g.R;
    const int64_t nkb = ceil_div(K, BK);
    double acc[4][NI][2];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

    if (TMA) {
        if (tid == 0) {
            for (int s = 0; s < NS; ++s) {
                mbar_init(&full[s], 1);
                mbar_init(&empty[s], 8);
            }
            mbar_fence_init();
        }
        __syncthreads();
        auto issue = [&](int slot, int64_t kb) {
            mbar_arrive_expect_tx(&full[slot], ABYTES + BBYTES);
            tma_load_3d(sA + slot * ATILE, &mapA, &full[slot], (int)(kb * BK), (int)m0, (int)i);
            bulk_g2s(sB + slot * BTILE, g.Bp + kb * BTILE, BBYTES, &full[slot]);
        };
        if (tid == 0) {
            tma_prefetch_desc(&mapA);
            for (int s = 0; s < NS && s < nkb; ++s) issue(s, s);
        }
        for (int64_t kb = 0; kb < nkb; ++kb) {
            if (tid == 0 && kb > 0) {
                const int64_t prev = kb - 1, nk = prev + NS;
                if (nk < nkb) {
                    const int ps = (int)(prev % NS);
                    mbar_wait(&empty[ps], (uint32_t)((prev / NS) & 1));
                    issue(ps, nk);
                }
            }
            const int stg = (int)(kb % NS);
            mbar_wait(&full[stg], (uint32_t)((kb / NS) & 1));
            mma_stage<NI>(sA + stg * ATILE, sB + stg * BTILE, acc, warp, r, q);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stg]);
        }
        __syncthreads();  // all MMA reads done before the epilogue reuses the ring
    } else {
        const double* A = g.F + i * g.n2 * g.n3;
        auto load = [&](int slot, int64_t kb) {
            double* dA = sA + slot * ATILE;
#pragma unroll
            for (int u = 0; u < ATILE / 256; ++u) {
                const int e = tid + 256 * u, line = e >> 4, col = e & 15;
                const int64_t m = m0 + line, k = kb * BK + col;
                const bool ok = (m < M) && (k < K);
                cp_async8(dA + swz(line, col), ok ? A + m * K + k : A, ok);
            }
            const double* src = g.Bp + kb * BTILE;
            double* dB = sB + slot * BTILE;
            for (int e = tid; e < BTILE / 2; e += 256)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dB + 2 * e)), "l"(src + 2 * e)
                             : "memory");
        };
#pragma unroll
        for (int s = 0; s < NS - 1; ++s) {
            if (s < nkb) load(s, s);
            cp_async_commit();
        }
        for (int64_t kb = 0; kb < nkb; ++kb) {
            cp_async_wait<NS - 2>();
            __syncthreads();
            const int stg = (int)(kb % NS);
            mma_stage<NI>(sA + stg * ATILE, sB + stg * BTILE, acc, warp, r, q);
            const int64_t nxt = kb + NS - 1;
            if (nxt < nkb) load((int)(nxt % NS), nxt);
            cp_async_commit();
        }
        cp_async_wait<0>();
        __syncthreads();
    }

    if (g.t1_out) {  // optional T1 rows for the Tucker-ALS single-hole products
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) {
            const int64_t j = m0 + warp * 32 + mi * 8 + r;
            if (j < M) {
                double* row = g.t1_out + ((g.i_off + i) * M + j) * R;
#pragma unroll
                for (int ni = 0; ni < NI; ++ni) {
                    const int c = ni * 8 + 2 * q;
                    if (c < R) row[c] = acc[mi][ni][0];
                    if (c + 1 < R) row[c + 1] = acc[mi][ni][1];
                }
            }
        }
    }

    // Epilogue on DMMA: P (r2 x R) = U2[m0:m0+256]^T T1_tile, rows in chunks of CH; leading
    // dimensions = 4 (mod 16) doubles make the fragment loads conflict-free (per half-warp).
    const int r2 = g.r2, r2p = (r2 + 7) & ~7;
    const int ldt = RP + ((4 - RP % 16) + 16) % 16, ldu = r2p + ((4 - r2p % 16) + 16) % 16;
    const int ring = NS * (ATILE + BTILE);
    const int CH = (BMR * (ldt + ldu) <= ring) ? BMR : (BMR / 2 * (ldt + ldu) <= ring ? BMR / 2 : BMR / 4);
    double* sT = sA;               // [CH][ldt]
    double* sU = sA + CH * ldt;    // [CH][ldu], zero-padded to r2p columns
    const int tb = r2p / 8, ntile = tb * NI;
    double pacc[8][2];
#pragma unroll
    for (int u = 0; u < 8; ++u) pacc[u][0] = pacc[u][1] = 0.0;
    for (int c0 = 0; c0 < BMR; c0 += CH) {
        for (int e = tid; e < CH * r2p; e += 256) {
            const int row = e / r2p, b = e - row * r2p;
            const int64_t j = m0 + c0 + row;
            const bool ok = (j < M && b < r2);
            cp_async8(sU + row * ldu + b, ok ? g.U2 + j * r2 + b : g.U2, ok);
        }
        cp_async_commit();
        if (warp * 32 >= c0 && warp * 32 < c0 + CH) {
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < NI; ++ni) {
                    const int row = warp * 32 + mi * 8 + r - c0, col = ni * 8 + 2 * q;
                    sT[row * ldt + col] = acc[mi][ni][0];
                    sT[row * ldt + col + 1] = acc[mi][ni][1];
                }
        }
        cp_async_wait<0>();
        __syncthreads();
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int t = warp + 8 * u;
            if (t < ntile) {
                const int b0 = (t / NI) * 8, cc0 = (t % NI) * 8;
                const double* pa = sU + q * ldu + b0 + r;
                const double* pb = sT + q * ldt + cc0 + r;
#pragma unroll 4
                for (int k = 0; k < CH; k += 4) dmma(pacc[u], pa[k * ldu], pb[k * ldt]);
            }
        }
        __syncthreads();
    }
    double* dst = g.out + ((size_t)(g.i_off + i) * g.JT + jt) * (size_t)(r2 * R);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const int t = warp + 8 * u;
        if (t < ntile) {
            const int b = (t / NI) * 8 + r, c = (t % NI) * 8 + 2 * q;
            if (b < r2) {
                if (c < R) dst[b * R + c] = pacc[u][0];
                if (c + 1 < R) dst[b * R + c + 1] = pacc[u][1];
            }
        }
    }
}

template <int NI, bool TMA>
size_t smem_bytes() {
    constexpr int NS = TMA ? STAGES : STAGES_C;
    return (size_t)NS * (ATILE + NI * 8 * BK) * 8 + 2 * NS * 8;
}
}  // namespace ttm1

// T2[i][o] = sum_jt part[i][jt][o] in index order.
__global__ void k_t2_reduce(const double* __restrict__ part, int JT, int64_t nout, int64_t total,
                            double* __restrict__ T2) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / nout, o = t % nout;
        const double* p = part + i * JT * nout + o;
        double s = p[0];
        for (int j = 1; j < JT; ++j) s += p[(int64_t)j * nout];
        T2[t] = s;
    }
}

template <int NI>
static int run_ttm12(const ttm1::Args12& a, int64_t n1, cudaStream_t st) {  // n1 = slabs in a.F
    const bool tma = (a.n3 % 2 == 0) && ((reinterpret_cast<uintptr_t>(a.F) & 15) == 0) && a.n3 >= ttm1::BK;
    CUtensorMap map;
    std::memset(&map, 0, sizeof(map));
    if (tma) {
        uint64_t dims[3] = {(uint64_t)a.n3, (uint64_t)a.n2, (uint64_t)n1};
        uint64_t strides[2] = {(uint64_t)(a.n3 * 8), (uint64_t)(a.n2 * a.n3 * 8)};
        uint32_t box[3] = {ttm1::BK, ttm1::BMR, 1};
        if (!make_tmap_f64(&map, a.F, 3, dims, strides, box)) return TUCKER_ERR_CUDA;
        const size_t sm = ttm1::smem_bytes<NI, true>();
        TK_CUDA(cudaFuncSetAttribute(ttm1::k_ttm12<NI, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        ttm1::k_ttm12<NI, true><<<dim3((unsigned)a.JT, (unsigned)n1), 256, sm, st>>>(map, a);
    } else {
        const size_t sm = ttm1::smem_bytes<NI, false>();
        TK_CUDA(cudaFuncSetAttribute(ttm1::k_ttm12<NI, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        ttm1::k_ttm12<NI, false><<<dim3((unsigned)a.JT, (unsigned)n1), 256, sm, st>>>(map, a);
    }
    TK_CHECK_LAUNCH();
    return TUCKER_OK;
}

static int launch_ttm12(const ttm1::Args12& a, int64_t n1, cudaStream_t st) {
    switch ((a.R + 7) / 8) {
        case 1: return run_ttm12<1>(a, n1, st);
        case 2: return run_ttm12<2>(a, n1, st);
        case 3: return run_ttm12<3>(a, n1, st);
        case 4: return run_ttm12<4>(a, n1, st);
        case 5: return run_ttm12<5>(a, n1, st);
        case 6: return run_ttm12<6>(a, n1, st);
        case 7: return run_ttm12<7>(a, n1, st);
        case 8: return run_ttm12<8>(a, n1, st);
        default: return TUCKER_ERR_UNSUPPORTED;
    }
}


static int64_t ttm_jt(const int64_t n[3]) { return ceil_div(n[1], ttm1::BMR); }

static size_t packed_u3_bytes(const int64_t n[3], int R) {
    return (size_t)ceil_div(n[2], ttm1::BK) * (size_t)(((R + 7) / 8) * 8) * ttm1::BK * 8;
}

size_t ttm_ws_bytes(const int64_t n[3], const int32_t r[3]) {
    const int64_t JT = ttm_jt(n);
    const size_t t2 = (size_t)n[0] * r[1] * r[2] * 8;
    return align_up(JT > 1 ? JT * t2 : 0, 256) + align_up(t2, 256) + align_up(packed_u3_bytes(n, r[2]), 256);
}

int launch_ttm_core(const int64_t n[3], const int32_t r[3], const double* F, const double* U1, const double* U2,
                    const double* U3, double* core, void* ws, size_t ws_bytes, cudaStream_t st) {
    return launch_ttm_core_impl(n, r, F, nullptr, U1, U2, U3, core, ws, ws_bytes, st);
}

// Tucker-ALS first pass: T1 = F x3 U3^T ((n1 n2) x r3, stored) and Y1 = T1 x2 U2^T (n1 x r2 x r3).
int launch_ttm_t1_y1(const int64_t n[3], const int32_t r[3], const double* F, const double* U2, const double* U3,
                     double* T1, double* Y1, void* ws, size_t ws_bytes, cudaStream_t st) {
    return launch_ttm_core_impl(n, r, F, nullptr, nullptr, U2, U3, nullptr, ws, ws_bytes, st, T1, Y1);
}

// Core with F either materialised (F != nullptr) or generated slab-chunk by slab-chunk (gen).
int launch_ttm_core_impl(const int64_t n[3], const int32_t r[3], const double* F, const FusedGen* gen,
                         const double* U1, const double* U2, const double* U3, double* core, void* ws,
                         size_t ws_bytes, cudaStream_t st, double* t1_out, double* t2_out, const Shard* shard,
                         const TtmI8* i8) {
    const bool sharded = gen && shard && shard->sharded();
    TK_PROF(TUCKER_PROF_TTM, st);
    const size_t chunk_b = gen ? align_up((size_t)gen->Pc * n[1] * n[2] * 8, 256) : 0;
    if (ws_bytes < ttm_ws_bytes(n, r) + chunk_b) return TUCKER_ERR_SIZE;
    if (r[1] > 64 || r[2] > 64) return TUCKER_ERR_UNSUPPORTED;
    const int64_t JT = ttm_jt(n);
    const size_t t2b = (size_t)n[0] * r[1] * r[2] * 8;
    char* w = static_cast<char*>(ws);
    double* chunk = reinterpret_cast<double*>(w);
    w += chunk_b;
    double* part = reinterpret_cast<double*>(w);
    w += align_up(JT > 1 ? JT * t2b : 0, 256);
    double* T2 = t2_out ? t2_out : reinterpret_cast<double*>(w);
    w += align_up(t2b, 256);
    double* Bp = reinterpret_cast<double*>(w);
    const int RP = ((r[2] + 7) / 8) * 8;
    ttm1::k_pack_u3<<<(unsigned)std::min<int64_t>(ceil_div(ceil_div(n[2], ttm1::BK) * RP * ttm1::BK, 256), 1024), 256, 0,
                      st>>>(U3, n[2], r[2], RP, Bp);
    TK_CHECK_LAUNCH();
    ttm1::Args12 a{F, Bp, U2, JT > 1 ? part : T2, n[1], n[2], r[2], r[1], (int)JT, 0, t1_out};
    // fused route: TTM1 of every generated slab chunk on the INT8 tensor cores (R22) when the caller
    // passes the route's exponent and a region large enough for the biggest chunk (T2 rows direct)
    int64_t nci[3] = {gen ? gen->Pc : 0, n[1], n[2]};
    const bool use_i8 = gen && i8 && !t1_out && ttm_i8_applies(nci, r, chunk) &&
                        i8->bytes >= ttm_i8_region_bytes(nci, r);
    if (sharded)  // rows of the other ranks' slabs stay zero (the all-reduce adds zeros)
        TK_CUDA(cudaMemsetAsync(JT > 1 && !use_i8 ? part : T2, 0, JT > 1 && !use_i8 ? JT * t2b : t2b, st));
    if (use_i8) {
        for (int64_t g0 = 0; g0 < n[0]; g0 += gen->Pc) {
            if (sharded && !shard->owns(g0 / gen->Pc)) continue;
            const int64_t pc = std::min<int64_t>(gen->Pc, n[0] - g0);
            ChunkGeo geo = gen->geo;
            geo.g0 = g0;
            geo.Pc = pc;
            TK_RC(launch_gen_chunk(geo, gen->kp, gen->cheb, gen->x2, chunk, st));
            const int64_t nc[3] = {pc, n[1], n[2]};
            TK_RC(launch_ttm12_i8(nc, r, chunk, U2, U3, i8->gmax, T2 + g0 * r[1] * r[2], i8->region, i8->bytes, st, 0,
                                  false));
        }
    } else if (!gen) {
        TK_RC(launch_ttm12(a, n[0], st));
    } else {
        for (int64_t g0 = 0; g0 < n[0]; g0 += gen->Pc) {
            if (sharded && !shard->owns(g0 / gen->Pc)) continue;
            const int64_t pc = std::min<int64_t>(gen->Pc, n[0] - g0);
            ChunkGeo geo = gen->geo;
            geo.g0 = g0;
            geo.Pc = pc;
            TK_RC(launch_gen_chunk(geo, gen->kp, gen->cheb, gen->x2, chunk, st));
            a.F = chunk;
            a.i_off = g0;
            TK_RC(launch_ttm12(a, pc, st));
        }
    }
    if (JT > 1 && !use_i8) {
        const int64_t nout = (int64_t)r[1] * r[2], total = n[0] * nout;
        k_t2_reduce<<<(unsigned)std::min<int64_t>(ceil_div(total, 256), 4096), 256, 0, st>>>(part, (int)JT, nout, total,
                                                                                              T2);
        TK_CHECK_LAUNCH();
    }
    if (sharded) {  // row (e): T2 rows are each computed by exactly one rank
        TK_CUDA(cudaStreamSynchronize(st));
        if (shard->allreduce(T2, n[0] * r[1] * r[2], TUCKER_DT_F64, TUCKER_RED_SUM) != 0) return TUCKER_ERR_COLLECTIVE;
    }
    if (!core) return TUCKER_OK;  // (Tucker-ALS: T1 / Y1 only)
    // TTM3: core (r1 x r2r3) = U1^T (r1 x n1) * T2 (n1 x r2r3)
    SmallGemm g3{r[0], (int64_t)r[1] * r[2], n[0], 1, U1, 1, r[0], 0, T2, (int64_t)r[1] * r[2], 1, 0, core,
                 (int64_t)r[1] * r[2], 1, 0};
    // split K = n1 over the (now free) TTM2 partials buffer
    TK_RC(launch_small_gemm_splitk(g3, JT > 1 ? part : nullptr, JT > 1 ? JT * t2b : 0, st));
    return TUCKER_OK;
}

// ---------------------------------------------------------------------------------- error
namespace errk {
constexpr int BM = 64, BN = 64, NT = 128;

// k -> (block, lane position) map shared by both operands.  Full 16-wide blocks are stored as is;
// a trailing partial block of <= 8 values is placed on the positions {0,1,4,5,8,9,12,13} that the
// first half-step (h = 0) of the K-major fragment loads reads, so the second half-step is skipped
// and no padded k is multiplied (R = 40 -> exactly 2.5 blocks).
__device__ __forceinline__ int kmap_inverse(int kb, int local, int full, int rem) {  // -> k or -1
    if (kb < full) return 16 * kb + local;
    if (rem > 8) return 16 * full + local;
    if (local & 2) return -1;
    return 16 * full + (local >> 2) * 2 + (local & 1);
}

__device__ __forceinline__ void kmap_forward(int k, int full, int rem, int& kb, int& local) {
    if (k < 16 * full) {
        kb = k >> 4;
        local = k & 15;
    } else {
        const int j = k - 16 * full;
        kb = full;
        local = rem > 8 ? j : (j >> 1) * 4 + (j & 1);
    }
}

struct ErrArgs {
    const double* F;   // n1 x n2 x n3
    const double* U2;  // n2 x r2
    const double* X;   // n1 x r2 x R   (X[i] = sum_a U1[i,a] core[a,:,:])
    const double* Up;  // packed U3: [ceil(n3/64)][KB][64][16], kmap + swizzle
    double* partial;   // 2 per CTA
    int64_t n2, n3;
    int r2, R, KB;
    int64_t i_off;     // global index of slab 0 of F (fused path: F is a chunk of slabs)
};

// Up[t][kb][line][local] (swizzled) = U3[64 t + line][kmap_inverse(kb, local)]  (0 if none)
__global__ void k_pack_u3_err(const double* __restrict__ U3, int64_t n3, int R, int KB, double* __restrict__ Up) {
    const int full = R / 16, rem = R % 16;
    const int64_t per = (int64_t)KB * BN * 16, tot = ceil_div(n3, BN) * per;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t tile = t / per;
        const int e = (int)(t % per), kb = e / (BN * 16), rr = e % (BN * 16), line = rr >> 4, col = rr & 15;
        const int k = kmap_inverse(kb, col, full, rem);
        const int64_t nn = tile * BN + line;
        Up[tile * per + kb * BN * 16 + swz(line, col)] = (nn < n3 && k >= 0 && k < R) ? U3[nn * R + k] : 0.0;
    }
}

__device__ __forceinline__ void bulk_g2s_e(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__host__ __device__ inline int ld_mod(int w, int target) {  // smallest ld >= w with ld % 16 == target
    return w + ((target - w % 16) + 16) % 16;
}

// W tiles for the error pass: for slab i and rows j0..j0+63,
//   W (64 x R) = U2[j0:j0+64] X[i]   (DMMA), stored in the k_err A-operand layout
//   Wp[(i * JE + jt)][kb][64][16] (kmap + swizzle, zeros elsewhere)
// so that k_err fetches a whole tile with one cp.async.bulk.  Fragment-load leading dimensions
// are 4 mod 16 doubles: a half-warp's 16 fragment addresses (4 rows x 4 k) hit 16 distinct
// 8-byte bank slots.  A CTA takes WSLABS slabs of one row tile: the U2 tile and the zero padding of
// the output tile are set up once (every slab writes the same positions), X[i] of the next slab is
// loaded while the current tile is stored.
constexpr int WSLABS = 4;
__global__ void __launch_bounds__(NT) k_err_w(const ErrArgs g, double* __restrict__ Wp, int64_t nslabs) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const int KB = g.KB, R = g.R, r2 = g.r2;
    const int r2p = (r2 + 7) & ~7, Rp = (R + 7) & ~7, ldu = ld_mod(r2p, 4), ldx = ld_mod(Rp, 4);
    double* sW = reinterpret_cast<double*>(smem_raw);  // [KB][BM][16]
    double* sU2 = sW + KB * BM * 16;                    // [BM][ldu]
    double* sX = sU2 + BM * ldu;                        // [r2p][ldx]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, r = lane >> 2, q = lane & 3;
    const int full16 = R / 16, rem = R % 16;
    const int64_t j0 = (int64_t)blockIdx.x * BM, M = g.n2;
    for (int e = tid; e < KB * BM * 16; e += NT) sW[e] = 0.0;
    for (int e = tid; e < BM * r2p; e += NT) {
        const int row = e / r2p, b = e - row * r2p;
        sU2[row * ldu + b] = (j0 + row < M && b < r2) ? g.U2[(j0 + row) * r2 + b] : 0.0;
    }
    for (int e = tid; e < r2p * ldx; e += NT) sX[e] = 0.0;  // padding rows / columns stay zero
    __syncthreads();  // (before any thread writes X values over the zeros)
    const int tnn = Rp / 8;  // <= 8 (R <= 64)
    const int mt0 = warp * 16;  // this warp's two 8-row m-tiles: BM / 8 = 8 tiles over 4 warps
    for (int64_t i = (int64_t)blockIdx.y * WSLABS; i < min(nslabs, (int64_t)(blockIdx.y + 1) * WSLABS); ++i) {
        const double* Xi = g.X + (g.i_off + i) * (int64_t)r2 * R;
        if ((R & 1) == 0) {  // X[i] is contiguous (r2 x R): coalesced 16-byte loads, a pair never straddles rows
            const double2* X2 = reinterpret_cast<const double2*>(Xi);
            for (int e = tid; e < r2 * R / 2; e += NT) {
                const int b = (2 * e) / R, c = 2 * e - b * R;
                const double2 v = X2[e];
                sX[b * ldx + c] = v.x;
                sX[b * ldx + c + 1] = v.y;
            }
        } else {
            for (int e = tid; e < r2 * R; e += NT) {
                const int b = e / R, c = e - b * R;
                sX[b * ldx + c] = Xi[e];
            }
        }
        __syncthreads();  // X ready; the previous tile's store is done with sW
        // 2 m-tiles x tnn n-tiles per warp, all accumulators live: 2 tnn independent DMMA chains
        double acc[2][8][2];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
            for (int nn = 0; nn < 8; ++nn) acc[mi][nn][0] = acc[mi][nn][1] = 0.0;
        for (int k = 0; k < r2p; k += 4) {
            const double a0 = sU2[(mt0 + r) * ldu + k + q], a1 = sU2[(mt0 + 8 + r) * ldu + k + q];
#pragma unroll
            for (int nn = 0; nn < 8; ++nn)
                if (nn < tnn) {
                    const double bb = sX[(k + q) * ldx + nn * 8 + r];
                    dmma(acc[0][nn], a0, bb);
                    dmma(acc[1][nn], a1, bb);
                }
        }
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
            for (int nn = 0; nn < 8; ++nn)
                if (nn < tnn)
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int c = nn * 8 + 2 * q + u;
                        if (c < R) {
                            int kb, local;
                            kmap_forward(c, full16, rem, kb, local);
                            sW[kb * BM * 16 + swz(mt0 + 8 * mi + r, local)] = acc[mi][nn][u];
                        }
                    }
        __syncthreads();  // W tile complete; sX free
        double2* dst = reinterpret_cast<double2*>(Wp + ((size_t)i * gridDim.x + blockIdx.x) * (size_t)(KB * BM * 16));
        const double2* src = reinterpret_cast<const double2*>(sW);
        for (int e = tid; e < KB * BM * 8; e += NT) dst[e] = src[e];
    }
}

// One CTA = slab i, rows j0..j0+63 (grid = (ceil(n2/64), n1)), 4 warps as 2 (M) x 2 (N) of
// 32 x 32; two CTAs per SM.
//   W tile (k_err_w) and U3 tiles (pre-packed) arrive by cp.async.bulk (mbarriers; U3 in a
//   2-slot ring);
//   loop over column tiles of 64: the F values of the tile are loaded into registers (fragment
//   layout, 16-byte evict-first loads) before its MMAs so HBM latency hides under them;
//   Ft tile = W U3^T on DMMA; sum (F - Ft)^2 and F^2 per thread; fixed-order block reduction.
__global__ void __launch_bounds__(NT, 2) k_err(const ErrArgs g, const double* __restrict__ Wp) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const int KB = g.KB, R = g.R;
    double* sA = reinterpret_cast<double*>(smem_raw);  // [KB][BM][16]
    double* sB = sA + KB * BM * 16;                    // [2][KB][BN][16]
    uint64_t* bar = reinterpret_cast<uint64_t*>(sB + 2 * KB * BN * 16);  // [0..1] U3 slots, [2] W
    __shared__ double red[40];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wm = warp >> 1, wn = warp & 1, r = lane >> 2, q = lane & 3;
    const int full16 = R / 16, rem = R % 16;
    const int64_t i = blockIdx.y, j0 = (int64_t)blockIdx.x * BM, M = g.n2, N = g.n3;
    const int ntiles = (int)ceil_div(N, BN);
    const uint32_t tbytes = (uint32_t)(KB * BN * 16 * 8), wbytes = (uint32_t)(KB * BM * 16 * 8);

    if (tid == 0) {
        for (int b = 0; b < 3; ++b) mbar_init(&bar[b], 1);
        mbar_fence_init();
    }
    __syncthreads();
    if (tid == 0) {
        mbar_arrive_expect_tx(&bar[2], wbytes);
        bulk_g2s_e(sA, Wp + ((size_t)i * gridDim.x + blockIdx.x) * (size_t)(KB * BM * 16), wbytes, &bar[2]);
        for (int t = 0; t < 2 && t < ntiles; ++t) {
            mbar_arrive_expect_tx(&bar[t], tbytes);
            bulk_g2s_e(sB + t * KB * BN * 16, g.Up + (int64_t)t * KB * BN * 16, tbytes, &bar[t]);
        }
    }
    const uint32_t sA32 = smem_u32(sA), sB32 = smem_u32(sB);
    // per-thread F row pointers (fragment rows), full-tile fast path when in range and aligned
    const bool rows_ok = (j0 + BM <= M);
    const bool vec2 = ((N & 1) == 0) && ((reinterpret_cast<uintptr_t>(g.F) & 15) == 0);
    const double* Fr = g.F + (i * M + j0 + wm * 32 + r) * N + wn * 32 + 2 * q;
    double sd = 0.0, sf = 0.0;
    mbar_wait(&bar[2], 0);
    for (int tile = 0; tile < ntiles; ++tile) {
        const int64_t n0 = (int64_t)tile * BN;
        // 1. F of this tile -> registers
        double f[4][4][2];
        if (rows_ok && vec2 && n0 + BN <= N) {
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) {
                    const double2 v = __ldcs(reinterpret_cast<const double2*>(Fr + (int64_t)mi * 8 * N + n0 + ni * 8));
                    f[mi][ni][0] = v.x;
                    f[mi][ni][1] = v.y;
                }
        } else {
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) {
                const int64_t row = j0 + wm * 32 + mi * 8 + r;
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) {
                    const int64_t col = n0 + wn * 32 + ni * 8 + 2 * q;
                    const double* src = Fr + (int64_t)mi * 8 * N + n0 + ni * 8;
                    f[mi][ni][0] = (row < M && col < N) ? __ldcs(src) : 0.0;
                    f[mi][ni][1] = (row < M && col + 1 < N) ? __ldcs(src + 1) : 0.0;
                }
            }
        }
        // 2. U3 tile ready
        const int slot = tile & 1;
        mbar_wait(&bar[slot], (uint32_t)((tile >> 1) & 1));
        // 3. Ft tile on DMMA
        const uint32_t tB0 = sB32 + (uint32_t)(slot * KB * BN * 16 * 8);
        // accumulators start at 0, not at -F: F's loads stay in flight under the MMAs (their
        // values are first needed in step 4)
        double acc[4][4][2];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
        for (int kb = 0; kb < KB; ++kb) {
            const uint32_t tA = sA32 + (uint32_t)(kb * BM * 16 * 8);
            const uint32_t tB = tB0 + (uint32_t)(kb * BN * 16 * 8);
            const int halves = (kb < full16 || rem > 8) ? 2 : 1;
            for (int h = 0; h < halves; ++h) {
                double a[4][2], b[4][2];
#pragma unroll
                for (int mi = 0; mi < 4; ++mi)
                    lds128_u32(a[mi][0], a[mi][1], tA + 8u * (uint32_t)swz_chunk(wm * 32 + mi * 8 + r, 2 * q + h));
#pragma unroll
                for (int ni = 0; ni < 4; ++ni)
                    lds128_u32(b[ni][0], b[ni][1], tB + 8u * (uint32_t)swz_chunk(wn * 32 + ni * 8 + r, 2 * q + h));
#pragma unroll
                for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
                    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                        for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], a[mi][s2], b[ni][s2]);
            }
        }
        __syncthreads();  // every warp is done with this slot
        if (tid == 0 && tile + 2 < ntiles) {
            mbar_arrive_expect_tx(&bar[slot], tbytes);
            bulk_g2s_e(sB + slot * KB * BN * 16, g.Up + (int64_t)(tile + 2) * KB * BN * 16, tbytes, &bar[slot]);
        }
        // 4. residual and norm (out-of-range positions hold f = 0 and acc = 0)
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int ni = 0; ni < 4; ++ni)
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const double d = f[mi][ni][u] - acc[mi][ni][u];
                    sd = fma(d, d, sd);
                    sf = fma(f[mi][ni][u], f[mi][ni][u], sf);
                }
    }
    sd = block_sum(sd, red);
    sf = block_sum(sf, red);
    if (tid == 0) {
        const int64_t b = (g.i_off + i) * gridDim.x + blockIdx.x;
        g.partial[2 * b] = sd;
        g.partial[2 * b + 1] = sf;
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

static size_t err_w_smem(const int32_t r[3]) {
    const int KB = (int)ceil_div(r[2], 16);
    const int r2p = (r[1] + 7) & ~7, Rp = (r[2] + 7) & ~7;
    return (size_t)KB * errk::BM * 16 * 8 +
           ((size_t)errk::BM * errk::ld_mod(r2p, 4) + (size_t)r2p * errk::ld_mod(Rp, 4)) * 8;
}
static size_t err_smem(const int32_t r[3]) {
    const int KB = (int)ceil_div(r[2], 16);
    // (rounded up to 1 KB: mbarriers at the end of an odd-sized region were seen to fault)
    return align_up((size_t)KB * (errk::BM + 2 * errk::BN) * 16 * 8 + 3 * 8, 1024);
}

static size_t packed_err_bytes(const int64_t n[3], const int32_t r[3]) {
    return (size_t)ceil_div(n[2], errk::BN) * ceil_div(r[2], 16) * errk::BN * 16 * 8;
}
static size_t packed_w_bytes(const int64_t n[3], const int32_t r[3], int64_t slabs) {
    return (size_t)slabs * ceil_div(n[1], errk::BM) * ceil_div(r[2], 16) * errk::BM * 16 * 8;
}

size_t err_ws_bytes(const int64_t n[3], const int32_t r[3]) { return err_ws_bytes_slabs(n, r, n[0]); }

size_t err_ws_bytes_slabs(const int64_t n[3], const int32_t r[3], int64_t slabs) {
    const int64_t nb = n[0] * ceil_div(n[1], errk::BM);
    return align_up((size_t)n[0] * r[1] * r[2] * 8, 256) + align_up((size_t)2 * nb * 8, 256) +
           align_up(packed_err_bytes(n, r), 256) + align_up(packed_w_bytes(n, r, slabs), 256);
}

int launch_error(const int64_t n[3], const int32_t r[3], const double* F, const double* U1, const double* U2,
                 const double* U3, const double* core, double* out3, void* ws, size_t ws_bytes, cudaStream_t st) {
    TK_PROF(TUCKER_PROF_ERROR, st);
    if (ttm_engine() == TUCKER_TTM_INT8_ERROR) {  // opt-in: the reconstruction on the INT8 tensor cores (R23)
        const int rc = launch_error_i8(n, r, F, U1, U2, U3, core, out3, ws, ws_bytes, st);
        if (rc != TUCKER_ERR_UNSUPPORTED) return rc;
    }
    return launch_error_impl(n, r, F, nullptr, U1, U2, U3, core, out3, ws, ws_bytes, st);
}

int launch_error_impl(const int64_t n[3], const int32_t r[3], const double* F, const FusedGen* gen, const double* U1,
                      const double* U2, const double* U3, const double* core, double* out3, void* ws, size_t ws_bytes,
                      cudaStream_t st, const Shard* shard) {
    const bool sharded = gen && shard && shard->sharded();
    const int64_t slabs = gen ? gen->Pc : n[0];
    const size_t chunk_b = gen ? align_up((size_t)gen->Pc * n[1] * n[2] * 8, 256) : 0;
    if (ws_bytes < err_ws_bytes_slabs(n, r, slabs) + chunk_b) return TUCKER_ERR_SIZE;
    if (r[1] > 64 || r[2] > 64) return TUCKER_ERR_UNSUPPORTED;
    const int64_t JE = ceil_div(n[1], errk::BM), nb = n[0] * JE;
    char* w = static_cast<char*>(ws);
    double* chunk = reinterpret_cast<double*>(w);
    w += chunk_b;
    double* X = reinterpret_cast<double*>(w);
    w += align_up((size_t)n[0] * r[1] * r[2] * 8, 256);
    double* partial = reinterpret_cast<double*>(w);
    w += align_up((size_t)2 * nb * 8, 256);
    double* Up = reinterpret_cast<double*>(w);
    w += align_up(packed_err_bytes(n, r), 256);
    double* Wp = reinterpret_cast<double*>(w);
    const int64_t r23 = (int64_t)r[1] * r[2];
    const int KB = (int)ceil_div(r[2], 16);
    // X (n1 x r2r3) = U1 (n1 x r1) * core (r1 x r2r3)
    SmallGemm gx{n[0], r23, r[0], 1, U1, r[0], 1, 0, core, r23, 1, 0, X, r23, 1, 0};
    TK_RC(launch_small_gemm(gx, st));
    const int64_t ptot = (int64_t)(packed_err_bytes(n, r) / 8);
    errk::k_pack_u3_err<<<(unsigned)std::min<int64_t>(ceil_div(ptot, 256), 1024), 256, 0, st>>>(U3, n[2], r[2], KB, Up);
    TK_CHECK_LAUNCH();
    const size_t smw = err_w_smem(r), sm = err_smem(r);
    TK_CUDA(cudaFuncSetAttribute(errk::k_err_w, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smw));
    TK_CUDA(cudaFuncSetAttribute(errk::k_err, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    auto block = [&](const double* Fb, int64_t ns, int64_t i_off) -> int {
        errk::ErrArgs a{Fb, U2, X, Up, partial, n[1], n[2], r[1], r[2], KB, i_off};
        const dim3 grid((unsigned)JE, (unsigned)ns);
        errk::k_err_w<<<dim3((unsigned)JE, (unsigned)ceil_div(ns, (int64_t)errk::WSLABS)), errk::NT, smw, st>>>(a, Wp, ns);
        TK_CHECK_LAUNCH();
        errk::k_err<<<grid, errk::NT, sm, st>>>(a, Wp);
        TK_CHECK_LAUNCH();
        return TUCKER_OK;
    };
    if (sharded) TK_CUDA(cudaMemsetAsync(partial, 0, (size_t)2 * nb * 8, st));  // others' tiles: zero
    if (!gen) {
        TK_RC(block(F, n[0], 0));
    } else {
        for (int64_t g0 = 0; g0 < n[0]; g0 += gen->Pc) {
            if (sharded && !shard->owns(g0 / gen->Pc)) continue;
            const int64_t pc = std::min<int64_t>(gen->Pc, n[0] - g0);
            ChunkGeo geo = gen->geo;
            geo.g0 = g0;
            geo.Pc = pc;
            TK_RC(launch_gen_chunk(geo, gen->kp, gen->cheb, gen->x2, chunk, st));
            TK_RC(block(chunk, pc, g0));
        }
    }
    if (sharded) {  // row (e): each (i, j-block) partial comes from exactly one rank
        TK_CUDA(cudaStreamSynchronize(st));
        if (shard->allreduce(partial, 2 * nb, TUCKER_DT_F64, TUCKER_RED_SUM) != 0) return TUCKER_ERR_COLLECTIVE;
    }
    errk::k_err_final<<<1, 1024, 0, st>>>(partial, nb, out3);
    TK_CHECK_LAUNCH();
    return TUCKER_OK;
}

}  // namespace tk
