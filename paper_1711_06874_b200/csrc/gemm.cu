// gemm.cu — strided batched FP64 GEMM on the tensor cores (DMMA), for the large dense contractions
// of the NEXT rows: the single-hole products of Tucker-ALS (f1) and the two streaming passes of
// the SVD-accurate HOSVD (f2).  C[b] (M x N) = A[b] (M x K) * B[b] (K x N) with arbitrary element
// strides (the operands are views of F, of factor matrices and of their transposes); `sub`
// selects C = C - A B (block Gram–Schmidt updates).
//
// CTA tile (32 WM) x (32 WN), WM x WN = 8 warps of 32 x 32; K-steps of 16 in a 4-stage cp.async
// ring.  Both operands are staged k-major per output line in the 128-byte-swizzled layout of the
// Gram kernels (A: [BM lines][16], B^T: [BN lines][16]) so the DMMA fragments load with
// conflict-free LDS.128 (k = 4q + s permutation, shared by both operands).  Global loads are
// 8-byte cp.async gathers whose thread mapping follows the unit-stride dimension (coalesced for
// either storage order).  Out-of-range elements are zero-filled; no split-K (callers split the
// contraction through the batch strides and add the partials in a fixed order).
#include "common.cuh"
#include "kernels.h"

namespace tk {
namespace dg {

constexpr int BK = 16, NT = 256;

// Element e of a [L lines][16 k] stage -> (line, col).  k-fast operands: 16 consecutive lanes read
// one line's 16 consecutive k (128 B).  Line-fast operands: a half-warp covers 8 consecutive lines x
// 2 adjacent k (two 64-B global segments) — in the swizzled layout those are 16 distinct 8-byte
// bank slots, so the cp.async shared-memory writes are conflict-free.
template <int L>
__device__ __forceinline__ void map_elem(int e, bool kfast, int& line, int& col) {
    if (kfast) {
        line = e >> 4;
        col = e & 15;
    } else {
        const int sub = e & 15, blk = e >> 4;
        line = (blk % (L / 8)) * 8 + (sub & 7);
        col = (blk / (L / 8)) * 2 + (sub >> 3);
    }
}

// MF: m8 fragments per warp (warp tile 8 MF x 32); WM x WN warps.  The skinny variant (WM = 1,
// WN = 8, MF = ceil(M / 8)) keeps the padding of a short M below 8 rows.
template <int WM, int WN, int MF, int STAGES>
__global__ void __launch_bounds__(NT, 2) k_dgemm(const SmallGemm g) {
    constexpr int BM = 8 * MF * WM, BN = 32 * WN;
    constexpr int AT = BM * BK, BT = BN * BK;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    double* sA = reinterpret_cast<double*>(smem_raw);
    double* sB = sA + STAGES * AT;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, r = lane >> 2, q = lane & 3;
    const int wm = warp / WN, wn = warp % WN;
    const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN, b = blockIdx.z;
    const double* A = g.A + b * g.sab;
    const double* B = g.B + b * g.sbb;
    const bool a_kfast = (g.sak == 1), b_kfast = (g.sbk == 1);
    const int64_t nkb = ceil_div(g.K, BK);

    auto load = [&](int slot, int64_t kb) {
        double* dA = sA + slot * AT;
        double* dB = sB + slot * BT;
        const int64_t k0 = kb * BK;
#pragma unroll
        for (int u = 0; u < (AT + NT - 1) / NT; ++u) {
            const int e = tid + NT * u;
            if (AT % NT != 0 && e >= AT) break;
            int line, col;
            map_elem<BM>(e, a_kfast, line, col);
            const int64_t m = m0 + line, k = k0 + col;
            const bool ok = (m < g.M) && (k < g.K);
            cp_async8(dA + swz(line, col), ok ? A + m * g.sam + k * g.sak : A, ok);
        }
#pragma unroll
        for (int u = 0; u < BT / NT; ++u) {
            const int e = tid + NT * u;
            int line, col;
            map_elem<BN>(e, b_kfast, line, col);
            const int64_t n = n0 + line, k = k0 + col;
            const bool ok = (n < g.N) && (k < g.K);
            cp_async8(dB + swz(line, col), ok ? B + k * g.sbk + n * g.sbn : B, ok);
        }
    };

    double acc[MF][4][2];
#pragma unroll
    for (int mi = 0; mi < MF; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < nkb) load(s, s);
        cp_async_commit();
    }
    for (int64_t kb = 0; kb < nkb; ++kb) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        const int stg = (int)(kb % STAGES);
        const double* tA = sA + stg * AT;
        const double* tB = sB + stg * BT;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            double a[MF][2], bb[4][2];
#pragma unroll
            for (int mi = 0; mi < MF; ++mi) lds128(a[mi][0], a[mi][1], tA + swz_chunk(wm * 8 * MF + mi * 8 + r, 2 * q + h));
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) lds128(bb[ni][0], bb[ni][1], tB + swz_chunk(wn * 32 + ni * 8 + r, 2 * q + h));
#pragma unroll
            for (int s = 0; s < 2; ++s)
#pragma unroll
                for (int mi = 0; mi < MF; ++mi)
#pragma unroll
                    for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], a[mi][s], bb[ni][s]);
        }
        const int64_t nxt = kb + STAGES - 1;
        if (nxt < nkb) load((int)(nxt % STAGES), nxt);
        cp_async_commit();
    }
    cp_async_wait<0>();
    double* C = g.C + b * g.scb;
#pragma unroll
    for (int mi = 0; mi < MF; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int64_t m = m0 + wm * 8 * MF + mi * 8 + r, n = n0 + wn * 32 + ni * 8 + 2 * q + u;
                if (m < g.M && n < g.N) {
                    double* c = C + m * g.scm + n * g.scn;
                    *c = g.sub ? *c - acc[mi][ni][u] : acc[mi][ni][u];
                }
            }
}

template <int WM, int WN, int MF = 4, int STAGES = 4>
static int run(const SmallGemm& g, cudaStream_t st) {
    constexpr int BM = 8 * MF * WM, BN = 32 * WN;
    const size_t sm = (size_t)STAGES * (BM + BN) * BK * sizeof(double);
    TK_CUDA(cudaFuncSetAttribute(k_dgemm<WM, WN, MF, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    const dim3 grid((unsigned)ceil_div(g.N, BN), (unsigned)ceil_div(g.M, BM), (unsigned)g.batch);
    k_dgemm<WM, WN, MF, STAGES><<<grid, NT, sm, st>>>(g);
    TK_CHECK_LAUNCH();
    return TUCKER_OK;
}

}  // namespace dg

// DMMA for contractions large enough to matter, the DFMA small-GEMM kernel otherwise.
int launch_gemm(const SmallGemm& g, cudaStream_t st) {
    if (g.M <= 0 || g.N <= 0 || g.batch <= 0) return TUCKER_OK;
    const double work = (double)g.M * g.N * g.K * g.batch;
    if (work < 4.0e7 || g.K < 16) return launch_small_gemm(g, st);
    if (g.batch > 65535 || ceil_div(g.M, 64) > 65535) return launch_small_gemm(g, st);
    // skinny shapes go to the one-warp-row kernel when it still fills two CTAs per SM
    const auto skinny_fills = [](int64_t n_long, int64_t batch) { return ceil_div(n_long, 128) * batch >= 2 * kNumSMs; };
    if (g.N <= 64 && g.M > g.N && skinny_fills(g.M, g.batch)) {  // skinny N: C^T = B^T A^T
        const SmallGemm t{g.N, g.M, g.K, g.batch, g.B, g.sbn, g.sbk, g.sbb, g.A, g.sak, g.sam, g.sab,
                          g.C, g.scn, g.scm, g.scb, g.sub};
        return launch_gemm(t, st);
    }
    if (g.M <= 64 && skinny_fills(g.N, g.batch)) {  // skinny M: one warp row of 8 MF rows, 256-wide N tiles
        switch ((g.M + 7) / 8) {
            case 1: return dg::run<1, 8, 1, 3>(g, st);
            case 2: return dg::run<1, 8, 2, 3>(g, st);
            case 3: return dg::run<1, 8, 3, 3>(g, st);
            case 4: return dg::run<1, 8, 4, 3>(g, st);
            case 5: return dg::run<1, 8, 5, 3>(g, st);
            case 6: return dg::run<2, 4, 3, 3>(g, st);  // 48 rows as two warp rows (no register spill)
            default: return dg::run<2, 4, 4, 4>(g, st);
        }
    }
    if (g.M <= 64 && g.N > g.M) return dg::run<2, 4>(g, st);  // 64 x 128 tiles
    return dg::run<4, 2>(g, st);                             // 128 x 64 tiles
}

}  // namespace tk
