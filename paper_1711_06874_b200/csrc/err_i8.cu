// err_i8.cu — a-6 (the relative Frobenius error E_FN) with the reconstruction on the INT8
// tensor cores.  E^2 ||F||^2 = sum_{p,k} (F[p,k] - Ft[p,k])^2 over the mode-3 fibres p = (i, j), with
// Ft[p, k] = sum_c W[p, c] U3[k, c] and W[p, :] = sum_b U2[j, b] X_i[b, :], X_i = sum_a U1[i, a] beta[a, :, :]
// (2 N r3 flops, FP64-bound on the DMMA pipe at r3 = 40).  Digit emulation as for TTM1 (ttm_i8.cu,
// DESIGN.md R22), here with the output per point (R23):
//
//   Z_k = rint(U3[k, :] 2^(46 - E_k)) per k (max_c |U3[k, c]| < 2^E_k) and Y_p = rint(W[p, :] 2^(46 - E_p))
//   per fibre, six balanced base-256 digits each; the 26 pairs s + t <= 6 summed exactly in int32 per
//   group d = s + t (TMEM), Ft = (hi + mid 2^-24 + lo 2^-32) 2^(E_p + E_k - 28) with the exact integers
//   hi = acc0 2^16 + acc1 2^8 + acc2, mid = acc3 2^16 + acc4 2^8 + acc5, lo = acc6 (|hi|, |mid| < 2^44);
//   the residual F - Ft and the sums of squares in FP64, fixed order per unit, fixed-order final sum.
//   Error of Ft: 2^-47 of |W[p,:]| |U3[k,:]| scales per rounded input plus <= 2^-52 per dropped term —
//   E moves by at most ~2^-46 (relative to ||F||), far inside T4.
//
// k_err_i8: persistent, one CTA per SM; unit = (k-tile of 128 k, chunk of 32 fibres), taken dynamically
// from a global counter in k-tile-major order (a CTA changes k-tile — reloads the 48 KB A image of U3
// digits — only a few times).  MMA: A = U3 digits (M = 128 k rows, K = r3 padded to 64), B = W digits
// of the chunk stacked by digit along N (N = 32 x digits paired), D group d at TMEM columns 32 d,
// two TMEM buffers (224 columns each).  Warps: 0 TMEM owner + MMA issuer, 1 loader (unit schedule,
// A image, F box {128 k, 32 fibres} by TMA and the chunk's W digit image by cp.async.bulk into a
// 4-stage ring; units are posted 6 ahead and their F boxes prefetched to L2), 2-9 epilogue (warp -> TMEM lane quarter and 16 of the 32 fibre columns).
#include "common.cuh"
#include "kernels.h"
#include "prof.h"

#include <cstring>

namespace tk {
namespace e8 {

constexpr int ND = 6, NGRP = 7;
constexpr int NS = 4;                       // stage ring
constexpr int FC = 32;                      // fibres per unit (MMA N per digit block)
constexpr int KT = 128;                     // k per unit (MMA M)
constexpr uint32_t ABLK = KT * 64;          // one U3 digit: 128 rows x 64 B (SWIZZLE_64B)
constexpr uint32_t AIMG = ND * ABLK;        // 48 KB per k-tile
constexpr uint32_t WBLK = FC * 64;          // one W digit of a chunk: 32 rows x 64 B
constexpr uint32_t WIMG = ND * WBLK;        // 12 KB per chunk
constexpr uint32_t FBYTES = FC * KT * 8;    // 32 KB F box
constexpr uint32_t STAGE = FBYTES + WIMG;
constexpr int NEPI = 8;                     // epilogue warps: 2 per TMEM lane quarter, 16 fibre columns each
constexpr int UG = 1024;                     // chunks per unit block (the block's W digits stay in L2 across its k-tiles)
constexpr int NT = 32 * (2 + NEPI);
constexpr int TQ = 8, TQ_CONSUMERS = 1 + NEPI;
constexpr int LA = 6;                        // units posted (and their F boxes prefetched to L2) ahead of the loads
constexpr uint64_t BIAS = 0x808080808080ull;
constexpr int MAX_R = 40;
constexpr size_t smem_bytes() { return (size_t)AIMG + (size_t)NS * STAGE + 1024; }

struct Args {
    const uint8_t* Aimg;      // [nkt][6][128][64] U3 digits (SWIZZLE_64B)
    const double* kscale;     // [nkt * 128]: 2^(E_k - 28) (0 past n3)
    const uint8_t* Wimg;      // [nfc][6][32][64] W digits (SWIZZLE_64B)
    const double* ps;         // [nfc * 32]: 2^E_p (0 past M)
    double* part;             // [units][NEPI][2]
    int64_t M, n3;
    int nkt, nfc;
    int64_t nunits;
    int* sched;
};

__device__ __forceinline__ uint64_t desc_sw64(uint32_t saddr) {  // K-major SWIZZLE_64B, SBO 512 B
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(512 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)4 << 61);
}
__device__ __forceinline__ uint32_t idesc_s8(int N) {  // D s32, A/B s8, K-major, M = 128
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_s8(uint32_t tmem, uint32_t a, uint32_t b, int N, uint32_t acc) {
    const uint64_t da = desc_sw64(a), db = desc_sw64(b);
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
        "l"(da), "l"(db), "r"(idesc_s8(N)), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t addr, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(addr));
}
__device__ __forceinline__ double i64_to_double(long long v) {  // exact for |v| < 2^51
    return __longlong_as_double(v + 0x4338000000000000LL) - 6755399441055744.0;
}
// unit u -> (k-tile, fibre chunk): blocks of UG chunks, k-tile-major inside a block (a block's W digits,
// 12 MB, stay in L2 while its k-tiles pass; a CTA changes k-tile about every UG / 148 units)
__device__ __forceinline__ void unit_of(int u, int nkt, int nfc, int& kt, int& fc) {
    const int per = nkt * UG, blk = u / per, r = u - blk * per;
    const int gsz = min(UG, nfc - blk * UG);  // chunks in this block (the last may be short)
    kt = r / gsz;
    fc = blk * UG + (r - kt * gsz);
}
// SWIZZLE_64B K-major byte offset of (row, byte c) in a block of 64-byte rows (512-byte atoms)
__host__ __device__ __forceinline__ uint32_t sw64(int row, int c) {
    return (uint32_t)((row >> 3) * 512 + (row & 7) * 64 + ((((c >> 4) ^ ((row >> 1) & 3)) << 4) | (c & 15)));
}

__global__ void __launch_bounds__(NT, 1) k_err_i8(const __grid_constant__ CUtensorMap mapF, const Args g) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    uint8_t* sA = smem;
    uint8_t* sS = smem + AIMG;
    __shared__ __align__(8) uint64_t afull, sfull[NS], sempty[NS], tfull[2], tempty[2], tq_full[TQ], tq_empty[TQ];
    __shared__ long long tq[TQ];
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        mbar_init(&afull, 1);
        for (int s = 0; s < NS; ++s) {
            mbar_init(&sfull[s], 1);
            mbar_init(&sempty[s], 1 + NEPI);  // MMA commit + the epilogue warps (F read)
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], NEPI);
        }
        for (int s = 0; s < TQ; ++s) {
            mbar_init(&tq_full[s], 1);
            mbar_init(&tq_empty[s], TQ_CONSUMERS);
        }
        mbar_fence_init();
        tma_prefetch_desc(&mapF);
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = tmem_base;
    auto next_unit = [&](int it) -> long long {
        const int slot = it % TQ;
        mbar_wait(&tq_full[slot], (uint32_t)(it / TQ) & 1u);
        const long long u = *reinterpret_cast<volatile long long*>(&tq[slot]);
        mbar_arrive(&tq_empty[slot]);
        return u;
    };

    if (warp == 0) {
        if (lane == 0) {  // MMA issuer
            int cur_kt = -1, reloads = 0;
            for (int it = 0;; ++it) {
                const long long u = next_unit(it);
                if (u < 0) break;
                const int kt = (int)((u >> 24) & 0xFFFF);
                if (kt != cur_kt) {
                    mbar_wait(&afull, (uint32_t)(reloads & 1));
                    ++reloads;
                    cur_kt = kt;
                }
                const int st = it % NS, buf = it & 1;
                mbar_wait(&tempty[buf], ((uint32_t)(it >> 1) & 1u) ^ 1u);
                mbar_wait(&sfull[st], (uint32_t)(it / NS) & 1u);
                fence_after();
                const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sS + st * STAGE + FBYTES);
                const uint32_t d0 = tmem + 256u * (uint32_t)buf;
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {  // K = 64 bytes of c (r3 <= 40, zero padded)
                    const uint32_t z = ks ? 1u : 0u, ka = a0 + 32u * ks, kb = b0 + 32u * ks;
                    // (U3 digit s, W digits t0..t1) -> TMEM columns 32 (s + t0): the first two set every
                    // column of the buffer (groups 0-5, group 6), the rest accumulate
                    mma_s8(d0, ka, kb, 6 * FC, z);                                   // s0, t0-5
                    mma_s8(d0 + 6 * FC, ka + ABLK, kb + 5 * WBLK, FC, z);             // s1, t5
                    mma_s8(d0 + FC, ka + ABLK, kb, 5 * FC, 1);                        // s1, t0-4
                    mma_s8(d0 + 2 * FC, ka + 2 * ABLK, kb, 5 * FC, 1);                // s2, t0-4
                    mma_s8(d0 + 3 * FC, ka + 3 * ABLK, kb, 4 * FC, 1);                // s3, t0-3
                    mma_s8(d0 + 4 * FC, ka + 4 * ABLK, kb, 3 * FC, 1);                // s4, t0-2
                    mma_s8(d0 + 5 * FC, ka + 5 * ABLK, kb, 2 * FC, 1);                // s5, t0-1
                }
                commit(&sempty[st]);
                commit(&tfull[buf]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // loader: unit schedule (posted LA units ahead, their F boxes prefetched to
                          // L2), A image, F box + W digits per unit
            int cur_kt = -1, posted = 0;
            bool done = false;
            long long ahead[TQ];
            for (int it = 0;; ++it) {
                while (!done && posted <= it + LA) {
                    const int slot = posted % TQ;
                    mbar_wait(&tq_empty[slot], ((uint32_t)(posted / TQ) & 1u) ^ 1u);
                    long long u = atomicAdd(g.sched, 1);
                    int kt = 0, fc = 0;
                    if (u >= g.nunits) u = -1;
                    else unit_of((int)u, g.nkt, g.nfc, kt, fc);
                    const long long pk = u < 0 ? -1 : (u << 40) | ((long long)kt << 24) | fc;  // unit, k-tile, chunk
                    tq[slot] = pk;
                    mbar_arrive(&tq_full[slot]);
                    ahead[slot] = pk;
                    ++posted;
                    if (u < 0) done = true;
                    else
                        asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];\n" ::"l"(
                                         reinterpret_cast<uint64_t>(&mapF)),
                                     "r"(kt * KT), "r"(fc * FC)
                                     : "memory");
                }
                const long long pk = ahead[it % TQ];
                if (pk < 0) break;
                const int kt = (int)((pk >> 24) & 0xFFFF), fc = (int)(pk & 0xFFFFFF);
                if (kt != cur_kt) {  // every MMA on the old A image done (unit it-1's stage released)
                    if (it > 0) mbar_wait(&sempty[(it - 1) % NS], (uint32_t)((it - 1) / NS) & 1u);
                    mbar_arrive_expect_tx(&afull, AIMG);
                    bulk_load(sA, g.Aimg + (size_t)kt * AIMG, AIMG, &afull);
                    cur_kt = kt;
                }
                const int st = it % NS;
                mbar_wait(&sempty[st], ((uint32_t)(it / NS) & 1u) ^ 1u);
                mbar_arrive_expect_tx(&sfull[st], STAGE);
                uint8_t* dst = sS + st * STAGE;
                tma_load_2d(dst, &mapF, &sfull[st], kt * KT, fc * FC);
                bulk_load(dst + FBYTES, g.Wimg + (size_t)fc * WIMG, WIMG, &sfull[st]);
            }
        }
    } else {  // epilogue: warp -> TMEM lanes 32 q (k rows) and fibre columns 16 h .. 16 h + 15
        const int ew = warp - 2, q = warp & 3, h = ew >> 2;
        const uint32_t tl = (uint32_t)(q * 32) << 16;
        const long long MAGIC = 0x4338000000000000LL;  // 1.5 2^52: (MAGIC + v) as a double is 1.5 2^52 + v
        for (int it = 0;; ++it) {
            long long pk = 0;
            if (lane == 0) pk = next_unit(it);
            pk = __shfl_sync(0xffffffffu, pk, 0);
            if (pk < 0) break;
            const int u = (int)(pk >> 40), kt = (int)((pk >> 24) & 0xFFFF), fc = (int)(pk & 0xFFFFFF);
            const int st = it % NS, buf = it & 1;
            const double sk = g.kscale[kt * KT + q * 32 + lane];
            const double* psc = g.ps + (int64_t)fc * FC + 16 * h;
            mbar_wait(&sfull[st], (uint32_t)(it / NS) & 1u);  // (F landed: the MMA has waited for it too)
            mbar_wait(&tfull[buf], (uint32_t)(it >> 1) & 1u);
            fence_after();
            const double* sF = reinterpret_cast<const double*>(sS + st * STAGE) + q * 32 + lane;
            double ae = 0.0, af = 0.0;
            uint32_t a[NGRP][16];  // both 8-column chunks in flight together
#pragma unroll
            for (int cc = 0; cc < 2; ++cc)
#pragma unroll
                for (int d = 0; d < NGRP; ++d)
                    tmem_ld8(tmem + tl + 256u * (uint32_t)buf + (uint32_t)(d * FC + 16 * h + 8 * cc),
                             *reinterpret_cast<uint32_t(*)[8]>(&a[d][8 * cc]));
            double scl[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) scl[e] = psc[e] * sk;
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[buf]);  // the accumulators are in registers
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                // hi = acc0 2^16 + acc1 2^8 + acc2 and mid likewise, exact in int64, + MAGIC: the bits
                // of the double 1.5 2^52 + hi (|hi| < 2^44)
                const long long hb = (long long)(int)a[0][e] * 65536 + (long long)(int)a[1][e] * 256 +
                                     ((long long)(int)a[2][e] + MAGIC);
                const long long mb = (long long)(int)a[3][e] * 65536 + (long long)(int)a[4][e] * 256 +
                                     ((long long)(int)a[5][e] + MAGIC);
                const double hi = __longlong_as_double(hb) - 6755399441055744.0;
                const double mid = __longlong_as_double(mb) - 6755399441055744.0;
                double t = fma(mid, 0x1p-24, hi);
                t = fma((double)(int)a[6][e], 0x1p-32, t);
                const double f = sF[(16 * h + e) * KT];
                const double r = fma(-t, scl[e], f);
                ae = fma(r, r, ae);
                af = fma(f, f, af);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sempty[st]);  // F read
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {  // fixed-order butterfly
                ae += __shfl_xor_sync(0xffffffffu, ae, o);
                af += __shfl_xor_sync(0xffffffffu, af, o);
            }
            if (lane == 0) {
                double* p = g.part + ((size_t)u * NEPI + ew) * 2;
                p[0] = ae;
                p[1] = af;
            }
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 0) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
    }
}

// U3 (n3 x R) -> per-k exponents and the A images: k-tile kt, digit s: rows k (128 x 64 B, SWIZZLE_64B),
// byte c = digit s of rint(U3[k, c] 2^(46 - E_k)) (0 for c >= R and k >= n3).  One warp per k.
__global__ void __launch_bounds__(256) k_u3_digits_err(const double* __restrict__ U3, int64_t n3, int R, int nkt,
                                                       uint8_t* __restrict__ img, double* __restrict__ kscale) {
    const int64_t k = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (k >= (int64_t)nkt * KT) return;
    const int kt = (int)(k / KT), kr = (int)(k % KT);
    double v0 = 0.0, v1 = 0.0;
    if (k < n3) {
        if (lane < R) v0 = U3[k * R + lane];
        if (lane + 32 < R) v1 = U3[k * R + lane + 32];
    }
    double mx = fmax(fabs(v0), fabs(v1));
    mx = warp_max(mx);
    int Ek = 0;
    if (mx > 0.0) frexp(mx, &Ek);
    if (lane == 0) kscale[k] = k < n3 ? ldexp(1.0, Ek - 28) : 0.0;
    const double sc = ldexp(1.0, 46 - Ek);
    for (int half = 0; half < 2; ++half) {
        const int c = lane + 32 * half;
        const uint64_t w = (uint64_t)(llrint((half ? v1 : v0) * sc) + (long long)BIAS);
        for (int s = 0; s < ND; ++s)
            img[(size_t)kt * AIMG + (size_t)s * ABLK + sw64(kr, c)] = (uint8_t)(((w >> (8 * (5 - s))) & 255u) ^ 0x80u);
    }
}

// W[p, :] = U2[j, :] X_i (fibre p = (i, j)), its scale 2^E_p and its digit image: chunk p / 32, digit t,
// row p % 32 (32 x 64 B blocks, SWIZZLE_64B).  One thread per fibre, X_i in shared memory.
__global__ void __launch_bounds__(256) k_w_digits(const double* __restrict__ U2, const double* __restrict__ X,
                                                  int64_t n2, int r2, int R, uint8_t* __restrict__ img,
                                                  double* __restrict__ ps) {
    extern __shared__ double sX[];  // r2 x R
    const int64_t i = blockIdx.y, j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int e = threadIdx.x; e < r2 * R; e += blockDim.x) sX[e] = X[i * r2 * R + e];
    __syncthreads();
    if (j >= n2) return;
    double w[MAX_R];
#pragma unroll
    for (int c = 0; c < MAX_R; ++c) w[c] = 0.0;
    for (int b = 0; b < r2; ++b) {
        const double u = U2[j * r2 + b];
#pragma unroll
        for (int c = 0; c < MAX_R; ++c)
            if (c < R) w[c] = fma(u, sX[b * R + c], w[c]);
    }
    double mx = 0.0;
#pragma unroll
    for (int c = 0; c < MAX_R; ++c) mx = fmax(mx, fabs(w[c]));
    int Ep = 0;
    if (mx > 0.0) frexp(mx, &Ep);
    const int64_t p = i * n2 + j;
    ps[p] = ldexp(1.0, Ep);
    const double sc = ldexp(1.0, 46 - Ep);
    const int fc = (int)(p / FC), rr = (int)(p % FC);
    uint8_t* base = img + (size_t)fc * WIMG;
    uint32_t lo[MAX_R], hi[MAX_R];  // X + bias: bytes 0-3 and 4-5 (digit t = byte 5 - t)
#pragma unroll
    for (int c = 0; c < MAX_R; ++c) {
        const uint64_t v = c < R ? (uint64_t)(llrint(w[c] * sc) + (long long)BIAS) : BIAS;
        lo[c] = (uint32_t)v;
        hi[c] = (uint32_t)(v >> 32);
    }
#pragma unroll
    for (int t = 0; t < ND; ++t) {
        const int m = 5 - t;  // byte of X + bias
#pragma unroll
        for (int u16 = 0; u16 < 4; ++u16) {  // 16 c per 16-byte unit (c >= R: digit 0)
            uint32_t wd[4];
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
                uint32_t word = 0;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int c = 16 * u16 + 4 * qq + e;
                    const uint32_t src = c < MAX_R ? (m < 4 ? lo[c] : hi[c]) : 0x80808080u;
                    word |= (((src >> (8 * (m & 3))) & 255u) ^ 0x80u) << (8 * e);
                }
                wd[qq] = word;
            }
            *reinterpret_cast<uint4*>(base + (size_t)t * WBLK + sw64(rr, 16 * u16)) = make_uint4(wd[0], wd[1], wd[2], wd[3]);
        }
    }
}

// Fixed-order two-level sum of the per-(unit, warp) partials: k_err_i8_sum1 reduces contiguous ranges
// (block b: pairs [b per, (b + 1) per), thread strided, tree in shared memory), k_err_i8_final the
// block sums in order; out3 = {E, ||F||, ||F - Ft||}.
constexpr int SUMB = 1024;
__global__ void __launch_bounds__(256) k_err_i8_sum1(const double* __restrict__ part, int64_t n, double* __restrict__ bs) {
    const int64_t per = (n + SUMB - 1) / SUMB, b0 = (int64_t)blockIdx.x * per, b1 = min(n, b0 + per);
    double se = 0.0, sf = 0.0;
    for (int64_t b = b0 + threadIdx.x; b < b1; b += blockDim.x) {
        se += part[2 * b];
        sf += part[2 * b + 1];
    }
    __shared__ double red[2][256];
    red[0][threadIdx.x] = se;
    red[1][threadIdx.x] = sf;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) {
            red[0][threadIdx.x] += red[0][threadIdx.x + o];
            red[1][threadIdx.x] += red[1][threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        bs[2 * blockIdx.x] = red[0][0];
        bs[2 * blockIdx.x + 1] = red[1][0];
    }
}
__global__ void __launch_bounds__(SUMB) k_err_i8_final(const double* __restrict__ bs, double* out3) {
    __shared__ double red[2][SUMB];
    red[0][threadIdx.x] = bs[2 * threadIdx.x];
    red[1][threadIdx.x] = bs[2 * threadIdx.x + 1];
    __syncthreads();
    for (int o = SUMB / 2; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) {
            red[0][threadIdx.x] += red[0][threadIdx.x + o];
            red[1][threadIdx.x] += red[1][threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double nf = sqrt(red[1][0]), nd = sqrt(red[0][0]);
        out3[0] = nd / nf;
        out3[1] = nf;
        out3[2] = nd;
    }
}

}  // namespace e8

bool err_i8_applies(const int64_t n[3], const int32_t r[3], const double* F) {
    return r[2] >= 1 && r[2] <= e8::MAX_R && r[1] <= 64 && n[2] % 2 == 0 && n[2] <= 16384 &&
           (reinterpret_cast<uintptr_t>(F) & 15) == 0;
}

size_t err_i8_ws_bytes(const int64_t n[3], const int32_t r[3]) {
    using namespace e8;
    const int64_t M = n[0] * n[1], nfc = ceil_div(M, (int64_t)FC), nkt = ceil_div(n[2], (int64_t)KT);
    return align_up((size_t)n[0] * r[1] * r[2] * 8, 256) + align_up((size_t)nfc * WIMG, 1024) +
           align_up((size_t)nfc * FC * 8, 256) + align_up((size_t)nkt * AIMG, 1024) + align_up((size_t)nkt * KT * 8, 256) +
           align_up((size_t)nkt * nfc * NEPI * 16, 256) + 256 + (size_t)SUMB * 16;
}

// out3 = {E, ||F||, ||F - Ft||} with Ft's reconstruction on the INT8 tensor cores (R23).  UNSUPPORTED when
// the shape does not apply or ws is too small (the caller then runs the DMMA error pass).
int launch_error_i8(const int64_t n[3], const int32_t r[3], const double* F, const double* U1, const double* U2,
                    const double* U3, const double* core, double* out3, void* ws, size_t ws_bytes, cudaStream_t st) {
    using namespace e8;
    if (!err_i8_applies(n, r, F) || ws_bytes < err_i8_ws_bytes(n, r)) return TUCKER_ERR_UNSUPPORTED;
    const int R = r[2];
    const int64_t M = n[0] * n[1], nfc = ceil_div(M, (int64_t)FC), nkt = ceil_div(n[2], (int64_t)KT);
    const int64_t r23 = (int64_t)r[1] * R, nunits = nkt * nfc;
    char* w = static_cast<char*>(ws);
    double* X = reinterpret_cast<double*>(w);
    w += align_up((size_t)n[0] * r23 * 8, 256);
    uint8_t* Wimg = reinterpret_cast<uint8_t*>(w);
    w += align_up((size_t)nfc * WIMG, 1024);
    double* ps = reinterpret_cast<double*>(w);
    w += align_up((size_t)nfc * FC * 8, 256);
    uint8_t* Aimg = reinterpret_cast<uint8_t*>(w);
    w += align_up((size_t)nkt * AIMG, 1024);
    double* kscale = reinterpret_cast<double*>(w);
    w += align_up((size_t)nkt * KT * 8, 256);
    double* part = reinterpret_cast<double*>(w);
    w += align_up((size_t)nunits * NEPI * 16, 256);
    int* sched = reinterpret_cast<int*>(w);
    // X (n1 x r2 r3) = U1 (n1 x r1) * core (r1 x r2 r3)
    SmallGemm gx{n[0], r23, r[0], 1, U1, r[0], 1, 0, core, r23, 1, 0, X, r23, 1, 0};
    TK_RC(launch_small_gemm(gx, st));
    k_u3_digits_err<<<(unsigned)ceil_div(nkt * KT, (int64_t)8), 256, 0, st>>>(U3, n[2], R, (int)nkt, Aimg, kscale);
    TK_CHECK_LAUNCH();
    if (M % FC) {  // rows past M: zero digits and scale
        TK_CUDA(cudaMemsetAsync(Wimg + (size_t)(nfc - 1) * WIMG, 0, WIMG, st));
        TK_CUDA(cudaMemsetAsync(ps + (nfc - 1) * FC, 0, FC * 8, st));
    }
    const size_t smx = (size_t)r23 * 8;
    TK_CUDA(cudaFuncSetAttribute(k_w_digits, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smx));
    k_w_digits<<<dim3((unsigned)ceil_div(n[1], (int64_t)256), (unsigned)n[0]), 256, smx, st>>>(U2, X, n[1], r[1], R,
                                                                                                 Wimg, ps);
    TK_CHECK_LAUNCH();
    TK_CUDA(cudaMemsetAsync(sched, 0, sizeof(int), st));
    PFN_tmapEncodeTiled enc = tmap_encoder();
    if (!enc) return TUCKER_ERR_CUDA;
    CUtensorMap map;  // F as M rows x n3 doubles, boxes of 128 k x 32 fibres (no swizzle; zero fill)
    std::memset(&map, 0, sizeof(map));
    cuuint64_t dims[2] = {(cuuint64_t)n[2], (cuuint64_t)M};
    cuuint64_t strides[1] = {(cuuint64_t)n[2] * 8};
    cuuint32_t box[2] = {KT, FC}, es[2] = {1, 1};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(F), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return report_cuda(cudaErrorInvalidValue, __FILE__, __LINE__);
    Args a{Aimg, kscale, Wimg, ps, part, M, n[2], (int)nkt, (int)nfc, nunits, sched};
    const size_t sm = smem_bytes();
    TK_CUDA(cudaFuncSetAttribute(k_err_i8, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k_err_i8<<<(unsigned)std::min<int64_t>(nunits, kNumSMs), NT, sm, st>>>(map, a);
    TK_CHECK_LAUNCH();
    double* bsum = reinterpret_cast<double*>(sched + 64);  // SUMB x 2 block sums
    k_err_i8_sum1<<<SUMB, 256, 0, st>>>(part, nunits * NEPI, bsum);
    TK_CHECK_LAUNCH();
    k_err_i8_final<<<1, SUMB, 0, st>>>(bsum, out3);
    TK_CHECK_LAUNCH();
    return TUCKER_OK;
}

}  // namespace tk
