// ttm_i8.cu — a-5 (the core by the TTM chain) with its dominant product on the INT8
// tensor cores: T1 = F x3 U3^T, i.e. T1[p, c] = sum_k F[p, k] U3[k, c] over the n1 n2 mode-3 fibres
// p = (i, j) of F — 2 N r3 flops, FP64-bound on the DMMA pipe at r3 = 40.  Digit (Ozaki-I) emulation:
//
//   X = rint(F 2^(46 - E)) with max |F| < 2^E (the tensor's global exponent, the one the INT8 Gram
//       route already scales by: DESIGN.md R20), |X| <= 2^46, and per column c of U3
//   Y = rint(U3 2^(46 - E_c)) with max_k |U3[k, c]| < 2^E_c.  Both are split into six balanced
//       base-256 digits, X = sum_s x_s 256^(5 - s), x_s in [-128, 127] (int8) — the bytes of
//       X + 0x808080808080 with their top bit flipped (one DFMA puts X + bias in the low 48 mantissa
//       bits: fma(F, 2^(46-E), 2^52 + bias)).
//   X Y = sum_{s,t} x_s y_t 256^(10 - s - t).  The 26 digit pairs with s + t <= 6 are formed on the
//       tensor cores (tcgen05 kind::i8, exact int32 accumulation: |sum| <= 6 * 128^2 * n3 < 2^31
//       for n3 <= 2^14), summed per group d = s + t in TMEM; the dropped pairs weigh
//       <= 2^-52 of max|X| max|Y| per term.  T1 = sum_d acc_d 2^(E + E_c - 12 - 8 d) in FP64.
//
// So T1 carries the input rounding 2^-47 max|F| (and 2^-47 max|U3[:, c]|) plus ~2^-52 per term —
// at the level of the FP64 DMMA product's own accumulation error (n3 2^-53).  DESIGN.md R22.
//
// k_ttm1_i8: persistent, one CTA per SM (minus the SMs a concurrent eigensolve needs), 128-fibre
// tiles (M = 128 TMEM lanes) taken dynamically from a global counter, warp-specialised:
//   warp 0      TMEM owner + MMA issuer (one thread): per K-step (32 k) one MMA per F digit s
//               (M = 128, N = NB x the U3 digits t paired with it, rounded up to 16; K = 32) into
//               TMEM columns NB s ..: pair (s, t) accumulates in group s + t; the epilogue zeroes
//               the accumulator before each tile;
//   warp 1      F loader and tile schedule: two TMA boxes (16 k x 128 fibres, SWIZZLE_128B, zero
//               fill past the edges) per K-step into a 5-stage ring (160 KB per SM), each stage
//               converted in place into its K-step's digit tiles and freed by the MMAs' commit;
//   warps 2-5   epilogue: tcgen05.ld of the 7 groups, Horner in FP64, T1 rows to HBM;
//   warp 6      B loader: the U3 digit image of each 128-k block (6 NB rows x 128 B, pre-swizzled
//               SWIZZLE_128B) by one cp.async.bulk into a 2-stage ring;
//   warps 7-22  converters: every K-step over all 16 warps (8 k of one fibre row per thread — every
//               warp takes every stage in order, so its parity waits are exact), F from the stage
//               through the swizzle (conflict-free), one DFMA + byte permutes per element, the
//               digit words stored over the rows just read in the SWIZZLE_128B K-major A layout
//               (two 128 x 128 B tiles per K-step: digits 0-3 and 4-5 as the 32-byte K chunks).
// T1 is written transposed (T1t[j][i][c], n2 x n1 r3) so that TTM2 is ONE DMMA GEMM
// U2^T (r2 x n2) T1t; TTM3 follows on T2 (0.3 % of the flops together).
#include "common.cuh"
#include "kernels.h"
#include "prof.h"

#include <cstring>

namespace tk {
namespace t8 {

constexpr int ND = 6;                      // base-256 digits per operand
constexpr int NGRP = 7;                    // TMEM groups d = s + t = 0..6
// One ring of NS stages, 32 KB each: a stage holds one K-step (32 k) of 128 fibres as two TMA
// boxes of F (SWIZZLE_128B, 16 doubles per row), then — converted in place by the converter warps —
// the same K-step as two SWIZZLE_128B A tiles of digits (tile 0: digits 0-3, tile 1: digits 4-5 as
// the 32-byte K chunks of a row), then it is freed by the MMAs' commit.
constexpr int NS = 5;
constexpr uint32_t ATILE = 128 * 128;      // one SWIZZLE_128B tile / F box: 128 rows x 128 bytes
constexpr uint32_t FBOX = ATILE;
constexpr uint32_t STAGE = 2 * ATILE;
constexpr int NCONV = 16;                  // converter warps (each K-step: 8 fibre rows x 32 k per warp)
constexpr int NT = 32 * (7 + NCONV);       // warps 0 MMA, 1 F loader, 2-5 epilogue, 6 B loader, 7.. converters
constexpr uint64_t BIAS = 0x808080808080ull;
constexpr int TQ = 4;                                        // tile-id ring depth
constexpr int TQ_CONSUMERS = 1 + 1 + 4 + NCONV;              // MMA, B loader, epilogue and converter warps
constexpr int MAX_R = 40;  // NB = r3 rounded up to 8, one MMA per digit (N = 6 NB <= 256)
constexpr int SB = 2, BK = 128;            // B ring: 128-k blocks (SWIZZLE_128B rows of 128 bytes)
constexpr size_t smem_bytes(int NB) {
    return (size_t)NS * STAGE + (size_t)SB * ND * NB * BK + 1024;
}

struct Args {
    const double* F;         // M x n3 (fibre-major, k contiguous)
    const uint8_t* Bimg;     // [nkb][ND * NB rows][128 B], SWIZZLE_128B image
    const double* colscale;  // [R]: 2^(E_c - 12)
    const uint32_t* gmax;    // high word of max |F| (the INT8 route's global exponent)
    double* T1;              // T1t: n2 x n1 x R (the TTM2 GEMM's K-major operand)
    int64_t M, n1, n2, n3;
    int R, NB, nks, nkb, ntiles;
    int* sched;  // tile counter (zero at launch): CTAs take tiles dynamically
};

__device__ __forceinline__ int exp_of(uint32_t hw) {  // E with max |F| < 2^E (gram_i8.cu row_exponent)
    const int ef = (int)(hw >> 20);
    return hw == 0u ? 0 : (ef == 0 ? -1022 : ef - 1022);
}
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {  // K-major SWIZZLE_128B, SBO 1024 B
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ uint64_t desc_sw64(uint32_t saddr) {  // K-major SWIZZLE_64B, SBO 512 B
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(512 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)4 << 61);
}
__device__ __forceinline__ uint32_t idesc_s8(int N) {  // D s32, A/B s8, K-major, M = 128
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_s8(uint32_t tmem, uint32_t a, uint32_t b, int N, uint32_t acc) {
    const uint64_t da = desc_sw128(a), db = desc_sw128(b);
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
__device__ __forceinline__ void tmem_st32_zero(uint32_t addr) {  // 32 columns of the warp's lanes := 0
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
        "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};\n" ::"r"(addr),
        "r"(0)
        : "memory");
}
// word of digit byte m (0 = least significant) of four elements' X + bias, top bits flipped
__device__ __forceinline__ uint32_t digit_word(uint32_t a, uint32_t b, uint32_t c, uint32_t d, int m) {
    const uint32_t sel = (uint32_t)m | ((uint32_t)(m + 4) << 4);
    return __byte_perm(__byte_perm(a, b, sel), __byte_perm(c, d, sel), 0x5410) ^ 0x80808080u;
}

__global__ void __launch_bounds__(NT, 1) k_ttm1_i8(const __grid_constant__ CUtensorMap mapF, const Args g) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    uint8_t* sS = smem;                    // the F / digit ring
    uint8_t* sB = smem + NS * STAGE;
    // ffull: F landed (TMA); afull: digits written (converters); sempty: MMAs done (commit)
    __shared__ __align__(8) uint64_t ffull[NS], afull[NS], sempty[NS], bfull[SB], bempty[SB], tfull, tempty;
    __shared__ __align__(8) uint64_t tq_full[TQ], tq_empty[TQ];
    __shared__ int tq[TQ];
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int NB = g.NB;
    const uint32_t bstage = (uint32_t)(ND * NB * BK);
    const int nks = g.nks;
    // Dynamic tile schedule: the F loader takes the next tile from the global counter and posts
    // it in a TQ-deep ring; every other role reads it there (a CTA whose SM is held by a
    // concurrent kernel — the mode-0 eigensolve on its side stream — then takes fewer tiles).
    auto next_tile = [&](int it) -> int {  // consumers: one thread per role unit
        const int slot = it % TQ;
        mbar_wait(&tq_full[slot], (uint32_t)(it / TQ) & 1u);
        const int t = *reinterpret_cast<volatile int*>(&tq[slot]);
        mbar_arrive(&tq_empty[slot]);
        return t;
    };
    auto next_tile_warp = [&](int it) -> int {
        int t = 0;
        if (lane == 0) t = next_tile(it);
        return __shfl_sync(0xffffffffu, t, 0);
    };
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&ffull[s], 1);
            mbar_init(&afull[s], NCONV);
            mbar_init(&sempty[s], 1);
        }
        for (int s = 0; s < SB; ++s) {
            mbar_init(&bfull[s], 1);
            mbar_init(&bempty[s], 1);
        }
        mbar_init(&tfull, 1);
        mbar_init(&tempty, 4);
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

    if (warp == 0) {
        if (lane == 0) {  // MMA issuer
            int as = 0, bs = 0;
            uint32_t aph = 0, bph = 0;
            const uint32_t tb = (uint32_t)(NB * BK);  // one digit block of B rows
            for (int it = 0;; ++it) {
                if (next_tile(it) < 0) break;
                mbar_wait(&tempty, it & 1);  // drained and zeroed by the epilogue
                fence_after();
                for (int ks = 0; ks < nks; ++ks) {
                    const int j = ks & 3;  // K-step within the 128-k B block
                    if (j == 0) mbar_wait(&bfull[bs], bph);
                    mbar_wait(&afull[as], aph);
                    fence_after();
                    const uint32_t a0 = smem_u32(sS + as * STAGE), a1 = a0 + ATILE;
                    const uint32_t b0 = smem_u32(sB + bs * bstage) + 32u * j;
                    // one MMA per digit s of F: B rows of digits t = 0 .. min(5, 6 - s) (N rounded
                    // up to 16: the extra rows land in columns of group 7, never read) into TMEM
                    // columns NB s ..: pair (s, t) accumulates in group s + t
#pragma unroll
                    for (int sd = 0; sd < ND; ++sd) {
                        const int nt = sd < 2 ? 6 : 7 - sd;
                        mma_s8(tmem + (uint32_t)(NB * sd), (sd < 4 ? a0 : a1) + 32u * (sd & 3), b0,
                               (nt * NB + 15) & ~15, 1u);
                    }
                    commit(&sempty[as]);
                    if (++as == NS) {
                        as = 0;
                        aph ^= 1;
                    }
                    if (j == 3 || ks == nks - 1) {
                        commit(&bempty[bs]);
                        if (++bs == SB) {
                            bs = 0;
                            bph ^= 1;
                        }
                    }
                }
                commit(&tfull);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // F loader: two SWIZZLE_128B boxes (16 k x 128 fibres) per K-step
            int fs = 0;
            uint32_t fph = 0;
            for (int it = 0;; ++it) {
                const int slot = it % TQ;
                mbar_wait(&tq_empty[slot], ((uint32_t)(it / TQ) & 1u) ^ 1u);
                int tile = atomicAdd(g.sched, 1);
                if (tile >= g.ntiles) tile = -1;
                tq[slot] = tile;
                mbar_arrive(&tq_full[slot]);
                if (tile < 0) break;
                for (int ks = 0; ks < nks; ++ks) {
                    const int k0 = ks * 32;
                    mbar_wait(&sempty[fs], fph ^ 1);
                    mbar_arrive_expect_tx(&ffull[fs], STAGE);
                    uint8_t* dst = sS + fs * STAGE;
                    tma_load_2d(dst, &mapF, &ffull[fs], k0, tile * 128);
                    tma_load_2d(dst + FBOX, &mapF, &ffull[fs], k0 + 16, tile * 128);
                    if (++fs == NS) {
                        fs = 0;
                        fph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 6) {
        if (lane == 0) {  // B loader
            int bs = 0;
            uint32_t bph = 0;
            for (int it = 0; next_tile(it) >= 0; ++it)
                for (int kb = 0; kb < g.nkb; ++kb) {
                    mbar_wait(&bempty[bs], bph ^ 1);
                    mbar_arrive_expect_tx(&bfull[bs], bstage);
                    bulk_load(sB + bs * bstage, g.Bimg + (size_t)kb * bstage, bstage, &bfull[bs]);
                    if (++bs == SB) {
                        bs = 0;
                        bph ^= 1;
                    }
                }
        }
    } else if (warp < 6) {  // epilogue: TMEM lanes 32 (warp % 4) ..
        const int lg = warp & 3, row = lg * 32 + lane;
        const double sE = ldexp(1.0, exp_of(*g.gmax));
        const uint32_t taddr = tmem + ((uint32_t)(lg * 32) << 16);
        const int ncol = (NGRP * NB + 16 + 31) & ~31;  // groups 0-6 and the rounding columns
        auto zero_tmem = [&]() {  // every MMA accumulates: the tile starts from zeros
            for (int c = 0; c < ncol; c += 32) tmem_st32_zero(taddr + (uint32_t)c);
            asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty);
        };
        zero_tmem();
        for (int it = 0;; ++it) {
            const int tile = next_tile_warp(it);
            if (tile < 0) break;
            mbar_wait(&tfull, it & 1);
            fence_after();
            const int64_t p = (int64_t)tile * 128 + row;  // fibre (i, j): T1t[j][i][:] (n2 x n1 R)
            const int64_t pi = p / g.n2, pj = p - pi * g.n2;
            double* out = g.T1 + (pj * g.n1 + pi) * g.R;
            for (int c0 = 0; c0 < g.R; c0 += 8) {
                uint32_t a[NGRP][8];
#pragma unroll
                for (int d = 0; d < NGRP; ++d) tmem_ld8(taddr + (uint32_t)(d * NB + c0), a[d]);
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
                if (p < g.M) {
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const int c = c0 + e;
                        if (c < g.R) {
                            double v = (double)(int)a[NGRP - 1][e];
#pragma unroll
                            for (int d = NGRP - 2; d >= 0; --d) v = fma(v, 0x1p-8, (double)(int)a[d][e]);
                            out[c] = v * (g.colscale[c] * sE);
                        }
                    }
                }
            }
            zero_tmem();
        }
    } else {  // converters: every K-step is split over all 16 warps (thread -> fibre row, 8-k quarter),
              // so every converter warp consumes every stage in order and its parity waits are exact
        // a quarter warp (one 16-byte access phase) = 8 consecutive rows of one quarter: distinct
        // swizzled chunks; a warp holds 8 whole rows (both boxes), which it alone reads and rewrites
        const int ct = tid - 224, qt = (ct >> 3) & 3, row = (ct & 7) | ((ct >> 5) << 3), h = qt >> 1;
        const int E = exp_of(*g.gmax);
        const double sc = ldexp(1.0, 46 - E);
        const double magic = 4503599627370496.0 + (double)BIAS;  // 2^52 + bias
        // this thread's 8 doubles: chunks 4 (qt % 2) .. +3 of its row in F box h (chunk u at u ^ (row % 8));
        // its digit bytes: 8 bytes at byte 8 (qt % 2) of unit 2 (s % 4) + h of its row (same swizzle)
        const uint32_t rbase = (uint32_t)((row >> 3) * 1024 + (row & 7) * 128);
        int fs = 0;
        uint32_t fph = 0;
        for (int it = 0;; ++it) {
            if (next_tile_warp(it) < 0) break;
            for (int ks = 0; ks < nks; ++ks) {
                mbar_wait(&ffull[fs], fph);
                const uint32_t st0 = smem_u32(sS + fs * STAGE) + rbase;
                const uint32_t f0 = st0 + h * FBOX;
                double x[8];
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n"
                                 : "=d"(x[2 * u]), "=d"(x[2 * u + 1])
                                 : "r"(f0 + (((uint32_t)(4 * (qt & 1) + u) ^ (uint32_t)(row & 7)) << 4))
                                 : "memory");
                __syncwarp();  // the digits overwrite the rows just read (this warp's own rows)
                uint32_t w[ND][2];  // [digit s][group of 4 k]
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    uint32_t lo[4], hi[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const long long b = __double_as_longlong(fma(x[4 * u + e], sc, magic));
                        lo[e] = (uint32_t)b;
                        hi[e] = (uint32_t)(b >> 32);
                    }
#pragma unroll
                    for (int m = 0; m < 4; ++m) w[5 - m][u] = digit_word(lo[0], lo[1], lo[2], lo[3], m);
#pragma unroll
                    for (int m = 0; m < 2; ++m) w[1 - m][u] = digit_word(hi[0], hi[1], hi[2], hi[3], m);
                }
#pragma unroll
                for (int sd = 0; sd < ND; ++sd) {
                    const uint32_t qq = (uint32_t)(2 * (sd & 3) + h) ^ (uint32_t)(row & 7);
                    const uint32_t addr = st0 + (uint32_t)(sd >> 2) * ATILE + (qq << 4) + 8u * (uint32_t)(qt & 1);
                    asm volatile("st.shared.v2.b32 [%0], {%1, %2};\n" ::"r"(addr), "r"(w[sd][0]), "r"(w[sd][1])
                                 : "memory");
                }
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&afull[fs]);
                if (++fs == NS) {
                    fs = 0;
                    fph ^= 1;
                }
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

// U3 (n3 x R, row-major) -> column exponents and the SWIZZLE_128B digit image of B:
// block kb (128 k) holds rows NB t + c (digit t of column c, most significant first), 128 bytes
// each (k = 128 kb .. + 127), 16-byte unit u of row r at unit u ^ (r % 8).  One CTA per column.
__global__ void __launch_bounds__(256) k_u3_digits(const double* __restrict__ U3, int64_t n3, int R, int NB,
                                                   uint8_t* __restrict__ img, double* __restrict__ colscale) {
    const int c = blockIdx.x;
    double mx = 0.0;
    for (int64_t k = threadIdx.x; k < n3; k += blockDim.x) mx = fmax(mx, fabs(U3[k * R + c]));
    __shared__ double red[32];
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        v = warp_max(v);
        if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    int Ec = 0;
    if (red[0] > 0.0) frexp(red[0], &Ec);  // max < 2^Ec
    if (threadIdx.x == 0) colscale[c] = ldexp(1.0, Ec - 12);
    const double sc = ldexp(1.0, 46 - Ec);
    const size_t bstage = (size_t)ND * NB * BK;
    for (int64_t k = threadIdx.x; k < n3; k += blockDim.x) {
        const uint64_t w = (uint64_t)(llrint(U3[k * R + c] * sc) + (long long)BIAS);
        const int64_t kb = k / BK;
        const int kc = (int)(k % BK);
        for (int t = 0; t < ND; ++t) {
            const int r = NB * t + c;
            const size_t off = (size_t)kb * bstage + (size_t)(r >> 3) * 1024 + (size_t)(r & 7) * 128 +
                               (size_t)((((kc >> 4) ^ (r & 7)) << 4) | (kc & 15));
            img[off] = (uint8_t)(((w >> (8 * (5 - t))) & 255u) ^ 0x80u);
        }
    }
}

// T2[i][b][c] = sum over the S K-slices of T2p[sl][b][i][c] (slice order)
__global__ void __launch_bounds__(256) k_t2_transpose(const double* __restrict__ T2p, int S, int64_t n1, int r2,
                                                      int R, double* __restrict__ T2) {
    const int64_t total = n1 * r2 * R;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / ((int64_t)r2 * R), o = t - i * r2 * R;
        const int b = (int)(o / R), c = (int)(o - (int64_t)b * R);
        const double* p = T2p + ((int64_t)b * n1 + i) * R + c;
        double v = p[0];
        for (int sl = 1; sl < S; ++sl) v += p[sl * total];
        T2[t] = v;
    }
}

}  // namespace t8

bool ttm_i8_applies(const int64_t n[3], const int32_t r[3], const double* F) {
    return r[2] >= 1 && r[2] <= t8::MAX_R && n[2] % 16 == 0 && n[2] <= 16384 &&
           (reinterpret_cast<uintptr_t>(F) & 15) == 0;
}

size_t ttm_i8_region_bytes(const int64_t n[3], const int32_t r[3]) {
    const int NB = ((r[2] + 7) / 8) * 8;
    const int64_t nkb = ceil_div(n[2], (int64_t)t8::BK);
    return align_up((size_t)n[0] * n[1] * r[2] * 8, 1024) + align_up((size_t)nkb * t8::ND * NB * t8::BK, 1024) +
           align_up((size_t)r[2] * 8, 256) + 256 + align_up((size_t)8 * n[0] * r[1] * r[2] * 8, 256);
}

// T2 (n1 x r2 x r3) = (F x3 U3^T) x2 U2^T with the first product on the INT8 tensor cores.
// gmax: the INT8 route's global exponent word (device); region: device scratch of
// ttm_i8_region_bytes.  UNSUPPORTED when the shape does not apply (the caller uses the DMMA TTM).
int launch_ttm12_i8(const int64_t n[3], const int32_t r[3], const double* F, const double* U2, const double* U3,
                    const uint32_t* gmax, double* T2, void* region, size_t region_bytes, cudaStream_t st,
                    int reserve_sms, bool profile) {
    using namespace t8;
    if (!ttm_i8_applies(n, r, F)) return TUCKER_ERR_UNSUPPORTED;
    if (region_bytes < ttm_i8_region_bytes(n, r)) return TUCKER_ERR_UNSUPPORTED;
    ProfScope prof(profile ? TUCKER_PROF_TTM : -1, st);
    const int R = r[2], NB = ((R + 7) / 8) * 8;
    const int64_t M = n[0] * n[1];
    const int64_t nkb = ceil_div(n[2], (int64_t)BK);
    char* w = static_cast<char*>(region);
    double* T1 = reinterpret_cast<double*>(w);
    w += align_up((size_t)M * R * 8, 1024);
    uint8_t* img = reinterpret_cast<uint8_t*>(w);
    const size_t img_bytes = (size_t)nkb * ND * NB * BK;
    w += align_up(img_bytes, 1024);
    double* colscale = reinterpret_cast<double*>(w);
    w += align_up((size_t)R * 8, 256);
    int* sched = reinterpret_cast<int*>(w);
    w += 256;
    TK_CUDA(cudaMemsetAsync(sched, 0, sizeof(int), st));
    double* part = reinterpret_cast<double*>(w);
    TK_CUDA(cudaMemsetAsync(img, 0, img_bytes, st));
    k_u3_digits<<<R, 256, 0, st>>>(U3, n[2], R, NB, img, colscale);
    TK_CHECK_LAUNCH();
    Args a{F, img, colscale, gmax, T1, M, n[0], n[1], n[2], R, NB, (int)ceil_div(n[2], (int64_t)32), (int)nkb,
           (int)ceil_div(M, (int64_t)128), sched};
    CUtensorMap map;  // F as M rows x n3 doubles, boxes of 16 k x 128 fibres (SWIZZLE_128B; zero fill)
    std::memset(&map, 0, sizeof(map));
    const uint64_t dims[2] = {(uint64_t)n[2], (uint64_t)M};
    const uint64_t strides[1] = {(uint64_t)n[2] * 8};
    const uint32_t box[2] = {16, 128};
    if (!make_tmap_f64(&map, F, 2, dims, strides, box)) return ::tk::report_cuda(cudaErrorInvalidValue, __FILE__, __LINE__);
    const size_t sm = smem_bytes(NB);
    TK_CUDA(cudaFuncSetAttribute(k_ttm1_i8, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    // one CTA per SM; `reserve_sms` SMs are left to a concurrent kernel (the mode-0 eigensolve's cluster,
    // which would otherwise wait for the whole persistent grid): the dynamic schedule absorbs it
    const int grid = (int)std::min<int64_t>(a.ntiles, std::max(kNumSMs - reserve_sms, kNumSMs / 2));
    k_ttm1_i8<<<grid, NT, sm, st>>>(map, a);
    TK_CHECK_LAUNCH();
    // TTM2 as one GEMM over the transposed T1, K = n2 split into S slices (a batch):
    // T2p[sl] (r2 x n1 R) = U2[slice]^T T1t[slice], then T2[i][b][c] = sum_sl T2p[sl][b][i][c] in
    // slice order (fixed, deterministic)
    const int S = n[1] % 8 == 0 ? 8 : 1;
    const int64_t Ks = n[1] / S, plane = n[0] * r[1] * R;
    const SmallGemm g2{r[1], n[0] * R, Ks, S, U2, 1, r[1], Ks * r[1], T1, n[0] * R, 1, Ks * n[0] * R,
                       part, n[0] * R, 1, plane, 0};
    TK_RC(launch_gemm(g2, st));
    k_t2_transpose<<<(unsigned)std::min<int64_t>(ceil_div(plane, 256), 4096), 256, 0, st>>>(part, S, n[0], r[1], R, T2);
    TK_CHECK_LAUNCH();
    return TUCKER_OK;
}

int& ttm_engine() {  // per calling thread (tucker_set_ttm_engine)
    static thread_local int engine = TUCKER_TTM_AUTO;
    return engine;
}

}  // namespace tk
