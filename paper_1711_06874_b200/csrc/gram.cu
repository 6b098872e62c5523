// gram.cu — a-3: per-mode Gram matrices G_m = F_(m) F_(m)^T.
//
// P:555-561 computes the HOSVD factors from "the SVD of the matrix unfolding A_(l)"; its left
// singular vectors are the eigenvectors of G_m, and P:581-585 identifies this O(n^{d+1}) step as
// the cost of the whole method.  G_m is invariant to the column order of the unfolding, so no
// unfolding is materialised: the three modes read F in place.
//   mode 0: F as n1 x (n2 n3) row-major; contraction index contiguous ("K-major").
//   mode 1: sum_i S_i S_i^T over slabs S_i = F[i,:,:] (n2 x n3), K-major, batched over i.
//   mode 2: F as B = (n1 n2) x n3 row-major, G = B^T B: contraction over the slow index
//           ("M-major").
//
// Kernel: SYRK on FP64 tensor cores.  B200 has no tcgen05 f64 kind, so the MMA is the legacy
// mma.sync m8n8k4 f64 (SASS DMMA.8x8x4); FP64 DFMA and DMMA share one pipe on GB100.
// Lower-triangular 128x128 output tiles x S split-K slices; each CTA = 8 MMA warps (64x32 warp
// tiles, 128 FP64 accumulators per lane); thread 0 also issues the TMA loads (cp.async.bulk.tensor,
// SWIZZLE_128B) into a 6-stage mbarrier ring.  Diagonal tiles load one operand (B = A).
// Split-K partial tiles go to the workspace and a fixed-order reduction writes both triangles —
// deterministic, no float atomics.  Shapes TMA cannot describe (odd n3 -> unaligned strides, or
// n_m < 128) take a cp.async (LDGSTS) variant of the same mainloop.
//
// Bank-conflict-free fragment loads (all LDS.128): K-major tiles use k = 4q + s per lane
// (q = lane & 3), which is a permutation of the 16 k of a stage shared by both operands; M-major
// tiles permute rows (m = 8r + mi for A, m = base(r) + ni for B) so that each lane reads
// consecutive doubles.  The epilogue undoes the permutation.
#include <cstdlib>

#include "common.cuh"
#include "fill_eval.cuh"
#include "kernels.h"
#include "prof.h"

namespace tk {
namespace gram {

constexpr int BM = 128;
constexpr int BK = 16;
constexpr int STAGES = 6;
constexpr int STAGES_G = 4;
constexpr int NCW = 8;  // MMA warps
constexpr int TILE = BM * BK;
constexpr uint32_t TILE_BYTES = TILE * 8;

struct Args {
    int mode;
    int64_t n1, n2, n3, n;
    int S;
    int64_t nkb;   // number of 16-wide k blocks
    int64_t nkb3;  // ceil(n3/16) (mode 1)
    const double* F;
    double* part;  // [T][S][BM*BM]
    int m3d;       // mode 2: 3-D tensor map (see make_mmajor_map)
};

__device__ __forceinline__ void tile_decode(int t, int& ti, int& tj) {
    int i = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while ((i + 1) * (i + 2) / 2 <= t) ++i;
    while (i * (i + 1) / 2 > t) --i;
    ti = i;
    tj = t - i * (i + 1) / 2;
}

__device__ __forceinline__ int mmajor_nbase(int r) {
    return (r & 1) * 8 + ((r >> 1) & 1) * 4 + (r >> 2) * 16;
}

// K-major stage: A, B = [128 lines (m)][16 k], swizzled.  Warp tile rows wm*64.., cols wn*32..
__device__ __forceinline__ void mma_kmajor(const double* A, const double* B, double (&acc)[8][4][2],
                                           int wm, int wn, int r, int q) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        double a[8][2], b[4][2];
#pragma unroll
        for (int mi = 0; mi < 8; ++mi)
            lds128(a[mi][0], a[mi][1], A + swz_chunk(wm * 64 + mi * 8 + r, 2 * q + h));
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
            lds128(b[ni][0], b[ni][1], B + swz_chunk(wn * 32 + ni * 8 + r, 2 * q + h));
#pragma unroll
        for (int s = 0; s < 2; ++s)
#pragma unroll
            for (int mi = 0; mi < 8; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], a[mi][s], b[ni][s]);
    }
}

// M-major stage: A, B = [8 boxes][16 lines (k)][16 m], swizzled per box.
__device__ __forceinline__ void mma_mmajor(const double* A, const double* B, double (&acc)[8][4][2],
                                           int wm, int wn, int r, int q) {
    const int mA = wm * 64 + r * 8;
    const int nB = wn * 32 + mmajor_nbase(r);
    const double* Ab = A + (mA >> 4) * (BK * 16);
    const double* Bb = B + (nB >> 4) * (BK * 16);
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        const int k = q + 4 * s;
        double a[8], b[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) lds128(a[2 * c], a[2 * c + 1], Ab + swz_chunk(k, ((mA & 15) >> 1) + c));
#pragma unroll
        for (int c = 0; c < 2; ++c) lds128(b[2 * c], b[2 * c + 1], Bb + swz_chunk(k, ((nB & 15) >> 1) + c));
#pragma unroll
        for (int mi = 0; mi < 8; ++mi)
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
    }
}

template <bool MMAJOR>
__device__ __forceinline__ void store_partial(double* P, const double (&acc)[8][4][2], int wm, int wn,
                                              int r, int q) {
#pragma unroll
    for (int mi = 0; mi < 8; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) {
            if (!MMAJOR) {
                const int row = wm * 64 + mi * 8 + r, col = wn * 32 + ni * 8 + 2 * q;
                *reinterpret_cast<double2*>(P + row * BM + col) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
            } else {
                const int row = wm * 64 + r * 8 + mi;
                P[row * BM + wn * 32 + mmajor_nbase(2 * q) + ni] = acc[mi][ni][0];
                P[row * BM + wn * 32 + mmajor_nbase(2 * q + 1) + ni] = acc[mi][ni][1];
            }
        }
}

// -------------------------------------------------------------------------------- TMA variant
// 8 MMA warps; thread 0 doubles as the TMA producer (a 9th warp would round the CTA up to 12
// warps for register allocation and cap the MMA warps at 168 registers).  Slot s of the ring is
// refilled at the top of the iteration after it was consumed, so the empty-barrier wait rarely
// blocks.
template <int MODE>
__device__ __forceinline__ void issue_stage(const CUtensorMap* map, const Args& a, uint64_t* bar, double* dA,
                                            double* dB, int ti, int tj, bool diag, int64_t kb) {
    mbar_arrive_expect_tx(bar, diag ? TILE_BYTES : 2 * TILE_BYTES);
    if (MODE == 0) {
        tma_load_2d(dA, map, bar, (int)(kb * BK), ti * BM);
        if (!diag) tma_load_2d(dB, map, bar, (int)(kb * BK), tj * BM);
    } else if (MODE == 1) {
        const int i = (int)(kb / a.nkb3), kk = (int)(kb % a.nkb3) * BK;
        tma_load_3d(dA, map, bar, kk, ti * BM, i);
        if (!diag) tma_load_3d(dB, map, bar, kk, tj * BM, i);
    } else if (a.m3d) {  // one 3-D box {16 m, 16 k, 8 m-chunks} lands as [8][16][16] directly
        tma_load_3d(dA, map, bar, 0, (int)(kb * BK), ti * (BM / 16));
        if (!diag) tma_load_3d(dB, map, bar, 0, (int)(kb * BK), tj * (BM / 16));
    } else {
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            tma_load_2d(dA + b * BK * 16, map, bar, ti * BM + 16 * b, (int)(kb * BK));
            if (!diag) tma_load_2d(dB + b * BK * 16, map, bar, tj * BM + 16 * b, (int)(kb * BK));
        }
    }
}

// Mode-2 (M-major) tensor map over a row-major (rows x n3) matrix: preferably the 3-D view
// {16, rows, n3/16} with strides {8 n3, 128} B and box {16, 16, 8} (one TMA per operand per
// stage); else the 2-D view with 8 boxes of {16, 16}.  Returns 0/1 = 3-D used, -1 on failure.
static int make_mmajor_map(CUtensorMap* map, const void* base, uint64_t rows, uint64_t n3) {
    if (n3 % 16 == 0) {
        uint64_t dims[3] = {16, rows, n3 / 16};
        uint64_t strides[2] = {n3 * 8, 128};
        uint32_t box[3] = {16, BK, BM / 16};
        if (make_tmap_f64(map, base, 3, dims, strides, box)) return 1;
    }
    uint64_t dims[2] = {n3, rows};
    uint64_t strides[1] = {n3 * 8};
    uint32_t box[2] = {16, BK};
    return make_tmap_f64(map, base, 2, dims, strides, box) ? 0 : -1;
}

// Mainloop over k-blocks [kb0, kb1) for output tile (ti, tj); `it0` is the ring iteration
// counter at entry (stages/parities continue across calls; the ring must be drained, i.e. every
// earlier iteration consumed, on entry).  Thread 0 produces, the 8 warps consume.
template <int MODE>
__device__ __forceinline__ void gram_consume(const CUtensorMap* map, const Args& a, int ti, int tj, bool diag,
                                             int64_t kb0, int64_t kb1, int64_t it0, double* sA, double* sB,
                                             uint64_t* full, uint64_t* empty, double (&acc)[8][4][2]) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wm = warp >> 2, wn = warp & 3, r = lane >> 2, q = lane & 3;
    // on a diagonal tile the warps whose 64 x 32 sub-tile lies strictly above the diagonal
    // (rows 0..63, columns 64..127) skip their MMA: only the lower triangle reaches G (saves
    // issue slots and power; the split-K wave is set by the full tiles)
    const bool upper = diag && wm == 0 && wn >= 2;
    const int64_t L = kb1 - kb0;
    if (threadIdx.x == 0)
        for (int64_t j = 0; j < STAGES && j < L; ++j) {
            const int slot = (int)((it0 + j) % STAGES);
            issue_stage<MODE>(map, a, &full[slot], sA + slot * TILE, sB + slot * TILE, ti, tj, diag, kb0 + j);
        }
    for (int64_t l = 0; l < L; ++l) {
        const int64_t it = it0 + l;
        if (threadIdx.x == 0 && l > 0) {
            const int64_t prev = it - 1, nl = l - 1 + STAGES;
            if (nl < L) {
                const int ps = (int)(prev % STAGES);
                mbar_wait(&empty[ps], (uint32_t)((prev / STAGES) & 1));
                issue_stage<MODE>(map, a, &full[ps], sA + ps * TILE, sB + ps * TILE, ti, tj, diag, kb0 + nl);
            }
        }
        const int stage = (int)(it % STAGES);
        mbar_wait(&full[stage], (uint32_t)((it / STAGES) & 1));
        const double* A = sA + stage * TILE;
        const double* B = diag ? A : sB + stage * TILE;
        if (!upper) {
            if (MODE == 2) mma_mmajor(A, B, acc, wm, wn, r, q);
            else mma_kmajor(A, B, acc, wm, wn, r, q);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
    }
}

template <int MODE>
__global__ void __launch_bounds__(NCW * 32, 1)
    k_gram_tma(const __grid_constant__ CUtensorMap map, const Args a) {
    extern __shared__ uint8_t smem_raw[];
    double* smem = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    double* sA = smem;
    double* sB = smem + STAGES * TILE;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * TILE);
    uint64_t* empty = full + STAGES;

    int ti, tj;
    tile_decode(blockIdx.x, ti, tj);
    const bool diag = (ti == tj);
    const int s = blockIdx.y;
    const int64_t kb0 = (int64_t)s * a.nkb / a.S, kb1 = (int64_t)(s + 1) * a.nkb / a.S;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], NCW);
        }
        mbar_fence_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) tma_prefetch_desc(&map);

    const int wm = warp >> 2, wn = warp & 3, r = lane >> 2, q = lane & 3;
    double acc[8][4][2];
#pragma unroll
    for (int mi = 0; mi < 8; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
    gram_consume<MODE>(&map, a, ti, tj, diag, kb0, kb1, 0, sA, sB, full, empty, acc);
    double* P = a.part + ((size_t)blockIdx.x * a.S + s) * (BM * BM);
    store_partial<MODE == 2>(P, acc, wm, wn, r, q);
}

// --------------------------------------------------------------- a-7 fused generate-and-Gram
// F is never materialised: plane chunks of F (mode 0 and 2: j-planes, layout [n1][Pc][n3];
// mode 1: i-planes, [Pc][n2][n3]; see fill_eval.cuh) are generated by all CTAs into a 2-slot ring
// sized to stay L2-resident (~2 x 32 MB), then consumed by the same TMA + DMMA mainloop as the
// materialised Gram (the chunk is the sub-tensor whose mode-m Gram is the chunk's contribution).
// One persistent cooperative grid, one CTA per SM: T x S MMA CTAs (output tile x split-K slice) and
// the remaining SMs as generator CTAs; per chunk c:
//     generators: chunk c+1 -> slot (c+1)&1   ||   MMA CTAs: consume chunk c from slot c&1
//     grid barrier
// (with fewer than 2 spare SMs every CTA generates before consuming).
// Accumulators stay in registers across all chunks; the split-K partials and the fixed-order
// k_gram_reduce are those of the materialised path.  Generic-proxy stores are ordered before the
// async-proxy (TMA) reads of other CTAs by fence.proxy.async + the release/acquire grid barrier.
struct FusedArgs {
    Args a;             // virtual chunk shape (see launch_gram_fused), nkb of one chunk, S, part
    ChunkGeo geo;       // g0 is set per chunk
    KParams kp;
    const double* cheb;
    const double* x2;
    double* slot[2];
    int64_t nchunks;
    unsigned int* bar;  // grid-barrier counter (zeroed before the launch)
    int nmma;           // CTAs 0..nmma-1: output tile x split-K slice (T x S)
    int ngen;           // CTAs nmma..: dedicated generators (0: every CTA generates)
};

__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int target) {
    asm volatile("fence.proxy.async.global;\n" ::: "memory");  // my generic stores -> async proxy
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(bar, 1u);
        unsigned int v;
        long long spins = 0;
        while (true) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(bar) : "memory");
            if (v >= target) break;
            __nanosleep(64);
            if (++spins > (1ll << 27)) __trap();  // ~10 s: never hang the GPU
        }
    }
    __syncthreads();
}

template <int MODE>
__global__ void __launch_bounds__(NCW * 32, 1)
    k_gram_fused(const __grid_constant__ CUtensorMap map0, const __grid_constant__ CUtensorMap map1,
                 const FusedArgs f) {
    extern __shared__ uint8_t smem_raw[];
    double* smem = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    double* sA = smem;
    double* sB = smem + STAGES * TILE;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * TILE);
    uint64_t* empty = full + STAGES;
    const Args& a = f.a;
    const int cta = blockIdx.x, ncta = gridDim.x;
    const bool mma = cta < f.nmma;
    const int T = f.nmma / a.S;
    const int tile = cta % T, s = cta / T;
    int ti = 0, tj = 0;
    if (mma) tile_decode(tile, ti, tj);
    const bool diag = (ti == tj);
    const int64_t kb0 = (int64_t)s * a.nkb / a.S, kb1 = (int64_t)(s + 1) * a.nkb / a.S;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wm = warp >> 2, wn = warp & 3, r = lane >> 2, q = lane & 3;

    if (threadIdx.x == 0 && mma) {
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], NCW);
        }
        mbar_fence_init();
        tma_prefetch_desc(&map0);
        tma_prefetch_desc(&map1);
    }
    __syncthreads();

    ChunkGeo geo = f.geo;
    const int64_t items = chunk_items(geo);
    // chunk 0: every CTA generates; later chunks: the generator CTAs (if any) while the MMA CTAs
    // consume the previous chunk, else everyone before consuming
    geo.g0 = 0;
    gen_chunk(geo, f.kp, f.cheb, f.x2, f.slot[0], (int64_t)cta * blockDim.x + threadIdx.x, items,
              (int64_t)ncta * blockDim.x);
    unsigned int nbar = 1;
    grid_barrier(f.bar, nbar * ncta);
    const bool gen_role = f.ngen > 0 ? !mma : true;
    const int gidx = f.ngen > 0 ? cta - f.nmma : cta, gcount = f.ngen > 0 ? f.ngen : ncta;

    double acc[8][4][2];
#pragma unroll
    for (int mi = 0; mi < 8; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
    int64_t it = 0;
    for (int64_t c = 0; c < f.nchunks; ++c) {
        if (gen_role && c + 1 < f.nchunks) {
            geo.g0 = (c + 1) * geo.Pc;
            gen_chunk(geo, f.kp, f.cheb, f.x2, f.slot[(c + 1) & 1], (int64_t)gidx * blockDim.x + threadIdx.x, items,
                      (int64_t)gcount * blockDim.x);
        }
        if (mma) {
            gram_consume<MODE>((c & 1) ? &map1 : &map0, a, ti, tj, diag, kb0, kb1, it, sA, sB, full, empty, acc);
            it += kb1 - kb0;
        }
        ++nbar;
        grid_barrier(f.bar, nbar * ncta);
    }
    if (mma) {
        double* P = a.part + ((size_t)tile * a.S + s) * (BM * BM);
        store_partial<MODE == 2>(P, acc, wm, wn, r, q);
    }
}

// -------------------------------------------------------------------------- cp.async variant
template <int MODE>
__device__ __forceinline__ void load_stage_generic(const Args& a, double* dA, double* dB, int ti,
                                                   int tj, bool diag, int64_t kb) {
    const int tid = threadIdx.x;
#pragma unroll
    for (int u = 0; u < TILE / 256; ++u) {
        const int e = tid + 256 * u;
#pragma unroll
        for (int op = 0; op < 2; ++op) {
            if (op == 1 && diag) break;
            const int64_t m0 = (op == 0 ? ti : tj) * (int64_t)BM;
            double* dst = op == 0 ? dA : dB;
            if (MODE == 0) {
                const int line = e >> 4, col = e & 15;
                const int64_t m = m0 + line, k = kb * BK + col, K = a.n2 * a.n3;
                const bool ok = (m < a.n) && (k < K);
                cp_async8(dst + swz(line, col), ok ? a.F + m * K + k : a.F, ok);
            } else if (MODE == 1) {
                const int line = e >> 4, col = e & 15;
                const int64_t i = kb / a.nkb3, kk = (kb % a.nkb3) * BK + col, j = m0 + line;
                const bool ok = (j < a.n2) && (kk < a.n3);
                cp_async8(dst + swz(line, col), ok ? a.F + (i * a.n2 + j) * a.n3 + kk : a.F, ok);
            } else {
                const int b = e >> 8, line = (e >> 4) & 15, col = e & 15;
                const int64_t m = m0 + b * 16 + col, kr = kb * BK + line;
                const bool ok = (m < a.n3) && (kr < a.n1 * a.n2);
                cp_async8(dst + b * BK * 16 + swz(line, col), ok ? a.F + kr * a.n3 + m : a.F, ok);
            }
        }
    }
}

template <int MODE>
__global__ void __launch_bounds__(NCW * 32, 1) k_gram_generic(const Args a) {
    extern __shared__ uint8_t smem_raw[];
    double* smem = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    double* sA = smem;
    double* sB = smem + STAGES_G * TILE;
    int ti, tj;
    tile_decode(blockIdx.x, ti, tj);
    const bool diag = (ti == tj);
    const int s = blockIdx.y;
    const int64_t kb0 = (int64_t)s * a.nkb / a.S, kb1 = (int64_t)(s + 1) * a.nkb / a.S;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wm = warp >> 2, wn = warp & 3, r = lane >> 2, q = lane & 3;

    double acc[8][4][2];
#pragma unroll
    for (int mi = 0; mi < 8; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

#pragma unroll
    for (int st = 0; st < STAGES_G - 1; ++st) {
        if (kb0 + st < kb1) load_stage_generic<MODE>(a, sA + st * TILE, sB + st * TILE, ti, tj, diag, kb0 + st);
        cp_async_commit();
    }
    for (int64_t kb = kb0; kb < kb1; ++kb) {
        cp_async_wait<STAGES_G - 2>();
        __syncthreads();
        const int stage = (int)((kb - kb0) % STAGES_G);
        const double* A = sA + stage * TILE;
        const double* B = diag ? A : sB + stage * TILE;
        if (MODE == 2) mma_mmajor(A, B, acc, wm, wn, r, q);
        else mma_kmajor(A, B, acc, wm, wn, r, q);
        const int64_t nxt = kb + STAGES_G - 1;
        if (nxt < kb1) {
            const int ns = (int)((nxt - kb0) % STAGES_G);
            load_stage_generic<MODE>(a, sA + ns * TILE, sB + ns * TILE, ti, tj, diag, nxt);
        }
        cp_async_commit();
    }
    cp_async_wait<0>();
    double* P = a.part + ((size_t)blockIdx.x * a.S + s) * (BM * BM);
    store_partial<MODE == 2>(P, acc, wm, wn, r, q);
}

// Fixed-order split-K reduction; writes G[row][col] and its mirror (exactly symmetric G).
__global__ void k_gram_reduce(const double* __restrict__ part, int S, int64_t n, double* __restrict__ G) {
    int ti, tj;
    tile_decode(blockIdx.y, ti, tj);
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < BM * BM; e += gridDim.x * blockDim.x) {
        const int row = e / BM, col = e % BM;
        if (ti == tj && row < col) continue;
        const int64_t gr = (int64_t)ti * BM + row, gc = (int64_t)tj * BM + col;
        if (gr >= n || gc >= n) continue;
        const double* p = part + (size_t)blockIdx.y * S * (BM * BM) + e;
        double sum = 0.0;
        for (int s = 0; s < S; ++s) sum += p[(size_t)s * (BM * BM)];
        G[gr * n + gc] = sum;
        G[gc * n + gr] = sum;
    }
}

struct Plan {
    int T, S;
    int64_t n, nkb, nkb3;
    bool tma;
};

static Plan make_plan(const int64_t n[3], int mode) {
    Plan p{};
    p.n = n[mode];
    const int nt = (int)ceil_div(p.n, BM);
    p.T = nt * (nt + 1) / 2;
    p.nkb3 = ceil_div(n[2], BK);
    if (mode == 0) p.nkb = ceil_div(n[1] * n[2], BK);
    else if (mode == 1) p.nkb = n[0] * p.nkb3;
    else p.nkb = ceil_div(n[0] * n[1], BK);
    // smallest number of waves w whose split count fills >= 97% of the SM slots
    const int64_t cap = std::max<int64_t>(1, p.nkb / 4);
    p.S = 1;
    for (int w = 1; w <= 64; ++w) {
        int64_t S = std::min<int64_t>((int64_t)kNumSMs * w / p.T, cap);
        if (S < 1) continue;
        const double waves = (double)ceil_div(p.T * S, kNumSMs);
        p.S = (int)S;
        if ((double)(p.T * S) / (kNumSMs * waves) >= 0.97 || S == cap) break;
    }
    p.tma = (n[2] % 2 == 0) && n[0] >= BM && n[1] >= BM && n[2] >= BM;
    return p;
}

static size_t smem_tma() { return (size_t)2 * STAGES * TILE * 8 + 2 * STAGES * 8 + 1024; }
static size_t smem_generic() { return (size_t)2 * STAGES_G * TILE * 8 + 1024; }

}  // namespace gram

size_t gram_ws_bytes(const int64_t n[3]) {
    size_t b = 0;
    for (int m = 0; m < 3; ++m) {
        gram::Plan p = gram::make_plan(n, m);
        b = std::max(b, (size_t)p.T * p.S * gram::BM * gram::BM * sizeof(double));
    }
    return b;
}

int launch_gram(const int64_t n[3], int mode, const double* F, double* G, void* ws, size_t ws_bytes,
                cudaStream_t st) {
    TK_PROF(TUCKER_PROF_DMMA_GRAM, st);
    using namespace gram;
    Plan p = make_plan(n, mode);
    if (ws_bytes < (size_t)p.T * p.S * BM * BM * sizeof(double)) return TUCKER_ERR_SIZE;
    Args a{};
    a.mode = mode;
    a.n1 = n[0]; a.n2 = n[1]; a.n3 = n[2];
    a.n = p.n;
    a.S = p.S;
    a.nkb = p.nkb;
    a.nkb3 = p.nkb3;
    a.F = F;
    a.part = static_cast<double*>(ws);
    dim3 grid((unsigned)p.T, (unsigned)p.S);
    if (p.tma) {
        CUtensorMap map;
        bool ok;
        if (mode == 0) {
            uint64_t dims[2] = {(uint64_t)(a.n2 * a.n3), (uint64_t)a.n1};
            uint64_t strides[1] = {(uint64_t)(a.n2 * a.n3 * 8)};
            uint32_t box[2] = {BK, BM};
            ok = make_tmap_f64(&map, F, 2, dims, strides, box);
        } else if (mode == 1) {
            uint64_t dims[3] = {(uint64_t)a.n3, (uint64_t)a.n2, (uint64_t)a.n1};
            uint64_t strides[2] = {(uint64_t)(a.n3 * 8), (uint64_t)(a.n2 * a.n3 * 8)};
            uint32_t box[3] = {BK, BM, 1};
            ok = make_tmap_f64(&map, F, 3, dims, strides, box);
        } else {
            const int m3 = make_mmajor_map(&map, F, (uint64_t)(a.n1 * a.n2), (uint64_t)a.n3);
            ok = m3 >= 0;
            a.m3d = m3 == 1;
        }
        if (!ok) return TUCKER_ERR_CUDA;
        const size_t sm = smem_tma();
        if (mode == 0) {
            TK_CUDA(cudaFuncSetAttribute(k_gram_tma<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            k_gram_tma<0><<<grid, NCW * 32, sm, st>>>(map, a);
        } else if (mode == 1) {
            TK_CUDA(cudaFuncSetAttribute(k_gram_tma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            k_gram_tma<1><<<grid, NCW * 32, sm, st>>>(map, a);
        } else {
            TK_CUDA(cudaFuncSetAttribute(k_gram_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            k_gram_tma<2><<<grid, NCW * 32, sm, st>>>(map, a);
        }
    } else {
        const size_t sm = smem_generic();
        if (mode == 0) {
            TK_CUDA(cudaFuncSetAttribute(k_gram_generic<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            k_gram_generic<0><<<grid, NCW * 32, sm, st>>>(a);
        } else if (mode == 1) {
            TK_CUDA(cudaFuncSetAttribute(k_gram_generic<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            k_gram_generic<1><<<grid, NCW * 32, sm, st>>>(a);
        } else {
            TK_CUDA(cudaFuncSetAttribute(k_gram_generic<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            k_gram_generic<2><<<grid, NCW * 32, sm, st>>>(a);
        }
    }
    TK_CHECK_LAUNCH();
    k_gram_reduce<<<dim3(16, (unsigned)p.T), 256, 0, st>>>(a.part, p.S, p.n, G);
    TK_CHECK_LAUNCH();
    return TUCKER_OK;
}

// ------------------------------------------------------------------------- a-7 fused launcher
// Chunk-size target in bytes; TUCKER_FUSED_CHUNK_KB (host environment) overrides it — a test
// knob that forces many chunks on small grids.
int64_t fused_chunk_target(int64_t dflt) {
    const char* e = std::getenv("TUCKER_FUSED_CHUNK_KB");
    if (e && *e) {
        const long long v = std::atoll(e);
        if (v > 0) return (int64_t)v << 10;
    }
    return dflt;
}

FusedGramPlan fused_gram_plan(const int64_t n[3], int mode) {
    FusedGramPlan f{};
    f.pa = (mode == 1) ? 0 : 1;
    const int64_t nr = f.pa == 0 ? n[1] : n[0];
    f.np = f.pa == 0 ? n[0] : n[1];
    const int64_t plane = nr * n[2];
    const int nt = (int)ceil_div(n[mode], gram::BM);
    f.T = nt * (nt + 1) / 2;
    f.S = std::max(1, kNumSMs / f.T);
    f.Pc = std::max<int64_t>(1, std::min<int64_t>(f.np, fused_chunk_target(32 << 20) / (plane * 8)));
    // at least ~16 k-blocks per CTA per chunk (pipeline restart amortisation)
    auto nkb = [&](int64_t pc) {
        return mode == 0 ? ceil_div(pc * n[2], gram::BK)
                         : mode == 1 ? pc * ceil_div(n[2], gram::BK) : ceil_div(n[0] * pc, gram::BK);
    };
    while (f.Pc < f.np && nkb(f.Pc) < 16 * (int64_t)f.S) f.Pc *= 2;
    f.Pc = std::min(f.Pc, f.np);
    f.nchunks = ceil_div(f.np, f.Pc);
    f.slot_elems = align_up((size_t)(f.Pc * plane), 128);
    f.part_bytes = (size_t)f.T * f.S * gram::BM * gram::BM * sizeof(double);
    return f;
}

int launch_gram_fused(const int64_t n[3], int mode, const KParams& kp, const double* cheb, const double* x2,
                      double* ring, double* part, unsigned int* bar, double* G, cudaStream_t st) {
    using namespace gram;
    if (n[2] % 2 != 0 || n[2] < BK) return TUCKER_ERR_UNSUPPORTED;
    const FusedGramPlan fp = fused_gram_plan(n, mode);
    if (fp.T * fp.S > kNumSMs) return TUCKER_ERR_UNSUPPORTED;
    int64_t vn[3] = {n[0], n[1], n[2]};
    if (fp.pa == 0) vn[0] = fp.Pc;
    else vn[1] = fp.Pc;
    FusedArgs f{};
    Args& a = f.a;
    a.mode = mode;
    a.n1 = vn[0]; a.n2 = vn[1]; a.n3 = vn[2];
    a.n = n[mode];
    a.S = fp.S;
    a.nkb3 = ceil_div(vn[2], BK);
    if (mode == 0) a.nkb = ceil_div(vn[1] * vn[2], BK);
    else if (mode == 1) a.nkb = vn[0] * a.nkb3;
    else a.nkb = ceil_div(vn[0] * vn[1], BK);
    a.F = ring;
    a.part = part;
    f.geo.pa = fp.pa;
    f.geo.n1 = n[0]; f.geo.n2 = n[1]; f.geo.n3 = n[2];
    f.geo.g0 = 0;
    f.geo.Pc = fp.Pc;
    f.geo.np = fp.np;
    f.geo.mirror = (kp.centred && n[2] % 8 == 0) ? 1 : 0;
    f.kp = kp;
    f.cheb = cheb;
    f.x2 = x2;
    f.slot[0] = ring;
    f.slot[1] = ring + fp.slot_elems;
    f.nchunks = fp.nchunks;
    f.bar = bar;
    CUtensorMap maps[2];
    for (int sl = 0; sl < 2; ++sl) {
        bool ok;
        if (mode == 0) {
            uint64_t dims[2] = {(uint64_t)(vn[1] * vn[2]), (uint64_t)vn[0]};
            uint64_t strides[1] = {(uint64_t)(vn[1] * vn[2] * 8)};
            uint32_t box[2] = {BK, BM};
            ok = make_tmap_f64(&maps[sl], f.slot[sl], 2, dims, strides, box);
        } else if (mode == 1) {
            uint64_t dims[3] = {(uint64_t)vn[2], (uint64_t)vn[1], (uint64_t)vn[0]};
            uint64_t strides[2] = {(uint64_t)(vn[2] * 8), (uint64_t)(vn[1] * vn[2] * 8)};
            uint32_t box[3] = {BK, BM, 1};
            ok = make_tmap_f64(&maps[sl], f.slot[sl], 3, dims, strides, box);
        } else {
            const int m3 = make_mmajor_map(&maps[sl], f.slot[sl], (uint64_t)(vn[0] * vn[1]), (uint64_t)vn[2]);
            ok = m3 >= 0;
            a.m3d = m3 == 1;
        }
        if (!ok) return TUCKER_ERR_CUDA;
    }
    TK_CUDA(cudaMemsetAsync(bar, 0, sizeof(unsigned int), st));
    f.nmma = fp.T * fp.S;
    f.ngen = (kNumSMs - f.nmma >= 2) ? kNumSMs - f.nmma : 0;
    const size_t sm = smem_tma();
    void* args[3] = {&maps[0], &maps[1], &f};
    const dim3 grid((unsigned)(f.nmma + f.ngen));
    const void* fn = mode == 0 ? (const void*)k_gram_fused<0> : mode == 1 ? (const void*)k_gram_fused<1>
                                                                          : (const void*)k_gram_fused<2>;
    TK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    TK_CUDA(cudaLaunchCooperativeKernel(fn, grid, dim3(NCW * 32), args, sm, st));
    TK_CHECK_LAUNCH();
    k_gram_reduce<<<dim3(16, (unsigned)fp.T), 256, 0, st>>>(part, fp.S, n[mode], G);
    TK_CHECK_LAUNCH();
    return TUCKER_OK;
}

}  // namespace tk
