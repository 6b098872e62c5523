// refine.cu — NEXT f2: beating the sqrt(eps) floor of the Gram route.
//
// The paper takes the SVD of each unfolding; the hot path forms G_m = F_(m) F_(m)^T,
// whose eigenvalues below ~1e-16 lambda_1 are rounding noise, so singular values below ~1e-8
// sigma_1 are lost (E plateaus near 1e-8).  This pass recovers SVD accuracy with a Rayleigh–Ritz
// step on F_(m) itself, starting from the Gram route's p = r + q leading eigenvectors V:
//   pass 1   Y = F_(m)^T V                 (N/n_m x p, stored column-major as Yt = Y^T)
//   BCGS2    Q = orth(Y)                    (block classical Gram–Schmidt twice: blocks of 8
//                                            columns, one pass over the earlier columns per
//                                            block projection, CGS2 inside a block; fixed-order
//                                            reductions; columns the Kahan–Parlett test finds
//                                            dependent on earlier blocks are replaced by
//                                            pseudo-random vectors and projected block-wise)
//   pass 2   B = F_(m) Q                    (n_m x p, split-K partials + fixed-order reduce)
//   SVD      B = U~ Sigma W^T               (one-sided Jacobi in a thread-block cluster: no
//                                            squaring, small singular values keep their accuracy)
// and U_m = U~[:, :r], sigma_m = Sigma[:r]; `iters` repeats the step from V = U~.  Every product
// is a plain FP64 contraction of F (no Gram), so the singular values are resolved down to
// ~eps sigma_1.  The streaming products run on the DMMA GEMM (gemm.cu).
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace tk {

namespace {
constexpr int kBlk = 4 * kNumSMs;  // CTAs of the CGS2 kernels
constexpr int kNT = 256;

__device__ __forceinline__ double hash_u(uint64_t idx) {  // SplitMix64 finaliser -> [-1,1)
    uint64_t z = idx * 0x9E3779B97F4A7C15ull + 0x2545F4914F6CDD1Dull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}

__device__ __forceinline__ void row_range(int64_t M, int64_t& b0, int64_t& b1) {
    b0 = (int64_t)blockIdx.x * M / gridDim.x;
    b1 = (int64_t)(blockIdx.x + 1) * M / gridDim.x;
}

// part[blk][j] = sum_{rows of blk} Q_j[row] y[row], j < k (columns of Yt are contiguous, length M).
__global__ void __launch_bounds__(kNT) k_cgs_dots(const double* __restrict__ Yt, int64_t M, int k,
                                                  double* __restrict__ part, const int* __restrict__ done,
                                                  const int* __restrict__ jstart) {
    if (*done) return;
    __shared__ double red[40];
    int64_t b0, b1;
    row_range(M, b0, b1);
    const double* y = Yt + (size_t)k * M;
    for (int j0 = *jstart; j0 < k; j0 += 8) {
        double acc[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] = 0.0;
        for (int64_t i = b0 + threadIdx.x; i < b1; i += kNT) {
            const double yi = y[i];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (j0 + u < k) acc[u] = fma(Yt[(size_t)(j0 + u) * M + i], yi, acc[u]);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const double s = block_sum(acc[u], red);
            if (threadIdx.x == 0 && j0 + u < k) part[(size_t)blockIdx.x * 64 + j0 + u] = s;
        }
    }
}

// h[j] = sum over blocks of part[blk][j] (j in [jstart, k)): one warp per j, lanes strided over the
// blocks, fixed shuffle tree (deterministic).
__global__ void __launch_bounds__(1024) k_reduce_h(const double* __restrict__ part, int nblk, int k,
                                                   const int* __restrict__ done, const int* __restrict__ jstart,
                                                   double* __restrict__ h) {
    if (*done) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int j = *jstart + warp; j < k; j += 32) {
        double s = 0.0;
        for (int b = lane; b < nblk; b += 32) s += part[(size_t)b * 64 + j];
        s = warp_sum(s);
        if (lane == 0) h[j] = s;
    }
}

// y -= Q h on this CTA's rows (j in [jstart, k)); npart[blk] = ||y||^2 of its rows.
__global__ void __launch_bounds__(kNT) k_cgs_update(double* __restrict__ Yt, int64_t M, int k,
                                                    const double* __restrict__ hg, double* __restrict__ npart,
                                                    const int* __restrict__ done, const int* __restrict__ jstart) {
    if (*done) return;
    __shared__ double h[64];
    __shared__ double red[40];
    const int js = *jstart;
    for (int j = threadIdx.x; j < k; j += kNT) h[j] = j < js ? 0.0 : hg[j];
    __syncthreads();
    int64_t b0, b1;
    row_range(M, b0, b1);
    double* y = Yt + (size_t)k * M;
    double ss = 0.0;
    for (int64_t i = b0 + threadIdx.x; i < b1; i += kNT) {
        double yi = y[i];
        for (int j = js; j < k; ++j) yi = fma(-h[j], Yt[(size_t)j * M + i], yi);
        y[i] = yi;
        ss = fma(yi, yi, ss);
    }
    ss = block_sum(ss, red);
    if (threadIdx.x == 0) npart[blockIdx.x] = ss;
}

// n1 = ||y'||^2 (after pass 1), n2 = ||y''||^2 (after pass 2), fixed-order sums.  Kahan–Parlett
// "twice is enough": accept y'' (normalised) if n2 >= n1 / 2; otherwise y was numerically in the
// span of the previous columns — replace it by a deterministic pseudo-random vector and run the
// two passes again (the last attempt is accepted unconditionally).
// `skip` is read only; `accepted` is written (by CTA 0) and read by the launches of the next
// attempt only — a kernel never reads a flag it writes.
__global__ void __launch_bounds__(kNT) k_cgs_finish(double* __restrict__ Yt, int64_t M, int k,
                                                    const double* __restrict__ npart, int nblk,
                                                    const int* __restrict__ skip, int* accepted, int last) {
    if (*skip) return;
    __shared__ double tot, tot1;
    if (threadIdx.x < 32) {  // lanes strided over the blocks, fixed shuffle tree
        double s = 0.0, s1 = 0.0;
        for (int b = threadIdx.x; b < nblk; b += 32) {
            s1 += npart[b];
            s += npart[nblk + b];
        }
        s = warp_sum(s);
        s1 = warp_sum(s1);
        if (threadIdx.x == 0) {
            tot = s;
            tot1 = s1;
        }
    }
    __syncthreads();
    int64_t b0, b1;
    row_range(M, b0, b1);
    double* y = Yt + (size_t)k * M;
    const bool ok = (tot > 1e-300 && tot >= 0.5 * tot1) || last;
    const double inv = tot > 0.0 ? 1.0 / sqrt(tot) : 0.0;
    for (int64_t i = b0 + threadIdx.x; i < b1; i += kNT) y[i] = ok ? y[i] * inv : hash_u(0x5eedull * (k + 1) + i);
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0 && ok) *accepted = 1;
}

// Eight block sums at once, bitwise equal to eight block_sum() calls (same shuffle trees, same
// warp order) with two barriers instead of sixteen.  red: >= 8 * 33 doubles.  Result in out[0..7]
// (valid on thread 0).
__device__ __forceinline__ void block_sum8(const double (&v)[8], double* red, double (&out)[8]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    double w[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) w[u] = warp_sum(v[u]);
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int u = 0; u < 8; ++u) red[u * 33 + warp] = w[u];
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            double t = lane < nw ? red[u * 33 + lane] : 0.0;
            out[u] = warp_sum(t);
        }
    }
}

// Lane-strided sum of nblk <= kBlk partials x[b * stride] (b = lane, lane + 32, ...) in the
// same order as the plain loop, with every load issued before the first add (one L2 round trip).
__device__ __forceinline__ double lane_sum_partials(const double* x, int nblk, int stride, int lane) {
    constexpr int kPer = (kBlk + 31) / 32;
    double v[kPer];
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        const int b = lane + 32 * q;
        v[q] = b < nblk ? x[(size_t)b * stride] : 0.0;
    }
    double sum = 0.0;
#pragma unroll
    for (int q = 0; q < kPer; ++q)
        if (lane + 32 * q < nblk) sum += v[q];
    return sum;
}

// The column-by-column CGS2 of one block (columns k in [c0, c0 + bb)) in a single cooperative
// launch: the same arithmetic as k_cgs_dots / k_reduce_h / k_cgs_update / k_cgs_finish (same row
// ranges, same fixed-order block and shuffle reductions — bitwise the same result), with grid-wide
// barriers instead of kernel boundaries.  Every CTA reduces the per-CTA partials itself (same
// order), so the projection coefficients and the accept decision need no broadcast.
// Three grid barriers per column (after each pass's dots, after the second update): a CTA's dots,
// update and normalisation touch only its own rows, with the same thread-to-row mapping, so the
// data needs no barrier; only the partials do.  They are double-buffered — part[] by pass,
// npart[] by attempt parity — so a fast CTA never overwrites partials a slow one still sums:
// part[pass] is rewritten only after the barrier that follows its last reader, and npart[par]
// only after the next attempt's second-update barrier.  part: 2 x nblk x 64, npart: 2 x 2 x nblk.
__global__ void __launch_bounds__(kNT, 4) k_cgs_block(double* __restrict__ Yt, int64_t M, int c0, int bb,
                                                      double* __restrict__ part, double* __restrict__ npart,
                                                      const int* __restrict__ jstart_all) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double red[8 * 33];
    __shared__ double h[64];
    __shared__ double tot_s, tot1_s;
    const int nblk = gridDim.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int64_t b0, b1;
    row_range(M, b0, b1);
    int seq = 0;  // attempts so far (npart parity)
    for (int k = c0; k < c0 + bb; ++k) {
        double* y = Yt + (size_t)k * M;
        for (int attempt = 0; attempt < 2; ++attempt, ++seq) {
            const int js = attempt == 0 ? jstart_all[k] : 0;  // a replaced column: full projection
            double* np = npart + (size_t)(seq & 1) * 2 * nblk;
            for (int pass = 0; pass < 2; ++pass) {
                if (k > 0) {
                    double* pp = part + (size_t)pass * nblk * 64;
                    // dots: pp[blk][j] over this CTA's rows (as k_cgs_dots)
                    for (int j0 = js; j0 < k; j0 += 8) {
                        double acc[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) acc[u] = 0.0;
#pragma unroll 4
                        for (int64_t i = b0 + threadIdx.x; i < b1; i += kNT) {
                            const double yi = y[i];
#pragma unroll
                            for (int u = 0; u < 8; ++u)
                                if (j0 + u < k) acc[u] = fma(Yt[(size_t)(j0 + u) * M + i], yi, acc[u]);
                        }
                        double sums[8];
                        block_sum8(acc, red, sums);
                        if (threadIdx.x == 0)
#pragma unroll
                            for (int u = 0; u < 8; ++u)
                                if (j0 + u < k) pp[(size_t)blockIdx.x * 64 + j0 + u] = sums[u];
                    }
                    grid.sync();
                    // h[j] = sum over blocks (as k_reduce_h: warp per j, lanes strided, shuffle tree)
                    for (int j = js + warp; j < k; j += kNT / 32) {
                        double sum = lane_sum_partials(pp + j, nblk, 64, lane);
                        sum = warp_sum(sum);
                        if (lane == 0) h[j] = sum;
                    }
                    for (int j = threadIdx.x; j < js; j += kNT) h[j] = 0.0;
                    __syncthreads();
                }
                // update (as k_cgs_update): y -= Q h, np[pass][blk] = ||y||^2 of this CTA's rows
                // four rows per thread at a time, every load before the first store (y aliases Yt,
                // so the compiler cannot hoist loads across the stores itself); per-row FMA order and
                // the row order of ss as in k_cgs_update
                double ss = 0.0;
                for (int64_t i0 = b0 + threadIdx.x; i0 < b1; i0 += 4 * kNT) {
                    double yr[4];
                    bool in[4];
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        in[r] = i0 + r * kNT < b1;
                        yr[r] = in[r] ? y[i0 + r * kNT] : 0.0;
                    }
#pragma unroll 2
                    for (int j = js; j < k; ++j) {
                        const double* qj = Yt + (size_t)j * M + i0;
                        const double hj = h[j];
#pragma unroll
                        for (int r = 0; r < 4; ++r)
                            if (in[r]) yr[r] = fma(-hj, qj[r * kNT], yr[r]);
                    }
#pragma unroll
                    for (int r = 0; r < 4; ++r)
                        if (in[r]) {
                            y[i0 + r * kNT] = yr[r];
                            ss = fma(yr[r], yr[r], ss);
                        }
                }
                ss = block_sum(ss, red);
                if (threadIdx.x == 0) np[pass * nblk + blockIdx.x] = ss;
            }
            grid.sync();
            // finish (as k_cgs_finish): Kahan-Parlett acceptance, normalise or replace
            if (threadIdx.x < 32) {
                double sum1 = lane_sum_partials(np, nblk, 1, lane);
                double sum = lane_sum_partials(np + nblk, nblk, 1, lane);
                sum = warp_sum(sum);
                sum1 = warp_sum(sum1);
                if (threadIdx.x == 0) {
                    tot_s = sum;
                    tot1_s = sum1;
                }
            }
            __syncthreads();
            const double tot = tot_s, tot1 = tot1_s;
            const bool ok = (tot > 1e-300 && tot >= 0.5 * tot1) || attempt == 1;
            const double inv = tot > 0.0 ? 1.0 / sqrt(tot) : 0.0;
            for (int64_t i0 = b0 + threadIdx.x; i0 < b1; i0 += 4 * kNT) {
                double yr[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) yr[r] = i0 + r * kNT < b1 ? y[i0 + r * kNT] : 0.0;
#pragma unroll
                for (int r = 0; r < 4; ++r)
                    if (i0 + r * kNT < b1) y[i0 + r * kNT] = ok ? yr[r] * inv : hash_u(0x5eedull * (k + 1) + i0 + r * kNT);
            }
            if (ok) {
                ++seq;
                break;
            }
        }
    }
}

// Start basis for the Rayleigh–Ritz steps: keep the Gram route's eigenvectors whose eigenvalue is
// resolved (lambda_k >= tau lambda_1, tau = 1e-12), replace the others by deterministic
// pseudo-random columns.  Unresolved Gram eigenvectors are not random: on symmetric grids they
// are exactly even or odd, and a basis made only of odd null vectors would miss the even tail
// directions that the refinement must find.
__global__ void k_seed_basis(double* __restrict__ V, int64_t n, int p, const double* __restrict__ lam) {
    const double l1 = lam[0];
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * p; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / p;
        const int k = (int)(t % p);
        if (!(lam[k] >= 1e-12 * l1)) V[t] = hash_u(0xba515ull * (k + 1) + (uint64_t)i);
    }
}

// Start basis for an ALS single-hole step: the current factor's r columns, then p - r
// deterministic pseudo-random guard columns (the Rayleigh–Ritz step then orthonormalises them).
__global__ void k_seed_from_factors(double* __restrict__ V, const double* __restrict__ U, int64_t n, int r, int p) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * p; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / p;
        const int k = (int)(t % p);
        V[t] = k < r ? U[i * r + k] : hash_u(0xa15ull * (k + 1) + (uint64_t)i);
    }
}

// Block projection coefficients, per-CTA partials: part[blk][j * bb + t] = sum over this CTA's rows
// of Q_j[i] Y_{c0+t}[i], j < c0, t < bb: a (c0 x rows) x (rows x bb) product on the FP64 tensor
// cores.  Rows are staged 32 at a time in shared memory (all column segments contiguous,
// coalesced) through a kDotStages-deep cp.async ring; warp w owns rows 4w..4w+3 of every tile —
// one m8n8k4 DMMA k-step per 8-row block of j (A = Q^T, B = Y_B), accumulators in registers
// across the tiles; the 8 warps' accumulators are summed in warp order at the end (fixed order).
// (A lane-per-j FMA version issued ~314 instructions per warp and tile — instruction-bound.)
// Dynamic shared memory: block_dots_smem(ncol).
constexpr int kDotStages = 3;
constexpr int kMaxJB = 8;  // c0 <= 64
__host__ __device__ constexpr int block_dots_ld(int ncol) { return ncol + 1; }
size_t block_dots_smem(int ncol) {
    const size_t ring = (size_t)kDotStages * 32 * block_dots_ld(ncol);
    const size_t red = (size_t)8 * kMaxJB * 64;
    return 8 * (ring > red ? ring : red);
}
__global__ void __launch_bounds__(kNT, 4) k_block_dots(const double* __restrict__ Yt, int64_t M, int c0, int bb,
                                                       double* __restrict__ part, const int* __restrict__ run) {
    if (run && !*run) return;
    extern __shared__ double dsm[];  // ring [stage][row][ld]; then the cross-warp sum [w][jb][64]
    int64_t b0, b1;
    row_range(M, b0, b1);
    const int ncol = c0 + bb, npair = c0 * bb, ld = block_dots_ld(ncol), njb = c0 / 8;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
    const int ntile = (int)((b1 - b0 + 31) / 32);
    auto issue = [&](int tt) {
        if (tt < ntile) {
            double* st = dsm + (size_t)(tt % kDotStages) * 32 * ld;
            const int64_t r0 = b0 + (int64_t)tt * 32;
            // lane = row of the tile, warp = first column; columns step by 8 (strength-reduced)
            const int i = threadIdx.x & 31, c0w = threadIdx.x >> 5;
            const bool v = r0 + i < b1;
            const double* src = Yt + (size_t)c0w * M + (v ? r0 + i : b0);
            double* dst = st + i * ld + c0w;
            for (int c = c0w; c < ncol; c += kNT / 32, src += (size_t)(kNT / 32) * M, dst += kNT / 32)
                cp_async8(dst, src, v);
        }
        cp_async_commit();  // (empty groups keep the wait count uniform)
    };
    double acc[kMaxJB][2];
#pragma unroll
    for (int jb = 0; jb < kMaxJB; ++jb) acc[jb][0] = acc[jb][1] = 0.0;
#pragma unroll
    for (int tt = 0; tt < kDotStages - 1; ++tt) issue(tt);
    for (int tt = 0; tt < ntile; ++tt) {
        cp_async_wait<kDotStages - 2>();
        __syncthreads();  // tile tt landed for all threads; tile tt-1's stage is free
        issue(tt + kDotStages - 1);
        const double* row = dsm + (size_t)(tt % kDotStages) * 32 * ld + (4 * warp + q) * ld;
        const double bv = g < bb ? row[c0 + g] : 0.0;  // B[k = q][n = g] = Y_{c0+g}[row]
#pragma unroll
        for (int jb = 0; jb < kMaxJB; ++jb)
            if (jb < njb) dmma(acc[jb], row[jb * 8 + g], bv);  // A[m = g][k = q] = Q_{8jb+g}[row]
    }
    cp_async_wait<0>();
    __syncthreads();
    double* red = dsm;  // [w][jb][lane][2]
#pragma unroll
    for (int jb = 0; jb < kMaxJB; ++jb)
        if (jb < njb) {
            red[((warp * kMaxJB + jb) * 32 + lane) * 2] = acc[jb][0];
            red[((warp * kMaxJB + jb) * 32 + lane) * 2 + 1] = acc[jb][1];
        }
    __syncthreads();
    for (int pr = threadIdx.x; pr < npair; pr += kNT) {
        // H[j][t]: j = 8 jb + g', t = 2 q' + u  ->  lane' = 4 g' + q'
        const int j = pr / bb, t = pr % bb, jb = j >> 3, gg = j & 7, qq = t >> 1, u = t & 1;
        double sum = 0.0;
        for (int w = 0; w < 8; ++w) sum += red[((w * kMaxJB + jb) * 32 + 4 * gg + qq) * 2 + u];
        part[(size_t)blockIdx.x * npair + pr] = sum;
    }
}

// Y_{c0+t}[i] -= sum_j Q_j[i] H[j][t] on this CTA's rows, then per-CTA partial squared norms of
// the updated block columns (cnpart[blk][t]).  H is held in shared memory with row stride 8
// (16-byte aligned pairs: one LDS.128 serves two block columns).
__global__ void __launch_bounds__(kNT, 4) k_block_update(double* __restrict__ Yt, int64_t M, int c0, int bb,
                                                      const double* __restrict__ H, double* __restrict__ cnpart,
                                                      const int* __restrict__ run) {
    if (run && !*run) return;
    __shared__ __align__(16) double h[64 * 8];
    __shared__ double red[40];
    for (int e = threadIdx.x; e < c0 * 8; e += kNT) {
        const int j = e >> 3, t = e & 7;
        h[e] = t < bb ? H[j * bb + t] : 0.0;
    }
    __syncthreads();
    int64_t b0, b1;
    row_range(M, b0, b1);
    double nrm[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) nrm[t] = 0.0;
    for (int64_t i = b0 + threadIdx.x; i < b1; i += kNT) {
        double y[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) y[t] = t < bb ? Yt[(size_t)(c0 + t) * M + i] : 0.0;
        // chunks of four Q values, the next chunk's loads issued before this chunk's FMAs (one
        // chunk always in flight); FMA order as before
        double q[4], qn[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) q[u] = u < c0 ? Yt[(size_t)u * M + i] : 0.0;
        for (int j0 = 0; j0 < c0; j0 += 4) {
#pragma unroll
            for (int u = 0; u < 4; ++u) qn[u] = j0 + 4 + u < c0 ? Yt[(size_t)(j0 + 4 + u) * M + i] : 0.0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (j0 + u >= c0) break;
                const double2* hj = reinterpret_cast<const double2*>(h + (j0 + u) * 8);
#pragma unroll
                for (int t2 = 0; t2 < 4; ++t2) {
                    const double2 hh = hj[t2];
                    y[2 * t2] = fma(-q[u], hh.x, y[2 * t2]);
                    y[2 * t2 + 1] = fma(-q[u], hh.y, y[2 * t2 + 1]);
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) q[u] = qn[u];
        }
#pragma unroll
        for (int t = 0; t < 8; ++t)
            if (t < bb) {
                Yt[(size_t)(c0 + t) * M + i] = y[t];
                nrm[t] = fma(y[t], y[t], nrm[t]);
            }
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        const double v = block_sum(nrm[t], red);
        if (threadIdx.x == 0) cnpart[(size_t)blockIdx.x * 8 + t] = v;
    }
}

// After the two inter-block passes: column t keeps its block-local projection start c0 when
// ||y''||^2 >= ||y'||^2 / 2 (Kahan–Parlett), else it is numerically in the span of the earlier
// blocks.  With dep != nullptr the failing columns are flagged (dep[t], dep[8] = any) for a
// block-wise replacement (k_block_replace + two more inter-block passes on those columns only);
// jstart[c0 + t] = 0 sends a column that fails anyway to the full column-by-column projection.
__global__ void k_block_check(const double* __restrict__ part1, const double* __restrict__ part2, int nblk, int bb,
                              int c0, int* __restrict__ jstart, int* __restrict__ dep, const int* __restrict__ run) {
    if (run && !*run) return;
    const int t = threadIdx.x >> 5, lane = threadIdx.x & 31;  // warp per column, lanes over blocks
    int bad = 0;
    if (t < bb) {
        double n1 = 0.0, n2 = 0.0;
        for (int b = lane; b < nblk; b += 32) {
            n1 += part1[(size_t)b * 8 + t];
            n2 += part2[(size_t)b * 8 + t];
        }
        n1 = warp_sum(n1);
        n2 = warp_sum(n2);
        const bool ok = n2 > 1e-300 && n2 >= 0.5 * n1;
        if (lane == 0) {
            jstart[c0 + t] = ok ? c0 : 0;
            if (dep) dep[t] = !ok;
            bad = !ok;
        }
    }
    const int any = __syncthreads_or(bad);
    if (dep && threadIdx.x == 0) dep[8] = any;
}

// Replace the flagged columns of the block by deterministic pseudo-random vectors (their content
// was dependent on the earlier blocks to working precision).
__global__ void __launch_bounds__(kNT) k_block_replace(double* __restrict__ Yt, int64_t M, int c0, int bb,
                                                       const int* __restrict__ dep) {
    if (!dep[8]) return;
    int64_t b0, b1;
    row_range(M, b0, b1);
    for (int t = 0; t < bb; ++t) {
        if (!dep[t]) continue;
        double* y = Yt + (size_t)(c0 + t) * M;
        for (int64_t i = b0 + threadIdx.x; i < b1; i += kNT) y[i] = hash_u(0x7e91ull * (c0 + t + 1) + i);
    }
}

// H[j][t] = sum_s part[s][j * bb + t] for the flagged columns t, 0 for the others (their update
// y -= Q H is then the identity).
__global__ void k_sum_partials_dep(const double* __restrict__ part, int S, int c0, int bb, const int* __restrict__ dep,
                                   double* __restrict__ out) {
    if (!dep[8]) return;
    const int lane = threadIdx.x & 31;
    const int64_t len = (int64_t)c0 * bb;
    for (int64_t o = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; o < len;
         o += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        double s = 0.0;
        for (int q = lane; q < S; q += 32) s += part[(size_t)q * len + o];
        s = warp_sum(s);
        if (lane == 0) out[o] = dep[o % bb] ? s : 0.0;
    }
}

// out[o] = sum_s part[s][o] for short outputs and many partials: warp per output, lanes strided
// over s, fixed shuffle tree.
__global__ void k_sum_partials_warp(const double* __restrict__ part, int S, int64_t len, double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    for (int64_t o = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; o < len;
         o += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        double s = 0.0;
        for (int q = lane; q < S; q += 32) s += part[(size_t)q * len + o];
        s = warp_sum(s);
        if (lane == 0) out[o] = s;
    }
}

// out[o] = sum_s part[s][o] (fixed order)
__global__ void k_sum_partials(const double* __restrict__ part, int S, int64_t len, double* __restrict__ out) {
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < len; o += (int64_t)gridDim.x * blockDim.x) {
        double s = part[o];
        for (int q = 1; q < S; ++q) s += part[(size_t)q * len + o];
        out[o] = s;
    }
}

struct RefLayout {
    size_t Yt, B, Bpart, V, dots, npart, flags, H, Hpart, cn, jst, total;
    int64_t Mmax;
    int S2;
};

constexpr int kSplit = 256;  // split-K factor of pass 2 (>= 6.9 waves of the skinny DMMA tiles at n_m = 1024)
constexpr int kBS = 8;      // block width of the block Gram–Schmidt

RefLayout ref_plan(const int64_t n[3], int p) {
    RefLayout L{};
    const int64_t N = n[0] * n[1] * n[2];
    const int64_t nmax = std::max(n[0], std::max(n[1], n[2]));
    L.Mmax = N / std::min(n[0], std::min(n[1], n[2]));
    size_t off = 0;
    L.Yt = off;
    off += align_up((size_t)p * L.Mmax * 8, 256);
    L.B = off;
    off += align_up((size_t)nmax * p * 8, 256);
    L.Bpart = off;
    // mode 1 (batched over i) needs n1 partials of n2 x p; modes 0, 2 need kSplit partials
    off += align_up((size_t)std::max<int64_t>(kSplit, n[0]) * nmax * p * 8, 256);
    L.V = off;
    off += align_up((size_t)nmax * p * 8, 256);
    L.dots = off;  // the cooperative CGS2 double-buffers both partial arrays
    off += align_up((size_t)2 * kBlk * 64 * 8, 256);
    L.npart = off;
    off += align_up((size_t)4 * kBlk * 8, 256);
    L.flags = off;
    off += 256;
    L.H = off;
    off += align_up((size_t)64 * kBS * 8, 256);
    L.Hpart = off;
    off += align_up((size_t)std::max(kSplit, kBlk) * 64 * kBS * 8, 256);
    L.cn = off;
    off += align_up((size_t)4 * kBlk * 8 * 8, 256);
    L.jst = off;  // jstart[64], jzero, dep[9] (at +80)
    off += align_up((size_t)(80 + 16) * sizeof(int), 256);
    L.total = off;
    return L;
}
}  // namespace

size_t refine_ws_bytes(const int64_t n[3], int p) { return ref_plan(n, p).total; }

int launch_seed_from_factors(double* V, const double* U, int64_t n, int r, int p, cudaStream_t st) {
    k_seed_from_factors<<<64, 256, 0, st>>>(V, U, n, r, p);
    TK_CHECK_LAUNCH();
    return TUCKER_OK;
}

// One or more Rayleigh–Ritz steps on F_(m) from V0 (n_m x p, dev; need not be orthonormal);
// lam0 (dev, p, nullable): V0's Gram eigenvalues, unresolved columns are replaced (k_seed_basis).
// Outputs U (n_m x r), sigma (r); ws >= refine_ws_bytes(n, p).
int launch_refine_mode(const int64_t n[3], int m, const double* F, const double* V0, const double* lam0, int p,
                       int r, int iters, double* U, double* sigma, void* ws, size_t ws_bytes, cudaStream_t st,
                       int* sweeps_out) {
    const RefLayout L = ref_plan(n, p);
    if (ws_bytes < L.total) return TUCKER_ERR_SIZE;
    if (p > 64 || r > p) return TUCKER_ERR_UNSUPPORTED;
    char* w = static_cast<char*>(ws);
    double* Yt = reinterpret_cast<double*>(w + L.Yt);
    double* B = reinterpret_cast<double*>(w + L.B);
    double* Bpart = reinterpret_cast<double*>(w + L.Bpart);
    double* V = reinterpret_cast<double*>(w + L.V);
    double* dots = reinterpret_cast<double*>(w + L.dots);
    double* npart = reinterpret_cast<double*>(w + L.npart);
    int* flags = reinterpret_cast<int*>(w + L.flags);
    double* H = reinterpret_cast<double*>(w + L.H);
    double* Hpart = reinterpret_cast<double*>(w + L.Hpart);
    double* cn = reinterpret_cast<double*>(w + L.cn);
    const int64_t n1 = n[0], n2 = n[1], n3 = n[2], nm = n[m];
    const int64_t M = n1 * n2 * n3 / nm;
    TK_CUDA(cudaMemcpyAsync(V, V0, (size_t)nm * p * 8, cudaMemcpyDeviceToDevice, st));
    if (lam0) {
        k_seed_basis<<<64, 256, 0, st>>>(V, nm, p, lam0);
        TK_CHECK_LAUNCH();
    }
    int nb_sm = 0, dev = 0;  // cooperative CGS2 needs all kBlk CTAs resident
    TK_CUDA(cudaGetDevice(&dev));
    int coop_attr = 0;
    TK_CUDA(cudaDeviceGetAttribute(&coop_attr, cudaDevAttrCooperativeLaunch, dev));
    TK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb_sm, k_cgs_block, kNT, 0));
    const bool coop_ok = coop_attr && nb_sm * kNumSMs >= kBlk;
    for (int it = 0; it < iters; ++it) {
        // ---- pass 1: Yt (p x M) = V^T F_(m)
        if (m == 0) {  // Yt[a][(j,k)] = sum_i V[i][a] F[i][(j,k)]
            SmallGemm g{p, M, n1, 1, V, 1, p, 0, F, M, 1, 0, Yt, M, 1, 0};
            TK_RC(launch_gemm(g, st));
        } else if (m == 1) {  // Yt[b][(i,k)] = sum_j V[j][b] F[i][j][k], batched over i
            SmallGemm g{p, n3, n2, n1, V, 1, p, 0, F, n3, 1, n2 * n3, Yt, M, 1, n3};
            TK_RC(launch_gemm(g, st));
        } else {  // Yt[c][(i,j)] = sum_k V[k][c] F[(i,j)][k]
            SmallGemm g{p, M, n3, 1, V, 1, p, 0, F, 1, n3, 0, Yt, M, 1, 0};
            TK_RC(launch_gemm(g, st));
        }
        // ---- block CGS2 of the p columns of Y (each column contiguous in Yt): blocks of kBS
        // columns; two inter-block passes (H = Q_<c0^T Y_B from per-CTA partials summed in a fixed
        // order, Y_B -= Q_<c0 H), then column-by-column CGS2 inside the block.
        // split of the M-long contractions: the largest divisor of M not above kSplit that keeps
        // chunks of >= 512
        int S = (int)std::min<int64_t>(kSplit, std::max<int64_t>(1, M / 512));
        while (M % S) --S;
        const int64_t Kc = M / S;
        int* jstart = reinterpret_cast<int*>(w + L.jst);
        int* jzero = jstart + 64;
        int* dep = jstart + 80;
        TK_CUDA(cudaMemsetAsync(jstart, 0, 65 * sizeof(int), st));
        for (int c0 = 0; c0 < p; c0 += kBS) {
            const int bb = std::min(kBS, p - c0);
            if (c0 > 0) {
                for (int pass = 0; pass < 2; ++pass) {
                    static const bool dots_attr = cudaFuncSetAttribute(k_block_dots,
                                                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                                       (int)block_dots_smem(64 + 8)) == cudaSuccess;
                    if (!dots_attr) return TUCKER_ERR_CUDA;
                    k_block_dots<<<kBlk, kNT, block_dots_smem(c0 + bb), st>>>(Yt, M, c0, bb, Hpart, nullptr);
                    TK_CHECK_LAUNCH();
                    k_sum_partials_warp<<<48, 256, 0, st>>>(Hpart, kBlk, (int64_t)c0 * bb, H);
                    TK_CHECK_LAUNCH();
                    k_block_update<<<kBlk, kNT, 0, st>>>(Yt, M, c0, bb, H, cn + (size_t)pass * kBlk * 8, nullptr);
                    TK_CHECK_LAUNCH();
                }
                k_block_check<<<1, 256, 0, st>>>(cn, cn + (size_t)kBlk * 8, kBlk, bb, c0, jstart, dep, nullptr);
                TK_CHECK_LAUNCH();
                // dependent columns: replaced and projected block-wise (each earlier column read
                // once per pass for the whole block, not once per column); device-side skip
                k_block_replace<<<kBlk, kNT, 0, st>>>(Yt, M, c0, bb, dep);
                TK_CHECK_LAUNCH();
                for (int pass = 0; pass < 2; ++pass) {
                    k_block_dots<<<kBlk, kNT, block_dots_smem(c0 + bb), st>>>(Yt, M, c0, bb, Hpart, dep + 8);
                    TK_CHECK_LAUNCH();
                    k_sum_partials_dep<<<48, 256, 0, st>>>(Hpart, kBlk, c0, bb, dep, H);
                    TK_CHECK_LAUNCH();
                    k_block_update<<<kBlk, kNT, 0, st>>>(Yt, M, c0, bb, H, cn + (size_t)(2 + pass) * kBlk * 8, dep + 8);
                    TK_CHECK_LAUNCH();
                }
                k_block_check<<<1, 256, 0, st>>>(cn + (size_t)2 * kBlk * 8, cn + (size_t)3 * kBlk * 8, kBlk, bb, c0,
                                                 jstart, nullptr, dep + 8);
                TK_CHECK_LAUNCH();
            }
            if (coop_ok) {  // one cooperative launch for the block's column-by-column CGS2
                void* args[] = {(void*)&Yt, (void*)&M, (void*)&c0, (void*)&bb, (void*)&dots, (void*)&npart,
                                (void*)&jstart};
                TK_CUDA(cudaLaunchCooperativeKernel((void*)k_cgs_block, dim3(kBlk), dim3(kNT), args, 0, st));
                TK_LAUNCHED();
                continue;
            }
            // flags[0] = 0 (attempt 0 always runs), flags[1] = attempt 0 accepted (attempt 1 skipped)
            for (int k = c0; k < c0 + bb; ++k) {
                TK_CUDA(cudaMemsetAsync(flags, 0, 3 * sizeof(int), st));
                for (int attempt = 0; attempt < 2; ++attempt) {
                    const int* skip = flags + attempt;
                    const int* js = attempt == 0 ? jstart + k : jzero;  // a replaced column: full projection
                    for (int pass = 0; pass < 2; ++pass) {
                        if (k > 0) {
                            k_cgs_dots<<<kBlk, kNT, 0, st>>>(Yt, M, k, dots, skip, js);
                            TK_CHECK_LAUNCH();
                            k_reduce_h<<<1, 1024, 0, st>>>(dots, kBlk, k, skip, js, H);
                            TK_CHECK_LAUNCH();
                        }
                        k_cgs_update<<<kBlk, kNT, 0, st>>>(Yt, M, k, H, npart + pass * kBlk, skip, js);
                        TK_CHECK_LAUNCH();
                    }
                    k_cgs_finish<<<kBlk, kNT, 0, st>>>(Yt, M, k, npart, kBlk, skip, flags + attempt + 1, attempt);
                    TK_CHECK_LAUNCH();
                }
            }
        }
        // ---- pass 2: B (n_m x p) = F_(m) Q, split over the contraction, fixed-order sum
        if (m == 0) {  // B[i][a] = sum_col F[i][col] Qt[a][col]
            SmallGemm g{n1, p, Kc, S, F, M, 1, Kc, Yt, 1, M, Kc, Bpart, p, 1, n1 * p};
            TK_RC(launch_gemm(g, st));
            k_sum_partials<<<256, 256, 0, st>>>(Bpart, S, n1 * p, B);
            TK_CHECK_LAUNCH();
        } else if (m == 1) {  // B_i[j][b] = sum_k F[i][j][k] Qt[b][(i,k)], batched over i
            SmallGemm g{n2, p, n3, n1, F, n3, 1, n2 * n3, Yt, 1, M, n3, Bpart, p, 1, n2 * p};
            TK_RC(launch_gemm(g, st));
            k_sum_partials<<<256, 256, 0, st>>>(Bpart, (int)n1, n2 * p, B);
            TK_CHECK_LAUNCH();
        } else {  // B[k][c] = sum_row F[row][k] Qt[c][row]
            SmallGemm g{n3, p, Kc, S, F, 1, n3, Kc * n3, Yt, 1, M, Kc, Bpart, p, 1, n3 * p};
            TK_RC(launch_gemm(g, st));
            k_sum_partials<<<256, 256, 0, st>>>(Bpart, S, n3 * p, B);
            TK_CHECK_LAUNCH();
        }
        // ---- SVD of B -> V (all p columns, sorted) and U, sigma (leading r)
        TK_RC(launch_svd_cluster(nm, p, r, B, V, U, sigma, sweeps_out, st));
    }
    return TUCKER_OK;
}

}  // namespace tk
