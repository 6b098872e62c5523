// eig_cluster.cu — a-4 Rayleigh–Ritz + CGS2 step of the block subspace iteration, run by ONE
// thread-block cluster whose CTAs each own 128 rows of the n x p basis.
//
// The HOSVD factor U_m is the top-r_m eigenbasis of G_m.  Per iteration (see eig.cu
// for the driver loop) one launch of this kernel: W = G V for the CTA's rows (gv_rows, DMMA; or
// from k_gemm_vg's Wt when G is not given), then:
//   H = V^T W            local 4x4-blocked partial sums over the CTA's rows, cluster-summed in
//                        rank order through distributed shared memory (deterministic; every
//                        CTA ends with the bitwise same H)
//   H = Q Theta Q^T      parallel cyclic Jacobi (jacobi.cuh), redundantly in every CTA
//   Vr = V Q, Y = W Q    in place, warp per row
//   rho_k = ||Y_k - theta_k Vr_k||  (k < r), cluster-summed
//   converged (rho_k <= 1e-14 theta_1 after >= 3 iterations) or last: sign rule R6 with two
//                        cluster reductions (column max, then first index >= max/2), write U,
//                        lambda, sigma
//   else V <- CGS2(Y)    column by column, projections and norms cluster-summed
// The basis never leaves shared memory inside an iteration; the only global traffic is loading
// V, W (n x p each) and storing the next V.  A 16-CTA cluster covers n <= 2048.
#include <cooperative_groups.h>

#include "common.cuh"
#include "jacobi.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace tk {
namespace eigc {

constexpr int RB = 128;   // rows per CTA
constexpr int P = 64;     // basis storage width (p <= 64)
constexpr int NT = 512;   // threads per CTA
constexpr int STG = 1088; // doubles per cluster-reduction stage buffer
constexpr int kMinIters = 3;
// Residual tolerance relative to theta_1: 1e-14 (SURVEY a-4), floored at 4 sqrt(n) eps — the
// rounding level of evaluating G v itself in FP64 (DESIGN reading R15); at n <= 1024 the floor
// is below 3e-14 and the 3-iteration minimum decides.
constexpr double kTol = 1e-14;
__host__ __device__ inline double res_tol(int64_t n) {
    return fmax(kTol, 4.0 * sqrt((double)n) * 2.220446049250313e-16);
}

// swizzled [RB][P] tile: conflict-free for both row-wise (fixed i) and column-wise (fixed j)
// warp accesses
__device__ __forceinline__ int sw(int i, int j) { return i * P + (j ^ (i & 15)); }

struct Smem {
    double H[P * (P + 1)];
    double Q[P * (P + 1)];
    double V[RB * P];
    double Y[RB * P];
    double stage[2][STG];
    double red[64];
    double theta[P];
    double vec[P];    // h / residuals / column stats (cluster-reduced)
    double tmp[16 * P];  // per-warp partials (16 warps x P)
    double cs[P / 2], sn[P / 2];
    int pa[P / 2], pb[P / 2];
    int order[P];
    int flag;
};

struct State {  // must match eig.cu
    int done;
    int iters;
    int converged;
    int sweeps;
    double resid;
    double lambda1;
};

struct Args {
    int64_t n;
    int p, r, it, last, orth_only;
    double* Vt;        // p x n (in: V; out: next V)
    const double* Wt;  // p x n  (G V, or G Omega when orth_only); unused when G is set
    const double* G;   // n x n (nullable): W = G V formed here, each CTA its own rows (see k_rr_cluster)
    double* U;         // n x r
    double* lambda;    // r (nullable)
    double* sigma;     // r (nullable)
    State* st;
};

enum { OP_SUM = 0, OP_MAX = 1, OP_MIN = 2 };

// Cluster all-reduce of `count` doubles from local smem `in` into local smem `out` (may alias).
// Fixed rank order 0..C-1: deterministic and identical in every CTA.  Stage buffers alternate
// by round so a buffer is rewritten only after the cluster barrier that follows its last remote
// read.
template <int OP>
__device__ void cl_reduce(cg::cluster_group& cl, Smem& s, int& round, const double* in, double* out, int count) {
    const unsigned C = cl.num_blocks();
    for (int base = 0; base < count; base += STG) {
        const int cnt = min(STG, count - base);
        double* stg = s.stage[round & 1];
        for (int x = threadIdx.x; x < cnt; x += blockDim.x) stg[x] = in[base + x];
        cl.sync();
        for (int x = threadIdx.x; x < cnt; x += blockDim.x) {
            double v[16];  // independent DSMEM loads first, then the fixed-order combine
#pragma unroll
            for (int rk = 0; rk < 16; ++rk)
                if (rk < (int)C) v[rk] = cl.map_shared_rank(stg, rk)[x];
            double acc = v[0];
#pragma unroll
            for (int rk = 1; rk < 16; ++rk)
                if (rk < (int)C) acc = OP == OP_SUM ? acc + v[rk] : OP == OP_MAX ? fmax(acc, v[rk]) : fmin(acc, v[rk]);
            out[base + x] = acc;
        }
        ++round;
    }
    __syncthreads();
}

__device__ __forceinline__ double hash_uniform(uint64_t idx) {  // SplitMix64 finaliser -> [-1,1)
    uint64_t z = idx * 0x9E3779B97F4A7C15ull + 0x2545F4914F6CDD1Dull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}

// Per-column partial sums over the CTA's rows: out[j] = sum_i f(i, j) for j < ncol, in a fixed
// order (8 row groups of 16, then groups in order).
template <typename Fn>
__device__ __forceinline__ void col_partials(Smem& s, int nrows, int ncol, double* out, Fn f) {
    const int t = threadIdx.x, j = t & (P - 1), part = t >> 6;  // 8 parts
    double acc = 0.0;
    if (j < ncol)
        for (int i = part * 16; i < min(nrows, part * 16 + 16); ++i) acc += f(i, j);
    s.tmp[part * P + j] = acc;
    __syncthreads();
    if (t < ncol) {
        double a = s.tmp[t];
        for (int q = 1; q < 8; ++q) a += s.tmp[q * P + t];
        out[t] = a;
    }
    __syncthreads();
}

// Cluster sum of the per-warp partials tmp[w][0..cnt) (16 warps) into vec[0..cnt): warps summed
// in order into the stage buffer, then the CTAs in rank order.  Deterministic, identical in every
// CTA; one cluster barrier.
__device__ __forceinline__ void warp_partials_cluster_sum(cg::cluster_group& cl, Smem& s, int& round, int cnt) {
    const unsigned C = cl.num_blocks();
    double* stg = s.stage[round & 1];
    __syncthreads();
    if (threadIdx.x < cnt) {
        double a = s.tmp[threadIdx.x];
        for (int w = 1; w < NT / 32; ++w) a += s.tmp[w * P + threadIdx.x];
        stg[threadIdx.x] = a;
    }
    cl.sync();
    if (threadIdx.x < cnt) {
        double v[16];
#pragma unroll
        for (int rk = 0; rk < 16; ++rk)
            if (rk < (int)C) v[rk] = cl.map_shared_rank(stg, rk)[threadIdx.x];
        double acc = v[0];
#pragma unroll
        for (int rk = 1; rk < 16; ++rk)
            if (rk < (int)C) acc += v[rk];
        s.vec[threadIdx.x] = acc;
    }
    ++round;
    __syncthreads();
}

// CGS2 of the p columns of Y (in place) over the cluster's distributed rows.  Warp w owns rows
// 8w..8w+7 for the projections; 4 lanes per row apply the update.
__device__ void cgs2_cluster(cg::cluster_group& cl, Smem& s, int& round, int p, int nrows, int64_t i0) {
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int r0 = warp * 8, r1 = min(nrows, r0 + 8);
    for (int k = 0; k < p; ++k) {
        for (int attempt = 0; attempt < 2; ++attempt) {
            for (int pass = 0; pass < 2 && k > 0; ++pass) {
                __syncwarp();  // the same warp updated these rows in the previous pass
                double a0 = 0.0, a1 = 0.0;
                for (int i = r0; i < r1; ++i) {
                    const double yk = s.Y[sw(i, k)];
                    a0 = fma(s.Y[sw(i, lane)], yk, a0);
                    a1 = fma(s.Y[sw(i, lane + 32)], yk, a1);
                }
                s.tmp[warp * P + lane] = a0;
                s.tmp[warp * P + lane + 32] = a1;
                warp_partials_cluster_sum(cl, s, round, k);
                {   // y_i -= sum_j h_j Y[i][j]: 4 lanes per row, j interleaved, fixed combine order
                    const int i = t >> 2, qd = t & 3;
                    double acc = 0.0;
                    if (i < nrows)
                        for (int j = qd; j < k; j += 4) acc = fma(s.vec[j], s.Y[sw(i, j)], acc);
                    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
                    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
                    if (i < nrows && qd == 0) s.Y[sw(i, k)] -= acc;
                }
            }
            // norm of column k (rows r0..r1 of each warp, lane-strided)
            __syncthreads();
            double ss = 0.0;
            if (lane < 8 && r0 + lane < r1) {
                const double y = s.Y[sw(r0 + lane, k)];
                ss = y * y;
            }
            ss = warp_sum(ss);
            if (lane == 0) s.tmp[warp * P] = ss;
            warp_partials_cluster_sum(cl, s, round, 1);
            const double tot = s.vec[0];
            if (tot > 1e-280) {
                const double inv = 1.0 / sqrt(tot);
                if (t < nrows) s.Y[sw(t, k)] *= inv;
                __syncthreads();
                break;
            }
            // exactly dependent column: deterministic pseudo-random replacement, retry
            if (t < nrows) s.Y[sw(t, k)] = hash_uniform(0x5eedull * (k + 1) + (uint64_t)(i0 + t));
            __syncthreads();
        }
    }
}

// W rows of this CTA, W[i][j] = sum_k G[i0 + i][k] V[k][j] (V = Vt^T: every CTA's rows, written by
// the previous launch; no CTA overwrites Vt before the cluster barrier of its first reduction, so
// all reads of this launch precede it), on DMMA (m8n8k4): warp w owns rows 8w .. 8w + 7 and all
// p <= 64 columns; k in chunks of GV_KC staged through the Jacobi scratch (H, Q: two stages),
// the next chunk's loads in flight under the current chunk's MMAs.  Forming W here, on the
// cluster's own SMs, makes one launch per iteration that needs no SMs beyond the cluster's (a
// persistent Gram on a concurrent stream holds every other SM).
constexpr int GV_KC = 16, GV_LD = GV_KC + 4;  // row stride 20 doubles: fragment loads 2 wavefronts
__device__ void gv_rows(const Args& a, Smem& s, int64_t i0, int nrows) {
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5, r = lane >> 2, q = lane & 3;
    const int64_t n = a.n;
    const int p = a.p;
    // two stages (s.H, s.Q), each: G chunk [RB][GV_LD] then V chunk [P][GV_LD]
    // per thread: 4 G values (rows t/4 .. of the 128 x 16 chunk) and 2 V values (64 x 16)
    double g4[4], v2[2];
    auto load = [&](int64_t k0) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = t + u * NT, i = e / GV_KC, kk = e % GV_KC;
            g4[u] = (i < nrows && k0 + kk < n) ? a.G[(i0 + i) * n + k0 + kk] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int e = t + u * NT, j = e / GV_KC, kk = e % GV_KC;
            v2[u] = (j < p && k0 + kk < n) ? a.Vt[(int64_t)j * n + k0 + kk] : 0.0;
        }
    };
    auto store = [&](double* b) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = t + u * NT;
            b[(e / GV_KC) * GV_LD + e % GV_KC] = g4[u];
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int e = t + u * NT;
            b[RB * GV_LD + (e / GV_KC) * GV_LD + e % GV_KC] = v2[u];
        }
    };
    double acc[8][2];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
    const int64_t nch = (n + GV_KC - 1) / GV_KC;
    load(0);
    store(s.H);
    __syncthreads();
    for (int64_t c = 0; c < nch; ++c) {
        if (c + 1 < nch) load((c + 1) * GV_KC);
        const double* b = (c & 1) ? s.Q : s.H;
#pragma unroll
        for (int kq = 0; kq < GV_KC; kq += 4) {
            const double av = b[(8 * warp + r) * GV_LD + kq + q];
#pragma unroll
            for (int nt = 0; nt < 8; ++nt)
                if (8 * nt < p) dmma(acc[nt], av, b[RB * GV_LD + (8 * nt + r) * GV_LD + kq + q]);
        }
        if (c + 1 < nch) store((c & 1) ? s.H : s.Q);
        __syncthreads();
    }
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int j = 8 * nt + 2 * q + u;
            s.Y[sw(8 * warp + r, j)] = j < p ? acc[nt][u] : 0.0;
        }
}

__global__ void __launch_bounds__(NT, 1) k_rr_cluster(Args a) {
    cg::cluster_group cl = cg::this_cluster();
    if (a.st->done) return;  // uniform across the cluster (written by an earlier launch)
    extern __shared__ __align__(16) uint8_t smem_raw[];
    Smem& s = *reinterpret_cast<Smem*>(smem_raw);  // (no integer casts: keeps LDS/STS addressing)
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int p = a.p, ld = jacobi_ld(p);
    const int64_t n = a.n;
    const int64_t i0 = (int64_t)cl.block_rank() * RB;
    const int64_t rem = n - i0;
    const int nrows = rem <= 0 ? 0 : (rem >= RB ? RB : (int)rem);
    int round = 0;

    // load V (unless orth_only) and W rows; zero padding
    for (int e = t; e < RB * P; e += NT) {
        const int j = e / RB, i = e % RB;
        const bool ok = i < nrows && j < p;
        if (!a.G) s.Y[sw(i, j)] = ok ? a.Wt[(size_t)j * n + i0 + i] : 0.0;
        if (!a.orth_only) s.V[sw(i, j)] = ok ? a.Vt[(size_t)j * n + i0 + i] : 0.0;
    }
    if (a.G) gv_rows(a, s, i0, nrows);  // W rows = G[i0 .., :] V (V of every CTA, from global)
    __syncthreads();

    if (!a.orth_only) {
        // 1. H = V^T W: lower-triangular 4x4 blocks (bi >= bj), 136 blocks, packed 16 per block
        double* hp = s.Q;  // scratch (2176 doubles)
        if (t < 136) {
            int bi = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
            while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
            while (bi * (bi + 1) / 2 > t) --bi;
            const int bj = t - bi * (bi + 1) / 2;
            double acc[4][4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
            for (int i = 0; i < nrows; ++i) {
                double va[4], wb[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) va[u] = s.V[sw(i, 4 * bi + u)];
#pragma unroll
                for (int v = 0; v < 4; ++v) wb[v] = s.Y[sw(i, 4 * bj + v)];
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int v = 0; v < 4; ++v) acc[u][v] = fma(va[u], wb[v], acc[u][v]);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) hp[t * 16 + u * 4 + v] = acc[u][v];
        }
        __syncthreads();
        cl_reduce<OP_SUM>(cl, s, round, hp, hp, 136 * 16);
        for (int e = t; e < 136 * 16; e += NT) {
            const int blk = e >> 4, u = (e >> 2) & 3, v = e & 3;
            int bi = (int)((sqrt(8.0 * blk + 1.0) - 1.0) * 0.5);
            while ((bi + 1) * (bi + 2) / 2 <= blk) ++bi;
            while (bi * (bi + 1) / 2 > blk) --bi;
            const int bj = blk - bi * (bi + 1) / 2;
            const int ra = 4 * bi + u, cb = 4 * bj + v;
            if (ra < p && cb < p && ra >= cb) {
                s.H[ra * ld + cb] = hp[e];
                s.H[cb * ld + ra] = hp[e];
            }
        }
        // 2. Jacobi (redundant per CTA, bitwise identical)
        __syncthreads();
        JacobiWork js{s.cs, s.sn, s.pa, s.pb, &s.flag, s.red};
        const int sweeps = jacobi_sym(s.H, s.Q, p, js, 60);
        sort_desc_diag(s.H, p, s.order);
        for (int k = t; k < p; k += NT) s.theta[k] = s.H[s.order[k] * ld + s.order[k]];
        __syncthreads();
        // Qs[a][k] = Q[a][order[k]] into H (P-wide rows)
        for (int e = t; e < P * P; e += NT) {
            const int aa = e / P, k = e % P;
            s.H[e] = (aa < p && k < p) ? s.Q[aa * ld + s.order[k]] : 0.0;
        }
        __syncthreads();
        // 3. Vr = V Qs, Y = W Qs (warp per row, in place)
        for (int i = warp; i < nrows; i += NT / 32) {
            double v0 = 0.0, v1 = 0.0, y0 = 0.0, y1 = 0.0;
            for (int aa = 0; aa < p; ++aa) {
                const double va = s.V[sw(i, aa)], wa = s.Y[sw(i, aa)];
                const double q0 = s.H[aa * P + lane], q1 = s.H[aa * P + lane + 32];
                v0 = fma(va, q0, v0);
                v1 = fma(va, q1, v1);
                y0 = fma(wa, q0, y0);
                y1 = fma(wa, q1, y1);
            }
            __syncwarp();
            s.V[sw(i, lane)] = v0;
            s.V[sw(i, lane + 32)] = v1;
            s.Y[sw(i, lane)] = y0;
            s.Y[sw(i, lane + 32)] = y1;
        }
        __syncthreads();
        // 4. residuals
        col_partials(s, nrows, a.r, s.vec, [&](int i, int k) {
            const double d = s.Y[sw(i, k)] - s.theta[k] * s.V[sw(i, k)];
            return d * d;
        });
        cl_reduce<OP_SUM>(cl, s, round, s.vec, s.vec, a.r);
        const double theta1 = s.theta[0];
        double rmax = 0.0;
        for (int k = 0; k < a.r; ++k) rmax = fmax(rmax, sqrt(s.vec[k]));
        const double rel = theta1 > 0.0 ? rmax / theta1 : 0.0;
        const bool conv = (a.it + 1 >= kMinIters) && (rel <= res_tol(n));
        if (conv || a.last) {
            // 5. sign rule R6 per column: max |u| (cluster max), then the first global index with
            //    |u_i| >= max/2 (cluster min of 2 i + [u_i < 0])
            if (t < a.r) {
                double mx = 0.0;
                for (int i = 0; i < nrows; ++i) mx = fmax(mx, fabs(s.V[sw(i, t)]));
                s.vec[t] = mx;
            }
            __syncthreads();
            cl_reduce<OP_MAX>(cl, s, round, s.vec, s.vec, a.r);
            if (t < a.r) {
                const double half = 0.5 * s.vec[t];
                double code = 1e300;
                for (int i = 0; i < nrows; ++i) {
                    const double v = s.V[sw(i, t)];
                    if (fabs(v) >= half) {
                        code = 2.0 * (double)(i0 + i) + (v < 0.0 ? 1.0 : 0.0);
                        break;
                    }
                }
                s.tmp[t] = code;
            }
            __syncthreads();
            cl_reduce<OP_MIN>(cl, s, round, s.tmp, s.tmp, a.r);
            for (int e = t; e < nrows * a.r; e += NT) {
                const int i = e / a.r, k = e % a.r;
                const double code = s.tmp[k];
                const bool flip = code < 1e299 && fmod(code, 2.0) == 1.0;
                const double v = s.V[sw(i, k)];
                a.U[(size_t)(i0 + i) * a.r + k] = flip ? -v : v;
            }
            if (cl.block_rank() == 0) {
                for (int k = t; k < a.r; k += NT) {
                    const double th = s.theta[k];
                    if (a.lambda) a.lambda[k] = th;
                    if (a.sigma) a.sigma[k] = th < 0.0 ? 0.0 : sqrt(th);  // NaN (poisoned input) propagates
                }
                if (t == 0) {
                    a.st->done = 1;
                    a.st->converged = conv ? 1 : 0;
                    a.st->iters = a.it + 1;
                    a.st->sweeps = sweeps;
                    a.st->resid = rel;
                    a.st->lambda1 = theta1;
                }
            }
            cl.sync();  // keep every CTA's shared memory alive until remote reads are done
            return;
        }
        if (cl.block_rank() == 0 && t == 0) {
            a.st->iters = a.it + 1;
            a.st->resid = rel;
            a.st->sweeps = sweeps;
        }
    }
    // 6. next basis V = CGS2(Y)
    cgs2_cluster(cl, s, round, p, nrows, i0);
    for (int e = t; e < p * RB; e += NT) {
        const int j = e / RB, i = e % RB;
        if (i < nrows) a.Vt[(size_t)j * n + i0 + i] = s.Y[sw(i, j)];
    }
    cl.sync();
}

// ------------------------------------------------------------------ NEXT f2: one-sided Jacobi SVD
// Left singular vectors and singular values of B (n x p, row-major, dev) by one-sided (Hestenes)
// Jacobi on its columns, rows distributed over the cluster like k_rr_cluster: per round of the
// round-robin ordering (jacobi.cuh) every CTA forms its partial (||b_a||^2, ||b_b||^2, b_a.b_b)
// for all pairs, one cluster reduction (rank order, deterministic) gives the same rotations in
// every CTA, and each CTA rotates its rows.  Unlike an eigensolver on B^T B this keeps small
// singular values to high relative accuracy (no squaring).  Outputs: Vout (n x p, columns sorted by
// descending sigma, normalised, sign rule R6), U (n x r = Vout's first r columns), sigma (r).
struct SvdArgs {
    int64_t n;
    int p, r;
    const double* B;
    double* Vout;
    double* U;
    double* sigma;
    int* sweeps_out;
};

__global__ void __launch_bounds__(NT, 1) k_svd_cluster(SvdArgs a) {
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(16) uint8_t smem_raw[];
    Smem& s = *reinterpret_cast<Smem*>(smem_raw);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nw = NT / 32;
    const int p = a.p;
    const int64_t n = a.n;
    const int64_t i0 = (int64_t)cl.block_rank() * RB;
    const int64_t rem = n - i0;
    const int nrows = rem <= 0 ? 0 : (rem >= RB ? RB : (int)rem);
    int round = 0;
    for (int e = t; e < RB * P; e += NT) {
        const int j = e / RB, i = e % RB;
        s.Y[sw(i, j)] = (i < nrows && j < p) ? a.B[(size_t)(i0 + i) * p + j] : 0.0;
    }
    __syncthreads();
    const int m = p + (p & 1), half = m / 2;
    const double eps = 2.220446049250313e-16;
    int sweep = 0;
    for (; sweep < 40; ++sweep) {
        int any = 0;
        for (int rd = 0; rd < m - 1; ++rd) {
            // partial (alpha, beta, gamma) of each pair over the local rows: warp per pair
            for (int w = warp; w < half; w += nw) {
                int pa, pb;
                rr_pair(rd, w, m, pa, pb);
                double al = 0.0, be = 0.0, ga = 0.0;
                if (pb < p)
                    for (int i = lane; i < nrows; i += 32) {
                        const double x = s.Y[sw(i, pa)], y = s.Y[sw(i, pb)];
                        al = fma(x, x, al);
                        be = fma(y, y, be);
                        ga = fma(x, y, ga);
                    }
                al = warp_sum(al);
                be = warp_sum(be);
                ga = warp_sum(ga);
                if (lane == 0) {
                    s.tmp[3 * w] = al;
                    s.tmp[3 * w + 1] = be;
                    s.tmp[3 * w + 2] = ga;
                }
            }
            __syncthreads();
            cl_reduce<OP_SUM>(cl, s, round, s.tmp, s.tmp, 3 * half);
            // identical rotations in every CTA; warp per pair applies it to the local rows
            for (int w = warp; w < half; w += nw) {
                int pa, pb;
                rr_pair(rd, w, m, pa, pb);
                if (pb >= p) continue;
                const double al = s.tmp[3 * w], be = s.tmp[3 * w + 1], ga = s.tmp[3 * w + 2];
                if (!(fabs(ga) > eps * sqrt(al * be)) || al == 0.0 || be == 0.0) continue;
                any = 1;
                const double zeta = (be - al) / (2.0 * ga);
                const double tt = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
                const double c = rsqrt(fma(tt, tt, 1.0)), sn = tt * c;
                for (int i = lane; i < nrows; i += 32) {
                    const double x = s.Y[sw(i, pa)], y = s.Y[sw(i, pb)];
                    s.Y[sw(i, pa)] = c * x - sn * y;
                    s.Y[sw(i, pb)] = sn * x + c * y;
                }
            }
            // every thread sees the same `any` (same reduced data); block barrier before the
            // next round reads the columns and overwrites tmp
            __syncthreads();
        }
        if (!__syncthreads_or(any)) break;
    }
    // column norms -> sigma, order, normalise, sign rule on the leading r (and all p) columns
    col_partials(s, nrows, p, s.vec, [&](int i, int k) {
        const double y = s.Y[sw(i, k)];
        return y * y;
    });
    cl_reduce<OP_SUM>(cl, s, round, s.vec, s.vec, p);
    for (int k = t; k < p; k += NT) s.theta[k] = sqrt(s.vec[k]);
    __syncthreads();
    for (int k = t; k < p; k += NT) {  // stable descending rank of sigma (NaN last: a permutation)
        auto key = [](double x) { return x == x ? x : -INFINITY; };
        const double v = key(s.theta[k]);
        int rank = 0;
        for (int j = 0; j < p; ++j) {
            const double w = key(s.theta[j]);
            rank += (w > v) || (w == v && j < k);
        }
        s.order[rank] = k;
    }
    __syncthreads();
    // normalise in place
    for (int e = t; e < nrows * p; e += NT) {
        const int i = e / p, k = e % p;
        const double sg = s.theta[k];
        if (sg > 0.0) s.Y[sw(i, k)] /= sg;
    }
    __syncthreads();
    // sign rule R6 on every output column (sorted position q -> source column order[q])
    if (t < p) {
        const int k = s.order[t];
        double mx = 0.0;
        for (int i = 0; i < nrows; ++i) mx = fmax(mx, fabs(s.Y[sw(i, k)]));
        s.vec[t] = mx;
    }
    __syncthreads();
    cl_reduce<OP_MAX>(cl, s, round, s.vec, s.vec, p);
    if (t < p) {
        const int k = s.order[t];
        const double halfm = 0.5 * s.vec[t];
        double code = 1e300;
        for (int i = 0; i < nrows; ++i) {
            const double v = s.Y[sw(i, k)];
            if (fabs(v) >= halfm) {
                code = 2.0 * (double)(i0 + i) + (v < 0.0 ? 1.0 : 0.0);
                break;
            }
        }
        s.tmp[t] = code;
    }
    __syncthreads();
    cl_reduce<OP_MIN>(cl, s, round, s.tmp, s.tmp, p);
    for (int e = t; e < nrows * p; e += NT) {
        const int i = e / p, q = e % p;
        const double code = s.tmp[q];
        const bool flip = code < 1e299 && fmod(code, 2.0) == 1.0;
        const double v = s.Y[sw(i, s.order[q])];
        const double o = flip ? -v : v;
        a.Vout[(size_t)(i0 + i) * p + q] = o;
        if (q < a.r) a.U[(size_t)(i0 + i) * a.r + q] = o;
    }
    if (cl.block_rank() == 0) {
        for (int q = t; q < a.r; q += NT) a.sigma[q] = s.theta[s.order[q]];
        if (t == 0 && a.sweeps_out) *a.sweeps_out = sweep + 1;
    }
    cl.sync();
}

}  // namespace eigc

// Cluster size for n rows (power of two, <= 16), or 0 when n is out of range.
int eig_cluster_size(int64_t n) {
    const int64_t c = ceil_div(n, eigc::RB);
    if (c > 16) return 0;
    int cs = 1;
    while (cs < c) cs <<= 1;
    return cs;
}

size_t eig_cluster_smem() { return sizeof(eigc::Smem); }

// Launch one Rayleigh–Ritz(+CGS2) step (orth_only = 1: CGS2 of Wt only).  Returns false if the
// cluster cannot be scheduled (caller falls back to the single-CTA path).
bool eig_cluster_supported(int64_t n) {
    const int cs = eig_cluster_size(n);
    if (cs == 0) return false;
    static int ok16 = -1;
    if (cudaFuncSetAttribute(eigc::k_rr_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)eig_cluster_smem()) != cudaSuccess)
        return false;
    if (cs > 8) {
        if (ok16 < 0) {
            ok16 = cudaFuncSetAttribute(eigc::k_rr_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                   cudaSuccess;
            if (ok16) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(cs);
                cfg.blockDim = dim3(eigc::NT);
                cfg.dynamicSmemBytes = eig_cluster_smem();
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = cs;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                int nc = 0;
                ok16 = cudaOccupancyMaxActiveClusters(&nc, eigc::k_rr_cluster, &cfg) == cudaSuccess && nc > 0;
            }
            cudaGetLastError();
        }
        return ok16 == 1;
    }
    return true;
}

int launch_svd_cluster(int64_t n, int p, int r, const double* B, double* Vout, double* U, double* sigma,
                       int* sweeps_out, cudaStream_t st) {
    if (!eig_cluster_supported(n) || p > eigc::P) return TUCKER_ERR_UNSUPPORTED;
    const int cs = eig_cluster_size(n);
    TK_CUDA(cudaFuncSetAttribute(eigc::k_svd_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)eig_cluster_smem()));
    if (cs > 8) TK_CUDA(cudaFuncSetAttribute(eigc::k_svd_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    eigc::SvdArgs a{n, p, r, B, Vout, U, sigma, sweeps_out};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(eigc::NT);
    cfg.dynamicSmemBytes = eig_cluster_smem();
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    TK_CUDA(cudaLaunchKernelEx(&cfg, eigc::k_svd_cluster, a));
    TK_CHECK_LAUNCH();
    return TUCKER_OK;
}

int launch_rr_cluster(int64_t n, int p, int r, int it, int last, int orth_only, double* Vt, const double* Wt,
                      double* U, double* lambda, double* sigma, void* state, cudaStream_t st, const double* G) {
    const int cs = eig_cluster_size(n);
    eigc::Args a{n, p, r, it, last, orth_only, Vt, Wt, G, U, lambda, sigma, static_cast<eigc::State*>(state)};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(eigc::NT);
    cfg.dynamicSmemBytes = eig_cluster_smem();
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    TK_CUDA(cudaLaunchKernelEx(&cfg, eigc::k_rr_cluster, a));
    TK_CHECK_LAUNCH();
    return TUCKER_OK;
}

}  // namespace tk
