// eig.cu — a-4: leading r eigenpairs of the symmetric PSD Gram matrix G_m.
//
// The HOSVD factor U_m is the top-r_m left singular subspace of the unfolding A_(m),
// i.e. the top-r_m eigenvectors of G_m; sigma = sqrt(max(lambda, 0)).
//
// Method (B200 design; the paper names no eigensolver): block subspace iteration with
// Rayleigh–Ritz on p = r + q columns (q = min(16, 64 - r)):
//   V_0 = orth(G Omega), Omega a fixed counter-hash block (deterministic); V_1 = orth(G V_0)
//   (cluster path: plain power steps until the last of the kMinIters iterations)
//   repeat: W = G V (multi-CTA DFMA GEMM); H = V^T W (p x p); H = Q Theta Q^T by parallel cyclic
//           Jacobi in shared memory (round-robin pairs, warp-parallel rotations, skip rule R7);
//           Vr = V Q, Y = W Q; residual rho_k = ||Y_k - theta_k Vr_k||;
//           stop when rho_k <= tol theta_1 for k < r after >= 3 iterations, else V = CGS2(Y).
// Small matrices (n <= 112) are diagonalised directly by the same shared-memory Jacobi.
// Outputs are sorted descending (stable) and sign-fixed by rule R6: the first entry with
// |u_i| >= max|u|/2 is made positive.  Everything is deterministic (fixed reduction orders).
#include "common.cuh"
#include "jacobi.cuh"
#include "kernels.h"
#include "prof.h"

namespace tk {
namespace eig {

constexpr int kMaxP = 64;
constexpr int kDirectMax = 112;  // whole-matrix Jacobi fits in shared memory up to here (207 KB)
constexpr int kThreads = 1024;
constexpr int kBatch = 8;
constexpr int kMaxIters = 96;
// Asynchronous completion (info == NULL): the iterations are enqueued up front, each exiting at
// once after convergence, but every launch of a converged solve still costs ~4 us on its side
// stream, ahead of the core that waits for U.  24 bounds them: the workloads
// converge in 3-8 iterations (tools/eig_iters_survey.py: at most 4 over configs 1-4, the f4
// kernels and Table 2's grids); a solve still unconverged there returns its last iterate, as the
// synchronous path does at kMaxIters (where NOCONV is reported).
constexpr int kMaxItersAsync = 24;
constexpr int kMinIters = 3;
// Residual tolerance relative to theta_1: 1e-14 (SURVEY a-4), floored at 4 sqrt(n) eps — the
// rounding level of evaluating G v itself in FP64 (DESIGN reading R15); at n <= 1024 the floor
// is below 3e-14 and the 3-iteration minimum decides.
constexpr double kTol = 1e-14;
__host__ __device__ inline double res_tol(int64_t n) {
    return fmax(kTol, 4.0 * sqrt((double)n) * 2.220446049250313e-16);
}

struct State {  // device-side status block
    int done;
    int iters;
    int converged;
    int sweeps;
    double resid;
    double lambda1;
};

__device__ __forceinline__ double hash_uniform(uint64_t idx) {  // SplitMix64 finaliser -> [-1,1)
    uint64_t z = idx * 0x9E3779B97F4A7C15ull + 0x2545F4914F6CDD1Dull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}

// Sign rule R6 on column vector u (n entries, stride `ld` in elements) — whole block.
__device__ void sign_fix_block(double* u, int64_t n, int64_t ld, double* red) {
    double mx = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) mx = fmax(mx, fabs(u[i * ld]));
    mx = warp_max(mx);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) t = fmax(t, red[w]);
        red[32] = t;
    }
    __syncthreads();
    const double half = 0.5 * red[32];
    int64_t first = INT64_MAX;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
        if (fabs(u[i * ld]) >= half) { first = i; break; }
    // block min of `first` (as double is exact for i < 2^53)
    double f = (double)first;
    for (int o = 16; o > 0; o >>= 1) f = fmin(f, __shfl_xor_sync(0xffffffffu, f, o));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = f;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = red[0];
        for (int w = 1; w < (int)(blockDim.x + 31) / 32; ++w) t = fmin(t, red[w]);
        red[32] = t;
    }
    __syncthreads();
    const int64_t istar = (int64_t)red[32];
    const bool flip = u[istar * ld] < 0.0;
    __syncthreads();
    if (flip)
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) u[i * ld] = -u[i * ld];
    __syncthreads();
}

// Two-pass classical Gram–Schmidt of the p rows of Yt (p x n) into Vt (orthonormal rows).
__device__ void cgs2_block(const double* Yt, double* Vt, int p, int64_t n, double* red, double* h) {
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int nw = (nt + 31) / 32;
    for (int k = 0; k < p; ++k) {
        double* v = Vt + (size_t)k * n;
        for (int64_t i = tid; i < n; i += nt) v[i] = Yt[(size_t)k * n + i];
        for (int attempt = 0; attempt < 2; ++attempt) {
            for (int pass = 0; pass < 2 && k > 0; ++pass) {
                for (int j0 = 0; j0 < k; j0 += 8) {
                    double part[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) part[u] = 0.0;
                    for (int64_t i = tid; i < n; i += nt) {
                        const double vi = v[i];
#pragma unroll
                        for (int u = 0; u < 8; ++u)
                            if (j0 + u < k) part[u] += Vt[(size_t)(j0 + u) * n + i] * vi;
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const double s = warp_sum(part[u]);
                        if (lane == 0) red[warp * 8 + u] = s;
                    }
                    __syncthreads();
                    if (tid < 8 && j0 + tid < k) {
                        double s = 0.0;
                        for (int w = 0; w < nw; ++w) s += red[w * 8 + tid];
                        h[j0 + tid] = s;
                    }
                    __syncthreads();
                }
                for (int64_t i = tid; i < n; i += nt) {
                    double vi = v[i];
                    for (int j = 0; j < k; ++j) vi -= h[j] * Vt[(size_t)j * n + i];
                    v[i] = vi;
                }
            }
            double ss = 0.0;
            for (int64_t i = tid; i < n; i += nt) ss += v[i] * v[i];
            ss = block_sum(ss, red);
            if (ss > 1e-280) {
                const double inv = 1.0 / sqrt(ss);
                for (int64_t i = tid; i < n; i += nt) v[i] *= inv;
                break;
            }
            // exactly dependent column: replace by a deterministic pseudo-random vector, retry
            for (int64_t i = tid; i < n; i += nt) v[i] = hash_uniform(0x5eedull * (k + 1) + (uint64_t)i);
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------------ kernels
__global__ void k_omega(double* Vt, int p, int64_t n) {
    const int64_t tot = (int64_t)p * n;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x)
        Vt[t] = hash_uniform((uint64_t)t);
}

// Warm start block: Vt[j][i] = V0[i][j] (j < r), pseudo-random for r <= j < p.
__global__ void k_seed_vt(double* Vt, const double* __restrict__ V0, int p, int r, int64_t n) {
    const int64_t tot = (int64_t)p * n;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(t / n);
        const int64_t i = t - (int64_t)j * n;
        Vt[t] = j < r ? V0[i * r + j] : hash_uniform((uint64_t)t);
    }
}

// Wt (p x n) = Vt (p x n) * G (n x n)   [= (G V)^T, G symmetric].  Tile 16 rows x 64 cols; K split
// into gridDim.z slices of kc (a multiple of 32): slice z writes Wt + z p n (k_vg_sum adds them).
__global__ void __launch_bounds__(256) k_gemm_vg(const double* __restrict__ Vt, const double* __restrict__ G,
                                                 double* __restrict__ Wt, int p, int64_t n, const State* st,
                                                 int64_t kc) {
    if (st && st->done) return;
    __shared__ double sV[16][33];
    __shared__ double sG[32][64];
    const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;  // ty 0..3 -> rows ty*4..ty*4+3
    const int64_t col = blockIdx.x * 64 + tx;
    const int row0 = blockIdx.y * 16;
    const int64_t kbeg = blockIdx.z * kc, kend = min(n, kbeg + kc);
    Wt += (size_t)blockIdx.z * p * n;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t k0 = kbeg; k0 < kend; k0 += 32) {
        for (int t = threadIdx.x; t < 16 * 32; t += 256) {
            const int rr = t / 32, kk = t % 32;
            sV[rr][kk] = (row0 + rr < p && k0 + kk < kend) ? Vt[(size_t)(row0 + rr) * n + k0 + kk] : 0.0;
        }
        for (int t = threadIdx.x; t < 32 * 64; t += 256) {
            const int kk = t / 64, cc = t % 64;
            const int64_t gc = blockIdx.x * 64 + cc;
            sG[kk][cc] = (k0 + kk < kend && gc < n) ? G[(size_t)(k0 + kk) * n + gc] : 0.0;
        }
        __syncthreads();
#pragma unroll 8
        for (int kk = 0; kk < 32; ++kk) {
            const double g = sG[kk][tx];
#pragma unroll
            for (int u = 0; u < 4; ++u) acc[u] = fma(sV[ty * 4 + u][kk], g, acc[u]);
        }
        __syncthreads();
    }
    if (col < n)
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (row0 + ty * 4 + u < p) Wt[(size_t)(row0 + ty * 4 + u) * n + col] = acc[u];
}

// Wt = sum_z part[z] in slice order (deterministic).
__global__ void __launch_bounds__(256) k_vg_sum(const double* __restrict__ part, int S, int64_t pn,
                                                double* __restrict__ Wt, const State* st) {
    if (st && st->done) return;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < pn; e += (int64_t)gridDim.x * blockDim.x) {
        double a = part[e];
        for (int z = 1; z < S; ++z) a += part[(int64_t)z * pn + e];
        Wt[e] = a;
    }
}

// K slices of W = G V: enough CTAs for the machine (the 16 x 64 output tiles of p x n are few),
// each slice >= 128 columns of K.
constexpr int kVgSlicesMax = 8;
static int vg_slices(int64_t n, int p) {
    const int64_t tiles = ceil_div(n, (int64_t)64) * ceil_div((int64_t)p, (int64_t)16);
    int S = (int)std::min<int64_t>(kVgSlicesMax, std::max<int64_t>(1, ceil_div((int64_t)2 * 148, tiles)));
    while (S > 1 && n / S < 128) --S;
    return S;
}

__global__ void __launch_bounds__(kThreads) k_orth(const double* Yt, double* Vt, int p, int64_t n) {
    __shared__ double red[8 * 32 + 40];
    __shared__ double h[kMaxP];
    cgs2_block(Yt, Vt, p, n, red, h);
}

struct RRArgs {
    int64_t n;
    int p, r, it, last;
    double* Vt;
    const double* Wt;
    double* VrT;
    double* YT;
    double* U;       // n x r output
    double* lambda;  // r (nullable)
    double* sigma;   // r (nullable)
    State* st;
};

// One Rayleigh–Ritz step (single CTA).
__global__ void __launch_bounds__(kThreads) k_rr(RRArgs a) {
    if (a.st->done) return;
    extern __shared__ double sm[];
    const int p = a.p, ld = jacobi_ld(p);
    const int64_t n = a.n;
    double* H = sm;
    double* Q = H + p * ld;
    double* red = Q + p * ld;          // 8*32 + 40
    double* h = red + 8 * 32 + 40;    // kMaxP
    double* cs = h + kMaxP;           // kMaxP/2 + 1
    double* sn = cs + kMaxP / 2 + 1;
    double* res = sn + kMaxP / 2 + 1;  // kMaxP
    int* ints = reinterpret_cast<int*>(res + kMaxP);
    int* arr = ints;                  // kMaxP + 1
    int* pp = arr + kMaxP + 2;
    int* qq = pp + kMaxP / 2 + 1;
    int* order = qq + kMaxP / 2 + 1;  // kMaxP
    int* flag = order + kMaxP;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x / 32;

    // 1. H = V^T W (lower triangle, mirrored)
    for (int pair = warp; pair < p * (p + 1) / 2; pair += nw) {
        int aa = (int)((sqrt(8.0 * pair + 1.0) - 1.0) * 0.5);
        while ((aa + 1) * (aa + 2) / 2 <= pair) ++aa;
        while (aa * (aa + 1) / 2 > pair) --aa;
        const int bb = pair - aa * (aa + 1) / 2;
        double s = 0.0;
        for (int64_t i = lane; i < n; i += 32) s += a.Vt[(size_t)aa * n + i] * a.Wt[(size_t)bb * n + i];
        s = warp_sum(s);
        if (lane == 0) { H[aa * ld + bb] = s; H[bb * ld + aa] = s; }
    }
    __syncthreads();
    // 2. Jacobi
    JacobiWork js{cs, sn, pp, qq, flag, red};
    const int sweeps = jacobi_sym(H, Q, p, js, 60);
    sort_desc_diag(H, p, order);
    // 3. VrT[k] = sum_a Q[a][order[k]] Vt[a],  YT[k] = sum_a Q[a][order[k]] Wt[a]
    for (int64_t i = tid; i < n; i += blockDim.x)
        for (int k0 = 0; k0 < p; k0 += 8) {
            double av[8], ay[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) av[u] = ay[u] = 0.0;
            for (int aa = 0; aa < p; ++aa) {
                const double v = a.Vt[(size_t)aa * n + i], w = a.Wt[(size_t)aa * n + i];
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (k0 + u < p) {
                        const double qv = Q[aa * ld + order[k0 + u]];
                        av[u] = fma(qv, v, av[u]);
                        ay[u] = fma(qv, w, ay[u]);
                    }
            }
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (k0 + u < p) {
                    a.VrT[(size_t)(k0 + u) * n + i] = av[u];
                    a.YT[(size_t)(k0 + u) * n + i] = ay[u];
                }
        }
    __syncthreads();
    // 4. residuals rho_k = ||Y_k - theta_k Vr_k|| for k < r
    for (int k = warp; k < a.r; k += nw) {
        const double th = H[order[k] * ld + order[k]];
        double s = 0.0;
        for (int64_t i = lane; i < n; i += 32) {
            const double d = a.YT[(size_t)k * n + i] - th * a.VrT[(size_t)k * n + i];
            s += d * d;
        }
        s = warp_sum(s);
        if (lane == 0) res[k] = sqrt(s);
    }
    __syncthreads();
    const double theta1 = H[order[0] * ld + order[0]];
    double rmax = 0.0;
    for (int k = 0; k < a.r; ++k) rmax = fmax(rmax, res[k]);
    const double rel = theta1 > 0.0 ? rmax / theta1 : 0.0;
    const bool conv = (a.it + 1 >= kMinIters) && (rel <= res_tol(n));
    if (conv || a.last) {
        // 5. outputs: U[:, k] = Vr_k (sign rule R6), lambda, sigma
        for (int k = 0; k < a.r; ++k) {
            sign_fix_block(a.VrT + (size_t)k * n, n, 1, red);
        }
        for (int64_t idx = tid; idx < n * a.r; idx += blockDim.x) {
            const int64_t i = idx / a.r;
            const int k = (int)(idx % a.r);
            a.U[idx] = a.VrT[(size_t)k * n + i];
        }
        for (int k = tid; k < a.r; k += blockDim.x) {
            const double th = H[order[k] * ld + order[k]];
            if (a.lambda) a.lambda[k] = th;
            if (a.sigma) a.sigma[k] = th < 0.0 ? 0.0 : sqrt(th);  // NaN (poisoned input) propagates
        }
        if (tid == 0) {
            a.st->done = 1;
            a.st->converged = conv ? 1 : 0;
            a.st->iters = a.it + 1;
            a.st->sweeps = sweeps;
            a.st->resid = rel;
            a.st->lambda1 = theta1;
        }
        return;
    }
    // 6. next basis V = CGS2(Y)
    cgs2_block(a.YT, a.Vt, p, n, red, h);
    if (tid == 0) { a.st->iters = a.it + 1; a.st->resid = rel; a.st->sweeps = sweeps; }
}

// Direct Jacobi of the whole n x n matrix (n <= kDirectMax), single CTA.
__global__ void __launch_bounds__(kThreads) k_direct(const double* G, int n, int r, double* U, double* lambda,
                                                     double* sigma, State* st) {
    extern __shared__ double sm[];
    double* H = sm;
    double* Q = H + n * jacobi_ld(n);
    double* red = Q + n * jacobi_ld(n);
    double* cs = red + 8 * 32 + 40;
    double* sn = cs + kDirectMax / 2 + 1;
    int* arr = reinterpret_cast<int*>(sn + kDirectMax / 2 + 1);
    int* pp = arr + kDirectMax + 2;
    int* qq = pp + kDirectMax / 2 + 1;
    int* order = qq + kDirectMax / 2 + 1;
    int* flag = order + kDirectMax;
    const int ld = jacobi_ld(n);
    for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) H[(idx / n) * ld + idx % n] = G[idx];
    __syncthreads();
    JacobiWork js{cs, sn, pp, qq, flag, red};
    const int sweeps = jacobi_sym(H, Q, n, js, 100);
    sort_desc_diag(H, n, order);
    // U (n x r) <- Q[:, order[k]], then sign rule per column (in place, stride r)
    for (int idx = threadIdx.x; idx < n * r; idx += blockDim.x) {
        const int i = idx / r, k = idx % r;
        U[idx] = Q[i * ld + order[k]];
    }
    __syncthreads();
    for (int k = 0; k < r; ++k) sign_fix_block(U + k, n, r, red);
    for (int k = threadIdx.x; k < r; k += blockDim.x) {
        const double th = H[order[k] * ld + order[k]];
        if (lambda) lambda[k] = th;
        if (sigma) sigma[k] = th < 0.0 ? 0.0 : sqrt(th);  // NaN (poisoned input) propagates
    }
    if (threadIdx.x == 0) {
        st->done = 1;
        st->converged = sweeps > 0 ? 1 : 0;
        st->iters = 0;
        st->sweeps = sweeps > 0 ? sweeps : -sweeps;
        st->resid = 0.0;
        st->lambda1 = H[order[0] * ld + order[0]];
    }
}

// Guard vectors q: 16 for small ranks; 8 from r = 32 on (the Jacobi and CGS2 costs grow as p^2,
// and at such ranks the spectra of the workloads are far down in the Gram's noise by then).
static int block_width(int64_t n, int r) {
    if (n <= kDirectMax) return (int)n;
    const int q = r >= 32 ? 8 : std::min(16, kMaxP - r);
    return (int)std::min<int64_t>(n, r + q);
}

static size_t rr_smem(int p) {
    return (size_t)(2 * p * jacobi_ld(p) + 8 * 32 + 40 + kMaxP + 2 * (kMaxP / 2 + 1) + kMaxP) * sizeof(double) +
           (size_t)(kMaxP + 2 + 2 * (kMaxP / 2 + 1) + kMaxP + 4) * sizeof(int);
}
static size_t direct_smem(int n) {
    return (size_t)(2 * n * jacobi_ld(n) + 8 * 32 + 40 + 2 * (kDirectMax / 2 + 1)) * sizeof(double) +
           (size_t)(kDirectMax + 2 + 2 * (kDirectMax / 2 + 1) + kDirectMax + 4) * sizeof(int);
}

}  // namespace eig

bool eig_rank_supported(int64_t n, int r) { return n <= eig::kDirectMax || r <= eig::kMaxP - 8; }

size_t eig_ws_bytes(int64_t n, int r) {
    using namespace eig;
    const int p = block_width(n, std::max(1, r));
    const int S = n > kDirectMax ? vg_slices(n, p) : 1;
    return align_up(sizeof(State), 256) + (4 + (S > 1 ? S : 0)) * align_up((size_t)p * n * sizeof(double), 256);
}

// Split form: launch_eig_begin enqueues the whole first pass (no host synchronisation; on the
// cluster path: start basis, the power steps and the first batch of Rayleigh-Ritz iterations,
// which usually converge — later launches of a converged solve exit at once), launch_eig_end
// synchronises, continues in batches while not converged, and reports.  launch_eig = both.
namespace eig {
struct Plan {
    int p, S;
    int64_t n;
    State* dst;
    double *Vt, *Wt, *VrT, *YT, *part;
};
static Plan eig_plan(int64_t n, int r, void* ws) {
    Plan q{};
    q.p = block_width(n, r);
    q.n = n;
    q.S = n > kDirectMax ? vg_slices(n, q.p) : 1;
    char* w = static_cast<char*>(ws);
    q.dst = reinterpret_cast<State*>(w);
    w += align_up(sizeof(State), 256);
    const size_t blk = align_up((size_t)q.p * n * sizeof(double), 256);
    q.Vt = reinterpret_cast<double*>(w);
    q.Wt = reinterpret_cast<double*>(w + blk);
    q.VrT = reinterpret_cast<double*>(w + 2 * blk);
    q.YT = reinterpret_cast<double*>(w + 3 * blk);
    q.part = reinterpret_cast<double*>(w + 4 * blk);  // S slices of p x n (blk apart: p n doubles each)
    return q;
}
// W = G V for the plan's Vt into its Wt (K-sliced when the output tiles are few); st_done: the
// solve's state (launches of a converged solve exit at once), or nullptr.
static int gemm_vg(const Plan& q, const double* G, const State* st_done, cudaStream_t st) {
    const int64_t n = q.n;
    const dim3 ggrid((unsigned)ceil_div(n, (int64_t)64), (unsigned)ceil_div((int64_t)q.p, (int64_t)16), (unsigned)q.S);
    const int64_t kc = ceil_div(ceil_div(n, (int64_t)q.S), (int64_t)32) * 32;
    if (q.S == 1) {
        k_gemm_vg<<<ggrid, 256, 0, st>>>(q.Vt, G, q.Wt, q.p, n, st_done, kc);
        TK_CHECK_LAUNCH();
        return TUCKER_OK;
    }
    k_gemm_vg<<<ggrid, 256, 0, st>>>(q.Vt, G, q.part, q.p, n, st_done, kc);
    TK_CHECK_LAUNCH();
    const int64_t pn = (int64_t)q.p * n;
    k_vg_sum<<<(unsigned)std::min<int64_t>(ceil_div(pn, (int64_t)256), 1024), 256, 0, st>>>(q.part, q.S, pn, q.Wt,
                                                                                            st_done);
    TK_CHECK_LAUNCH();
    return TUCKER_OK;
}
}  // namespace eig

int launch_eig_begin(int64_t n, const double* G, int r, double* U, double* lambda, double* sigma, void* ws,
                     size_t ws_bytes, cudaStream_t st, const double* V0) {
    TK_PROF(TUCKER_PROF_EIG, st);
    using namespace eig;
    if (r < 1 || r > n) return TUCKER_ERR_RANK;
    if (n > kDirectMax && r > kMaxP - 8) return TUCKER_ERR_UNSUPPORTED;
    if (ws_bytes < eig_ws_bytes(n, r)) return TUCKER_ERR_SIZE;
    const Plan q = eig_plan(n, r, ws);
    const int p = q.p;
    State* dst = q.dst;
    double *Vt = q.Vt, *Wt = q.Wt;
    TK_CUDA(cudaMemsetAsync(dst, 0, sizeof(State), st));
    if (n <= kDirectMax) {
        const size_t sm = direct_smem((int)n);
        TK_CUDA(cudaFuncSetAttribute(k_direct, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        k_direct<<<1, kThreads, sm, st>>>(G, (int)n, r, U, lambda, sigma, dst);
        TK_CHECK_LAUNCH();
    } else if (eig_cluster_supported(n)) {
        // cluster path (n <= 2048): W = G V on many CTAs, Rayleigh–Ritz + CGS2 in one cluster
        if (V0) {
            k_seed_vt<<<64, 256, 0, st>>>(Vt, V0, p, r, n);
        } else {
            k_omega<<<64, 256, 0, st>>>(Vt, p, n);
        }
        TK_CHECK_LAUNCH();
        // one cluster launch per iteration: W = G V is formed inside it (the cluster's own SMs)
        TK_RC(launch_rr_cluster(n, p, r, 0, 0, 1, Vt, Wt, U, lambda, sigma, dst, st, G));
        // iterations 1 .. kMinIters-2 are plain power steps (V <- CGS2(G V), no Rayleigh–Ritz):
        // the Ritz rotation does not change the subspace, and a single Jacobi solve of the dense
        // H at the end replaces the per-iteration ones (a warm start skips them)
        for (int w = 1; w < kMinIters - 1 && !V0; ++w)
            TK_RC(launch_rr_cluster(n, p, r, 0, 0, 1, Vt, Wt, U, lambda, sigma, dst, st, G));
        for (int it = kMinIters - 1; it < kMinIters + 3; ++it)  // first batch: 4 Rayleigh-Ritz steps
            TK_RC(launch_rr_cluster(n, p, r, it, it == kMaxIters - 1 ? 1 : 0, 0, Vt, Wt, U, lambda, sigma, dst, st,
                                    G));
    } else {
        k_omega<<<64, 256, 0, st>>>(Vt, p, n);
        TK_CHECK_LAUNCH();
        TK_RC(gemm_vg(q, G, nullptr, st));
        k_orth<<<1, kThreads, 0, st>>>(Wt, Vt, p, n);
        TK_CHECK_LAUNCH();
        const size_t sm = rr_smem(p);
        TK_CUDA(cudaFuncSetAttribute(k_rr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        for (int it = 0; it < kBatch; ++it) {
            TK_RC(gemm_vg(q, G, dst, st));
            RRArgs a{n, p, r, it, it == kMaxIters - 1 ? 1 : 0, Vt, Wt, q.VrT, q.YT, U, lambda, sigma, dst};
            k_rr<<<1, kThreads, sm, st>>>(a);
            TK_CHECK_LAUNCH();
        }
    }
    return TUCKER_OK;
}

int launch_eig_end(int64_t n, const double* G, int r, double* U, double* lambda, double* sigma, void* ws,
                   cudaStream_t st, tucker_info* info, int slot) {
    TK_PROF(TUCKER_PROF_EIG, st);
    using namespace eig;
    const Plan q = eig_plan(n, r, ws);
    const int p = q.p;
    State* dst = q.dst;
    State hs;
    TK_CUDA(cudaMemcpyAsync(&hs, dst, sizeof(State), cudaMemcpyDeviceToHost, st));
    TK_CUDA(cudaStreamSynchronize(st));
    if (n > kDirectMax) {  // continue in batches while not converged
        const bool cl = eig_cluster_supported(n);
        int it = cl ? kMinIters + 3 : kBatch;
        if (!cl) {
            const size_t sm = rr_smem(p);
            TK_CUDA(cudaFuncSetAttribute(k_rr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        }
        while (!hs.done && it < kMaxIters) {
            for (int b = 0; b < kBatch && it < kMaxIters; ++b, ++it) {
                if (cl) {
                    TK_RC(launch_rr_cluster(n, p, r, it, it == kMaxIters - 1 ? 1 : 0, 0, q.Vt, q.Wt, U, lambda, sigma,
                                            dst, st, G));
                } else {
                    TK_RC(gemm_vg(q, G, dst, st));
                    RRArgs a{n, p, r, it, it == kMaxIters - 1 ? 1 : 0, q.Vt, q.Wt, q.VrT, q.YT, U, lambda, sigma, dst};
                    const size_t sm = rr_smem(p);
                    k_rr<<<1, kThreads, sm, st>>>(a);
                    TK_CHECK_LAUNCH();
                }
            }
            TK_CUDA(cudaMemcpyAsync(&hs, dst, sizeof(State), cudaMemcpyDeviceToHost, st));
            TK_CUDA(cudaStreamSynchronize(st));
        }
    }
    if (info) {
        info->iters[slot] = hs.iters;
        info->converged[slot] = hs.converged;
        info->block[slot] = p;
        info->sweeps[slot] = hs.sweeps;
        info->resid[slot] = hs.resid;
        info->lambda1[slot] = hs.lambda1;
        // resolved count k_res = #{k <= r : lambda_k >= 1e-12 lambda_1} (R14)
        double ev[128];
        const double* src = lambda ? lambda : sigma;
        const int rr = src ? std::min(r, 128) : 0;
        if (rr) {
            TK_CUDA(cudaMemcpyAsync(ev, src, (size_t)rr * 8, cudaMemcpyDeviceToHost, st));
            TK_CUDA(cudaStreamSynchronize(st));
        }
        int k = src ? 0 : -1;
        for (int i = 0; i < rr; ++i) {
            const double lam = lambda ? ev[i] : ev[i] * ev[i];
            const double l1 = lambda ? ev[0] : ev[0] * ev[0];
            k += lam >= 1e-12 * l1 ? 1 : 0;
        }
        info->k_resolved[slot] = k;
    }
    return hs.converged ? TUCKER_OK : TUCKER_ERR_NOCONV;
}

// Asynchronous completion (no host synchronisation; CUDA-Graph capturable): the remaining
// iterations up to kMaxItersAsync are enqueued unconditionally — every launch of a converged solve exits
// at once (the state's `done` flag), so the cost of the unneeded ones is their launch latency.
int launch_eig_rest(int64_t n, const double* G, int r, double* U, double* lambda, double* sigma, void* ws,
                    cudaStream_t st) {
    TK_PROF(TUCKER_PROF_EIG, st);
    using namespace eig;
    if (n <= kDirectMax) return TUCKER_OK;  // the direct Jacobi finished in launch_eig_begin
    const Plan q = eig_plan(n, r, ws);
    const int p = q.p;
    const bool cl = eig_cluster_supported(n);
    if (!cl) {
        const size_t sm = rr_smem(p);
        TK_CUDA(cudaFuncSetAttribute(k_rr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    }
    for (int it = cl ? kMinIters + 3 : kBatch; it < kMaxItersAsync; ++it) {
        const int last = it == kMaxItersAsync - 1 ? 1 : 0;
        if (cl) {
            TK_RC(launch_rr_cluster(n, p, r, it, last, 0, q.Vt, q.Wt, U, lambda, sigma, q.dst, st, G));
        } else {
            TK_RC(gemm_vg(q, G, q.dst, st));
            RRArgs a{n, p, r, it, last, q.Vt, q.Wt, q.VrT, q.YT, U, lambda, sigma, q.dst};
            k_rr<<<1, kThreads, rr_smem(p), st>>>(a);
            TK_CHECK_LAUNCH();
        }
    }
    return TUCKER_OK;
}

int launch_eig(int64_t n, const double* G, int r, double* U, double* lambda, double* sigma, void* ws,
               size_t ws_bytes, cudaStream_t st, tucker_info* info, int slot, const double* V0) {
    TK_RC(launch_eig_begin(n, G, r, U, lambda, sigma, ws, ws_bytes, st, V0));
    return launch_eig_end(n, G, r, U, lambda, sigma, ws, st, info, slot);
}

}  // namespace tk
