// jacobi.cuh — shared-memory parallel cyclic Jacobi for a small symmetric matrix (a-4's
// Rayleigh–Ritz solve and the direct path for n <= 96).
//
// Rotations of Golub & Van Loan Alg. 8.4.2; parallel ordering = round-robin ("circle method"):
// in round s = 0..m-2 player m-1 meets s and, for w = 1..m/2-1, player (s+w) mod (m-1) meets
// (s-w) mod (m-1), so every pair meets exactly once per sweep and the m/2 rotations of a round
// commute.  The pairing is computed in closed form (no serial bookkeeping thread).  Skip rule R7:
// rotate (a,b) only if |h_ab| > max(eps sqrt|h_aa h_bb|, eps max_i|h_ii| / p) — the absolute floor
// lets the rounding-noise block converge.  The test is evaluated on squares.  The off-diagonal pair entry is set to
// exactly 0 after its rotation.  A warp owns pairs warp, warp+nw, ...: its lanes compute their
// rotations in parallel and the warp rotates their rows; then all warps rotate columns — two
// barriers per round (requires half <= 32 * nwarps); H and Q use an odd leading
// dimension (bank-conflict-free column sweeps).
#pragma once

#include "common.cuh"

namespace tk {

struct JacobiWork {  // shared-memory scratch; sizes for m <= 2*kHalfMax players
    double* cs;      // m/2
    double* sn;      // m/2
    int* pa;         // m/2  (-1: no rotation)
    int* pb;         // m/2
    int* flag;       // 1
    double* red;     // >= 33
};

__device__ __forceinline__ void rr_pair(int s, int w, int m, int& a, int& b) {
    if (w == 0) {
        a = s;
        b = m - 1;
    } else {
        const int mm = m - 1;  // 0 <= s < mm, 0 < w < mm: one conditional subtraction each
        a = s + w;
        a -= a >= mm ? mm : 0;
        b = s - w + mm;
        b -= b >= mm ? mm : 0;
    }
    if (a > b) { const int t = a; a = b; b = t; }
}

// Leading dimension used for H and Q: the smallest odd number >= p, so that column-wise warp
// accesses (consecutive rows, fixed column) hit distinct shared-memory banks.
__host__ __device__ __forceinline__ int jacobi_ld(int p) { return p | 1; }

// Diagonalise H (p x p, leading dimension ld = jacobi_ld(p)) in place; Q (p x p, same ld)
// accumulates the rotations (Q := Q J).  If `init_q`, Q starts as the identity.  Returns the
// number of sweeps (negative if the cap was hit).  Every thread of the block must call it.
__device__ inline int jacobi_sym(double* H, double* Q, int p, JacobiWork js, int max_sweeps, bool init_q = true) {
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
    const int ld = jacobi_ld(p);
    const int m = p + (p & 1), half = m / 2;
    const double eps = 2.220446049250313e-16;
    if (init_q)
        for (int i = warp; i < p; i += nw)
            for (int j = lane; j < p; j += 32) Q[i * ld + j] = (i == j) ? 1.0 : 0.0;
    if (p < 2) {
        __syncthreads();
        return 1;
    }
    for (int sweep = 0; sweep < max_sweeps; ++sweep) {
        double dm = 0.0;
        for (int i = tid; i < p; i += nt) dm = fmax(dm, fabs(H[i * ld + i]));
        dm = warp_max(dm);
        __syncthreads();  // previous readers of red / flag are done
        if (lane == 0) js.red[warp] = dm;
        if (tid == 0) *js.flag = 0;
        __syncthreads();
        double dmax = 0.0;
        for (int w = 0; w < nw; ++w) dmax = fmax(dmax, js.red[w]);
        const double floor_abs = eps * dmax / (double)p;
        for (int s = 0; s < m - 1; ++s) {
            // (1)+(2) warp `warp` owns pairs warp + l*nw (l = 0, 1, ...): lane l computes the
            //     rotation of its pair (all of the warp's pairs in parallel), publishes it for the
            //     column phase, and the warp rotates rows a, b of each of its pairs.  Rows of
            //     different pairs are disjoint, so no barrier is needed before the row update.
            {
                const int w = warp + lane * nw;
                int a = 0, b = 0, rot = 0;
                double c = 1.0, sn = 0.0;
                if (w < half) {
                    rr_pair(s, w, m, a, b);
                    if (b < p) {
                        const double apq = H[a * ld + b], app = H[a * ld + a], aqq = H[b * ld + b];
                        // |apq| > max(eps sqrt|app aqq|, floor) tested on squares (no sqrt); the
                        // rotation t = sign(tau) / (|tau| + sqrt(1 + tau^2)), tau = d / h, d = aqq - app,
                        // h = 2 apq, is formed as t = sign(d) h / (|d| + sqrt(d^2 + h^2)): one sqrt,
                        // one division, one rsqrt on the dependent chain
                        const double apq2 = apq * apq;
                        if (apq2 > fmax(eps * eps * fabs(app * aqq), floor_abs * floor_abs)) {
                            const double d = aqq - app, h = 2.0 * apq;
                            const double t = copysign(1.0, d) * h / (fabs(d) + sqrt(fma(d, d, h * h)));
                            c = rsqrt(fma(t, t, 1.0));
                            sn = t * c;
                            rot = 1;
                        }
                    }
                    js.pa[w] = rot ? a : -1;
                    js.pb[w] = b;
                    js.cs[w] = c;
                    js.sn[w] = sn;
                }
                if (__any_sync(0xffffffffu, rot) && lane == 0) *js.flag = 1;
                __syncwarp();  // all lanes' reads of H precede the row updates
                const int mine = (half - warp + nw - 1) / nw;  // pairs owned by this warp
                for (int l = 0; l < mine; ++l) {
                    const int rl = __shfl_sync(0xffffffffu, rot, l);
                    if (!rl) continue;
                    const int al = __shfl_sync(0xffffffffu, a, l), bl = __shfl_sync(0xffffffffu, b, l);
                    const double cl = __shfl_sync(0xffffffffu, c, l), sl = __shfl_sync(0xffffffffu, sn, l);
                    for (int j = lane; j < p; j += 32) {
                        const double x = H[al * ld + j], y = H[bl * ld + j];
                        H[al * ld + j] = cl * x - sl * y;
                        H[bl * ld + j] = sl * x + cl * y;
                    }
                }
            }
            __syncthreads();
            // (3) columns: H <- H J, Q <- Q J (warp per pair, lanes over rows); the rotated pair
            //     entry becomes exactly 0
            for (int w = warp; w < half; w += nw) {
                const int a = js.pa[w];
                if (a < 0) continue;
                const int b = js.pb[w];
                const double c = js.cs[w], sn = js.sn[w];
                for (int i = lane; i < p; i += 32) {
                    const double x = H[i * ld + a], y = H[i * ld + b];
                    double na = c * x - sn * y, nb = sn * x + c * y;
                    if (i == a) nb = 0.0;
                    if (i == b) na = 0.0;
                    H[i * ld + a] = na;
                    H[i * ld + b] = nb;
                    const double xq = Q[i * ld + a], yq = Q[i * ld + b];
                    Q[i * ld + a] = c * xq - sn * yq;
                    Q[i * ld + b] = sn * xq + c * yq;
                }
            }
            __syncthreads();
        }
        if (!*js.flag) return sweep + 1;
    }
    return -max_sweeps;
}

// Stable descending order of the diagonal of H (ld = jacobi_ld(p)): order[rank] = index.
__device__ __forceinline__ void sort_desc_diag(const double* H, int p, int* order) {
    const int ld = jacobi_ld(p);
    // NaN (a poisoned input, R18 window check) sorts last: a total order, so `order` is
    // always a permutation
    auto key = [](double x) { return x == x ? x : -INFINITY; };
    for (int k = threadIdx.x; k < p; k += blockDim.x) {
        const double v = key(H[k * ld + k]);
        int rank = 0;
        for (int j = 0; j < p; ++j) {
            const double w = key(H[j * ld + j]);
            rank += (w > v) || (w == v && j < k);
        }
        order[rank] = k;
    }
    __syncthreads();
}

}  // namespace tk
