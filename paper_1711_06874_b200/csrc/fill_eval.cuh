// fill_eval.cuh — a-2 point evaluation C(r) shared by the materialised fill (fill.cu) and the
// fused generate-and-contract paths (gram.cu, ttm.cu): Matérn closed forms nu = 1/2, 3/2, 5/2
// (P:353-358), general nu through the K_nu Chebyshev table (see fill.cu), p-Slater
// (P:1029-1031), the Matérn spectral density (NEXT f4).  Every path evaluates F
// bitwise identically.
#pragma once

#include "common.cuh"
#include "kernels.h"

namespace tk {

// ------------------------------------------------------------------------- K_nu Chebyshev table
// e^z K_nu(z) = int_0^inf exp(-2 z sinh^2(t/2)) cosh(nu t) dt, trapezoid h = 1/32, summed until a
// node k has f_k < f_{k-1} and f_k < 1e-18 (running sum) (the last node counted is that k).
// Warp-cooperative form (all 32 lanes call it with the same nu, z): lane L takes nodes 32 b + L + 1
// of batch b; the stopping node is found with a warp prefix sum.  Returns the integral on every lane.
__device__ inline double scaled_besselk_trapz_warp(double nu, double z) {
    const double h = 1.0 / 32.0;
    const int lane = threadIdx.x & 31;
    double sum = 0.5, prev = 1.0;  // sum of the nodes counted so far, f of the last node of the batch before
    for (int b = 0; b < 200000 / 32; ++b) {
        const double t = (32 * b + lane + 1) * h;
        const double sh = sinh(0.5 * t);
        const double f = exp(-2.0 * z * sh * sh) * cosh(nu * t);
        double pre = f;  // inclusive prefix sum over the lanes
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, pre, o);
            if (lane >= o) pre += y;
        }
        const double fup = __shfl_up_sync(0xffffffffu, f, 1);  // every lane takes part
        const double fprev = lane == 0 ? prev : fup;
        const bool stop = f < fprev && f < 1e-18 * (sum + pre);
        const unsigned m = __ballot_sync(0xffffffffu, stop);
        if (m) {
            const int ls = __ffs(m) - 1;  // first stopping node of the batch: nodes up to it count
            return h * (sum + __shfl_sync(0xffffffffu, pre, ls));
        }
        sum += __shfl_sync(0xffffffffu, pre, 31);
        prev = __shfl_sync(0xffffffffu, f, 31);
    }
    return h * sum;
}
__device__ inline double scaled_besselk_trapz(double nu, double z) {
    const double h = 1.0 / 32.0;
    double sum = 0.5, prev = 1.0;
    for (int k = 1; k < 200000; ++k) {
        double t = k * h;
        double sh = sinh(0.5 * t);
        double f = exp(-2.0 * z * sh * sh) * cosh(nu * t);
        sum += f;
        if (f < prev && f < 1e-18 * sum) break;
        prev = f;
    }
    return h * sum;
}

// ----------------------------------------------------------------------------- point kernels

__device__ __forceinline__ double cheb_eval(const double* c, double x) {
    // y = c0/2 + sum_{m>=1} c_m T_m(x)  (Clenshaw)
    double b1 = 0.0, b2 = 0.0, x2 = 2.0 * x;
#pragma unroll
    for (int m = kChebN - 1; m >= 1; --m) {
        double b0 = fma(x2, b1, c[m] - b2);
        b2 = b1;
        b1 = b0;
    }
    return fma(x, b1, 0.5 * c[0] - b2);
}

__device__ __forceinline__ double eval_point(const KParams& kp, const double* cheb, double r2) {
    if (kp.family == TUCKER_MATERN_SPECTRAL)  // C (alpha^2 + rho^2)^{-(nu + 3/2)}
        return __dmul_rn(kp.sigma2, pow(__dadd_rn(kp.alpha2, r2), kp.mexp));
    const double r = __dsqrt_rn(r2);
    if (kp.family == TUCKER_SLATER) {
        double rp = (kp.p == 1.0) ? r : (kp.p == 2.0) ? r2 : pow(r, kp.p);
        return __dmul_rn(kp.sigma2, exp(__dmul_rn(-kp.lambda, rp)));
    }
    if (r == 0.0) return kp.sigma2;  // R4: C(0) = sigma^2
    const double z = __ddiv_rn(__dmul_rn(kp.sqrt2nu, r), kp.ell);
    const double e = exp(-z);
    switch (kp.closed) {
        case 1: return __dmul_rn(kp.sigma2, e);
        case 2: return __dmul_rn(kp.sigma2, __dmul_rn(__dadd_rn(1.0, z), e));
        case 3: {
            double poly = __dadd_rn(__dadd_rn(1.0, z), __ddiv_rn(__dmul_rn(z, z), 3.0));
            return __dmul_rn(kp.sigma2, __dmul_rn(poly, e));
        }
        default: break;
    }
    int ex;
    double m = frexp(z, &ex);  // z = m 2^ex, m in [1/2,1): interval j = ex - 1
    int j = ex - 1 - kChebJmin;
    if (j >= 0 && j < kChebIntervals) return e * cheb_eval(cheb + j * kChebN, 4.0 * m - 3.0);
    return e * (kp.pref * pow(z, kp.nu) * scaled_besselk_trapz(kp.nu, z));
}

__device__ __forceinline__ void st_v4(double* p, double a, double b, double c, double d) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};\n" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d)
                 : "memory");
}


__host__ __device__ inline bool grid_centred(const tucker_grid& g) {
    return (g.lo[0] == -g.hi[0]) && (g.lo[1] == -g.hi[1]) && (g.lo[2] == -g.hi[2]);
}

// ------------------------------------------------------------------ plane chunks (a-7 fused)
// A chunk holds planes g0 .. g0+Pc-1 of one axis of F:
//   pa = 0 (i-planes): layout [Pc][n2][n3], element (p, j, k) = F[g0+p, j, k]
//   pa = 1 (j-planes): layout [n1][Pc][n3], element (i, p, k) = F[i, g0+p, k]
// Planes at or beyond np are zero.  Values are bitwise those of the materialised fill (same nodes,
// same association order r^2 = (x^2 + y^2) + z^2, same eval_point).  On centred grids with
// n3 % 8 == 0 an item is (plane, row < ceil(nr/2), k-quad < n3/8): 4 evaluations, 4 mirrored
// 256-bit stores (rows a and nr-1-a, k and n3-1-k); otherwise an item is one element.

__host__ __device__ __forceinline__ int64_t chunk_items(const ChunkGeo& c) {
    const int64_t nr = c.pa == 0 ? c.n2 : c.n1;
    return c.mirror ? c.Pc * ((nr + 1) / 2) * (c.n3 / 8) : c.Pc * nr * c.n3;
}

__device__ __forceinline__ void gen_chunk(const ChunkGeo& c, const KParams& kp, const double* cheb,
                                          const double* __restrict__ x2, double* __restrict__ out, int64_t lo,
                                          int64_t hi, int64_t step) {
    const double* xa = x2;
    const double* xb = x2 + c.n1;
    const double* xc = x2 + c.n1 + c.n2;
    const int64_t nr = c.pa == 0 ? c.n2 : c.n1, n3 = c.n3;
    if (c.mirror) {
        const int64_t hr = (nr + 1) / 2, q3 = n3 / 8;
        for (int64_t it = lo; it < hi; it += step) {
            const int64_t t = it % q3, pr = it / q3, a = pr % hr, p = pr / hr;
            const int64_t g = c.g0 + p, k0 = 4 * t;
            double v[4] = {0.0, 0.0, 0.0, 0.0};
            if (g < c.np) {
                const double s = c.pa == 0 ? __dadd_rn(xa[g], xb[a]) : __dadd_rn(xa[a], xb[g]);
#pragma unroll
                for (int u = 0; u < 4; ++u) v[u] = eval_point(kp, cheb, __dadd_rn(s, xc[k0 + u]));
            }
            const int64_t a2 = nr - 1 - a;
            const int64_t r0 = c.pa == 0 ? (p * nr + a) : (a * c.Pc + p);
            const int64_t r1 = c.pa == 0 ? (p * nr + a2) : (a2 * c.Pc + p);
            st_v4(out + r0 * n3 + k0, v[0], v[1], v[2], v[3]);
            st_v4(out + r0 * n3 + (n3 - 4 - k0), v[3], v[2], v[1], v[0]);
            st_v4(out + r1 * n3 + k0, v[0], v[1], v[2], v[3]);
            st_v4(out + r1 * n3 + (n3 - 4 - k0), v[3], v[2], v[1], v[0]);
        }
    } else {
        for (int64_t it = lo; it < hi; it += step) {
            const int64_t k = it % n3, pr = it / n3;
            int64_t p, a, row;
            if (c.pa == 0) { a = pr % nr; p = pr / nr; row = p * nr + a; }
            else { p = pr % c.Pc; a = pr / c.Pc; row = a * c.Pc + p; }
            const int64_t g = c.g0 + p;
            double v = 0.0;
            if (g < c.np) {
                const double s = c.pa == 0 ? __dadd_rn(xa[g], xb[a]) : __dadd_rn(xa[a], xb[g]);
                v = eval_point(kp, cheb, __dadd_rn(s, xc[k]));
            }
            out[row * n3 + k] = v;
        }
    }
}

// Host: kernel parameters for the point kernels (closed-form dispatch per DESIGN R-readings).
KParams make_kparams(const tucker_kernel& kn);

// Host: enqueue k_nodes (squared nodes x^2 of the three axes, R2) and, for general nu, the
// K_nu Chebyshev table.  nodes_x2 holds n1+n2+n3 doubles, cheb kChebIntervals*kChebN.
int launch_fill_prep(const tucker_grid& g, const tucker_kernel& kn, const KParams& kp, double* nodes_x2,
                     double* cheb, cudaStream_t st);

int launch_gen_chunk(const ChunkGeo& geo, const KParams& kp, const double* cheb, const double* x2, double* out,
                     cudaStream_t st);

}  // namespace tk
