// fill.cu — a-1 grid nodes and a-2 function-tensor fill F[i,j,k] = C(||x_ijk||).
//
// Kernel families: Matérn eq. (Matern) P:353-358 (closed forms for nu = 1/2, 3/2, 5/2, P:365-366
// and the half-integer K_nu), general nu through a hand-written K_nu; p-Slater eq. (exp_p)
// P:1029-1031.
//
// General-nu K_nu: g(z) = e^z z^nu K_nu(z) is smooth on every dyadic
// interval [2^j, 2^{j+1}); a per-call table of degree-20 Chebyshev coefficients of
// pref * g (pref = sigma2 2^{1-nu}/Gamma(nu)) is built on the device from node values computed by
// the trapezoid rule on K_nu(z) = int_0^inf e^{-z cosh t} cosh(nu t) dt with h = 1/32 — the paper's
// own sinc-quadrature device.  Each point then costs one exp and a Clenshaw sum
// (~21 DFMA), C = e^{-z} * cheb_j(4m - 3) where z = m 2^{j+1}, m in [1/2, 1).  Points outside the
// table range fall back to the per-point trapezoid sum.
//
// Store path: on centred grids (lo = -hi on every axis) F is even in every index, so the kernel
// evaluates one octant and writes each value to its 8 mirror images with 256-bit stores
// (st.global.v4.f64 -> STG.E.ENL2.256); reversed positions stay inside the same cache lines.
#include "common.cuh"
#include "fill_eval.cuh"
#include "kernels.h"
#include "prof.h"

namespace tk {

// ------------------------------------------------------------------------------------------ a-1
__global__ void k_nodes(double c0, double s0, int64_t n0, double c1, double s1, int64_t n1,
                        double c2, double s2, int64_t n2, double* x2) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t tot = n0 + n1 + n2;
    if (t >= tot) return;
    double c, s;
    int64_t n, i;
    if (t < n0) { c = c0; s = s0; n = n0; i = t; }
    else if (t < n0 + n1) { c = c1; s = s1; n = n1; i = t - n0; }
    else { c = c2; s = s2; n = n2; i = t - n0 - n1; }
    double m = (double)(2 * i - (n - 1));
    double x = __dadd_rn(c, __dmul_rn(s, m));  // R2: c + s (2i - (n-1)), no contraction
    x2[t] = __dmul_rn(x, x);
}

// One block per dyadic interval j = kChebJmin + blockIdx.x; warp k < 21 computes the node value at
// x_k = cos(pi (k+1/2)/21) (warp-cooperative trapezoid), then thread m the coefficient
// c_m = 2/21 sum_k g_k cos(pi m (k+1/2)/21).
__global__ void __launch_bounds__(kChebN * 32) k_cheb_table(double nu, double pref, double* table) {
    __shared__ double g[kChebN];
    const int j = kChebJmin + blockIdx.x;
    const int k = threadIdx.x >> 5;
    const double xk = cospi((k + 0.5) / kChebN);
    const double z = ldexp(1.5 + 0.5 * xk, j);
    const double v = scaled_besselk_trapz_warp(nu, z);
    if ((threadIdx.x & 31) == 0) g[k] = pref * pow(z, nu) * v;
    __syncthreads();
    if (threadIdx.x < kChebN) {
        const int m = threadIdx.x;
        double c = 0.0;
        for (int t = 0; t < kChebN; ++t) c += g[t] * cospi(m * (t + 0.5) / kChebN);
        table[blockIdx.x * kChebN + m] = c * (2.0 / kChebN);
    }
}

// Octant fill with 8-fold mirrored 256-bit stores.  Requires lo = -hi on all axes and
// n3 % 8 == 0.  Item = (i < h1, j < h2, quad t < n3/8); 4 consecutive k per thread.
// mx (nullable; centred grids with n3 / 2 <= kFillMaxK): also the row maxima of the three
// unfoldings as high words of |F| (the INT8 Gram's row scaling, bitwise what k_i8_rowmax computes
// from the stored tensor) for the first half of every axis — rows i (mx[0..n1)), j (mx[n1..)),
// k (mx[n1+n2..)); the caller mirrors them.  mode 2 through shared-memory maxima flushed once per
// CTA, modes 0 and 1 through one global atomic per distinct row and warp.
constexpr int kFillMaxK = 4096;
template <bool kMax>
__global__ void __launch_bounds__(256) k_fill_octant(KParams kp, const double* __restrict__ cheb_g,
                                                     const double* __restrict__ x2,
                                                     int64_t n1, int64_t n2, int64_t n3,
                                                     double* __restrict__ F, uint32_t* __restrict__ mx) {
    __shared__ double cheb[kChebIntervals * kChebN];
    __shared__ uint32_t smk[kMax ? kFillMaxK : 1];
    if (kp.family == TUCKER_MATERN && kp.closed == 0)
        for (int t = threadIdx.x; t < kChebIntervals * kChebN; t += blockDim.x) cheb[t] = cheb_g[t];
    if (kMax)
        for (int t = threadIdx.x; t < n3 / 2; t += blockDim.x) smk[t] = 0u;
    __syncthreads();
    const double* xa = x2;
    const double* xb = x2 + n1;
    const double* xc = x2 + n1 + n2;
    const int64_t h1 = (n1 + 1) / 2, h2 = (n2 + 1) / 2, q3 = n3 / 8;
    const int64_t total = h1 * h2 * q3;
    int64_t t_cur = -1;  // (kMax) k-chunk whose maxima km holds
    uint32_t km[4] = {0u, 0u, 0u, 0u};
    for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < total;
         it += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = it % q3;
        const int64_t ij = it / q3;
        const int64_t j = ij % h2, i = ij / h2;
        const int64_t k0 = 4 * t;
        const double s = __dadd_rn(xa[i], xb[j]);
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = eval_point(kp, cheb, __dadd_rn(s, xc[k0 + u]));
        const int64_t rows[4] = {i * n2 + j, i * n2 + (n2 - 1 - j), (n1 - 1 - i) * n2 + j,
                                 (n1 - 1 - i) * n2 + (n2 - 1 - j)};
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            double* row = F + rows[w] * n3;
            st_v4(row + k0, v[0], v[1], v[2], v[3]);
            st_v4(row + (n3 - 4 - k0), v[3], v[2], v[1], v[0]);
        }
        if (kMax) {
            // mode 2: per-thread maxima of its 4 k's, kept in registers while its k-chunk stays
            // the same (always, when q3 divides the grid stride) and flushed to shared memory
            if (t != t_cur) {
                if (t_cur >= 0)
#pragma unroll
                    for (int u = 0; u < 4; ++u) atomicMax(&smk[4 * t_cur + u], km[u]);
                t_cur = t;
#pragma unroll
                for (int u = 0; u < 4; ++u) km[u] = 0u;
            }
            uint32_t hm = 0u;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t h = (uint32_t)__double2hiint(v[u]) & 0x7FFFFFFFu;
                hm = max(hm, h);
                km[u] = max(km[u], h);
            }
            // modes 0 and 1: one reduction and two atomics per distinct (i, j) and warp
            const unsigned grp = __match_any_sync(__activemask(), ij);
            const uint32_t m = __reduce_max_sync(grp, hm);
            if ((int)(threadIdx.x & 31) == __ffs(grp) - 1) {
                atomicMax(mx + i, m);
                atomicMax(mx + n1 + j, m);
            }
        }
    }
    if (kMax) {
        if (t_cur >= 0)
#pragma unroll
            for (int u = 0; u < 4; ++u) atomicMax(&smk[4 * t_cur + u], km[u]);
        __syncthreads();
        for (int t = threadIdx.x; t < n3 / 2; t += blockDim.x)
            if (smk[t]) atomicMax(mx + n1 + n2 + t, smk[t]);
    }
}

// Mirror the first-half row maxima to the second half of every axis (centred grids).
__global__ void k_fill_mirror_max(uint32_t* mx, int64_t n1, int64_t n2, int64_t n3) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t* m;
    int64_t n, idx;
    if (t < n1) { m = mx; n = n1; idx = t; }
    else if (t < n1 + n2) { m = mx + n1; n = n2; idx = t - n1; }
    else if (t < n1 + n2 + n3) { m = mx + n1 + n2; n = n3; idx = t - n1 - n2; }
    else return;
    if (idx >= (n + 1) / 2) m[idx] = m[n - 1 - idx];
}

// General fill: one point per thread (any grid, any n3).
__global__ void __launch_bounds__(256) k_fill_general(KParams kp, const double* __restrict__ cheb_g,
                                                      const double* __restrict__ x2,
                                                      int64_t n1, int64_t n2, int64_t n3,
                                                      double* __restrict__ F) {
    __shared__ double cheb[kChebIntervals * kChebN];
    if (kp.family == TUCKER_MATERN && kp.closed == 0)
        for (int t = threadIdx.x; t < kChebIntervals * kChebN; t += blockDim.x) cheb[t] = cheb_g[t];
    __syncthreads();
    const int64_t N = n1 * n2 * n3;
    for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < N;
         it += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = it % n3;
        const int64_t ij = it / n3;
        const int64_t j = ij % n2, i = ij / n2;
        const double r2 = __dadd_rn(__dadd_rn(x2[i], x2[n1 + j]), x2[n1 + n2 + k]);
        F[it] = eval_point(kp, cheb, r2);
    }
}

// Standalone plane-chunk generation (fused TTM / error passes, a-7).
__global__ void __launch_bounds__(256) k_gen_chunk(ChunkGeo geo, KParams kp, const double* __restrict__ cheb,
                                                   const double* __restrict__ x2, double* __restrict__ out) {
    const int64_t items = chunk_items(geo);
    gen_chunk(geo, kp, cheb, x2, out, blockIdx.x * (int64_t)blockDim.x + threadIdx.x, items,
              (int64_t)gridDim.x * blockDim.x);
}

int launch_gen_chunk(const ChunkGeo& geo, const KParams& kp, const double* cheb, const double* x2, double* out,
                     cudaStream_t st) {
    const int64_t items = chunk_items(geo);
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(ceil_div(items, 256), (int64_t)kNumSMs * 16));
    k_gen_chunk<<<(unsigned)blocks, 256, 0, st>>>(geo, kp, cheb, x2, out);
    TK_CHECK_LAUNCH();
    return TUCKER_OK;
}

// --------------------------------------------------------------------------------- launcher
KParams make_kparams(const tucker_kernel& kn) {
    KParams kp{};
    kp.family = kn.family;
    kp.sigma2 = kn.sigma2;
    kp.ell = kn.ell;
    kp.nu = kn.nu;
    kp.lambda = kn.lambda;
    kp.p = kn.p;
    kp.sqrt2nu = sqrt(2.0 * kn.nu);
    kp.closed = 0;
    if (kn.family == TUCKER_MATERN && !(kn.flags & TUCKER_FORCE_GENERAL_BESSEL)) {
        if (kn.nu == 0.5) kp.closed = 1;
        else if (kn.nu == 1.5) kp.closed = 2;
        else if (kn.nu == 2.5) kp.closed = 3;
    }
    if (kn.family == TUCKER_MATERN && kp.closed == 0) kp.pref = kn.sigma2 * (pow(2.0, 1.0 - kn.nu) / tgamma(kn.nu));
    if (kn.family == TUCKER_MATERN_SPECTRAL) {
        kp.alpha2 = kn.lambda * kn.lambda;
        kp.mexp = -(kn.nu + 1.5);
    }
    return kp;
}

int launch_fill_prep(const tucker_grid& g, const tucker_kernel& kn, const KParams& kp, double* nodes_x2,
                     double* cheb, cudaStream_t st) {
    const int64_t n1 = g.n[0], n2 = g.n[1], n3 = g.n[2];
    double c[3], s[3];
    for (int a = 0; a < 3; ++a) {  // host: exactly the oracle's expressions (R2)
        c[a] = (g.lo[a] + g.hi[a]) * 0.5;
        s[a] = (g.hi[a] - g.lo[a]) / (2.0 * (double)(g.n[a] - 1));
    }
    const int64_t tot = n1 + n2 + n3;
    k_nodes<<<(unsigned)ceil_div(tot, 256), 256, 0, st>>>(c[0], s[0], n1, c[1], s[1], n2, c[2], s[2], n3, nodes_x2);
    TK_CHECK_LAUNCH();
    if (kn.family == TUCKER_MATERN && kp.closed == 0) {
        k_cheb_table<<<kChebIntervals, kChebN * 32, 0, st>>>(kn.nu, kp.pref, cheb);
        TK_CHECK_LAUNCH();
    }
    return TUCKER_OK;
}

bool fill_rowmax_supported(const tucker_grid& g) {
    return grid_centred(g) && g.n[2] % 8 == 0 && g.n[2] / 2 <= kFillMaxK;
}

int launch_fill(const tucker_grid& g, const tucker_kernel& kn, double* F, double* nodes_x2, double* cheb,
                cudaStream_t st, uint32_t* mx) {
    TK_PROF(TUCKER_PROF_FILL, st);
    const int64_t n1 = g.n[0], n2 = g.n[1], n3 = g.n[2];
    const KParams kp = make_kparams(kn);
    if (mx && !fill_rowmax_supported(g)) return TUCKER_ERR_UNSUPPORTED;
    TK_RC(launch_fill_prep(g, kn, kp, nodes_x2, cheb, st));
    if (grid_centred(g) && n3 % 8 == 0) {
        const int64_t items = ((n1 + 1) / 2) * ((n2 + 1) / 2) * (n3 / 8);
        const int64_t blocks = std::min<int64_t>(ceil_div(items, 256), (int64_t)kNumSMs * 16);
        if (mx) {
            TK_CUDA(cudaMemsetAsync(mx, 0, (size_t)(n1 + n2 + n3) * 4, st));
            k_fill_octant<true><<<(unsigned)blocks, 256, 0, st>>>(kp, cheb, nodes_x2, n1, n2, n3, F, mx);
            TK_CHECK_LAUNCH();
            k_fill_mirror_max<<<(unsigned)ceil_div(n1 + n2 + n3, 256), 256, 0, st>>>(mx, n1, n2, n3);
        } else {
            k_fill_octant<false><<<(unsigned)blocks, 256, 0, st>>>(kp, cheb, nodes_x2, n1, n2, n3, F, nullptr);
        }
    } else {
        const int64_t blocks = std::min<int64_t>(ceil_div(n1 * n2 * n3, 256), (int64_t)kNumSMs * 16);
        k_fill_general<<<(unsigned)blocks, 256, 0, st>>>(kp, cheb, nodes_x2, n1, n2, n3, F);
    }
    TK_CHECK_LAUNCH();
    return TUCKER_OK;
}

}  // namespace tk
