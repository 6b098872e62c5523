// sym.cu — NEXT f3: the symmetry-exploiting variant of the whole path for centred grids
// (not in the paper).
//
// On a centred grid (lo = -hi on every axis, nodes mirror-exact by R2) F is even in each index:
// F[i,j,k] = F[n1-1-i, j, k] = ... .  Let h_m = ceil(n_m / 2) and the per-index weights w_i = 2
// (w = 1 for the middle index of an odd axis), and define the weighted octant tensor
//     F_w[i,j,k] = sqrt(w_i w_j w_k) F[i,j,k],   i < h1, j < h2, k < h3.
// Then, exactly:
//   * the mode-m Gram H_m of F_w equals D G_m^{oct} D (D = diag sqrt(w)), whose nonzero spectrum
//     is that of G_m; every eigenvector of G_m with nonzero eigenvalue is even (G_m P = G_m for
//     the reversal P), u = D^{-1} y extended by u_{n-1-i} = u_i, with y the eigenvector of H_m;
//     odd eigenvectors have eigenvalue 0 (rank F_(m) <= h_m), so r_m <= h_m is required;
//   * beta = F x1 U1^T x2 U2^T x3 U3^T = F_w x1 Y1^T x2 Y2^T x3 Y3^T (Y_m = the y's);
//   * ||F - F~||^2 = ||F_w - F_w~||^2 and ||F|| = ||F_w||.
// So the hot path runs unchanged on F_w (N/8 points): Grams cost 1/16, TTM and error 1/8; on a
// cubic isotropic grid (equal n, boxes and ranks) one Gram and one eigensolve serve all three
// modes (F is then symmetric under index permutations: G_1 = G_2 = G_3).  The
// factors are expanded and sign-fixed by rule R6 on the full vector (k_expand_sym), and the core
// is formed from the sign-fixed y's so that it matches the returned U.
#include "common.cuh"
#include "fill_eval.cuh"
#include "kernels.h"

namespace tk {

namespace {
constexpr double kSqrt2 = 1.4142135623730951;

__device__ __forceinline__ bool is_mid(int64_t i, int64_t n) { return (n & 1) && i == (n - 1) / 2; }

// F_w (h1 x h2 x h3, C order).  Values = the materialised fill's (same nodes, same association
// order) times the exact weight {1, sqrt2, 2, 2 sqrt2}[# non-middle indices].  An item is 4
// consecutive k of one (i, j) row (one index decomposition per 4 evaluations; 256-bit stores when
// h3 % 4 == 0).
__global__ void __launch_bounds__(256) k_fill_sym(KParams kp, const double* __restrict__ cheb_g,
                                                  const double* __restrict__ x2, int64_t n1, int64_t n2,
                                                  int64_t n3, double* __restrict__ Fw) {
    __shared__ double cheb[kChebIntervals * kChebN];
    if (kp.family == TUCKER_MATERN && kp.closed == 0)
        for (int t = threadIdx.x; t < kChebIntervals * kChebN; t += blockDim.x) cheb[t] = cheb_g[t];
    __syncthreads();
    const double* xa = x2;
    const double* xb = x2 + n1;
    const double* xc = x2 + n1 + n2;
    const int64_t h1 = (n1 + 1) / 2, h2 = (n2 + 1) / 2, h3 = (n3 + 1) / 2, q3 = (h3 + 3) / 4;
    const int64_t total = h1 * h2 * q3;
    const double wtab[4] = {1.0, kSqrt2, 2.0, 2.0 * kSqrt2};
    const bool vec = (h3 % 4) == 0;
    for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < total; it += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = it % q3, ij = it / q3, j = ij % h2, i = ij / h2;
        const int cij = (is_mid(i, n1) ? 0 : 1) + (is_mid(j, n2) ? 0 : 1);
        const double s = __dadd_rn(xa[i], xb[j]);
        const int64_t k0 = 4 * t;
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t k = k0 + u;
            v[u] = 0.0;
            if (k < h3) v[u] = eval_point(kp, cheb, __dadd_rn(s, xc[k])) * wtab[cij + (is_mid(k, n3) ? 0 : 1)];
        }
        double* row = Fw + (i * h2 + j) * h3;
        if (vec) {
            st_v4(row + k0, v[0], v[1], v[2], v[3]);
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (k0 + u < h3) row[k0 + u] = v[u];
        }
    }
}

// Column k of Y (h x r): u_i = y_i / sqrt(w_i); sign rule R6 on the full even vector (its first
// index with |u_i| >= max|u|/2 lies in the first half); U[i][k] = U[n-1-i][k] = s u_i and
// y_i <- s y_i.  One CTA per column.
__global__ void __launch_bounds__(256) k_expand_sym(double* __restrict__ Y, int64_t h, int64_t n, int r,
                                                    double* __restrict__ U) {
    __shared__ double red[40];
    const int k = blockIdx.x;
    double mx = 0.0;
    for (int64_t i = threadIdx.x; i < h; i += blockDim.x) {
        const double u = is_mid(i, n) ? Y[i * r + k] : Y[i * r + k] / kSqrt2;
        mx = fmax(mx, fabs(u));
    }
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    double m = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
    __syncthreads();
    double first = 1e300;
    for (int64_t i = threadIdx.x; i < h; i += blockDim.x) {
        const double u = is_mid(i, n) ? Y[i * r + k] : Y[i * r + k] / kSqrt2;
        if (fabs(u) >= 0.5 * m) {
            first = (double)i;
            break;
        }
    }
    for (int o = 16; o > 0; o >>= 1) first = fmin(first, __shfl_xor_sync(0xffffffffu, first, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = first;
    __syncthreads();
    double f = 1e300;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) f = fmin(f, red[w]);
    const int64_t i0 = (int64_t)f;
    const double s = (Y[i0 * r + k] < 0.0) ? -1.0 : 1.0;
    __syncthreads();
    for (int64_t i = threadIdx.x; i < h; i += blockDim.x) {
        const double y = s * Y[i * r + k];
        const double u = is_mid(i, n) ? y : y / kSqrt2;
        U[i * r + k] = u;
        U[(n - 1 - i) * r + k] = u;
        Y[i * r + k] = y;
    }
}

struct SymLayout {
    size_t nodes, cheb, Fw, Y[3], G, mx, scratch, total, scratch_bytes;
    int64_t h[3];
};

SymLayout sym_plan(const tucker_grid& g, const int32_t r[3]) {
    SymLayout L{};
    for (int a = 0; a < 3; ++a) L.h[a] = (g.n[a] + 1) / 2;
    size_t off = 0;
    L.nodes = off;
    off += align_up((size_t)(g.n[0] + g.n[1] + g.n[2]) * 8, 256);
    L.cheb = off;
    off += align_up((size_t)kChebIntervals * kChebN * 8, 256);
    L.Fw = off;
    off += align_up((size_t)L.h[0] * L.h[1] * L.h[2] * 8, 1024);
    for (int a = 0; a < 3; ++a) {
        L.Y[a] = off;
        off += align_up((size_t)L.h[a] * r[a] * 8, 256);
    }
    const int64_t hm = std::max(L.h[0], std::max(L.h[1], L.h[2]));
    L.G = off;
    off += align_up((size_t)hm * hm * 8, 256);
    L.mx = off;
    off += align_up((size_t)(L.h[0] + L.h[1] + L.h[2]) * 8, 256);
    L.scratch = off;
    size_t s = gram_auto_ws_bytes(L.h);
    for (int a = 0; a < 3; ++a) s = std::max(s, eig_ws_bytes(L.h[a], r[a]));
    s = std::max(s, ttm_ws_bytes(L.h, r));
    s = std::max(s, err_ws_bytes(L.h, r));
    L.scratch_bytes = align_up(s, 256);
    off += L.scratch_bytes;
    L.total = off;
    return L;
}
}  // namespace

size_t sym_ws_bytes(const tucker_grid& g, const int32_t r[3]) { return sym_plan(g, r).total; }

int launch_hosvd_sym(const tucker_grid& g, const tucker_kernel& kn, const int32_t r[3], double* const U[3],
                     double* core, double* const sigma[3], double* err3, void* ws, size_t ws_bytes, cudaStream_t st,
                     tucker_info* info) {
    const SymLayout L = sym_plan(g, r);
    if (ws_bytes < L.total) return TUCKER_ERR_SIZE;
    for (int a = 0; a < 3; ++a)
        if (r[a] > L.h[a]) return TUCKER_ERR_RANK;
    char* w = static_cast<char*>(ws);
    double* x2 = reinterpret_cast<double*>(w + L.nodes);
    double* cheb = reinterpret_cast<double*>(w + L.cheb);
    double* Fw = reinterpret_cast<double*>(w + L.Fw);
    double* G = reinterpret_cast<double*>(w + L.G);
    void* scr = w + L.scratch;
    const KParams kp = make_kparams(kn);
    TK_RC(launch_fill_prep(g, kn, kp, x2, cheb, st));
    const int64_t tot = L.h[0] * L.h[1] * ((L.h[2] + 3) / 4);
    k_fill_sym<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(tot, 256), (int64_t)kNumSMs * 16)), 256, 0,
                 st>>>(kp, cheb, x2, g.n[0], g.n[1], g.n[2], Fw);
    TK_CHECK_LAUNCH();
    uint32_t* mx = reinterpret_cast<uint32_t*>(w + L.mx);
    if (gram_use_i8(L.h)) TK_RC(launch_gram_i8_rowmax(L.h, Fw, mx, st));
    double* Y[3];
    int worst = TUCKER_OK;
    // cubic isotropic grid and equal ranks: F is symmetric under index permutations, so the three
    // mode Grams are equal (up to the rounding of r^2's summation order) — one Gram and one
    // eigensolve serve all modes
    const bool iso = g.n[0] == g.n[1] && g.n[1] == g.n[2] && g.lo[0] == g.lo[1] && g.lo[1] == g.lo[2] &&
                     g.hi[0] == g.hi[1] && g.hi[1] == g.hi[2] && r[0] == r[1] && r[1] == r[2];
    for (int m = 0; m < 3; ++m) {
        Y[m] = reinterpret_cast<double*>(w + L.Y[m]);
        if (iso && m > 0) {
            TK_CUDA(cudaMemcpyAsync(Y[m], Y[0], (size_t)L.h[m] * r[m] * 8, cudaMemcpyDeviceToDevice, st));
            TK_CUDA(cudaMemcpyAsync(U[m], U[0], (size_t)g.n[m] * r[m] * 8, cudaMemcpyDeviceToDevice, st));
            TK_CUDA(cudaMemcpyAsync(sigma[m], sigma[0], (size_t)r[m] * 8, cudaMemcpyDeviceToDevice, st));
            if (info) {
                info->iters[m] = info->iters[0];
                info->converged[m] = info->converged[0];
                info->block[m] = info->block[0];
                info->sweeps[m] = info->sweeps[0];
                info->resid[m] = info->resid[0];
                info->lambda1[m] = info->lambda1[0];
            }
            continue;
        }
        TK_RC(launch_gram_auto(L.h, m, Fw, G, mx, scr, L.scratch_bytes, st));
        const int rc = launch_eig(L.h[m], G, r[m], Y[m], nullptr, sigma[m], scr, L.scratch_bytes, st, info, m);
        if (rc == TUCKER_ERR_NOCONV) worst = rc;
        else if (rc != TUCKER_OK) return rc;
        k_expand_sym<<<(unsigned)r[m], 256, 0, st>>>(Y[m], L.h[m], g.n[m], r[m], U[m]);
        TK_CHECK_LAUNCH();
    }
    TK_RC(launch_ttm_core(L.h, r, Fw, Y[0], Y[1], Y[2], core, scr, L.scratch_bytes, st));
    if (err3) TK_RC(launch_error(L.h, r, Fw, Y[0], Y[1], Y[2], core, err3, scr, L.scratch_bytes, st));
    return worst;
}

}  // namespace tk
