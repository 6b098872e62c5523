// multigrid.cu — NEXT f4 (alternative): multigrid Tucker.  "HOSVD only at the
// coarsest grid level n_0 << n"; "the initial guess for the ALS procedure is computed at each
// refined level by the interpolation of the dominating Tucker subspaces obtained from the previous
// coarser grid", so the fine levels cost O(n^3) (the TTM passes of ALS) instead of the O(n^4) of
// the HOSVD.  This file holds the prolongation: each factor column, a smooth function of the node
// coordinate, is interpolated from the coarse nodes to the fine ones by 4-point Lagrange (cubic)
// interpolation (one-sided stencils at the ends); the orchestration (fill per level, coarsest
// HOSVD, prolongation + orthonormalisation by the cluster SVD, ALS sweeps) is in api.cu.
#include "common.cuh"
#include "kernels.h"

namespace tk {

// Uf (nf x r) <- cubic interpolation of the columns of Uc (nc x r) from the coarse nodes xc to the
// fine nodes xf (both increasing, same interval).  One thread per fine entry.
__global__ void k_prolong(const double* __restrict__ Uc, const double* __restrict__ xc, int64_t nc,
                          double* __restrict__ Uf, const double* __restrict__ xf, int64_t nf, int r) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nf * r; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / r;
        const int c = (int)(t % r);
        const double x = xf[i];
        // interval of x: the largest k with xc[k] <= x (binary search), stencil k-1 .. k+2 clamped
        int64_t lo = 0, hi = nc - 1;
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (xc[mid] <= x) lo = mid;
            else hi = mid;
        }
        const int m = nc < 4 ? (int)nc : 4;
        int64_t s0 = lo - 1;
        if (s0 < 0) s0 = 0;
        if (s0 + m > nc) s0 = nc - m;
        double v = 0.0;
        for (int a = 0; a < m; ++a) {
            double w = 1.0;
            for (int b = 0; b < m; ++b)
                if (b != a) w *= (x - xc[s0 + b]) / (xc[s0 + a] - xc[s0 + b]);
            v = fma(w, Uc[(s0 + a) * r + c], v);
        }
        Uf[t] = v;
    }
}

// Node coordinates of one axis (the a-1 formula, R2: c + s (2i - (n-1))).
__global__ void k_axis_nodes(double* x, int64_t n, double lo, double hi) {
    const double c = (lo + hi) * 0.5, s = (hi - lo) / (2.0 * (double)(n - 1));
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = __dadd_rn(c, __dmul_rn(s, (double)(2 * i - (n - 1))));
}

int launch_prolong(const double* Uc, int64_t nc, double lo, double hi, double* Uf, int64_t nf, int r, double* xbuf,
                   cudaStream_t st) {
    double* xc = xbuf;
    double* xf = xbuf + nc;
    k_axis_nodes<<<(unsigned)ceil_div(nc, 256), 256, 0, st>>>(xc, nc, lo, hi);
    TK_CHECK_LAUNCH();
    k_axis_nodes<<<(unsigned)ceil_div(nf, 256), 256, 0, st>>>(xf, nf, lo, hi);
    TK_CHECK_LAUNCH();
    k_prolong<<<(unsigned)std::min<int64_t>(ceil_div(nf * r, 256), 4096), 256, 0, st>>>(Uc, xc, nc, Uf, xf, nf, r);
    TK_CHECK_LAUNCH();
    return TUCKER_OK;
}

}  // namespace tk
