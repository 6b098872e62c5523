// als.cu — NEXT f1: Tucker-ALS (HOOI) sweeps on the GPU.
//
// The paper's Tucker algorithm is HOSVD followed by ALS: for each mode m in turn the
// single-hole tensor Y_m = F x_{q != m} U_q^T (n_m x r_a x r_b) is formed and U_m is replaced by the
// leading r_m left singular vectors of its unfolding Y_(m).  One sweep streams F twice:
//   pass A (k_ttm12, fused, TMA + DMMA):  T1 = F x3 U3^T (stored, n1 n2 x r3) and Y1 = T1 x2 U2^T
//   Y1 -> singular vectors -> U1
//   Y2[j] = U1^T T1[:, j, :]       (batched DMMA GEMM over j)    -> singular vectors -> U2
//   pass B: Z = U1^T F_(1)          (r1 x n2 n3, DMMA GEMM streaming F, gemm.cu)
//   Y3[:, a, :] = Z[a]^T U2          (batched over a)              -> singular vectors -> U3
// and after the last sweep the core beta[a,b,c] = sum_k U3[k,c] Y3[k,a,b] (no extra pass).
// Singular vectors without a Gram (the f2 machinery of refine.cu on the virtual n_m x r_a x r_b
// tensor Y_m): from V = [current U_m | 8 pseudo-random guard columns], one Rayleigh–Ritz step
// Z = Y_(m)^T V, Q = CGS2(Z), B = Y_(m) Q, U_m = leading left singular vectors of B by one-sided
// Jacobi.  Forming Y_(m) Y_(m)^T would square the conditioning and bury every direction below
// ~sqrt(eps) sigma_1 (the HOSVD Gram route's noise floor, R14): at 1024^3, r = 40 that made ALS
// *raise* E (5.4e-9 -> 1.1e-8), which HOOI started from HOSVD cannot do in exact arithmetic.
// Fallback to the Gram + eigensolver (warm-started) where the SVD kernels do not apply
// (n_m > 2048, or r_a r_b < p).
// sigma_m are the singular values of the last single-hole unfoldings.  Everything reuses the
// hot-path kernels; nothing here runs on the host except launches.
#include "common.cuh"
#include "kernels.h"

namespace tk {

namespace {
struct AlsLayout {
    size_t G, T1Z, Y1, Y2, Y3, V0, scratch, total, scratch_bytes;
};

// Rayleigh–Ritz block width of the Gram-free single-hole SVD (r + 8 guard columns, <= 56), or 0
// when the SVD route does not apply to mode m.
int als_svd_p(const int64_t n[3], const int32_t r[3], int m) {
    const int64_t ra = m == 0 ? r[1] : r[0], rb = m == 2 ? r[1] : r[2];
    const int64_t p = std::min<int64_t>(n[m], std::min<int64_t>(r[m] + 8, 56));
    if (n[m] > 2048 || ra * rb < p || p < r[m]) return 0;
    return (int)p;
}

AlsLayout als_plan(const int64_t n[3], const int32_t r[3]) {
    AlsLayout L{};
    size_t off = 0;
    const int64_t nmax = std::max(n[0], std::max(n[1], n[2]));
    L.G = off;
    off += align_up((size_t)nmax * nmax * 8, 256);
    L.T1Z = off;
    off += align_up(std::max((size_t)n[0] * n[1] * r[2], (size_t)r[0] * n[1] * n[2]) * 8, 256);
    L.Y1 = off;
    off += align_up((size_t)n[0] * r[1] * r[2] * 8, 256);
    L.Y2 = off;
    off += align_up((size_t)n[1] * r[0] * r[2] * 8, 256);
    L.Y3 = off;
    off += align_up((size_t)n[2] * r[0] * r[1] * 8, 256);
    L.V0 = off;
    off += align_up((size_t)nmax * 64 * 8, 256);
    L.scratch = off;
    size_t s = ttm_ws_bytes(n, r);
    const int64_t v1[3] = {n[0], r[1], r[2]}, v2[3] = {n[1], r[0], r[2]}, v3[3] = {n[2], r[0], r[1]};
    s = std::max(s, gram_ws_bytes(v1));
    s = std::max(s, gram_ws_bytes(v2));
    s = std::max(s, gram_ws_bytes(v3));
    for (int m = 0; m < 3; ++m) s = std::max(s, eig_ws_bytes(n[m], r[m]));
    const int64_t* vv[3] = {v1, v2, v3};
    for (int m = 0; m < 3; ++m)
        if (const int p = als_svd_p(n, r, m)) s = std::max(s, refine_ws_bytes(vv[m], p));
    L.scratch_bytes = align_up(s, 256);
    off += L.scratch_bytes;
    L.total = off;
    return L;
}
}  // namespace

size_t als_ws_bytes(const int64_t n[3], const int32_t r[3]) { return als_plan(n, r).total; }

int launch_als(const int64_t n[3], const int32_t r[3], const double* F, double* const U[3], double* core,
               double* const sigma[3], int sweeps, void* ws, size_t ws_bytes, cudaStream_t st, tucker_info* info) {
    const AlsLayout L = als_plan(n, r);
    if (ws_bytes < L.total) return TUCKER_ERR_SIZE;
    char* w = static_cast<char*>(ws);
    double* G = reinterpret_cast<double*>(w + L.G);
    double* T1 = reinterpret_cast<double*>(w + L.T1Z);
    double* Z = T1;  // T1 is dead once Y2 is formed
    double* Y1 = reinterpret_cast<double*>(w + L.Y1);
    double* Y2 = reinterpret_cast<double*>(w + L.Y2);
    double* Y3 = reinterpret_cast<double*>(w + L.Y3);
    void* scr = w + L.scratch;
    const size_t sb = L.scratch_bytes;
    const int64_t r1 = r[0], r2 = r[1], r3 = r[2], n1 = n[0], n2 = n[1], n3 = n[2];
    int worst = TUCKER_OK;
    double* V0 = reinterpret_cast<double*>(w + L.V0);
    auto solve = [&](int m, const double* Y, int64_t ra, int64_t rb) -> int {
        const int64_t v[3] = {n[m], ra, rb};
        if (const int p = als_svd_p(n, r, m)) {  // Gram-free: one Rayleigh–Ritz step on Y_(m)
            TK_RC(launch_seed_from_factors(V0, U[m], n[m], r[m], p, st));
            TK_RC(launch_refine_mode(v, 0, Y, V0, nullptr, p, r[m], 1, U[m], sigma[m], scr, sb, st, nullptr));
            if (info) {
                info->iters[m] = 1;
                info->converged[m] = 1;
                info->block[m] = p;
            }
            return TUCKER_OK;
        }
        TK_RC(launch_gram(v, 0, Y, G, scr, sb, st));
        // warm start from the current factor (the previous sweep's, or the caller's initial one)
        const int rc = launch_eig(n[m], G, r[m], U[m], nullptr, sigma[m], scr, sb, st, info, m, U[m]);
        if (rc == TUCKER_ERR_NOCONV) worst = rc;
        else if (rc != TUCKER_OK) return rc;
        return TUCKER_OK;
    };
    for (int s = 0; s < sweeps; ++s) {
        // mode 1: pass A gives T1 and Y1
        TK_RC(launch_ttm_t1_y1(n, r, F, U[1], U[2], T1, Y1, scr, sb, st));
        TK_RC(solve(0, Y1, r2, r3));
        // mode 2: Y2[j] (r1 x r3) = U1^T (r1 x n1) * T1[:, j, :] (n1 x r3, row stride n2 r3)
        SmallGemm g2{r1, r3, n1, n2, U[0], 1, r1, 0, T1, n2 * r3, 1, r3, Y2, r3, 1, r1 * r3};
        TK_RC(launch_gemm(g2, st));
        TK_RC(solve(1, Y2, r1, r3));
        // mode 3: pass B, Z (r1 x n2 n3) = U1^T F_(1); Y3[:, a, :] (n3 x r2) = Z[a]^T (n3 x n2) U2
        SmallGemm gz{r1, n2 * n3, n1, 1, U[0], 1, r1, 0, F, n2 * n3, 1, 0, Z, n2 * n3, 1, 0};
        TK_RC(launch_gemm(gz, st));
        SmallGemm g3{n3, r2, n2, r1, Z, 1, n3, n2 * n3, U[1], r2, 1, 0, Y3, r1 * r2, 1, r2};
        TK_RC(launch_gemm(g3, st));
        TK_RC(solve(2, Y3, r1, r2));
    }
    // core (r1 r2 x r3) = Y3_(3)^T (r1 r2 x n3) * U3 (n3 x r3)
    SmallGemm gc{r1 * r2, r3, n3, 1, Y3, 1, r1 * r2, 0, U[2], r3, 1, 0, core, r3, 1, 0};
    TK_RC(launch_gemm(gc, st));
    return worst;
}

}  // namespace tk
