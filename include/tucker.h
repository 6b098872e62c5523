/*
 * tucker.h — C-ABI of the B200-native (sm_100a) Tucker/HOSVD hot path of arXiv 1711.06874,
 * "Tucker tensor analysis of Matérn functions in spatial statistics".
 *
 * Citations: "P:n" is line n of the paper's LaTeX source; "R<k>" are the readings of
 * ambiguous passages listed in DESIGN.md §3.
 *
 * The path:
 *   a-1 grid nodes             x_i = -b + (i-1)h, h = 2b/(n-1)
 *   a-2 function-tensor fill   F[i,j,k] = C(||x_ijk||), Matérn / Slater
 *   a-3 per-mode Gram          G_m = F_(m) F_(m)^T  (the SVD of the unfolding A_(l))
 *   a-4 top-r eigenvectors     U_m = leading r_m eigenvectors of G_m, sigma = sqrt(lambda)
 *   a-5 core                   beta = F x1 U1^T x2 U2^T x3 U3^T
 *   a-6 error                  E = ||F - beta x1 U1 x2 U2 x3 U3|| / ||F||
 *
 * Conventions (all entry points):
 *   - Device pointers ("dev") are CUDA device memory owned by the caller; the library never
 *     allocates or frees caller memory.  All scratch comes from the caller's workspace `ws`
 *     (device, >= tucker_workspace_size() bytes, 256-byte aligned).
 *   - Work is enqueued on `stream` (a cudaStream_t; NULL = legacy default stream).  Entry points
 *     are asynchronous unless stated.  tucker_hosvd / tucker_hosvd_rowmax synchronise only when
 *     `info` is non-NULL (then per mode, to test and report eigensolver convergence); with
 *     info == NULL they never touch the host (CUDA-Graph capturable) and cannot report NOCONV or
 *     TUCKER_ERR_INPUT (a bad input then shows as NaN outputs).
 *   - Tensors are FP64, C order (n1 x n2 x n3, k fastest).  Factor U_m is n_m x r_m row-major
 *     (column c = c-th factor vector).  The core is r1 x r2 x r3 C order.
 *   - Validation happens before any launch.  Errors are returned as TUCKER_* codes; no exception
 *     crosses the ABI.  Functions are reentrant across threads: the only mutable library state is
 *     per calling thread (the Gram engine of tucker_set_gram_engine, the two side streams the
 *     HOSVD overlaps its eigensolves on, the launch counter, the opt-in stage timer) besides a
 *     one-time driver entry-point lookup.
 */
#ifndef TUCKER_B200_H
#define TUCKER_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define TUCKER_API __attribute__((visibility("default")))
#else
#define TUCKER_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Axes-parallel box prod_m [lo_m, hi_m] with n_m collocation nodes per axis.
 * Node i of axis m (i = 0..n_m-1) is c + s*(2i-(n_m-1)), c = (lo+hi)/2, s = (hi-lo)/(2(n_m-1)):
 * the paper's -b + (i-1)h, evaluated in a form that is bitwise mirror-exact (R2). */
typedef struct {
    int64_t n[3];
    double lo[3], hi[3];
} tucker_grid;

enum { TUCKER_MATERN = 0, TUCKER_SLATER = 1, TUCKER_MATERN_SPECTRAL = 2 };

/* Kernel parameters.
 *   TUCKER_MATERN: C(r) = sigma2 * 2^{1-nu}/Gamma(nu) * z^nu K_nu(z), z = sqrt(2 nu) r / ell
 *                  (eq. Matern; sigma2 per R3; C(0) = sigma2, R4).  nu in {0.5,1.5,2.5}
 *                  (compared exactly) uses the closed forms e^{-z}, (1+z)e^{-z}, (1+z+z^2/3)e^{-z}
 *                  unless TUCKER_FORCE_GENERAL_BESSEL is set.
 *   TUCKER_SLATER: C(r) = sigma2 * exp(-lambda r^p), 0 < p <= 2 (eq. exp_p; p = 2 is
 *                  the Gaussian).
 *   TUCKER_MATERN_SPECTRAL (NEXT f4): the Matérn spectral density f(rho) = sigma2 (alpha^2 +
 *                  rho^2)^{-(nu + 3/2)} (eq. SD_matern, d = 3, C = sigma2 by R17) with
 *                  alpha = `lambda` > 0, nu > 0; rho = ||x|| on the (frequency) grid.
 * `flags` may hold TUCKER_FORCE_GENERAL_BESSEL. */
typedef struct {
    int32_t family;
    int32_t flags;
    double sigma2, ell, nu, lambda, p;
} tucker_kernel;

enum {
    TUCKER_FORCE_GENERAL_BESSEL = 2, /* kernel flag: evaluate half-integer nu through K_nu */
};

enum {
    TUCKER_OK = 0,
    TUCKER_ERR_INVALID_ARG = 1, /* null pointer, n_m < 2, lo >= hi, bad mode                */
    TUCKER_ERR_DOMAIN = 2,      /* sigma2<=0, ell<=0, nu<=0, lambda<=0, p not in (0,2]       */
    TUCKER_ERR_RANK = 3,        /* r_m < 1 or r_m > n_m                                      */
    TUCKER_ERR_SIZE = 4,        /* workspace too small / size overflow                       */
    TUCKER_ERR_NOCONV = 5,      /* eigensolver hit its iteration cap (best iterate returned) */
    TUCKER_ERR_CUDA = 6,        /* a CUDA runtime/driver call failed                         */
    TUCKER_ERR_UNSUPPORTED = 7, /* e.g. r_m too large for the eigensolver block (r_m > 56)   */
    TUCKER_ERR_COLLECTIVE = 8,  /* the caller's all-reduce callback reported a failure       */
    TUCKER_ERR_INPUT = 9        /* F not finite, or caller row maxima that do not bound F     */
};

/* Per-mode eigensolver report (host struct, optional). */
typedef struct {
    int32_t iters[3];     /* subspace iterations (0 = direct Jacobi on G_m)                   */
    int32_t converged[3]; /* 1 if every leading-r_m Ritz residual met the tolerance           */
    int32_t block[3];     /* subspace block width p_m                                          */
    int32_t sweeps[3];    /* Jacobi sweeps of the last Rayleigh-Ritz solve                    */
    double resid[3];      /* max_{k<=r_m} ||G v_k - theta_k v_k|| / theta_1                   */
    double lambda1[3];    /* theta_1 (largest eigenvalue of G_m)                              */
    int32_t k_resolved[3]; /* #{k <= r_m : lambda_k >= 1e-12 lambda_1}: the resolved leading
                              eigenpairs (R14; past it the Gram route's noise)  */
    int32_t moduli[3];     /* INT8 Gram route: moduli the exact Gram of mode m was formed with
                              (16, or 15 / 14 where the row-norm bound of DESIGN.md R21 allows it);
                              0 for the FP64 DMMA engine.  Set by tucker_hosvd,
                              tucker_hosvd_rowmax, tucker_hosvd_prepared (untouched elsewhere) */
} tucker_info;

/* Workspace bytes needed by tucker_hosvd / tucker_error / tucker_gram / tucker_eig /
 * tucker_ttm_core / tucker_approximate for this grid and ranks (r may be NULL: ranks
 * min(n_m, 56)).  Depends on the calling thread's Gram engine (set it first). */
TUCKER_API size_t tucker_workspace_size(const tucker_grid* grid, const int32_t r[3]);
/* Workspace bytes tucker_fill / tucker_fill_rowmax need (the nodes and the K_nu table; a few KB). */
TUCKER_API size_t tucker_workspace_size_fill(const tucker_grid* grid);

/* a-1 + a-2: F (dev, n1*n2*n3 doubles) <- collocation tensor of `kernel` on `grid`
 * (P:981-997).  Uses ws (>= tucker_workspace_size_fill) for the nodes and the K_nu Chebyshev
 * table. */
TUCKER_API int tucker_fill(const tucker_grid* grid, const tucker_kernel* kernel, double* F, void* ws,
                size_t ws_bytes, void* stream);

/* a-3: G (dev, n_m x n_m, both triangles) <- F_(m) F_(m)^T for mode m in {0,1,2}
 * (P:555-561).  Deterministic (fixed-order split-K reduction). */
TUCKER_API int tucker_gram(const tucker_grid* grid, int32_t mode, const double* F, double* G, void* ws,
                size_t ws_bytes, void* stream);

/* a-3 on the INT8 tensor cores (tcgen05 kind::i8): the same G as tucker_gram, to FP64 accuracy by
 * modular emulation (R18).  Every row a_i of F_(m) is scaled by 2^(b - E_i)
 * (max_k |a_ik| < 2^E_i, b <= 50) and rounded to integers X; S = X X^T is formed exactly from its
 * residues modulo 16 pairwise-coprime moduli (int8 Gram matrices on the tensor cores, exact int32
 * accumulation) and reconstructed by the Chinese remainder theorem; G_ij = fl(2^(E_i+E_j-2b) S_ij),
 * one rounding.  Deterministic and independent of the launch configuration.  Workspace:
 * tucker_workspace_size_i8 (residues of up to 8 GiB of the unfolding at a time, partials).
 * TUCKER_ERR_UNSUPPORTED if some n_m > 16384.  A value outside the scheme's window (NaN / Inf in
 * F) makes every entry of G NaN. */
TUCKER_API size_t tucker_workspace_size_i8(const tucker_grid* grid);
/* The INT8 Gram's modular scheme for an unfolding with K columns (host only, no GPU): the 16
 * moduli (moduli[16], host) and the integer width b (*b, host) used by tucker_gram_i8 —
 * pairwise coprime odd p_l <= 253 with prod p_l > 2 K 2^(2b), b <= 50.  Returns TUCKER_OK. */
TUCKER_API int tucker_i8_scheme(int64_t K, int32_t* moduli, int32_t* b);
/* Which INT8 residue layout the materialised Grams of `grid` use under the calling thread's engine
 * (host only): *shared = 1 for the shared layout (R20: one residue pass serves the three
 * modes, ONE exponent E = the largest row exponent scales the whole tensor, b = the scheme's width
 * for the largest K), 0 for the per-mode row-scaled layout (R18; b of mode 0's K — each mode uses
 * its own).  The shared layout applies when n3 % 16 == 0 and the 16 N-byte residue tensor fits the
 * cap (40 GiB); TUCKER_GRAM_INT8_ROWSCALED forces the per-mode layout.  UNSUPPORTED if the INT8
 * engine does not apply. */
TUCKER_API int tucker_i8_layout(const tucker_grid* grid, int32_t* shared, int32_t* b);
/* Gram engine of tucker_gram, tucker_hosvd and tucker_approximate, per calling thread (set it
 * before sizing workspaces: tucker_workspace_size depends on it).  TUCKER_GRAM_AUTO
 * (default): the INT8 emulation where supported (every n_m <= 16384), DMMA otherwise. */
enum { TUCKER_GRAM_AUTO = 0, TUCKER_GRAM_DMMA = 1, TUCKER_GRAM_INT8 = 2, TUCKER_GRAM_INT8_ROWSCALED = 3 };
TUCKER_API int tucker_set_gram_engine(int32_t engine);
TUCKER_API int32_t tucker_get_gram_engine(void);
/* TTM engine of the core on the INT8 hosvd route (tucker_hosvd, tucker_hosvd_rowmax,
 * tucker_hosvd_prepared, tucker_approximate with INT8 Grams in the shared layout), per calling
 * thread.  TUCKER_TTM_AUTO (default): the first product T1 = F x3 U3^T (P:578-579, 2 N r3 flops)
 * on the INT8 tensor cores by six balanced base-256 digits per operand, the 26 digit pairs of
 * weight >= 256^-6 (R22: input rounding 2^-47 of max|F| and of each column's max|U3|,
 * truncation <= 2^-52 per term), where r3 <= 48, n3 % 16 == 0 and n3 <= 16384; the FP64 DMMA TTM
 * otherwise.  TUCKER_TTM_DMMA forces the DMMA TTM.  TUCKER_TTM_INT8_ERROR = AUTO plus the error
 * pass's reconstruction Ft = W U3^T on the INT8 tensor cores (tucker_error; R23: the same
 * digit scheme, E within 2^-46 of the FP64 pass) — opt-in: measured slower than the DMMA error pass.
 * INVALID_ARG for other values. */
enum { TUCKER_TTM_AUTO = 0, TUCKER_TTM_DMMA = 1, TUCKER_TTM_INT8_ERROR = 2 };
TUCKER_API int tucker_set_ttm_engine(int32_t engine);
TUCKER_API int32_t tucker_get_ttm_engine(void);
TUCKER_API int tucker_gram_i8(const tucker_grid* grid, int32_t mode, const double* F, double* G, void* ws,
                size_t ws_bytes, void* stream);

/* a-4: leading r eigenpairs of a symmetric PSD n x n matrix G (dev): U (dev, n x r row-major,
 * sorted by descending eigenvalue, sign rule R6), lambda (dev, r).  Synchronises `stream`.
 * `info_mode` (host, nullable) receives {iters, converged, block, sweeps, resid, lambda1} in
 * slot 0 of a tucker_info. */
TUCKER_API int tucker_eig(int64_t n, const double* G, int32_t r, double* U, double* lambda, void* ws,
               size_t ws_bytes, void* stream, tucker_info* info_mode);

/* a-5: core (dev, r1*r2*r3) <- F x1 U1^T x2 U2^T x3 U3^T for given factors (dev). */
TUCKER_API int tucker_ttm_core(const tucker_grid* grid, const int32_t r[3], const double* F, const double* U1,
                    const double* U2, const double* U3, double* core, void* ws, size_t ws_bytes,
                    void* stream);

/* a-3..a-5: truncated HOSVD of F (dev).  Outputs (dev): U1,U2,U3 (n_m x r_m), core, and
 * sigma_m (dev, r_m) = sqrt(max(lambda_m,0)).  `info` (host) may be NULL (asynchronous call, see
 * the conventions).  Errors: INVALID_ARG, RANK, SIZE, UNSUPPORTED (r_m > 56 with n_m > 112, or
 * r_2 / r_3 > 64 — checked before any launch), NOCONV and INPUT (info != NULL only), CUDA. */
TUCKER_API int tucker_hosvd(const tucker_grid* grid, const int32_t r[3], const double* F, double* U1,
                 double* U2, double* U3, double* core, double* sigma1, double* sigma2,
                 double* sigma3, void* ws, size_t ws_bytes, void* stream, tucker_info* info);

/* a-2 + the INT8 route's row scaling in one pass: tucker_fill, and rowmax (dev, n1+n2+n3 uint32)
 * <- per row of each unfolding the largest high 32-bit word of |F| (sign cleared): rows i of
 * F_(1) at [0, n1), rows j of F_(2) at [n1, n1+n2), rows k of F_(3) at [n1+n2, n1+n2+n3) — the
 * exponents R18 scales each row by.  Centred grids with n3 % 8 == 0 and n3 <= 8192 only (the
 * octant fill), else TUCKER_ERR_UNSUPPORTED (use tucker_fill).  Workspace as tucker_fill. */
TUCKER_API int tucker_fill_rowmax(const tucker_grid* grid, const tucker_kernel* kernel, double* F, uint32_t* rowmax,
                       void* ws, size_t ws_bytes, void* stream);

/* tucker_hosvd with the row maxima of F supplied (rowmax from tucker_fill_rowmax of this very F):
 * on the INT8 Gram route the row-maxima pass over F is skipped, the results are bitwise those of
 * tucker_hosvd.  rowmax == NULL, or the DMMA route: tucker_hosvd.  The maxima are verified where
 * they are used: a row maximum that does not bound its row (a stale rowmax) is detected by the
 * residue kernel, which then makes the Grams NaN — TUCKER_ERR_INPUT with info != NULL, NaN outputs
 * without. */
TUCKER_API int tucker_hosvd_rowmax(const tucker_grid* grid, const int32_t r[3], const double* F,
                        const uint32_t* rowmax, double* U1, double* U2, double* U3, double* core,
                        double* sigma1, double* sigma2, double* sigma3, void* ws, size_t ws_bytes,
                        void* stream, tucker_info* info);

/* a-2 + the INT8 route's inputs in one pass (centred grids with n3 % 16 == 0 under the shared
 * residue layout, R20; else TUCKER_ERR_UNSUPPORTED): F (dev) <- the collocation tensor, and into
 * ws — the tucker_hosvd workspace of (grid, r), the calling thread's engine — the global exponent
 * and the residue planes of F.  The octant fill evaluates N/8 values (F is even in every index)
 * and converts each to its residues once, storing value and residue bytes at the 8 mirrored
 * positions: the residue pass over F is gone.  Before the fill, the unfoldings' largest row norms
 * (the rows nearest the centre: C(r) is non-increasing in r) choose the moduli per mode (DESIGN.md
 * R21): 14 where (2^(b-E) max ||a_i|| + sqrt(K)/2)^2 < P_14 / 2, else 15 where it is < P_15 / 2 — the
 * Gram is still exact — else 16; planes no mode reads are not written.  Follow it with tucker_hosvd_prepared
 * on the same F and ws. */
TUCKER_API int tucker_fill_prepare(const tucker_grid* grid, const tucker_kernel* kernel, const int32_t r[3], double* F,
                        void* ws, size_t ws_bytes, void* stream);
/* tucker_hosvd on a workspace prepared by tucker_fill_prepare for this very F (the caller guarantees
 * it; nothing of F is re-read for the Grams): the row-maxima and residue passes are skipped, the
 * results are those tucker_hosvd computes on the shared layout.  A value outside the scheme's window
 * still trips the flag (TUCKER_ERR_INPUT with info, NaN without).  Same outputs and errors as
 * tucker_hosvd, plus UNSUPPORTED where tucker_fill_prepare is.  The prepared residue planes are
 * only read: the workspace can serve further calls on the same F. */
TUCKER_API int tucker_hosvd_prepared(const tucker_grid* grid, const int32_t r[3], const double* F, double* U1,
                          double* U2, double* U3, double* core, double* sigma1, double* sigma2, double* sigma3,
                          void* ws, size_t ws_bytes, void* stream, tucker_info* info);

/* a-6: out3 (dev, 3 doubles) <- {E, ||F||, ||F - Ft||} with Ft = core x1 U1 x2 U2 x3 U3
 * (P:1016-1025).  Deterministic (fixed-order reduction, no float atomics). */
TUCKER_API int tucker_error(const tucker_grid* grid, const int32_t r[3], const double* F, const double* U1,
                 const double* U2, const double* U3, const double* core, double* out3, void* ws,
                 size_t ws_bytes, void* stream);

/* Whole path with HOST outputs (the end-to-end call a user makes): fill F into the caller's
 * device buffer F (dev, n1*n2*n3), HOSVD, error; then copy U_m, core, sigma_m and
 * {E, ||F||, ||F-Ft||} to the host buffers (any host memory; pinned is faster) and synchronise.
 * Host buffers: U_h[m] (n_m*r_m), core_h (r1*r2*r3), sigma_h[m] (r_m), err_h (3). */
TUCKER_API int tucker_approximate(const tucker_grid* grid, const tucker_kernel* kernel, const int32_t r[3],
                       double* F, double* const U_h[3], double* core_h, double* const sigma_h[3],
                       double* err_h, void* ws, size_t ws_bytes, void* stream, tucker_info* info);

/* ------------------------------------------------------------------------------------------
 * a-7 fused generate-and-contract (BASELINE config 5's 2048^3 path): F is never materialised.
 * The function tensor is regenerated from `grid` + `kernel` (bitwise the values tucker_fill
 * would store) in plane chunks: for the Gram, chunks of ~32 MB are generated by a persistent
 * cooperative grid into an L2-resident two-slot ring and consumed by the same TMA + DMMA tiles as
 * tucker_gram (one grid barrier per chunk); for the core and the error, chunks of i-slabs
 * (~1 GiB) are generated ahead of the fused TTM / error kernels.  Results equal the
 * materialised path's up to the summation order of the Gram (split points differ).
 * Workspace (dev, caller-owned) >= tucker_workspace_size_fused(grid, r); no F argument.
 * Requirements: n3 even and >= 16 (TMA strides), ranks r_m <= 56.  Errors as above, plus
 * TUCKER_ERR_UNSUPPORTED when the cooperative grid cannot be made resident.
 */
TUCKER_API size_t tucker_workspace_size_fused(const tucker_grid* grid, const int32_t r[3]);

/* a-3 fused: G (dev, n_m x n_m, both triangles) <- F_(m) F_(m)^T with F generated on the fly. */
TUCKER_API int tucker_gram_fused(const tucker_grid* grid, const tucker_kernel* kernel, int32_t mode, double* G,
                      void* ws, size_t ws_bytes, void* stream);

/* a-3..a-5 fused: truncated HOSVD of the function tensor of (grid, kernel); outputs as
 * tucker_hosvd (dev U_m n_m x r_m, core r1*r2*r3, sigma_m r_m); `info` (host) may be NULL. */
TUCKER_API int tucker_hosvd_fused(const tucker_grid* grid, const tucker_kernel* kernel, const int32_t r[3],
                       double* U1, double* U2, double* U3, double* core, double* sigma1, double* sigma2,
                       double* sigma3, void* ws, size_t ws_bytes, void* stream, tucker_info* info);

/* a-6 fused: out3 (dev) <- {E, ||F||, ||F - Ft||} with F regenerated chunk by chunk. */
TUCKER_API int tucker_error_fused(const tucker_grid* grid, const tucker_kernel* kernel, const int32_t r[3],
                       const double* U1, const double* U2, const double* U3, const double* core, double* out3,
                       void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------------------------
 * Row (e): ONE fused HOSVD (a-7, F never stored) sharded over `nshards` ranks,
 * one process per GPU.  Every rank makes the same call with its own `shard` in [0, nshards).
 * The work units — the residue super-chunks of each mode's unfolding (INT8 Gram route) and the
 * i-slab chunks of the core and of the error — go round-robin to the ranks; the exchange steps
 * (§8(e): "Grams: all-reduce of the n_m x n_m partials", "TTM1: ... all-reduce of r-sized
 * intermediates", "Error: a scalar all-reduce") are all-reduces the CALLER performs through
 * `allreduce` (e.g. torch.distributed over NCCL):
 *   - per mode, the exact per-modulus residue sums of the Gram (int32, SUM; 16 x tiles x 512 x 256),
 *     then folded mod p_l and reconstructed by the CRT on every rank;
 *   - non-centred grids only: the row maxima of the three unfoldings (int32, MAX);
 *   - T2 = F x2 U2^T x3 U3^T (n1 x r2 r3 doubles, SUM; rows off a rank's slabs are zero);
 *   - with err3 != NULL, the per-tile error partials (doubles, SUM; zero off the rank's slabs).
 * Integer sums are exact and the floating-point ones add zeros, so every rank returns the bitwise
 * result of tucker_hosvd_fused (+ tucker_error_fused).  The eigensolves are replicated.
 * allreduce(user, ws_offset, count, dtype, op): reduce `count` elements of `dtype` in place at
 * byte offset `ws_offset` of `ws` (device memory of this rank) across the ranks; called from the
 * calling host thread after `stream` has been synchronised, the same number of times and in the
 * same order on every rank; must return 0 when the reduced data is in place.  nshards == 1 never
 * calls it (it may then be NULL).
 * Workspace >= tucker_workspace_size_fused(grid, r).  Requires the INT8 fused Gram route
 * (n_m <= 16384, engine not forced to DMMA): else TUCKER_ERR_UNSUPPORTED.  Errors as
 * tucker_hosvd_fused, plus INVALID_ARG (nshards < 1, shard out of range, nshards > 1 and no
 * callback) and TUCKER_ERR_COLLECTIVE (the callback returned non-zero; the call stops there).
 */
enum { TUCKER_DT_INT32 = 0, TUCKER_DT_F64 = 1 };
enum { TUCKER_RED_SUM = 0, TUCKER_RED_MAX = 1 };
typedef int (*tucker_allreduce_fn)(void* user, int64_t ws_offset, int64_t count, int32_t dtype, int32_t op);
TUCKER_API int tucker_hosvd_fused_sharded(const tucker_grid* grid, const tucker_kernel* kernel, const int32_t r[3],
                       int32_t shard, int32_t nshards, tucker_allreduce_fn allreduce, void* user, double* U1,
                       double* U2, double* U3, double* core, double* sigma1, double* sigma2, double* sigma3,
                       double* err3, void* ws, size_t ws_bytes, void* stream, tucker_info* info);

/* ------------------------------------------------------------------------------------------
 * NEXT f1: Tucker-ALS (HOOI) sweeps, the paper's second stage after HOSVD: for each
 * mode m in turn U_m <- leading r_m left singular vectors of the single-hole unfolding
 * (F x_{q != m} U_q^T)_(m) (top eigenvectors of its Gram), modes 1, 2, 3 in order; `sweeps`
 * (>= 1) sweeps; then core = F x1 U1^T x2 U2^T x3 U3^T with the final factors.
 *   F (dev, n1 x n2 x n3), U_m (dev, n_m x r_m, in: initial factors, e.g. tucker_hosvd's; out:
 *   refined, sign rule R6), core (dev out), sigma_m (dev out: singular values of the last
 *   single-hole unfoldings).  Workspace (dev) >= tucker_workspace_size_als(grid, r).
 *   Errors: INVALID_ARG (null, sweeps < 1), RANK, SIZE, UNSUPPORTED (r_2 or r_3 > 64, r_m > 56),
 *   NOCONV (best iterate returned), CUDA.  Synchronises `stream` once per mode and sweep. */
TUCKER_API size_t tucker_workspace_size_als(const tucker_grid* grid, const int32_t r[3]);
TUCKER_API int tucker_als(const tucker_grid* grid, const int32_t r[3], const double* F, double* U1, double* U2,
               double* U3, double* core, double* sigma1, double* sigma2, double* sigma3, int32_t sweeps,
               void* ws, size_t ws_bytes, void* stream, tucker_info* info);

/* ------------------------------------------------------------------------------------------
 * NEXT f3: symmetry-exploiting HOSVD for centred grids (lo = -hi on every axis; not in the paper).
 * F is even in each index, so the path runs on the weighted octant tensor
 * F_w[i,j,k] = sqrt(w_i w_j w_k) F[i,j,k] (i < ceil(n1/2) ..., w = 2, or 1 for the middle index of
 * an odd axis): its mode-m Grams have the nonzero spectrum of G_m, their eigenvectors y give the
 * (even) factors u = y / sqrt(w) mirrored to full length, and core and error equal those of F
 * (f3).  Outputs as tucker_hosvd (full-length U_m, sign rule R6 on the full vector,
 * core consistent with them) plus err3 (dev, nullable) = {E, ||F||, ||F - Ft||}.
 * On a cubic isotropic grid (equal n_m, boxes and ranks) the three mode Grams are equal and one
 * Gram + eigensolve serves all modes (U1 = U2 = U3).
 * Requires r_m <= ceil(n_m/2) (the odd eigenvectors have eigenvalue 0): else TUCKER_ERR_RANK.
 * Non-centred grid: TUCKER_ERR_UNSUPPORTED.  Workspace >= tucker_workspace_size_sym(grid, r);
 * no F argument (the octant is generated into the workspace, N/8 doubles). */
TUCKER_API size_t tucker_workspace_size_sym(const tucker_grid* grid, const int32_t r[3]);
TUCKER_API int tucker_hosvd_sym(const tucker_grid* grid, const tucker_kernel* kernel, const int32_t r[3],
                     double* U1, double* U2, double* U3, double* core, double* sigma1, double* sigma2,
                     double* sigma3, double* err3, void* ws, size_t ws_bytes, void* stream, tucker_info* info);

/* ------------------------------------------------------------------------------------------
 * NEXT f2: SVD-accurate HOSVD (beats the Gram route's sqrt(eps) floor; P:557-561 takes the SVD
 * of each unfolding).  Per mode: the Gram route's p = min(n_m, r_m + 8, 56) leading eigenvectors
 * V, then `iters` (>= 1) Rayleigh–Ritz steps on F_(m) itself: Y = F_(m)^T V, Q = CGS2(Y),
 * B = F_(m) Q, U~ Sigma = one-sided-Jacobi SVD of B, V = U~ (no Gram, so singular values are
 * resolved down to ~eps sigma_1 instead of ~1e-8 sigma_1).  Outputs as tucker_hosvd (sigma_m from
 * the SVD of B).  Requires n_m <= 2048, r_m <= 56.  Workspace >= tucker_workspace_size_accurate. */
TUCKER_API size_t tucker_workspace_size_accurate(const tucker_grid* grid, const int32_t r[3]);
TUCKER_API int tucker_hosvd_accurate(const tucker_grid* grid, const int32_t r[3], const double* F, double* U1,
                          double* U2, double* U3, double* core, double* sigma1, double* sigma2, double* sigma3,
                          int32_t iters, void* ws, size_t ws_bytes, void* stream, tucker_info* info);

/* ------------------------------------------------------------------------------------------
 * Multigrid Tucker (the paper's alternative whose cost is linear in the tensor size):
 * the function tensor of (grid, kernel) on a sequence of dyadically refined grids (n -> ceil(n/2)
 * per axis, the same box) from the coarsest level with every n_m <= n0 (never below r_m or 4
 * nodes) up to `grid`; HOSVD only at the coarsest level; at each finer level the previous level's
 * factor columns are interpolated to the new nodes (4-point Lagrange in the node coordinate),
 * orthonormalised (one-sided Jacobi SVD) and refined by `sweeps` (>= 1) Tucker-ALS sweeps on that
 * level's tensor (tucker_als).  F (dev, n1 x n2 x n3) receives the finest tensor (the call fills
 * it); outputs as tucker_als (U_m, core, sigma_m of the last single-hole unfoldings).
 * levels_out (host, nullable) <- the number of levels.  Workspace >= tucker_workspace_size_multigrid.
 * Errors: INVALID_ARG (null, sweeps < 1, n0 < 4), DOMAIN, RANK, SIZE, UNSUPPORTED (r_m > 56, r_2 or
 * r_3 > 64), NOCONV (best iterate), CUDA. */
TUCKER_API size_t tucker_workspace_size_multigrid(const tucker_grid* grid, const int32_t r[3], int32_t n0);
TUCKER_API int tucker_multigrid(const tucker_grid* grid, const tucker_kernel* kernel, const int32_t r[3], int32_t n0,
                     int32_t sweeps, double* F, double* U1, double* U2, double* U3, double* core, double* sigma1,
                     double* sigma2, double* sigma3, void* ws, size_t ws_bytes, void* stream, tucker_info* info,
                     int32_t* levels_out);

/* Number of kernel launches enqueued by this thread's most recent entry-point call. */
/* Opt-in per-stage device timing: while enabled, CUDA events are recorded on the launching stream
 * around each stage's launches (off by default: no events, no overhead).  tucker_profile_read
 * synchronises the recorded events, writes the total milliseconds and the number of timed calls of
 * each stage into ms[TUCKER_PROF_NSTAGES] / count[TUCKER_PROF_NSTAGES] (host) and clears them. */
enum {
    TUCKER_PROF_FILL = 0,
    TUCKER_PROF_I8_ROWMAX = 1,   /* INT8 Gram: row maxima of the three unfoldings            */
    TUCKER_PROF_I8_RESIDUES = 2, /* INT8 Gram: scaled rounding + residues mod 16 moduli       */
    TUCKER_PROF_I8_GEMM = 3,     /* INT8 Gram: tcgen05 kind::i8 residue Grams (k_i8_gemm)     */
    TUCKER_PROF_I8_CRT = 4,      /* INT8 Gram: chunk fold + Chinese-remainder reconstruction  */
    TUCKER_PROF_DMMA_GRAM = 5,   /* DMMA Gram (k_gram_tma / k_gram + reduction)                */
    TUCKER_PROF_EIG = 6,
    TUCKER_PROF_TTM = 7,
    TUCKER_PROF_ERROR = 8,
    TUCKER_PROF_NSTAGES = 9
};
TUCKER_API int tucker_profile_enable(int32_t on);
TUCKER_API int tucker_profile_read(double* ms, int64_t* count);

TUCKER_API int64_t tucker_last_launch_count(void);

TUCKER_API const char* tucker_strerror(int code);

#ifdef __cplusplus
}
#endif
#endif /* TUCKER_B200_H */
