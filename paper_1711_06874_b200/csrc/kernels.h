// kernels.h — internal launch interfaces between api.cu and the kernel files (not exported).
#pragma once

#include <algorithm>
#include <functional>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/tucker.h"

namespace tk {

// K_nu Chebyshev table: dyadic intervals [2^j, 2^{j+1}), j = kChebJmin .. kChebJmin+kChebIntervals-1
constexpr int kChebN = 21;  // degree 20
constexpr int kChebJmin = -16;
constexpr int kChebIntervals = 25;  // z in [2^-16, 2^9)

// Point-kernel parameters (a-2; fill_eval.cuh evaluates them).
struct KParams {
    int family;
    int closed;  // 0 general, 1: nu=1/2, 2: nu=3/2, 3: nu=5/2
    int centred; // lo = -hi on every axis (set by the caller from the grid)
    double sigma2, ell, sqrt2nu, lambda, p, nu, pref;
    double alpha2, mexp;  // spectral density: alpha^2 and -(nu + 3/2)
};

// Plane chunk of F for the fused paths (a-7; layout and generation in fill_eval.cuh).
struct ChunkGeo {
    int pa;
    int mirror;
    int64_t n1, n2, n3;
    int64_t g0, Pc, np;
};

int launch_fill(const tucker_grid& g, const tucker_kernel& k, double* F, double* nodes_x2,
                double* cheb, cudaStream_t st, uint32_t* mx = nullptr);
// fill + row maxima (launch_fill with mx) is available on centred grids with n3 % 8 == 0, n3 <= 8192
bool fill_rowmax_supported(const tucker_grid& g);

// Gram G_m (n_m x n_m, both triangles) of the mode-m unfolding of F.
size_t gram_ws_bytes(const int64_t n[3]);
int launch_gram(const int64_t n[3], int mode, const double* F, double* G, void* ws, size_t ws_bytes,
                cudaStream_t st);

// a-3 on the INT8 tensor cores (gram_i8.cu): modular emulation of the FP64 Gram.
bool gram_i8_supported(const int64_t n[3]);
int gram_i8_scheme(int64_t K, int32_t* moduli, int32_t* b);
size_t gram_i8_ws_bytes(const int64_t n[3]);
// Row maxima of the three unfoldings (n1 + n2 + n3 u64 bit patterns of non-negative doubles).
int launch_gram_i8_rowmax(const int64_t n[3], const double* F, uint32_t* mx, cudaStream_t st);
// mx: row maxima from launch_gram_i8_rowmax, or nullptr (computed into the workspace).
int launch_gram_i8(const int64_t n[3], int mode, const double* F, double* G, const uint32_t* mx,
                   void* ws, size_t ws_bytes, cudaStream_t st);
// The three Grams through one pipeline (residues of the next job overlap the current int8 GEMM);
// after_mode(m) runs on `st` once G_m is complete (e.g. the eigensolver).  ws: gram_i8_ws_bytes,
// disjoint from anything after_mode uses.
int launch_gram_i8_modes(const int64_t n[3], const double* F, double* G, void* ws, size_t ws_bytes, cudaStream_t st,
                         const std::function<int(int)>& after_mode);
// Row (e): one fused HOSVD sharded over `count` ranks.  Work units (residue super-chunks of a
// mode's unfolding, i-slab chunks of the core and the error) go round-robin to the ranks; the
// partial results are exact integer residue sums (Grams) or sums with zeros off the owner
// (T2 rows, error partials), combined by the caller's all-reduce — so every rank ends with the
// bitwise result of the single-GPU call.  allreduce(ptr, count, dtype, op) runs after the stream
// has been synchronised (dtype TUCKER_DT_*, op TUCKER_RED_*).
struct Shard {
    int index = 0, count = 1;
    std::function<int(void*, int64_t, int, int)> allreduce;
    bool owns(int64_t unit) const { return count <= 1 || unit % count == index; }
    bool sharded() const { return count > 1; }
};

// a-7 with the INT8 Gram (F never stored): generator of the plane chunks.
struct I8Gen {
    KParams kp;
    const double* cheb;
    const double* x2;
};
bool gram_i8_fused_supported(const int64_t n[3]);
size_t gram_i8_fused_ws_bytes(const int64_t n[3]);
int launch_gram_i8_fused_modes(const int64_t n[3], const I8Gen& gen, double* G, void* ws, size_t ws_bytes,
                               cudaStream_t st, int m_first, int m_last, const std::function<int(int)>& after_mode,
                               const Shard* shard = nullptr);
// Device int of the INT8 workspace: 1 if an input value fell outside the scheme window (stale
// row maxima or non-finite F; the Gram is then NaN), reset at the start of every Gram call.
const int* gram_i8_flag_slot(const int64_t n[3], const void* ws);
// Moduli per mode of the INT8 Grams formed in ws (shared layout: k_i8_nmod's device slots, copied
// asynchronously on st — valid after the stream synchronises; per-mode layout: 16).
int gram_i8_moduli(const int64_t n[3], const void* ws, int32_t* out, cudaStream_t st);
// prep: 0 nothing precomputed; 1 the row maxima are already in the workspace's slot
// (gram_i8_rowmax_slot; e.g. written by the fill) — the row-maxima pass is skipped; 2 the shared
// layout's residues and global exponent are already in the workspace (launch_fill_prepare of this
// F) — the row-maxima and residue passes are skipped.
int launch_gram_i8_hosvd(const int64_t n[3], const double* F, double* const G[3], void* ws, size_t ws_bytes,
                         cudaStream_t st, const std::function<int(const int*, int)>& on_phase, int prep = 0);
// The fill and the shared residues in one octant pass (centred grid, n3 % 16 == 0, shared layout):
// F, the global exponent and the residue planes of the INT8 workspace i8ws (gram_i8_hosvd_ws_bytes).
bool fill_prepare_supported(const tucker_grid& g);
int launch_fill_prepare(const tucker_grid& g, const tucker_kernel& kn, double* F, double* nodes_x2, double* cheb,
                        void* i8ws, size_t i8ws_bytes, cudaStream_t st);
size_t gram_i8_hosvd_ws_bytes(const int64_t n[3]);
uint32_t* gram_i8_rowmax_slot(const int64_t n[3], void* ws);
// Per-device non-blocking side streams of the library (which = 0, 1, 2; created once per thread).
cudaStream_t side_stream(int which);
// Engine selection (tucker_set_gram_engine): TUCKER_GRAM_AUTO / _DMMA / _INT8.
int& gram_engine();
// TTM engine of the INT8 hosvd route (tucker_set_ttm_engine): TUCKER_TTM_AUTO / _DMMA.
int& ttm_engine();
// a-5 with T1 = F x3 U3^T on the INT8 tensor cores (ttm_i8.cu, R22): T2 out; UNSUPPORTED
// when the shape does not apply or `region` is too small (the caller then runs the DMMA TTM).
bool ttm_i8_applies(const int64_t n[3], const int32_t r[3], const double* F);
size_t ttm_i8_region_bytes(const int64_t n[3], const int32_t r[3]);
int launch_ttm12_i8(const int64_t n[3], const int32_t r[3], const double* F, const double* U2, const double* U3,
                    const uint32_t* gmax, double* T2, void* region, size_t region_bytes, cudaStream_t st,
                    int reserve_sms = 0, bool profile = true);
// INT8 TTM context for the fused route's slab chunks (launch_ttm_core_impl): the route's global
// exponent word and a free device region.
struct TtmI8 {
    const uint32_t* gmax;
    void* region;
    size_t bytes;
};
bool gram_i8_fused_ttm_scratch(const int64_t n[3], void* ws, const uint32_t** gmax, void** region, size_t* bytes);
// The INT8 shared route's global exponent word (and its residue region): false when the
// materialised Grams do not use the shared layout.
// a-6 with the reconstruction W U3^T on the INT8 tensor cores (err_i8.cu, R23); UNSUPPORTED
// when the shape does not apply or ws is too small (the caller then runs the DMMA error pass).
bool err_i8_applies(const int64_t n[3], const int32_t r[3], const double* F);
size_t err_i8_ws_bytes(const int64_t n[3], const int32_t r[3]);
int launch_error_i8(const int64_t n[3], const int32_t r[3], const double* F, const double* U1, const double* U2,
                    const double* U3, const double* core, double* out3, void* ws, size_t ws_bytes, cudaStream_t st);
bool gram_i8_ttm_scratch(const int64_t n[3], void* ws, const uint32_t** gmax, void** region, size_t* bytes);
bool gram_use_i8(const int64_t n[3]);
// Materialised INT8 Grams of this grid use the shared residue layout (one residue pass, one global
// exponent; R20) — and its integer width b.
bool gram_i8_shared_layout(const int64_t n[3]);
int gram_i8_shared_bits(const int64_t n[3]);
size_t gram_auto_ws_bytes(const int64_t n[3]);
int launch_gram_auto(const int64_t n[3], int mode, const double* F, double* G, const uint32_t* mx,
                     void* ws, size_t ws_bytes, cudaStream_t st);

// a-7 fused generate-and-Gram (F never materialised).  KParams / ChunkGeo: fill_eval.cuh.
struct FusedGramPlan {
    int pa;              // plane axis of the chunks (0: i-planes, 1: j-planes)
    int T, S;            // output tiles, split-K factor (T*S <= SMs: one cooperative wave)
    int64_t np, Pc;      // planes on that axis, planes per chunk
    int64_t nchunks;
    size_t slot_elems;   // doubles per ring slot (two slots)
    size_t part_bytes;   // split-K partials
};
FusedGramPlan fused_gram_plan(const int64_t n[3], int mode);
int64_t fused_chunk_target(int64_t dflt);  // TUCKER_FUSED_CHUNK_KB test override
int launch_gram_fused(const int64_t n[3], int mode, const KParams& kp, const double* cheb, const double* x2,
                      double* ring, double* part, unsigned int* bar, double* G, cudaStream_t st);

// Top-r eigenpairs of a symmetric PSD n x n matrix (dev).  iters/resid/... reported in `info`
// slot `slot`.
size_t eig_ws_bytes(int64_t n, int r);
// Split form: begin enqueues the first pass without host synchronisation, end synchronises,
// continues while not converged and reports (launch_eig = begin + end).
// V0 (dev, n x r row-major, nullable): warm start (Tucker-ALS: the previous factor) — the start
// block is [V0, pseudo-random columns] and the power steps before the first Rayleigh–Ritz step are
// skipped (V0 already spans the target subspace approximately; convergence is still decided by
// the Ritz residuals).
bool eig_rank_supported(int64_t n, int r);  // r <= 56 unless n is small enough for the direct Jacobi
int launch_eig_begin(int64_t n, const double* G, int r, double* U, double* lambda, double* sigma, void* ws,
                     size_t ws_bytes, cudaStream_t st, const double* V0 = nullptr);
int launch_eig_end(int64_t n, const double* G, int r, double* U, double* lambda, double* sigma, void* ws,
                   cudaStream_t st, tucker_info* info, int slot);
// Asynchronous completion of launch_eig_begin (no host synchronisation): enqueues the remaining
// iterations (each exits at once after convergence).  Convergence is not reported.
int launch_eig_rest(int64_t n, const double* G, int r, double* U, double* lambda, double* sigma, void* ws,
                    cudaStream_t st);
int launch_eig(int64_t n, const double* G, int r, double* U, double* lambda, double* sigma,
               void* ws, size_t ws_bytes, cudaStream_t st, tucker_info* info, int slot, const double* V0 = nullptr);

// Cluster Rayleigh–Ritz step (eig_cluster.cu); n <= 2048.
bool eig_cluster_supported(int64_t n);
int eig_cluster_size(int64_t n);
// G (nullable): W = G V formed inside the cluster kernel (Wt unused) — one launch per iteration.
int launch_rr_cluster(int64_t n, int p, int r, int it, int last, int orth_only, double* Vt, const double* Wt,
                      double* U, double* lambda, double* sigma, void* state, cudaStream_t st,
                      const double* G = nullptr);

// NEXT f2: left singular vectors of B (n x p, n <= 2048, p <= 64) by one-sided Jacobi in a cluster.
int launch_svd_cluster(int64_t n, int p, int r, const double* B, double* Vout, double* U, double* sigma,
                       int* sweeps_out, cudaStream_t st);

// Multigrid Tucker (multigrid.cu): Uf (nf x r) <- cubic interpolation of Uc's columns from the nc
// nodes to the nf nodes of [lo, hi] (xbuf: nc + nf doubles of scratch).
int launch_prolong(const double* Uc, int64_t nc, double lo, double hi, double* Uf, int64_t nf, int r, double* xbuf,
                   cudaStream_t st);

// NEXT f2: Rayleigh–Ritz steps on F_(m) from the Gram route's V (refine.cu).
size_t refine_ws_bytes(const int64_t n[3], int p);
int launch_refine_mode(const int64_t n[3], int m, const double* F, const double* V0, const double* lam0, int p,
                       int r, int iters, double* U, double* sigma, void* ws, size_t ws_bytes, cudaStream_t st,
                       int* sweeps_out);
// V (n x p) <- [U (n x r) | p - r deterministic pseudo-random columns] (ALS start basis).
int launch_seed_from_factors(double* V, const double* U, int64_t n, int r, int p, cudaStream_t st);

// Core beta = F x1 U1^T x2 U2^T x3 U3^T.
size_t ttm_ws_bytes(const int64_t n[3], const int32_t r[3]);
int launch_ttm_core(const int64_t n[3], const int32_t r[3], const double* F, const double* U1,
                    const double* U2, const double* U3, double* core, void* ws, size_t ws_bytes,
                    cudaStream_t st);

// Fused (F never materialised) variants of the core and the error: F is generated as chunks of
// Pc i-slabs ([Pc][n2][n3], fill_eval.cuh) into the head of the workspace.
struct FusedGen {
    ChunkGeo geo;  // pa = 0; g0/Pc set per chunk
    KParams kp;
    const double* cheb;
    const double* x2;
    int64_t Pc;
};
int launch_ttm_core_impl(const int64_t n[3], const int32_t r[3], const double* F, const FusedGen* gen,
                         const double* U1, const double* U2, const double* U3, double* core, void* ws,
                         size_t ws_bytes, cudaStream_t st, double* t1_out = nullptr, double* t2_out = nullptr,
                         const Shard* shard = nullptr, const TtmI8* i8 = nullptr);
// Tucker-ALS (f1): T1 = F x3 U3^T ((n1 n2) x r3) and Y1 = T1 x2 U2^T (n1 x r2 x r3), both stored.
int launch_ttm_t1_y1(const int64_t n[3], const int32_t r[3], const double* F, const double* U2, const double* U3,
                     double* T1, double* Y1, void* ws, size_t ws_bytes, cudaStream_t st);
int launch_error_impl(const int64_t n[3], const int32_t r[3], const double* F, const FusedGen* gen, const double* U1,
                      const double* U2, const double* U3, const double* core, double* out3, void* ws, size_t ws_bytes,
                      cudaStream_t st, const Shard* shard = nullptr);
size_t err_ws_bytes_slabs(const int64_t n[3], const int32_t r[3], int64_t slabs);

// NEXT f1: Tucker-ALS sweeps from initial factors U (in/out); core and sigma of the last sweep.
size_t als_ws_bytes(const int64_t n[3], const int32_t r[3]);
int launch_als(const int64_t n[3], const int32_t r[3], const double* F, double* const U[3], double* core,
               double* const sigma[3], int sweeps, void* ws, size_t ws_bytes, cudaStream_t st, tucker_info* info);

// NEXT f3: symmetry-exploiting path on centred grids (sym.cu): the hot path on the weighted
// octant tensor, factors expanded to full length.  err3 (dev, nullable) <- {E, ||F||, ||F-Ft||}.
size_t sym_ws_bytes(const tucker_grid& g, const int32_t r[3]);
int launch_hosvd_sym(const tucker_grid& g, const tucker_kernel& kn, const int32_t r[3], double* const U[3],
                     double* core, double* const sigma[3], double* err3, void* ws, size_t ws_bytes, cudaStream_t st,
                     tucker_info* info);

// Relative Frobenius error {E, ||F||, ||F-Ft||}.
size_t err_ws_bytes(const int64_t n[3], const int32_t r[3]);
int launch_error(const int64_t n[3], const int32_t r[3], const double* F, const double* U1,
                 const double* U2, const double* U3, const double* core, double* out3, void* ws,
                 size_t ws_bytes, cudaStream_t st);

// Small strided batched GEMM (DFMA): C[b](M x N) = A[b](M x K) * B[b](K x N); element strides.
struct SmallGemm {
    int64_t M, N, K, batch;
    const double* A;
    int64_t sam, sak, sab;
    const double* B;
    int64_t sbk, sbn, sbb;
    double* C;
    int64_t scm, scn, scb;
    int sub;  // 0: C = A B;  1: C = C - A B
};
int launch_small_gemm(const SmallGemm& p, cudaStream_t st);
// The same for one long-K product with few output tiles: K split into slices (a batch into `scratch`),
// then summed in slice order (deterministic); the plain kernel when it does not apply.
int launch_small_gemm_splitk(const SmallGemm& p, double* scratch, size_t scratch_bytes, cudaStream_t st);
// Same contract on the FP64 tensor cores (gemm.cu) when the contraction is large; falls back to
// launch_small_gemm for small ones.
int launch_gemm(const SmallGemm& p, cudaStream_t st);

}  // namespace tk
