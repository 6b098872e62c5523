// api.cu — the extern "C" boundary declared in include/tucker.h: argument validation,
// workspace planning, stage orchestration on the caller's stream.  Host C++ only; every step of
// the numerical path runs in the kernels of fill.cu / gram.cu / eig.cu / ttm.cu.
#include <cmath>
#include <cstring>

#include "common.cuh"
#include "fill_eval.cuh"
#include "kernels.h"
#include "prof.h"

#include <cstdio>
#include <cstdlib>

namespace tk {

int64_t& launch_counter() {
    static thread_local int64_t c = 0;
    return c;
}

int report_cuda(cudaError_t e, const char* file, int line) {
    static const bool dbg = std::getenv("TUCKER_DEBUG") != nullptr;
    if (dbg) std::fprintf(stderr, "tucker: CUDA error at %s:%d: %s\n", file, line, cudaGetErrorString(e));
    return TUCKER_ERR_CUDA;
}

PFN_tmapEncodeTiled tmap_encoder() {
    static PFN_tmapEncodeTiled fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_tmapEncodeTiled>(p);
    }
    return fn;
}

bool make_tmap_f64(CUtensorMap* map, const void* base, int rank, const uint64_t* dims,
                   const uint64_t* strides_bytes, const uint32_t* box) {
    PFN_tmapEncodeTiled enc = tmap_encoder();
    if (!enc) return false;
    cuuint64_t d[5], s[4];
    cuuint32_t b[5], e[5];
    for (int i = 0; i < rank; ++i) {
        d[i] = dims[i];
        b[i] = box[i];
        e[i] = 1;
    }
    for (int i = 0; i + 1 < rank; ++i) s[i] = strides_bytes[i];
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, (cuuint32_t)rank, const_cast<void*>(base), d, s, b, e,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

namespace {

int check_grid(const tucker_grid* g) {
    if (!g) return TUCKER_ERR_INVALID_ARG;
    for (int a = 0; a < 3; ++a) {
        if (g->n[a] < 2) return TUCKER_ERR_INVALID_ARG;
        if (!(g->lo[a] < g->hi[a]) || !std::isfinite(g->lo[a]) || !std::isfinite(g->hi[a]))
            return TUCKER_ERR_INVALID_ARG;
        if (g->n[a] > (int64_t)1 << 20) return TUCKER_ERR_SIZE;
    }
    const double N = (double)g->n[0] * (double)g->n[1] * (double)g->n[2];
    if (N * 8.0 > 9.0e18) return TUCKER_ERR_SIZE;
    return TUCKER_OK;
}

int check_kernel(const tucker_kernel* k) {
    if (!k) return TUCKER_ERR_INVALID_ARG;
    if (!(k->sigma2 > 0.0) || !std::isfinite(k->sigma2)) return TUCKER_ERR_DOMAIN;
    if (k->family == TUCKER_MATERN) {
        if (!(k->nu > 0.0) || !(k->ell > 0.0) || !std::isfinite(k->nu) || !std::isfinite(k->ell))
            return TUCKER_ERR_DOMAIN;
        if (k->nu > 50.0) return TUCKER_ERR_DOMAIN;
        return TUCKER_OK;
    }
    if (k->family == TUCKER_SLATER) {
        if (!(k->lambda > 0.0) || !(k->p > 0.0) || !(k->p <= 2.0) || !std::isfinite(k->lambda))
            return TUCKER_ERR_DOMAIN;
        return TUCKER_OK;
    }
    if (k->family == TUCKER_MATERN_SPECTRAL) {
        if (!(k->lambda > 0.0) || !(k->nu > 0.0) || !std::isfinite(k->lambda) || !std::isfinite(k->nu))
            return TUCKER_ERR_DOMAIN;
        return TUCKER_OK;
    }
    return TUCKER_ERR_INVALID_ARG;
}

int check_ranks(const tucker_grid* g, const int32_t* r) {
    if (!r) return TUCKER_ERR_INVALID_ARG;
    for (int a = 0; a < 3; ++a)
        if (r[a] < 1 || r[a] > g->n[a]) return TUCKER_ERR_RANK;
    return TUCKER_OK;
}

// Workspace layout (all 256-byte aligned):
//   [nodes x^2 (n1+n2+n3)] [K_nu table] [G (max n_m^2)] [row maxima (n1+n2+n3), INT8 Gram]
//   [scratch = max(gram, eig, ttm, err)] [device outputs of tucker_approximate: U1 U2 U3 core
//   sigma1..3 err3]
struct Layout {
    size_t nodes, cheb, G, i8, i8_bytes, eig, eig_bytes, t2, scratch, outs, total;
    size_t scratch_bytes, g_bytes;
};

Layout plan(const tucker_grid* g, const int32_t* rin) {
    int32_t r[3];
    for (int a = 0; a < 3; ++a) r[a] = rin ? rin[a] : (int32_t)std::min<int64_t>(g->n[a], 56);
    const int64_t* n = g->n;
    Layout L{};
    size_t off = 0;
    L.nodes = off;
    off += align_up((size_t)(n[0] + n[1] + n[2]) * 8, 256);
    L.cheb = off;
    off += align_up((size_t)kChebIntervals * kChebN * 8, 256);
    L.G = off;
    const int64_t nmax = std::max(n[0], std::max(n[1], n[2]));
    L.g_bytes = align_up((size_t)nmax * nmax * 8, 256);
    off += (gram_use_i8(n) ? 3 : 1) * L.g_bytes;  // INT8 route: one G per mode (eigensolves overlap)
    const bool i8 = gram_use_i8(n);
    L.i8 = off;
    L.i8_bytes = i8 ? align_up(gram_i8_hosvd_ws_bytes(n), 1024) : 0;  // INT8 Gram pipeline (own region)
    off += L.i8_bytes;
    if (i8) {  // the eigensolves run beside the Grams and the core's first two products: own regions
        size_t e = 0;
        for (int a = 0; a < 3; ++a) e = std::max(e, eig_ws_bytes(n[a], r[a]));
        L.eig = off;
        L.eig_bytes = align_up(e, 256);
        off += 3 * L.eig_bytes;  // one per mode: the three eigensolves are in flight together
        L.t2 = off;
        off += align_up((size_t)n[0] * r[1] * r[2] * 8, 256);
    }
    L.scratch = off;
    size_t s = i8 ? 0 : gram_ws_bytes(n);
    if (!i8)
        for (int a = 0; a < 3; ++a) s = std::max(s, eig_ws_bytes(n[a], r[a]));
    s = std::max(s, ttm_ws_bytes(n, r));
    s = std::max(s, std::max(err_ws_bytes(n, r), err_i8_ws_bytes(n, r)));
    s = std::max(s, ttm_i8_region_bytes(n, r));  // the INT8 TTM's T1 / digit image / TTM2 partials
    L.scratch_bytes = align_up(s, 256);
    off += L.scratch_bytes;
    L.outs = off;
    size_t o = 0;
    for (int a = 0; a < 3; ++a) o += align_up((size_t)n[a] * r[a] * 8, 256) + align_up((size_t)r[a] * 8, 256);
    o += align_up((size_t)r[0] * r[1] * r[2] * 8, 256) + 256;
    off += o;
    L.total = off;
    return L;
}

inline char* at(void* ws, size_t off) { return static_cast<char*>(ws) + off; }

// Rank limits of the eigensolver and the core, checked before any launch (r_m <= n_m is
// check_ranks'): the subspace block needs r_m <= 56 once n_m exceeds the direct-Jacobi size, the
// core's fused TTM needs r_2, r_3 <= 64.
int check_hosvd_limits(const tucker_grid* g, const int32_t* r) {
    for (int a = 0; a < 3; ++a)
        if (!eig_rank_supported(g->n[a], r[a])) return TUCKER_ERR_UNSUPPORTED;
    if (r[1] > 64 || r[2] > 64) return TUCKER_ERR_UNSUPPORTED;
    return TUCKER_OK;
}

// info == nullptr: asynchronous (no host synchronisation, CUDA-Graph capturable; convergence and
// input-window failures are not reported — a failed input shows as NaN outputs).  info != nullptr:
// the eigensolves are completed with host synchronisations and reported, and the call returns
// TUCKER_ERR_INPUT if the INT8 route saw a value outside its window.
int hosvd_impl(const tucker_grid* g, const int32_t* r, const double* F, double* const U[3], double* core,
               double* const sig[3], void* ws, size_t ws_bytes, cudaStream_t st, tucker_info* info,
               int prep = 0) {
    const Layout L = plan(g, r);
    if (ws_bytes < L.total) return TUCKER_ERR_SIZE;
    TK_RC(check_hosvd_limits(g, r));
    const bool sync = info != nullptr;
    double* G = reinterpret_cast<double*>(at(ws, L.G));
    void* scr = at(ws, L.scratch);
    int worst = TUCKER_OK;
    auto eig_mode = [&](int m) -> int {
        if (!sync) {
            TK_RC(launch_eig_begin(g->n[m], G, r[m], U[m], nullptr, sig[m], scr, L.scratch_bytes, st));
            return launch_eig_rest(g->n[m], G, r[m], U[m], nullptr, sig[m], scr, st);
        }
        const int rc = launch_eig(g->n[m], G, r[m], U[m], nullptr, sig[m], scr, L.scratch_bytes, st, info, m);
        if (rc == TUCKER_ERR_NOCONV) worst = rc;
        else if (rc != TUCKER_OK) return rc;
        return TUCKER_OK;
    };
    if (L.i8_bytes) {
        // INT8-emulated Grams (row maxima once per F), modes in the order 2, 1, 0.  Each eigensolve
        // runs on a side stream while the next Gram runs on `st` (one G per mode; the eigensolver is
        // latency-bound on one cluster); the last one (mode 0: U1) runs beside the core's first two
        // products (which need U2, U3 only); the third product waits for it.
        // one side stream per mode (A: mode 2, C: mode 1, B: mode 0 beside TTM1 + TTM2): the
        // persistent int8 Gram holds every SM, so the solves of modes 2 and 1 mostly run after the
        // last Gram — side by side, not one after the other
        cudaStream_t sideA = side_stream(0), sideB = side_stream(1), sideC = side_stream(2);
        if (!sideA || !sideB || !sideC) return TUCKER_ERR_CUDA;
        cudaEvent_t ev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
        auto cleanup = [&]() {
            for (cudaEvent_t e : ev)
                if (e) cudaEventDestroy(e);
        };
        for (int i = 0; i < 6; ++i)
            if (cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming) != cudaSuccess) {
                cleanup();
                return TUCKER_ERR_CUDA;
            }
        double* Gm[3] = {G, reinterpret_cast<double*>(at(ws, L.G + L.g_bytes)),
                         reinterpret_cast<double*>(at(ws, L.G + 2 * L.g_bytes))};
        void* escr[3] = {at(ws, L.eig), at(ws, L.eig + L.eig_bytes), at(ws, L.eig + 2 * L.eig_bytes)};
        double* T2 = reinterpret_cast<double*>(at(ws, L.t2));
        auto side_of = [&](int m) { return m == 0 ? sideB : (m == 1 ? sideC : sideA); };
        auto eig_end = [&](int m) -> int {  // host waits for the solve (its first pass is long queued)
            if (!sync) return launch_eig_rest(g->n[m], Gm[m], r[m], U[m], nullptr, sig[m], escr[m], side_of(m));
            const int rc = launch_eig_end(g->n[m], Gm[m], r[m], U[m], nullptr, sig[m], escr[m], side_of(m), info, m);
            if (rc == TUCKER_ERR_NOCONV) worst = rc;
            else if (rc != TUCKER_OK) return rc;
            return TUCKER_OK;
        };
        // each eigensolve's first pass is enqueued as soon as its Gram is: it runs beside the next
        // Gram's residue kernels
        bool side_used = false;  // side-stream work enqueued: joined into `st` on every exit path
        int rc = launch_gram_i8_hosvd(g->n, F, Gm, at(ws, L.i8), L.i8_bytes, st, [&](const int* ms, int cnt) -> int {
            side_used = true;
            for (int i = 0; i < cnt; ++i) {
                const int m = ms[i];
                if (cudaEventRecord(ev[m], st) != cudaSuccess || cudaStreamWaitEvent(side_of(m), ev[m], 0) != cudaSuccess)
                    return TUCKER_ERR_CUDA;
                TK_RC(launch_eig_begin(g->n[m], Gm[m], r[m], U[m], nullptr, sig[m], escr[m], L.eig_bytes, side_of(m)));
            }
            return TUCKER_OK;
        }, prep);
        if (rc == TUCKER_OK) rc = eig_end(2);
        if (rc == TUCKER_OK) rc = eig_end(1);
        // U3 final on side A, U2 on side C -> TTM1 + TTM2 on `st`, beside the mode-0 eigensolve on side B
        if (rc == TUCKER_OK && (cudaEventRecord(ev[3], sideA) != cudaSuccess ||
                                cudaEventRecord(ev[5], sideC) != cudaSuccess ||
                                cudaStreamWaitEvent(st, ev[3], 0) != cudaSuccess ||
                                cudaStreamWaitEvent(st, ev[5], 0) != cudaSuccess))
            rc = TUCKER_ERR_CUDA;
        if (rc == TUCKER_OK) {  // TTM1 on the INT8 tensor cores where it applies (R22), else DMMA
            rc = TUCKER_ERR_UNSUPPORTED;
            const uint32_t* gm = nullptr;
            void* reg = nullptr;
            size_t rb = 0;
            // (its scratch is the general one, free here: the residue planes stay intact, so a prepared
            // workspace can serve another tucker_hosvd_prepared call)
            if (ttm_engine() != TUCKER_TTM_DMMA && gram_i8_ttm_scratch(g->n, at(ws, L.i8), &gm, &reg, &rb))
                // the mode-0 eigensolve runs beside it on side stream B: leave it its SMs (one CTA,
                // or one thread-block cluster per iteration)
                rc = launch_ttm12_i8(g->n, r, F, U[1], U[2], gm, T2, scr, L.scratch_bytes, st,
                                     g->n[0] <= 112 ? 1 : (eig_cluster_supported(g->n[0]) ? eig_cluster_size(g->n[0]) : 0));
            if (rc == TUCKER_ERR_UNSUPPORTED)
                rc = launch_ttm_core_impl(g->n, r, F, nullptr, nullptr, U[1], U[2], nullptr, scr, L.scratch_bytes, st,
                                          nullptr, T2);
        }
        if (rc == TUCKER_OK) rc = eig_end(0);
        if (rc == TUCKER_OK && (cudaEventRecord(ev[4], sideB) != cudaSuccess ||
                                cudaStreamWaitEvent(st, ev[4], 0) != cudaSuccess))
            rc = TUCKER_ERR_CUDA;
        if (rc != TUCKER_OK && side_used) {
            // an error after side-stream work was enqueued: `st` must not run ahead of it (the
            // caller may free U or ws once the stream is idle)
            cudaEventRecord(ev[3], sideA);
            cudaEventRecord(ev[4], sideB);
            cudaEventRecord(ev[5], sideC);
            cudaStreamWaitEvent(st, ev[3], 0);
            cudaStreamWaitEvent(st, ev[4], 0);
            cudaStreamWaitEvent(st, ev[5], 0);
        }
        cleanup();
        TK_RC(rc);
        // TTM3: core (r1 x r2 r3) = U1^T (r1 x n1) * T2 (n1 x r2 r3)
        SmallGemm g3{r[0], (int64_t)r[1] * r[2], g->n[0], 1, U[0], 1, r[0], 0, T2, (int64_t)r[1] * r[2], 1, 0, core,
                     (int64_t)r[1] * r[2], 1, 0};
        TK_RC(launch_small_gemm_splitk(g3, static_cast<double*>(scr), L.scratch_bytes, st));  // scr is free again
        if (sync) {  // input-window check of the INT8 route (stale row maxima, non-finite F)
            int bad = 0;
            TK_RC(gram_i8_moduli(g->n, at(ws, L.i8), info->moduli, st));
            TK_CUDA(cudaMemcpyAsync(&bad, gram_i8_flag_slot(g->n, at(ws, L.i8)), sizeof(int), cudaMemcpyDeviceToHost, st));
            TK_CUDA(cudaStreamSynchronize(st));
            if (bad) return TUCKER_ERR_INPUT;
        }
        return worst;
    } else {
        if (info)
            for (int m = 0; m < 3; ++m) info->moduli[m] = 0;  // FP64 DMMA Grams
        for (int m = 0; m < 3; ++m) {
            TK_RC(launch_gram(g->n, m, F, G, scr, L.scratch_bytes, st));
            TK_RC(eig_mode(m));
        }
    }
    TK_RC(launch_ttm_core(g->n, r, F, U[0], U[1], U[2], core, scr, L.scratch_bytes, st));
    return worst;
}

// ---------------------------------------------------------------- a-7 fused (F never stored)
// Slab chunk (i-planes) for the fused core / error passes: about 1 GiB, and at least two waves
// of k_ttm12 CTAs when the grid allows it.
int64_t fused_slab_chunk(const int64_t n[3]) {
    const int64_t plane = n[1] * n[2] * 8;
    const int64_t target = fused_chunk_target((int64_t)1 << 30);
    int64_t pc = std::max<int64_t>(1, target / plane);
    const int64_t jt = ceil_div(n[1], 256);
    if (target == ((int64_t)1 << 30)) pc = std::max<int64_t>(pc, ceil_div(2 * kNumSMs, jt));
    return std::min<int64_t>(pc, n[0]);
}

// Fused workspace: [nodes x^2][K_nu table][G][scratch]; scratch = max(fused Gram ring + partials
// + barrier, eigensolver, chunk + core, chunk + error).
struct FusedLayout {
    size_t nodes, cheb, G, i8, i8_bytes, scratch, total, scratch_bytes;
    int64_t pc_slab;
};

bool fused_use_i8(const int64_t n[3]) { return gram_use_i8(n) && gram_i8_fused_supported(n); }

FusedLayout plan_fused(const tucker_grid* g, const int32_t* rin) {
    int32_t r[3];
    for (int a = 0; a < 3; ++a) r[a] = rin ? rin[a] : (int32_t)std::min<int64_t>(g->n[a], 56);
    const int64_t* n = g->n;
    FusedLayout L{};
    size_t off = 0;
    L.nodes = off;
    off += align_up((size_t)(n[0] + n[1] + n[2]) * 8, 256);
    L.cheb = off;
    off += align_up((size_t)kChebIntervals * kChebN * 8, 256);
    L.G = off;
    const int64_t nmax = std::max(n[0], std::max(n[1], n[2]));
    off += align_up((size_t)nmax * nmax * 8, 1024);
    // INT8 Gram (F never stored): residues, chunk buffer, row maxima; its own region (the row
    // maxima live across the three modes and their eigensolves)
    L.i8 = off;
    L.i8_bytes = fused_use_i8(n) ? align_up(gram_i8_fused_ws_bytes(n), 1024) : 0;
    off += L.i8_bytes;
    L.scratch = off;
    size_t s = 0;
    for (int m = 0; m < 3; ++m) {
        if (!L.i8_bytes) {
            const FusedGramPlan fp = fused_gram_plan(n, m);
            s = std::max(s, 2 * align_up(fp.slot_elems * 8, 1024) + align_up(fp.part_bytes, 256) + 256);
        }
        s = std::max(s, eig_ws_bytes(n[m], r[m]));
    }
    L.pc_slab = fused_slab_chunk(n);
    const size_t chunk = align_up((size_t)L.pc_slab * n[1] * n[2] * 8, 256);
    s = std::max(s, chunk + ttm_ws_bytes(n, r));
    s = std::max(s, chunk + err_ws_bytes_slabs(n, r, L.pc_slab));
    L.scratch_bytes = align_up(s, 256);
    off += L.scratch_bytes;
    L.total = off;
    return L;
}

KParams fused_kparams(const tucker_grid* g, const tucker_kernel* k) {
    KParams kp = make_kparams(*k);
    kp.centred = grid_centred(*g) ? 1 : 0;
    return kp;
}

int fused_gram_into(const tucker_grid* g, int m, const KParams& kp, const FusedLayout& L, void* ws, double* G,
                    cudaStream_t st) {
    const FusedGramPlan fp = fused_gram_plan(g->n, m);
    char* scr = at(ws, L.scratch);
    double* ring = reinterpret_cast<double*>(scr);
    double* part = reinterpret_cast<double*>(scr + 2 * align_up(fp.slot_elems * 8, 1024));
    unsigned int* bar = reinterpret_cast<unsigned int*>(scr + 2 * align_up(fp.slot_elems * 8, 1024) +
                                                        align_up(fp.part_bytes, 256));
    return launch_gram_fused(g->n, m, kp, reinterpret_cast<const double*>(at(ws, L.cheb)),
                             reinterpret_cast<const double*>(at(ws, L.nodes)), ring, part, bar, G, st);
}

FusedGen fused_gen(const tucker_grid* g, const KParams& kp, const FusedLayout& L, void* ws) {
    FusedGen f{};
    f.geo.pa = 0;
    f.geo.mirror = (kp.centred && g->n[2] % 8 == 0) ? 1 : 0;
    f.geo.n1 = g->n[0];
    f.geo.n2 = g->n[1];
    f.geo.n3 = g->n[2];
    f.geo.np = g->n[0];
    f.geo.g0 = 0;
    f.geo.Pc = L.pc_slab;
    f.kp = kp;
    f.cheb = reinterpret_cast<const double*>(at(ws, L.cheb));
    f.x2 = reinterpret_cast<const double*>(at(ws, L.nodes));
    f.Pc = L.pc_slab;
    return f;
}

}  // namespace
}  // namespace tk

using namespace tk;

extern "C" {

size_t tucker_workspace_size(const tucker_grid* grid, const int32_t r[3]) {
    if (check_grid(grid) != TUCKER_OK) return 0;
    return plan(grid, r).total;
}

size_t tucker_workspace_size_fill(const tucker_grid* grid) {
    if (check_grid(grid) != TUCKER_OK) return 0;
    return plan(grid, nullptr).G;  // nodes + K_nu table (the leading regions of every layout)
}

int tucker_fill(const tucker_grid* grid, const tucker_kernel* kernel, double* F, void* ws, size_t ws_bytes,
                void* stream) {
    launch_counter() = 0;
    TK_RC(check_grid(grid));
    TK_RC(check_kernel(kernel));
    if (!F || !ws) return TUCKER_ERR_INVALID_ARG;
    const Layout L = plan(grid, nullptr);
    if (ws_bytes < L.G) return TUCKER_ERR_SIZE;
    return launch_fill(*grid, *kernel, F, reinterpret_cast<double*>(at(ws, L.nodes)),
                       reinterpret_cast<double*>(at(ws, L.cheb)), static_cast<cudaStream_t>(stream));
}

int tucker_fill_rowmax(const tucker_grid* grid, const tucker_kernel* kernel, double* F, uint32_t* rowmax, void* ws,
                       size_t ws_bytes, void* stream) {
    launch_counter() = 0;
    TK_RC(check_grid(grid));
    TK_RC(check_kernel(kernel));
    if (!F || !rowmax || !ws) return TUCKER_ERR_INVALID_ARG;
    if (!fill_rowmax_supported(*grid)) return TUCKER_ERR_UNSUPPORTED;
    const Layout L = plan(grid, nullptr);
    if (ws_bytes < L.G) return TUCKER_ERR_SIZE;
    return launch_fill(*grid, *kernel, F, reinterpret_cast<double*>(at(ws, L.nodes)),
                       reinterpret_cast<double*>(at(ws, L.cheb)), static_cast<cudaStream_t>(stream), rowmax);
}

int tucker_gram(const tucker_grid* grid, int32_t mode, const double* F, double* G, void* ws, size_t ws_bytes,
                void* stream) {
    launch_counter() = 0;
    TK_RC(check_grid(grid));
    if (mode < 0 || mode > 2 || !F || !G || !ws) return TUCKER_ERR_INVALID_ARG;
    return launch_gram_auto(grid->n, mode, F, G, nullptr, ws, ws_bytes, static_cast<cudaStream_t>(stream));
}

int tucker_set_gram_engine(int32_t engine) {
    if (engine != TUCKER_GRAM_AUTO && engine != TUCKER_GRAM_DMMA && engine != TUCKER_GRAM_INT8 &&
        engine != TUCKER_GRAM_INT8_ROWSCALED)
        return TUCKER_ERR_INVALID_ARG;
    gram_engine() = engine;
    return TUCKER_OK;
}

int32_t tucker_get_gram_engine(void) { return gram_engine(); }

int tucker_set_ttm_engine(int32_t engine) {
    if (engine != TUCKER_TTM_AUTO && engine != TUCKER_TTM_DMMA && engine != TUCKER_TTM_INT8_ERROR)
        return TUCKER_ERR_INVALID_ARG;
    ttm_engine() = engine;
    return TUCKER_OK;
}

int32_t tucker_get_ttm_engine(void) { return ttm_engine(); }

size_t tucker_workspace_size_i8(const tucker_grid* grid) {
    if (check_grid(grid) != TUCKER_OK || !gram_i8_supported(grid->n)) return 0;
    return gram_i8_ws_bytes(grid->n);
}

int tucker_i8_layout(const tucker_grid* grid, int32_t* shared, int32_t* b) {
    TK_RC(check_grid(grid));
    if (!shared || !b) return TUCKER_ERR_INVALID_ARG;
    if (!gram_use_i8(grid->n)) return TUCKER_ERR_UNSUPPORTED;
    *shared = gram_i8_shared_layout(grid->n) ? 1 : 0;
    int32_t mods[16];
    const int64_t* n = grid->n;
    const int64_t K0 = n[1] * n[2];
    if (*shared) {
        *b = gram_i8_shared_bits(n);
    } else {
        gram_i8_scheme(K0, mods, b);  // per mode: b of mode 0's K (each mode uses its own K)
    }
    return TUCKER_OK;
}

int tucker_i8_scheme(int64_t K, int32_t* moduli, int32_t* b) {
    if (K < 1 || !moduli || !b) return TUCKER_ERR_INVALID_ARG;
    return gram_i8_scheme(K, moduli, b);
}

int tucker_gram_i8(const tucker_grid* grid, int32_t mode, const double* F, double* G, void* ws, size_t ws_bytes,
                   void* stream) {
    launch_counter() = 0;
    TK_RC(check_grid(grid));
    if (mode < 0 || mode > 2 || !F || !G || !ws) return TUCKER_ERR_INVALID_ARG;
    if (!gram_i8_supported(grid->n)) return TUCKER_ERR_UNSUPPORTED;
    return launch_gram_i8(grid->n, mode, F, G, nullptr, ws, ws_bytes, static_cast<cudaStream_t>(stream));
}

int tucker_eig(int64_t n, const double* G, int32_t r, double* U, double* lambda, void* ws, size_t ws_bytes,
               void* stream, tucker_info* info_mode) {
    launch_counter() = 0;
    if (n < 1 || !G || !U || !ws) return TUCKER_ERR_INVALID_ARG;
    if (r < 1 || r > n) return TUCKER_ERR_RANK;
    return launch_eig(n, G, r, U, lambda, nullptr, ws, ws_bytes, static_cast<cudaStream_t>(stream), info_mode, 0);
}

int tucker_ttm_core(const tucker_grid* grid, const int32_t r[3], const double* F, const double* U1,
                    const double* U2, const double* U3, double* core, void* ws, size_t ws_bytes, void* stream) {
    launch_counter() = 0;
    TK_RC(check_grid(grid));
    TK_RC(check_ranks(grid, r));
    if (!F || !U1 || !U2 || !U3 || !core || !ws) return TUCKER_ERR_INVALID_ARG;
    if (r[2] > 64) return TUCKER_ERR_UNSUPPORTED;
    return launch_ttm_core(grid->n, r, F, U1, U2, U3, core, ws, ws_bytes, static_cast<cudaStream_t>(stream));
}

int tucker_hosvd(const tucker_grid* grid, const int32_t r[3], const double* F, double* U1, double* U2, double* U3,
                 double* core, double* sigma1, double* sigma2, double* sigma3, void* ws, size_t ws_bytes,
                 void* stream, tucker_info* info) {
    launch_counter() = 0;
    TK_RC(check_grid(grid));
    TK_RC(check_ranks(grid, r));
    if (!F || !U1 || !U2 || !U3 || !core || !sigma1 || !sigma2 || !sigma3 || !ws) return TUCKER_ERR_INVALID_ARG;
    if (info) std::memset(info, 0, sizeof(*info));
    double* const U[3] = {U1, U2, U3};
    double* const S[3] = {sigma1, sigma2, sigma3};
    return hosvd_impl(grid, r, F, U, core, S, ws, ws_bytes, static_cast<cudaStream_t>(stream), info);
}

int tucker_hosvd_rowmax(const tucker_grid* grid, const int32_t r[3], const double* F, const uint32_t* rowmax,
                        double* U1, double* U2, double* U3, double* core, double* sigma1, double* sigma2,
                        double* sigma3, void* ws, size_t ws_bytes, void* stream, tucker_info* info) {
    launch_counter() = 0;
    TK_RC(check_grid(grid));
    TK_RC(check_ranks(grid, r));
    if (!F || !U1 || !U2 || !U3 || !core || !sigma1 || !sigma2 || !sigma3 || !ws) return TUCKER_ERR_INVALID_ARG;
    if (info) std::memset(info, 0, sizeof(*info));
    double* const U[3] = {U1, U2, U3};
    double* const S[3] = {sigma1, sigma2, sigma3};
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const Layout L = plan(grid, r);
    if (ws_bytes < L.total) return TUCKER_ERR_SIZE;
    const bool use = rowmax && L.i8_bytes;
    if (use)
        TK_CUDA(cudaMemcpyAsync(gram_i8_rowmax_slot(grid->n, at(ws, L.i8)), rowmax,
                                (size_t)(grid->n[0] + grid->n[1] + grid->n[2]) * 4, cudaMemcpyDeviceToDevice, st));
    return hosvd_impl(grid, r, F, U, core, S, ws, ws_bytes, st, info, use);
}

int tucker_fill_prepare(const tucker_grid* grid, const tucker_kernel* kernel, const int32_t r[3], double* F, void* ws,
                        size_t ws_bytes, void* stream) {
    launch_counter() = 0;
    TK_RC(check_grid(grid));
    TK_RC(check_kernel(kernel));
    TK_RC(check_ranks(grid, r));
    if (!F || !ws) return TUCKER_ERR_INVALID_ARG;
    const Layout L = plan(grid, r);
    if (ws_bytes < L.total) return TUCKER_ERR_SIZE;
    if (!L.i8_bytes || !fill_prepare_supported(*grid)) return TUCKER_ERR_UNSUPPORTED;
    return launch_fill_prepare(*grid, *kernel, F, reinterpret_cast<double*>(at(ws, L.nodes)),
                               reinterpret_cast<double*>(at(ws, L.cheb)), at(ws, L.i8), L.i8_bytes,
                               static_cast<cudaStream_t>(stream));
}

int tucker_hosvd_prepared(const tucker_grid* grid, const int32_t r[3], const double* F, double* U1, double* U2,
                          double* U3, double* core, double* sigma1, double* sigma2, double* sigma3, void* ws,
                          size_t ws_bytes, void* stream, tucker_info* info) {
    launch_counter() = 0;
    TK_RC(check_grid(grid));
    TK_RC(check_ranks(grid, r));
    if (!F || !U1 || !U2 || !U3 || !core || !sigma1 || !sigma2 || !sigma3 || !ws) return TUCKER_ERR_INVALID_ARG;
    const Layout L = plan(grid, r);
    if (ws_bytes < L.total) return TUCKER_ERR_SIZE;
    if (!L.i8_bytes || !fill_prepare_supported(*grid)) return TUCKER_ERR_UNSUPPORTED;
    if (info) std::memset(info, 0, sizeof(*info));
    double* const U[3] = {U1, U2, U3};
    double* const S[3] = {sigma1, sigma2, sigma3};
    return hosvd_impl(grid, r, F, U, core, S, ws, ws_bytes, static_cast<cudaStream_t>(stream), info, 2);
}

int tucker_error(const tucker_grid* grid, const int32_t r[3], const double* F, const double* U1, const double* U2,
                 const double* U3, const double* core, double* out3, void* ws, size_t ws_bytes, void* stream) {
    launch_counter() = 0;
    TK_RC(check_grid(grid));
    TK_RC(check_ranks(grid, r));
    if (!F || !U1 || !U2 || !U3 || !core || !out3 || !ws) return TUCKER_ERR_INVALID_ARG;
    return launch_error(grid->n, r, F, U1, U2, U3, core, out3, ws, ws_bytes, static_cast<cudaStream_t>(stream));
}

int tucker_approximate(const tucker_grid* grid, const tucker_kernel* kernel, const int32_t r[3], double* F,
                       double* const U_h[3], double* core_h, double* const sigma_h[3], double* err_h, void* ws,
                       size_t ws_bytes, void* stream, tucker_info* info) {
    launch_counter() = 0;
    TK_RC(check_grid(grid));
    TK_RC(check_kernel(kernel));
    TK_RC(check_ranks(grid, r));
    if (!F || !U_h || !core_h || !sigma_h || !err_h || !ws) return TUCKER_ERR_INVALID_ARG;
    for (int a = 0; a < 3; ++a)
        if (!U_h[a] || !sigma_h[a]) return TUCKER_ERR_INVALID_ARG;
    const Layout L = plan(grid, r);
    if (ws_bytes < L.total) return TUCKER_ERR_SIZE;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (info) std::memset(info, 0, sizeof(*info));
    // device outputs live in the tail of the workspace
    char* o = at(ws, L.outs);
    double *Ud[3], *Sd[3];
    for (int a = 0; a < 3; ++a) {
        Ud[a] = reinterpret_cast<double*>(o);
        o += align_up((size_t)grid->n[a] * r[a] * 8, 256);
        Sd[a] = reinterpret_cast<double*>(o);
        o += align_up((size_t)r[a] * 8, 256);
    }
    double* cored = reinterpret_cast<double*>(o);
    o += align_up((size_t)r[0] * r[1] * r[2] * 8, 256);
    double* errd = reinterpret_cast<double*>(o);

    // on centred grids the fill also writes the INT8 route's inputs: the shared residues (one octant
    // pass, R20) or at least the row maxima — one or two passes over F fewer
    int prep = 0;
    if (L.i8_bytes && fill_prepare_supported(*grid)) {
        TK_RC(launch_fill_prepare(*grid, *kernel, F, reinterpret_cast<double*>(at(ws, L.nodes)),
                                  reinterpret_cast<double*>(at(ws, L.cheb)), at(ws, L.i8), L.i8_bytes, st));
        prep = 2;
    } else {
        const bool mx_fused = L.i8_bytes && fill_rowmax_supported(*grid);
        TK_RC(launch_fill(*grid, *kernel, F, reinterpret_cast<double*>(at(ws, L.nodes)),
                          reinterpret_cast<double*>(at(ws, L.cheb)), st,
                          mx_fused ? gram_i8_rowmax_slot(grid->n, at(ws, L.i8)) : nullptr));
        prep = mx_fused ? 1 : 0;
    }
    const int64_t c0 = launch_counter();
    const int rc = hosvd_impl(grid, r, F, Ud, cored, Sd, ws, ws_bytes, st, info, prep);
    if (rc != TUCKER_OK && rc != TUCKER_ERR_NOCONV) return rc;
    const int64_t c1 = launch_counter();
    (void)c0;
    (void)c1;
    TK_RC(launch_error(grid->n, r, F, Ud[0], Ud[1], Ud[2], cored, errd, at(ws, L.scratch), L.scratch_bytes, st));
    for (int a = 0; a < 3; ++a) {
        TK_CUDA(cudaMemcpyAsync(U_h[a], Ud[a], (size_t)grid->n[a] * r[a] * 8, cudaMemcpyDeviceToHost, st));
        TK_CUDA(cudaMemcpyAsync(sigma_h[a], Sd[a], (size_t)r[a] * 8, cudaMemcpyDeviceToHost, st));
    }
    TK_CUDA(cudaMemcpyAsync(core_h, cored, (size_t)r[0] * r[1] * r[2] * 8, cudaMemcpyDeviceToHost, st));
    TK_CUDA(cudaMemcpyAsync(err_h, errd, 3 * 8, cudaMemcpyDeviceToHost, st));
    TK_CUDA(cudaStreamSynchronize(st));
    return rc;
}

size_t tucker_workspace_size_fused(const tucker_grid* grid, const int32_t r[3]) {
    if (check_grid(grid) != TUCKER_OK) return 0;
    return plan_fused(grid, r).total;
}

int tucker_gram_fused(const tucker_grid* grid, const tucker_kernel* kernel, int32_t mode, double* G, void* ws,
                      size_t ws_bytes, void* stream) {
    launch_counter() = 0;
    TK_RC(check_grid(grid));
    TK_RC(check_kernel(kernel));
    if (mode < 0 || mode > 2 || !G || !ws) return TUCKER_ERR_INVALID_ARG;
    const int32_t r1[3] = {1, 1, 1};  // the Gram alone: no rank-dependent scratch
    const FusedLayout L = plan_fused(grid, r1);
    if (ws_bytes < L.total) return TUCKER_ERR_SIZE;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const KParams kp = fused_kparams(grid, kernel);
    TK_RC(launch_fill_prep(*grid, *kernel, kp, reinterpret_cast<double*>(at(ws, L.nodes)),
                           reinterpret_cast<double*>(at(ws, L.cheb)), st));
    if (L.i8_bytes) {
        const I8Gen gen{kp, reinterpret_cast<const double*>(at(ws, L.cheb)),
                        reinterpret_cast<const double*>(at(ws, L.nodes))};
        return launch_gram_i8_fused_modes(grid->n, gen, G, at(ws, L.i8), L.i8_bytes, st, mode, mode,
                                          [](int) { return (int)TUCKER_OK; });
    }
    return fused_gram_into(grid, mode, kp, L, ws, G, st);
}

int tucker_hosvd_fused(const tucker_grid* grid, const tucker_kernel* kernel, const int32_t r[3], double* U1,
                       double* U2, double* U3, double* core, double* sigma1, double* sigma2, double* sigma3, void* ws,
                       size_t ws_bytes, void* stream, tucker_info* info) {
    launch_counter() = 0;
    TK_RC(check_grid(grid));
    TK_RC(check_kernel(kernel));
    TK_RC(check_ranks(grid, r));
    if (!U1 || !U2 || !U3 || !core || !sigma1 || !sigma2 || !sigma3 || !ws) return TUCKER_ERR_INVALID_ARG;
    const FusedLayout L = plan_fused(grid, r);
    if (ws_bytes < L.total) return TUCKER_ERR_SIZE;
    if (info) std::memset(info, 0, sizeof(*info));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const KParams kp = fused_kparams(grid, kernel);
    TK_RC(launch_fill_prep(*grid, *kernel, kp, reinterpret_cast<double*>(at(ws, L.nodes)),
                           reinterpret_cast<double*>(at(ws, L.cheb)), st));
    double* const U[3] = {U1, U2, U3};
    double* const S[3] = {sigma1, sigma2, sigma3};
    double* G = reinterpret_cast<double*>(at(ws, L.G));
    void* scr = at(ws, L.scratch);
    int worst = TUCKER_OK;
    auto eig_mode = [&](int m) -> int {
        const int rc = launch_eig(grid->n[m], G, r[m], U[m], nullptr, S[m], scr, L.scratch_bytes, st, info, m);
        if (rc == TUCKER_ERR_NOCONV) worst = rc;
        else if (rc != TUCKER_OK) return rc;
        return TUCKER_OK;
    };
    if (L.i8_bytes) {
        const I8Gen gen{kp, reinterpret_cast<const double*>(at(ws, L.cheb)),
                        reinterpret_cast<const double*>(at(ws, L.nodes))};
        TK_RC(launch_gram_i8_fused_modes(grid->n, gen, G, at(ws, L.i8), L.i8_bytes, st, 0, 2, eig_mode));
    } else {
        for (int m = 0; m < 3; ++m) {
            TK_RC(fused_gram_into(grid, m, kp, L, ws, G, st));
            TK_RC(eig_mode(m));
        }
    }
    const FusedGen gen = fused_gen(grid, kp, L, ws);
    TtmI8 ti{nullptr, nullptr, 0};
    const bool i8t = L.i8_bytes && ttm_engine() != TUCKER_TTM_DMMA &&
                     gram_i8_fused_ttm_scratch(grid->n, at(ws, L.i8), &ti.gmax, &ti.region, &ti.bytes);
    TK_RC(launch_ttm_core_impl(grid->n, r, nullptr, &gen, U1, U2, U3, core, scr, L.scratch_bytes, st, nullptr, nullptr,
                               nullptr, i8t ? &ti : nullptr));
    return worst;
}

int tucker_hosvd_fused_sharded(const tucker_grid* grid, const tucker_kernel* kernel, const int32_t r[3], int32_t shard,
                               int32_t nshards, tucker_allreduce_fn allreduce, void* user, double* U1, double* U2,
                               double* U3, double* core, double* sigma1, double* sigma2, double* sigma3, double* err3,
                               void* ws, size_t ws_bytes, void* stream, tucker_info* info) {
    launch_counter() = 0;
    if (nshards < 1 || shard < 0 || shard >= nshards || (nshards > 1 && !allreduce)) return TUCKER_ERR_INVALID_ARG;
    TK_RC(check_grid(grid));
    TK_RC(check_kernel(kernel));
    TK_RC(check_ranks(grid, r));
    if (!U1 || !U2 || !U3 || !core || !sigma1 || !sigma2 || !sigma3 || !ws) return TUCKER_ERR_INVALID_ARG;
    const FusedLayout L = plan_fused(grid, r);
    if (ws_bytes < L.total) return TUCKER_ERR_SIZE;
    if (!L.i8_bytes) return TUCKER_ERR_UNSUPPORTED;  // the shardable Gram is the INT8 fused route
    if (info) std::memset(info, 0, sizeof(*info));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Shard sh;
    sh.index = shard;
    sh.count = nshards;
    char* const wsb = static_cast<char*>(ws);
    sh.allreduce = [&](void* p, int64_t count, int dtype, int op) -> int {
        const int64_t off = static_cast<char*>(p) - wsb;
        return allreduce(user, off, count, dtype, op);
    };
    const KParams kp = fused_kparams(grid, kernel);
    TK_RC(launch_fill_prep(*grid, *kernel, kp, reinterpret_cast<double*>(at(ws, L.nodes)),
                           reinterpret_cast<double*>(at(ws, L.cheb)), st));
    double* const U[3] = {U1, U2, U3};
    double* const S[3] = {sigma1, sigma2, sigma3};
    double* G = reinterpret_cast<double*>(at(ws, L.G));
    void* scr = at(ws, L.scratch);
    int worst = TUCKER_OK;
    auto eig_mode = [&](int m) -> int {  // replicated: the same G on every rank gives the same U_m
        const int rc = launch_eig(grid->n[m], G, r[m], U[m], nullptr, S[m], scr, L.scratch_bytes, st, info, m);
        if (rc == TUCKER_ERR_NOCONV) worst = rc;
        else if (rc != TUCKER_OK) return rc;
        return TUCKER_OK;
    };
    const I8Gen ig{kp, reinterpret_cast<const double*>(at(ws, L.cheb)), reinterpret_cast<const double*>(at(ws, L.nodes))};
    TK_RC(launch_gram_i8_fused_modes(grid->n, ig, G, at(ws, L.i8), L.i8_bytes, st, 0, 2, eig_mode, &sh));
    const FusedGen gen = fused_gen(grid, kp, L, ws);
    TtmI8 ti{nullptr, nullptr, 0};  // the same INT8 TTM as tucker_hosvd_fused (bitwise the same T2 rows)
    const bool i8t = L.i8_bytes && ttm_engine() != TUCKER_TTM_DMMA &&
                     gram_i8_fused_ttm_scratch(grid->n, at(ws, L.i8), &ti.gmax, &ti.region, &ti.bytes);
    TK_RC(launch_ttm_core_impl(grid->n, r, nullptr, &gen, U1, U2, U3, core, scr, L.scratch_bytes, st, nullptr, nullptr,
                               &sh, i8t ? &ti : nullptr));
    if (err3)
        TK_RC(launch_error_impl(grid->n, r, nullptr, &gen, U1, U2, U3, core, err3, scr, L.scratch_bytes, st, &sh));
    return worst;
}

int tucker_error_fused(const tucker_grid* grid, const tucker_kernel* kernel, const int32_t r[3], const double* U1,
                       const double* U2, const double* U3, const double* core, double* out3, void* ws,
                       size_t ws_bytes, void* stream) {
    launch_counter() = 0;
    TK_RC(check_grid(grid));
    TK_RC(check_kernel(kernel));
    TK_RC(check_ranks(grid, r));
    if (!U1 || !U2 || !U3 || !core || !out3 || !ws) return TUCKER_ERR_INVALID_ARG;
    const FusedLayout L = plan_fused(grid, r);
    if (ws_bytes < L.total) return TUCKER_ERR_SIZE;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const KParams kp = fused_kparams(grid, kernel);
    TK_RC(launch_fill_prep(*grid, *kernel, kp, reinterpret_cast<double*>(at(ws, L.nodes)),
                           reinterpret_cast<double*>(at(ws, L.cheb)), st));
    const FusedGen gen = fused_gen(grid, kp, L, ws);
    TK_PROF(TUCKER_PROF_ERROR, st);
    return launch_error_impl(grid->n, r, nullptr, &gen, U1, U2, U3, core, out3, at(ws, L.scratch), L.scratch_bytes,
                             st);
}

size_t tucker_workspace_size_als(const tucker_grid* grid, const int32_t r[3]) {
    if (check_grid(grid) != TUCKER_OK || !r || check_ranks(grid, r) != TUCKER_OK) return 0;
    return als_ws_bytes(grid->n, r);
}

int tucker_als(const tucker_grid* grid, const int32_t r[3], const double* F, double* U1, double* U2, double* U3,
               double* core, double* sigma1, double* sigma2, double* sigma3, int32_t sweeps, void* ws,
               size_t ws_bytes, void* stream, tucker_info* info) {
    launch_counter() = 0;
    TK_RC(check_grid(grid));
    TK_RC(check_ranks(grid, r));
    if (!F || !U1 || !U2 || !U3 || !core || !sigma1 || !sigma2 || !sigma3 || !ws || sweeps < 1)
        return TUCKER_ERR_INVALID_ARG;
    if (r[1] > 64 || r[2] > 64) return TUCKER_ERR_UNSUPPORTED;
    if (info) std::memset(info, 0, sizeof(*info));
    double* const U[3] = {U1, U2, U3};
    double* const S[3] = {sigma1, sigma2, sigma3};
    return launch_als(grid->n, r, F, U, core, S, sweeps, ws, ws_bytes, static_cast<cudaStream_t>(stream), info);
}

// ---------------------------------------------------------------- multigrid Tucker
namespace {
constexpr int kMgMaxLevels = 12;
struct MgPlan {
    int L;                      // levels, 0 = coarsest .. L-1 = the caller's grid
    int64_t n[kMgMaxLevels][3];
    size_t off_fill, off_x, off_Fc, off_U[2], off_V, off_sig, off_sub, sub_bytes, total;
    int64_t nmax;
};

// Dyadic coarsening n -> ceil(n/2) per axis (n = 2m - 1 grids nest exactly), down to the first
// level whose every n_m <= n0, never below r_m (the coarsest HOSVD needs r_m <= n_m) or 4 nodes.
MgPlan mg_plan(const tucker_grid* g, const int32_t* r, int32_t n0) {
    MgPlan P{};
    int64_t lev[kMgMaxLevels][3];
    int L = 0;
    int64_t cur[3] = {g->n[0], g->n[1], g->n[2]};
    for (;;) {
        for (int a = 0; a < 3; ++a) lev[L][a] = cur[a];
        ++L;
        if (L == kMgMaxLevels || std::max(cur[0], std::max(cur[1], cur[2])) <= n0) break;
        int64_t nx[3];
        bool ok = true;
        for (int a = 0; a < 3; ++a) {
            nx[a] = (cur[a] + 1) / 2;
            ok &= nx[a] >= std::max<int64_t>(r[a], 4);
        }
        if (!ok) break;
        for (int a = 0; a < 3; ++a) cur[a] = nx[a];
    }
    P.L = L;
    for (int l = 0; l < L; ++l)
        for (int a = 0; a < 3; ++a) P.n[l][a] = lev[L - 1 - l][a];
    const int64_t* nf = g->n;
    P.nmax = std::max(nf[0], std::max(nf[1], nf[2]));
    size_t off = 0;
    P.off_fill = off;
    off += align_up(plan(g, nullptr).G, 256);  // nodes + K_nu table of the finest grid (covers all)
    P.off_x = off;
    off += align_up((size_t)2 * P.nmax * 8, 256);
    P.off_Fc = off;
    size_t fc = 0;
    for (int l = 0; l + 1 < L; ++l) fc = std::max(fc, (size_t)(P.n[l][0] * P.n[l][1] * P.n[l][2]) * 8);
    off += align_up(fc, 256);
    for (int s = 0; s < 2; ++s) {
        P.off_U[s] = off;
        for (int a = 0; a < 3; ++a) off += align_up((size_t)P.nmax * r[a] * 8, 256);
    }
    P.off_V = off;  // prolonged factor (SVD input) and the SVD's full output
    off += 2 * align_up((size_t)P.nmax * 64 * 8, 256);
    P.off_sig = off;
    off += align_up((size_t)3 * 64 * 8, 256);
    P.off_sub = off;
    size_t sub = 0;
    for (int l = 0; l < L; ++l) {
        tucker_grid gl = *g;
        for (int a = 0; a < 3; ++a) gl.n[a] = P.n[l][a];
        sub = std::max(sub, l == 0 ? plan(&gl, r).total : als_ws_bytes(gl.n, r));
    }
    P.sub_bytes = align_up(sub, 256);
    off += P.sub_bytes;
    P.total = off;
    return P;
}
}  // namespace

size_t tucker_workspace_size_multigrid(const tucker_grid* grid, const int32_t r[3], int32_t n0) {
    if (check_grid(grid) != TUCKER_OK || !r || check_ranks(grid, r) != TUCKER_OK || n0 < 4) return 0;
    return mg_plan(grid, r, n0).total;
}

int tucker_multigrid(const tucker_grid* grid, const tucker_kernel* kernel, const int32_t r[3], int32_t n0,
                     int32_t sweeps, double* F, double* U1, double* U2, double* U3, double* core, double* sigma1,
                     double* sigma2, double* sigma3, void* ws, size_t ws_bytes, void* stream, tucker_info* info,
                     int32_t* levels_out) {
    launch_counter() = 0;
    TK_RC(check_grid(grid));
    TK_RC(check_kernel(kernel));
    TK_RC(check_ranks(grid, r));
    if (!F || !U1 || !U2 || !U3 || !core || !sigma1 || !sigma2 || !sigma3 || !ws || sweeps < 1 || n0 < 4)
        return TUCKER_ERR_INVALID_ARG;
    if (r[1] > 64 || r[2] > 64) return TUCKER_ERR_UNSUPPORTED;
    const MgPlan P = mg_plan(grid, r, n0);
    if (ws_bytes < P.total) return TUCKER_ERR_SIZE;
    for (int a = 0; a < 3; ++a)
        if (r[a] > 56 || P.n[0][a] < r[a]) return TUCKER_ERR_UNSUPPORTED;
    if (info) std::memset(info, 0, sizeof(*info));
    if (levels_out) *levels_out = P.L;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    char* w = static_cast<char*>(ws);
    double* nodes = reinterpret_cast<double*>(w + P.off_fill);
    const Layout Lf = plan(grid, nullptr);
    double* cheb = reinterpret_cast<double*>(w + P.off_fill + Lf.cheb);
    double* xbuf = reinterpret_cast<double*>(w + P.off_x);
    double* Fc = reinterpret_cast<double*>(w + P.off_Fc);
    double* Ubuf[2][3];
    for (int s = 0; s < 2; ++s) {
        size_t o = P.off_U[s];
        for (int a = 0; a < 3; ++a) {
            Ubuf[s][a] = reinterpret_cast<double*>(w + o);
            o += align_up((size_t)P.nmax * r[a] * 8, 256);
        }
    }
    double* V = reinterpret_cast<double*>(w + P.off_V);
    double* Vo = reinterpret_cast<double*>(w + P.off_V + align_up((size_t)P.nmax * 64 * 8, 256));
    double* sig = reinterpret_cast<double*>(w + P.off_sig);
    void* sub = w + P.off_sub;
    double* const Uout[3] = {U1, U2, U3};
    double* const Sout[3] = {sigma1, sigma2, sigma3};
    int worst = TUCKER_OK;
    double* const* Ucur = Ubuf[0];
    for (int l = 0; l < P.L; ++l) {
        tucker_grid gl = *grid;
        for (int a = 0; a < 3; ++a) gl.n[a] = P.n[l][a];
        const bool finest = l == P.L - 1;
        double* Fl = finest ? F : Fc;
        TK_RC(launch_fill(gl, *kernel, Fl, nodes, cheb, st));
        double* const* Unext = finest ? Uout : Ubuf[(l + 1) & 1];
        if (l == 0) {  // HOSVD at the coarsest level only
            int rc = hosvd_impl(&gl, r, Fl, Unext, core, Sout, sub, P.sub_bytes, st, info);
            if (rc == TUCKER_ERR_NOCONV) worst = rc;
            else if (rc != TUCKER_OK) return rc;
            if (P.L == 1) return worst;
        } else {  // prolongate the previous level's subspaces, orthonormalise, ALS sweeps
            for (int a = 0; a < 3; ++a) {
                TK_RC(launch_prolong(Ucur[a], P.n[l - 1][a], grid->lo[a], grid->hi[a], V, gl.n[a], r[a], xbuf, st));
                TK_RC(launch_svd_cluster(gl.n[a], r[a], r[a], V, Vo, Unext[a], sig + 64 * a, nullptr, st));
            }
            const int rc = launch_als(gl.n, r, Fl, Unext, core, Sout, sweeps, sub, P.sub_bytes, st, info);
            if (rc == TUCKER_ERR_NOCONV) worst = rc;
            else if (rc != TUCKER_OK) return rc;
        }
        Ucur = Unext;
    }
    return worst;
}

size_t tucker_workspace_size_sym(const tucker_grid* grid, const int32_t r[3]) {
    if (check_grid(grid) != TUCKER_OK || !r) return 0;
    return sym_ws_bytes(*grid, r);
}

int tucker_hosvd_sym(const tucker_grid* grid, const tucker_kernel* kernel, const int32_t r[3], double* U1,
                     double* U2, double* U3, double* core, double* sigma1, double* sigma2, double* sigma3,
                     double* err3, void* ws, size_t ws_bytes, void* stream, tucker_info* info) {
    launch_counter() = 0;
    TK_RC(check_grid(grid));
    TK_RC(check_kernel(kernel));
    TK_RC(check_ranks(grid, r));
    if (!U1 || !U2 || !U3 || !core || !sigma1 || !sigma2 || !sigma3 || !ws) return TUCKER_ERR_INVALID_ARG;
    if (!grid_centred(*grid)) return TUCKER_ERR_UNSUPPORTED;
    for (int a = 0; a < 3; ++a)
        if (r[a] > (grid->n[a] + 1) / 2) return TUCKER_ERR_RANK;
    if (info) std::memset(info, 0, sizeof(*info));
    double* const U[3] = {U1, U2, U3};
    double* const S[3] = {sigma1, sigma2, sigma3};
    return launch_hosvd_sym(*grid, *kernel, r, U, core, S, err3, ws, ws_bytes, static_cast<cudaStream_t>(stream),
                            info);
}

// NEXT f2 layout: [G][V (n_max x p)][scratch]
static int accurate_p(int64_t n, int r) { return (int)std::min<int64_t>(n, std::min(r + 8, 56)); }

// [G][V, its Gram eigenvalues][INT8 Gram region (if that engine is in effect)][scratch]
static size_t accurate_plan(const tucker_grid* g, const int32_t* r, size_t* offV, size_t* offS, size_t* offI8 = nullptr,
                            size_t* i8_bytes = nullptr) {
    const int64_t* n = g->n;
    const int64_t nmax = std::max(n[0], std::max(n[1], n[2]));
    size_t off = align_up((size_t)nmax * nmax * 8, 256);
    *offV = off;
    off += align_up((size_t)nmax * 64 * 8, 256) + 64 * 8;
    off = align_up(off, 1024);
    const size_t ib = gram_use_i8(n) ? align_up(gram_i8_ws_bytes(n), 1024) : 0;
    if (offI8) *offI8 = off;
    if (i8_bytes) *i8_bytes = ib;
    off += ib;
    *offS = off;
    size_t s = ib ? 0 : gram_ws_bytes(n);
    int pmax = 1;
    for (int a = 0; a < 3; ++a) {
        const int p = accurate_p(n[a], r[a]);
        pmax = std::max(pmax, p);
        s = std::max(s, eig_ws_bytes(n[a], p));
    }
    s = std::max(s, refine_ws_bytes(n, pmax));
    s = std::max(s, ttm_ws_bytes(n, r));
    return off + align_up(s, 256);
}

size_t tucker_workspace_size_accurate(const tucker_grid* grid, const int32_t r[3]) {
    if (check_grid(grid) != TUCKER_OK || !r || check_ranks(grid, r) != TUCKER_OK) return 0;
    size_t a, b;
    return accurate_plan(grid, r, &a, &b);
}

int tucker_hosvd_accurate(const tucker_grid* grid, const int32_t r[3], const double* F, double* U1, double* U2,
                          double* U3, double* core, double* sigma1, double* sigma2, double* sigma3, int32_t iters,
                          void* ws, size_t ws_bytes, void* stream, tucker_info* info) {
    launch_counter() = 0;
    TK_RC(check_grid(grid));
    TK_RC(check_ranks(grid, r));
    if (!F || !U1 || !U2 || !U3 || !core || !sigma1 || !sigma2 || !sigma3 || !ws || iters < 1)
        return TUCKER_ERR_INVALID_ARG;
    for (int a = 0; a < 3; ++a)
        if (r[a] > 56 || grid->n[a] > 2048) return TUCKER_ERR_UNSUPPORTED;
    size_t offV, offS, offI8, i8_bytes;
    const size_t total = accurate_plan(grid, r, &offV, &offS, &offI8, &i8_bytes);
    if (ws_bytes < total) return TUCKER_ERR_SIZE;
    if (info) std::memset(info, 0, sizeof(*info));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    double* G = static_cast<double*>(ws);
    double* V = reinterpret_cast<double*>(at(ws, offV));
    const int64_t nmx = std::max(grid->n[0], std::max(grid->n[1], grid->n[2]));
    double* lam = V + align_up((size_t)nmx * 64 * 8, 256) / 8;
    void* scr = at(ws, offS);
    const size_t sb = total - offS;
    double* const U[3] = {U1, U2, U3};
    double* const S[3] = {sigma1, sigma2, sigma3};
    int worst = TUCKER_OK;
    auto after = [&](int m) -> int {  // Gram route's subspace, then the Rayleigh-Ritz steps on F_(m)
        const int p = accurate_p(grid->n[m], r[m]);
        const int rc = launch_eig(grid->n[m], G, p, V, lam, nullptr, scr, sb, st, info, m);
        if (rc == TUCKER_ERR_NOCONV) worst = rc;
        else if (rc != TUCKER_OK) return rc;
        return launch_refine_mode(grid->n, m, F, V, lam, p, r[m], iters, U[m], S[m], scr, sb, st, nullptr);
    };
    if (i8_bytes) {
        TK_RC(launch_gram_i8_modes(grid->n, F, G, at(ws, offI8), i8_bytes, st, after));
    } else {
        for (int m = 0; m < 3; ++m) {
            TK_RC(launch_gram(grid->n, m, F, G, scr, sb, st));
            TK_RC(after(m));
        }
    }
    TK_RC(launch_ttm_core(grid->n, r, F, U1, U2, U3, core, scr, sb, st));
    return worst;
}

int64_t tucker_last_launch_count(void) { return launch_counter(); }

const char* tucker_strerror(int code) {
    switch (code) {
        case TUCKER_OK: return "ok";
        case TUCKER_ERR_INVALID_ARG: return "invalid argument (null pointer, n < 2, lo >= hi, bad mode)";
        case TUCKER_ERR_DOMAIN: return "kernel parameter outside its domain";
        case TUCKER_ERR_RANK: return "rank out of range (r < 1 or r > n)";
        case TUCKER_ERR_SIZE: return "workspace too small or size overflow";
        case TUCKER_ERR_NOCONV: return "eigensolver did not converge (best iterate returned)";
        case TUCKER_ERR_CUDA: return "CUDA runtime/driver error";
        case TUCKER_ERR_UNSUPPORTED: return "unsupported configuration";
        case TUCKER_ERR_COLLECTIVE: return "the caller's all-reduce callback failed";
        case TUCKER_ERR_INPUT: return "input not finite, or row maxima that do not bound F";
        default: return "unknown error code";
    }
}

}  // extern "C"
