"""Thin ctypes binding of the C-ABI in include/tucker.h (argument marshalling only).

Every numerical step runs in libtucker_b200.so (hand-written sm_100a CUDA).  PyTorch provides the
device memory and the stream; there is no CPU or PyTorch fallback: if the native library is
missing or no CUDA device is present, the calls raise.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TUCKER_LIB_PATH") or os.path.join(_PKG, "libtucker_b200.so")  # (env: A/B runs)

MATERN, SLATER, MATERN_SPECTRAL = 0, 1, 2
GRAM_AUTO, GRAM_DMMA, GRAM_INT8, GRAM_INT8_ROWSCALED = 0, 1, 2, 3
FORCE_GENERAL_BESSEL = 2
ERRORS = {0: "TUCKER_OK", 1: "TUCKER_ERR_INVALID_ARG", 2: "TUCKER_ERR_DOMAIN", 3: "TUCKER_ERR_RANK",
          4: "TUCKER_ERR_SIZE", 5: "TUCKER_ERR_NOCONV", 6: "TUCKER_ERR_CUDA", 7: "TUCKER_ERR_UNSUPPORTED",
          8: "TUCKER_ERR_COLLECTIVE", 9: "TUCKER_ERR_INPUT"}
EXPORTS = ("tucker_workspace_size", "tucker_workspace_size_fill", "tucker_fill", "tucker_fill_prepare",
           "tucker_hosvd_prepared", "tucker_fill_rowmax", "tucker_hosvd_rowmax", "tucker_gram", "tucker_eig", "tucker_ttm_core",
           "tucker_hosvd", "tucker_error", "tucker_approximate", "tucker_workspace_size_fused",
           "tucker_gram_fused", "tucker_hosvd_fused", "tucker_error_fused", "tucker_hosvd_fused_sharded",
           "tucker_workspace_size_als",
           "tucker_als", "tucker_workspace_size_sym", "tucker_hosvd_sym", "tucker_workspace_size_accurate",
           "tucker_hosvd_accurate", "tucker_workspace_size_i8", "tucker_gram_i8", "tucker_i8_scheme", "tucker_i8_layout",
           "tucker_set_gram_engine", "tucker_get_gram_engine", "tucker_set_ttm_engine", "tucker_get_ttm_engine", "tucker_profile_enable", "tucker_profile_read",
           "tucker_workspace_size_multigrid", "tucker_multigrid", "tucker_last_launch_count", "tucker_strerror")


class TuckerError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        super().__init__(f"{where}: {ERRORS.get(code, code)} ({_strerror(code)})")


class CGrid(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64 * 3), ("lo", ctypes.c_double * 3), ("hi", ctypes.c_double * 3)]


class CKernel(ctypes.Structure):
    _fields_ = [("family", ctypes.c_int32), ("flags", ctypes.c_int32), ("sigma2", ctypes.c_double),
                ("ell", ctypes.c_double), ("nu", ctypes.c_double), ("lam", ctypes.c_double),
                ("p", ctypes.c_double)]


class CInfo(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int32 * 3), ("converged", ctypes.c_int32 * 3), ("block", ctypes.c_int32 * 3),
                ("sweeps", ctypes.c_int32 * 3), ("resid", ctypes.c_double * 3), ("lambda1", ctypes.c_double * 3),
                ("k_resolved", ctypes.c_int32 * 3), ("moduli", ctypes.c_int32 * 3)]

    def as_dict(self) -> dict:
        return {k: list(getattr(self, k)) for k, _ in self._fields_}


_lib = None


# tucker_allreduce_fn(user, ws_offset, count, dtype, op) -> 0 on success
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                ctypes.c_int32)
DT_INT32, DT_F64 = 0, 1
RED_SUM, RED_MAX = 0, 1


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load the native library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"native library not built: {path} (run python -m paper_1711_06874_b200.build)")
    lib = ctypes.CDLL(path)
    P, vp, i32, i64, sz = ctypes.POINTER, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    pg, pk, pi = P(CGrid), P(CKernel), P(CInfo)
    pr = P(ctypes.c_int32)
    sig = {
        "tucker_workspace_size": (sz, [pg, pr]),
        "tucker_workspace_size_fill": (sz, [pg]),
        "tucker_fill": (ctypes.c_int, [pg, pk, vp, vp, sz, vp]),
        "tucker_fill_rowmax": (ctypes.c_int, [pg, pk, vp, vp, vp, sz, vp]),
        "tucker_fill_prepare": (ctypes.c_int, [pg, pk, pr, vp, vp, sz, vp]),
        "tucker_hosvd_prepared": (ctypes.c_int, [pg, pr, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp, pi]),
        "tucker_hosvd_rowmax": (ctypes.c_int, [pg, pr, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp, pi]),
        "tucker_gram": (ctypes.c_int, [pg, i32, vp, vp, vp, sz, vp]),
        "tucker_workspace_size_i8": (sz, [pg]),
        "tucker_gram_i8": (ctypes.c_int, [pg, i32, vp, vp, vp, sz, vp]),
        "tucker_i8_scheme": (ctypes.c_int, [i64, P(ctypes.c_int32), P(ctypes.c_int32)]),
        "tucker_i8_layout": (ctypes.c_int, [pg, P(ctypes.c_int32), P(ctypes.c_int32)]),
        "tucker_set_gram_engine": (ctypes.c_int, [i32]),
        "tucker_get_gram_engine": (i32, []),
        "tucker_set_ttm_engine": (ctypes.c_int, [i32]),
        "tucker_get_ttm_engine": (i32, []),
        "tucker_profile_enable": (ctypes.c_int, [i32]),
        "tucker_profile_read": (ctypes.c_int, [P(ctypes.c_double), P(ctypes.c_int64)]),
        "tucker_eig": (ctypes.c_int, [i64, vp, i32, vp, vp, vp, sz, vp, pi]),
        "tucker_ttm_core": (ctypes.c_int, [pg, pr, vp, vp, vp, vp, vp, vp, sz, vp]),
        "tucker_hosvd": (ctypes.c_int, [pg, pr, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp, pi]),
        "tucker_error": (ctypes.c_int, [pg, pr, vp, vp, vp, vp, vp, vp, vp, sz, vp]),
        "tucker_approximate": (ctypes.c_int, [pg, pk, pr, vp, P(vp), vp, P(vp), vp, vp, sz, vp, pi]),
        "tucker_workspace_size_fused": (sz, [pg, pr]),
        "tucker_gram_fused": (ctypes.c_int, [pg, pk, i32, vp, vp, sz, vp]),
        "tucker_hosvd_fused": (ctypes.c_int, [pg, pk, pr, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp, pi]),
        "tucker_error_fused": (ctypes.c_int, [pg, pk, pr, vp, vp, vp, vp, vp, vp, sz, vp]),
        "tucker_hosvd_fused_sharded": (ctypes.c_int, [pg, pk, pr, i32, i32, ALLREDUCE_FN, vp, vp, vp, vp, vp, vp,
                                                      vp, vp, vp, vp, sz, vp, pi]),
        "tucker_workspace_size_als": (sz, [pg, pr]),
        "tucker_als": (ctypes.c_int, [pg, pr, vp, vp, vp, vp, vp, vp, vp, vp, i32, vp, sz, vp, pi]),
        "tucker_workspace_size_sym": (sz, [pg, pr]),
        "tucker_hosvd_sym": (ctypes.c_int, [pg, pk, pr, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp, pi]),
        "tucker_workspace_size_accurate": (sz, [pg, pr]),
        "tucker_hosvd_accurate": (ctypes.c_int, [pg, pr, vp, vp, vp, vp, vp, vp, vp, vp, i32, vp, sz, vp, pi]),
        "tucker_workspace_size_multigrid": (sz, [pg, pr, i32]),
        "tucker_multigrid": (ctypes.c_int, [pg, pk, pr, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp, pi,
                                            P(ctypes.c_int32)]),
        "tucker_last_launch_count": (i64, []),
        "tucker_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def _strerror(code: int) -> str:
    try:
        return load().tucker_strerror(code).decode()
    except Exception:  # pragma: no cover
        return "?"


def _check(code: int, where: str) -> int:
    if code != 0:
        raise TuckerError(code, where)
    return code


def cgrid(g) -> CGrid:
    c = CGrid()
    for a in range(3):
        c.n[a], c.lo[a], c.hi[a] = int(g.n[a]), float(g.lo[a]), float(g.hi[a])
    return c


def ckernel(k) -> CKernel:
    return CKernel(int(k.family), int(getattr(k, "flags", 0)), float(k.sigma2), float(k.ell), float(k.nu),
                   float(k.lam), float(k.p))


def cranks(r) -> ctypes.Array:
    return (ctypes.c_int32 * 3)(*[int(v) for v in r])


def _ptr(t: torch.Tensor) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _dev(t: torch.Tensor, name: str):
    if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise ValueError(f"{name} must be a contiguous float64 CUDA tensor")


def last_launch_count() -> int:
    return int(load().tucker_last_launch_count())


def workspace_bytes(grid, ranks=None) -> int:
    lib = load()
    g = cgrid(grid)
    return int(lib.tucker_workspace_size(ctypes.byref(g), cranks(ranks) if ranks is not None else None))


def workspace(grid, ranks=None, device="cuda") -> torch.Tensor:
    return torch.empty(workspace_bytes(grid, ranks), dtype=torch.uint8, device=device)


def workspace_fill(grid, device="cuda") -> torch.Tensor:
    """The few-KB workspace of tucker_fill / tucker_fill_rowmax (nodes, K_nu table)."""
    n = int(load().tucker_workspace_size_fill(ctypes.byref(cgrid(grid))))
    return torch.empty(n, dtype=torch.uint8, device=device)


# -------------------------------------------------------------------------------- entry points
def fill(grid, kernel, F: torch.Tensor | None = None, ws: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    lib = load()
    shape = tuple(int(v) for v in grid.n)
    if F is None:
        F = torch.empty(shape, dtype=torch.float64, device="cuda")
    _dev(F, "F")
    ws = ws if ws is not None else workspace_fill(grid)
    g, k = cgrid(grid), ckernel(kernel)
    _check(lib.tucker_fill(ctypes.byref(g), ctypes.byref(k), _ptr(F), _ptr(ws), ws.numel(), _stream(stream)),
           "tucker_fill")
    return F


def fill_rowmax(grid, kernel, F: torch.Tensor | None = None, ws: torch.Tensor | None = None, stream=None):
    """tucker_fill_rowmax: (F, rowmax) — the fill plus the INT8 route's per-row maxima (centred grids,
    n3 % 8 == 0, n3 <= 8192; TuckerError UNSUPPORTED otherwise)."""
    lib = load()
    shape = tuple(int(v) for v in grid.n)
    if F is None:
        F = torch.empty(shape, dtype=torch.float64, device="cuda")
    _dev(F, "F")
    mx = torch.empty(int(sum(shape)), dtype=torch.int32, device=F.device)  # uint32 bit patterns (< 2^31)
    ws = ws if ws is not None else workspace_fill(grid)
    g, k = cgrid(grid), ckernel(kernel)
    _check(lib.tucker_fill_rowmax(ctypes.byref(g), ctypes.byref(k), _ptr(F), _ptr(mx), _ptr(ws), ws.numel(),
                                  _stream(stream)), "tucker_fill_rowmax")
    return F, mx


def fill_prepare(grid, kernel, ranks, F: torch.Tensor | None = None, ws: torch.Tensor | None = None, stream=None):
    """tucker_fill_prepare: (F, ws) — the fill plus the INT8 route's shared residues written into the
    HOSVD workspace `ws` of (grid, ranks); follow with hosvd_prepared(grid, ranks, F, ws)."""
    lib = load()
    shape = tuple(int(v) for v in grid.n)
    if F is None:
        F = torch.empty(shape, dtype=torch.float64, device="cuda")
    _dev(F, "F")
    ws = ws if ws is not None else workspace(grid, ranks)
    g, k = cgrid(grid), ckernel(kernel)
    _check(lib.tucker_fill_prepare(ctypes.byref(g), ctypes.byref(k), cranks(ranks), _ptr(F), _ptr(ws), ws.numel(),
                                   _stream(stream)), "tucker_fill_prepare")
    return F, ws


def hosvd_prepared(grid, ranks, F: torch.Tensor, ws: torch.Tensor, stream=None, sync: bool = True) -> HosvdResult:
    """tucker_hosvd_prepared on a workspace from fill_prepare of this F."""
    lib = load()
    _dev(F, "F")
    r = tuple(int(v) for v in ranks)
    U = [torch.empty((int(grid.n[m]), r[m]), dtype=torch.float64, device=F.device) for m in range(3)]
    S = [torch.empty(r[m], dtype=torch.float64, device=F.device) for m in range(3)]
    core = torch.empty(r, dtype=torch.float64, device=F.device)
    info = CInfo()
    g = cgrid(grid)
    rc = lib.tucker_hosvd_prepared(ctypes.byref(g), cranks(r), _ptr(F), _ptr(U[0]), _ptr(U[1]), _ptr(U[2]),
                                   _ptr(core), _ptr(S[0]), _ptr(S[1]), _ptr(S[2]), _ptr(ws), ws.numel(),
                                   _stream(stream), ctypes.byref(info) if sync else None)
    if rc not in (0, 5):
        _check(rc, "tucker_hosvd_prepared")
    return HosvdResult(U, core, S, info.as_dict(), rc)


def gram(grid, mode: int, F: torch.Tensor, ws: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    lib = load()
    _dev(F, "F")
    n = int(grid.n[mode])
    G = torch.empty((n, n), dtype=torch.float64, device=F.device)
    ws = ws if ws is not None else workspace(grid)
    g = cgrid(grid)
    _check(lib.tucker_gram(ctypes.byref(g), int(mode), _ptr(F), _ptr(G), _ptr(ws), ws.numel(), _stream(stream)),
           "tucker_gram")
    return G


def set_gram_engine(engine: int) -> None:
    """Gram engine of gram / hosvd / approximate: GRAM_AUTO (INT8 emulation where supported),
    GRAM_DMMA or GRAM_INT8.  Process-wide; size workspaces after setting it."""
    _check(load().tucker_set_gram_engine(int(engine)), "tucker_set_gram_engine")


def get_gram_engine() -> int:
    return int(load().tucker_get_gram_engine())


TTM_AUTO, TTM_DMMA, TTM_INT8_ERROR = 0, 1, 2


def set_ttm_engine(engine: int) -> None:
    """TTM engine of the INT8 hosvd route's core: TTM_AUTO (T1 = F x3 U3^T on the INT8 tensor cores
    by base-256 digits where it applies, R22), TTM_DMMA (the FP64 tensor-core TTM) or
    TTM_INT8_ERROR (AUTO plus the error pass's reconstruction on the INT8 tensor cores, R23; opt-in)."""
    _check(load().tucker_set_ttm_engine(int(engine)), "tucker_set_ttm_engine")


def get_ttm_engine() -> int:
    return int(load().tucker_get_ttm_engine())


PROF_STAGES = ("fill", "i8_rowmax", "i8_residues", "i8_gemm", "i8_crt", "dmma_gram", "eig", "ttm", "error")


def profile_enable(on: bool = True) -> None:
    """Record CUDA events around each stage's launches (on the launching stream) until disabled."""
    _check(load().tucker_profile_enable(1 if on else 0), "tucker_profile_enable")


def profile_read() -> dict:
    """{stage: (total ms, timed calls)} since the last read; synchronises the recorded events."""
    n = len(PROF_STAGES)
    ms, cnt = (ctypes.c_double * n)(), (ctypes.c_int64 * n)()
    _check(load().tucker_profile_read(ms, cnt), "tucker_profile_read")
    return {PROF_STAGES[i]: (ms[i], cnt[i]) for i in range(n)}


def i8_scheme(K: int) -> tuple:
    """(moduli, b) of the INT8 Gram's modular scheme for K unfolding columns (host query)."""
    mod, b = (ctypes.c_int32 * 16)(), ctypes.c_int32()
    _check(load().tucker_i8_scheme(int(K), mod, ctypes.byref(b)), "tucker_i8_scheme")
    return list(mod), int(b.value)


def i8_layout(grid) -> tuple:
    """(shared, b): whether the materialised INT8 Grams of `grid` use the shared residue layout
    (one global exponent, R20) and its integer width b (host query)."""
    sh, b = ctypes.c_int32(), ctypes.c_int32()
    _check(load().tucker_i8_layout(ctypes.byref(cgrid(grid)), ctypes.byref(sh), ctypes.byref(b)), "tucker_i8_layout")
    return bool(sh.value), int(b.value)


def workspace_i8(grid) -> torch.Tensor:
    lib = load()
    g = cgrid(grid)
    n = lib.tucker_workspace_size_i8(ctypes.byref(g))
    if n == 0:
        raise TuckerError(7, "tucker_workspace_size_i8")
    return torch.empty(n, dtype=torch.uint8, device="cuda")


def gram_i8(grid, mode: int, F: torch.Tensor, ws: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """a-3 on the INT8 tensor cores (modular emulation of the FP64 Gram, R18)."""
    lib = load()
    _dev(F, "F")
    n = int(grid.n[mode])
    G = torch.empty((n, n), dtype=torch.float64, device=F.device)
    ws = ws if ws is not None else workspace_i8(grid)
    g = cgrid(grid)
    _check(lib.tucker_gram_i8(ctypes.byref(g), int(mode), _ptr(F), _ptr(G), _ptr(ws), ws.numel(), _stream(stream)),
           "tucker_gram_i8")
    return G


def eig(G: torch.Tensor, r: int, ws: torch.Tensor | None = None, stream=None, check: bool = True):
    lib = load()
    _dev(G, "G")
    n = G.shape[0]
    U = torch.empty((n, r), dtype=torch.float64, device=G.device)
    lam = torch.empty(r, dtype=torch.float64, device=G.device)
    if ws is None:
        ws = workspace(type("g", (), {"n": (n, 2, 2), "lo": (-1, -1, -1), "hi": (1, 1, 1)}), (r, 1, 1))
    info = CInfo()
    rc = lib.tucker_eig(n, _ptr(G), int(r), _ptr(U), _ptr(lam), _ptr(ws), ws.numel(), _stream(stream),
                        ctypes.byref(info))
    if check and rc not in (0, 5):
        _check(rc, "tucker_eig")
    return U, lam, info.as_dict(), rc


def ttm_core(grid, ranks, F, U1, U2, U3, ws=None, stream=None) -> torch.Tensor:
    lib = load()
    for t, nm in ((F, "F"), (U1, "U1"), (U2, "U2"), (U3, "U3")):
        _dev(t, nm)
    core = torch.empty(tuple(int(v) for v in ranks), dtype=torch.float64, device=F.device)
    ws = ws if ws is not None else workspace(grid, ranks)
    g = cgrid(grid)
    _check(lib.tucker_ttm_core(ctypes.byref(g), cranks(ranks), _ptr(F), _ptr(U1), _ptr(U2), _ptr(U3), _ptr(core),
                               _ptr(ws), ws.numel(), _stream(stream)), "tucker_ttm_core")
    return core


@dataclass
class HosvdResult:
    U: list
    core: torch.Tensor
    sigma: list
    info: dict
    rc: int


def hosvd(grid, ranks, F: torch.Tensor, ws: torch.Tensor | None = None, stream=None,
          rowmax: torch.Tensor | None = None, sync: bool = True) -> HosvdResult:
    """tucker_hosvd, or tucker_hosvd_rowmax when `rowmax` (from fill_rowmax of this F) is given.
    sync=False passes info = NULL: the call is asynchronous (no host synchronisation, capturable in
    a CUDA Graph) and `info` stays empty."""
    lib = load()
    _dev(F, "F")
    dev = F.device
    r = tuple(int(v) for v in ranks)
    U = [torch.empty((int(grid.n[m]), r[m]), dtype=torch.float64, device=dev) for m in range(3)]
    S = [torch.empty(r[m], dtype=torch.float64, device=dev) for m in range(3)]
    core = torch.empty(r, dtype=torch.float64, device=dev)
    ws = ws if ws is not None else workspace(grid, r)
    info = CInfo()
    g = cgrid(grid)
    if rowmax is not None:
        if not (rowmax.is_cuda and rowmax.dtype == torch.int32 and rowmax.is_contiguous()):
            raise ValueError("rowmax must be a contiguous int32 CUDA tensor (from fill_rowmax)")
        rc = lib.tucker_hosvd_rowmax(ctypes.byref(g), cranks(r), _ptr(F), _ptr(rowmax), _ptr(U[0]), _ptr(U[1]),
                                     _ptr(U[2]), _ptr(core), _ptr(S[0]), _ptr(S[1]), _ptr(S[2]), _ptr(ws),
                                     ws.numel(), _stream(stream), ctypes.byref(info) if sync else None)
    else:
        rc = lib.tucker_hosvd(ctypes.byref(g), cranks(r), _ptr(F), _ptr(U[0]), _ptr(U[1]), _ptr(U[2]), _ptr(core),
                              _ptr(S[0]), _ptr(S[1]), _ptr(S[2]), _ptr(ws), ws.numel(), _stream(stream),
                              ctypes.byref(info) if sync else None)
    if rc not in (0, 5):
        _check(rc, "tucker_hosvd")
    return HosvdResult(U, core, S, info.as_dict(), rc)


def error(grid, ranks, F, U, core, ws=None, stream=None) -> torch.Tensor:
    lib = load()
    out = torch.empty(3, dtype=torch.float64, device=F.device)
    ws = ws if ws is not None else workspace(grid, ranks)
    g = cgrid(grid)
    _check(lib.tucker_error(ctypes.byref(g), cranks(ranks), _ptr(F), _ptr(U[0]), _ptr(U[1]), _ptr(U[2]),
                            _ptr(core), _ptr(out), _ptr(ws), ws.numel(), _stream(stream)), "tucker_error")
    return out


# ------------------------------------------------------------------ NEXT f1: Tucker-ALS
def als(grid, ranks, F: torch.Tensor, U_init, sweeps: int, ws: torch.Tensor | None = None, stream=None) -> HosvdResult:
    """Tucker-ALS sweeps from initial factors U_init (copied); returns refined U, core,
    sigma of the last single-hole unfoldings."""
    lib = load()
    _dev(F, "F")
    r = tuple(int(v) for v in ranks)
    U = [u[:, : r[m]].contiguous().clone() for m, u in enumerate(U_init)]
    S = [torch.empty(r[m], dtype=torch.float64, device=F.device) for m in range(3)]
    core = torch.empty(r, dtype=torch.float64, device=F.device)
    if ws is None:
        g0 = cgrid(grid)
        ws = torch.empty(int(lib.tucker_workspace_size_als(ctypes.byref(g0), cranks(r))), dtype=torch.uint8,
                         device=F.device)
    info = CInfo()
    g = cgrid(grid)
    rc = lib.tucker_als(ctypes.byref(g), cranks(r), _ptr(F), _ptr(U[0]), _ptr(U[1]), _ptr(U[2]), _ptr(core),
                        _ptr(S[0]), _ptr(S[1]), _ptr(S[2]), int(sweeps), _ptr(ws), ws.numel(), _stream(stream),
                        ctypes.byref(info))
    if rc not in (0, 5):
        _check(rc, "tucker_als")
    return HosvdResult(U, core, S, info.as_dict(), rc)


# ------------------------------------------------------------------ multigrid Tucker
def multigrid(grid, kernel, ranks, n0: int = 64, sweeps: int = 2, F: torch.Tensor | None = None,
              ws: torch.Tensor | None = None, stream=None):
    """tucker_multigrid: HOSVD on the coarsest dyadic level (every n_m <= n0), then per finer level
    interpolated factors + `sweeps` ALS sweeps; returns (HosvdResult, F, levels)."""
    lib = load()
    r = tuple(int(v) for v in ranks)
    shape = tuple(int(v) for v in grid.n)
    if F is None:
        F = torch.empty(shape, dtype=torch.float64, device="cuda")
    _dev(F, "F")
    U = [torch.empty((shape[m], r[m]), dtype=torch.float64, device=F.device) for m in range(3)]
    S = [torch.empty(r[m], dtype=torch.float64, device=F.device) for m in range(3)]
    core = torch.empty(r, dtype=torch.float64, device=F.device)
    g, k = cgrid(grid), ckernel(kernel)
    if ws is None:
        nb = int(lib.tucker_workspace_size_multigrid(ctypes.byref(g), cranks(r), int(n0)))
        if nb == 0:
            raise TuckerError(1, "tucker_workspace_size_multigrid")
        ws = torch.empty(nb, dtype=torch.uint8, device=F.device)
    info = CInfo()
    lev = ctypes.c_int32()
    rc = lib.tucker_multigrid(ctypes.byref(g), ctypes.byref(k), cranks(r), int(n0), int(sweeps), _ptr(F), _ptr(U[0]),
                              _ptr(U[1]), _ptr(U[2]), _ptr(core), _ptr(S[0]), _ptr(S[1]), _ptr(S[2]), _ptr(ws),
                              ws.numel(), _stream(stream), ctypes.byref(info), ctypes.byref(lev))
    if rc not in (0, 5):
        _check(rc, "tucker_multigrid")
    return HosvdResult(U, core, S, info.as_dict(), rc), F, int(lev.value)


# ------------------------------------------------------------------ NEXT f2: SVD-accurate HOSVD
def hosvd_accurate(grid, ranks, F: torch.Tensor, iters: int = 1, ws: torch.Tensor | None = None,
                   stream=None) -> HosvdResult:
    lib = load()
    _dev(F, "F")
    r = tuple(int(v) for v in ranks)
    U = [torch.empty((int(grid.n[m]), r[m]), dtype=torch.float64, device=F.device) for m in range(3)]
    S = [torch.empty(r[m], dtype=torch.float64, device=F.device) for m in range(3)]
    core = torch.empty(r, dtype=torch.float64, device=F.device)
    g = cgrid(grid)
    if ws is None:
        ws = torch.empty(int(lib.tucker_workspace_size_accurate(ctypes.byref(g), cranks(r))), dtype=torch.uint8,
                         device=F.device)
    info = CInfo()
    rc = lib.tucker_hosvd_accurate(ctypes.byref(g), cranks(r), _ptr(F), _ptr(U[0]), _ptr(U[1]), _ptr(U[2]),
                                   _ptr(core), _ptr(S[0]), _ptr(S[1]), _ptr(S[2]), int(iters), _ptr(ws), ws.numel(),
                                   _stream(stream), ctypes.byref(info))
    if rc not in (0, 5):
        _check(rc, "tucker_hosvd_accurate")
    return HosvdResult(U, core, S, info.as_dict(), rc)


# ------------------------------------------------------------------ NEXT f3: symmetric variant
def hosvd_sym(grid, kernel, ranks, ws: torch.Tensor | None = None, stream=None):
    """Symmetry-exploiting HOSVD + error on a centred grid (weighted octant); returns
    (HosvdResult, err3 tensor {E, ||F||, ||F-Ft||})."""
    lib = load()
    r = tuple(int(v) for v in ranks)
    U = [torch.empty((int(grid.n[m]), r[m]), dtype=torch.float64, device="cuda") for m in range(3)]
    S = [torch.empty(r[m], dtype=torch.float64, device="cuda") for m in range(3)]
    core = torch.empty(r, dtype=torch.float64, device="cuda")
    err = torch.empty(3, dtype=torch.float64, device="cuda")
    g, k = cgrid(grid), ckernel(kernel)
    if ws is None:
        ws = torch.empty(int(lib.tucker_workspace_size_sym(ctypes.byref(g), cranks(r))), dtype=torch.uint8,
                         device="cuda")
    info = CInfo()
    rc = lib.tucker_hosvd_sym(ctypes.byref(g), ctypes.byref(k), cranks(r), _ptr(U[0]), _ptr(U[1]), _ptr(U[2]),
                              _ptr(core), _ptr(S[0]), _ptr(S[1]), _ptr(S[2]), _ptr(err), _ptr(ws), ws.numel(),
                              _stream(stream), ctypes.byref(info))
    if rc not in (0, 5):
        _check(rc, "tucker_hosvd_sym")
    return HosvdResult(U, core, S, info.as_dict(), rc), err


# ------------------------------------------------------------------ a-7 fused (F never stored)
def workspace_bytes_fused(grid, ranks=None) -> int:
    lib = load()
    g = cgrid(grid)
    return int(lib.tucker_workspace_size_fused(ctypes.byref(g), cranks(ranks) if ranks is not None else None))


def workspace_fused(grid, ranks=None, device="cuda") -> torch.Tensor:
    return torch.empty(workspace_bytes_fused(grid, ranks), dtype=torch.uint8, device=device)


def gram_fused(grid, kernel, mode: int, ws: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    lib = load()
    n = int(grid.n[mode])
    G = torch.empty((n, n), dtype=torch.float64, device="cuda")
    ws = ws if ws is not None else workspace_fused(grid)
    g, k = cgrid(grid), ckernel(kernel)
    _check(lib.tucker_gram_fused(ctypes.byref(g), ctypes.byref(k), int(mode), _ptr(G), _ptr(ws), ws.numel(),
                                 _stream(stream)), "tucker_gram_fused")
    return G


def hosvd_fused(grid, kernel, ranks, ws: torch.Tensor | None = None, stream=None) -> HosvdResult:
    lib = load()
    r = tuple(int(v) for v in ranks)
    U = [torch.empty((int(grid.n[m]), r[m]), dtype=torch.float64, device="cuda") for m in range(3)]
    S = [torch.empty(r[m], dtype=torch.float64, device="cuda") for m in range(3)]
    core = torch.empty(r, dtype=torch.float64, device="cuda")
    ws = ws if ws is not None else workspace_fused(grid, r)
    info = CInfo()
    g, k = cgrid(grid), ckernel(kernel)
    rc = lib.tucker_hosvd_fused(ctypes.byref(g), ctypes.byref(k), cranks(r), _ptr(U[0]), _ptr(U[1]), _ptr(U[2]),
                                _ptr(core), _ptr(S[0]), _ptr(S[1]), _ptr(S[2]), _ptr(ws), ws.numel(),
                                _stream(stream), ctypes.byref(info))
    if rc not in (0, 5):
        _check(rc, "tucker_hosvd_fused")
    return HosvdResult(U, core, S, info.as_dict(), rc)


@dataclass
class ShardedResult:
    U: list
    core: torch.Tensor
    sigma: list
    err: torch.Tensor | None
    info: dict
    rc: int
    exchanges: list  # (ws_offset, count, dtype, op) of every all-reduce, in call order


def hosvd_fused_sharded(grid, kernel, ranks, shard: int, nshards: int, group=None, with_error: bool = True,
                        ws: torch.Tensor | None = None, stream=None) -> ShardedResult:
    """Row (e): this rank's share of ONE fused HOSVD (+ error) sharded over `nshards` ranks
    (tucker_hosvd_fused_sharded).  The exchange steps are torch.distributed all-reduces on views of
    the workspace (`group`: the process group; NCCL over NVLink in production, gloo in the
    one-GPU tests) — argument marshalling only, the arithmetic is the library's."""
    lib = load()
    r = tuple(int(v) for v in ranks)
    U = [torch.empty((int(grid.n[m]), r[m]), dtype=torch.float64, device="cuda") for m in range(3)]
    S = [torch.empty(r[m], dtype=torch.float64, device="cuda") for m in range(3)]
    core = torch.empty(r, dtype=torch.float64, device="cuda")
    err = torch.empty(3, dtype=torch.float64, device="cuda") if with_error else None
    ws = ws if ws is not None else workspace_fused(grid, r)
    exchanges, failure = [], []

    def _allreduce(user, off, count, dtype, op):
        try:
            import torch.distributed as dist
            tdt, esz = (torch.int32, 4) if dtype == DT_INT32 else (torch.float64, 8)
            view = ws[off: off + count * esz].view(tdt)
            dist.all_reduce(view, op=dist.ReduceOp.MAX if op == RED_MAX else dist.ReduceOp.SUM, group=group)
            torch.cuda.synchronize()
            exchanges.append((int(off), int(count), int(dtype), int(op)))
            return 0
        except Exception as e:  # reported to the library as TUCKER_ERR_COLLECTIVE
            failure.append(e)
            return 1

    cb = ALLREDUCE_FN(_allreduce)
    info = CInfo()
    g, k = cgrid(grid), ckernel(kernel)
    rc = lib.tucker_hosvd_fused_sharded(ctypes.byref(g), ctypes.byref(k), cranks(r), int(shard), int(nshards), cb,
                                        None, _ptr(U[0]), _ptr(U[1]), _ptr(U[2]), _ptr(core), _ptr(S[0]),
                                        _ptr(S[1]), _ptr(S[2]), _ptr(err) if err is not None else None, _ptr(ws),
                                        ws.numel(), _stream(stream), ctypes.byref(info))
    if failure:
        raise TuckerError(8, f"tucker_hosvd_fused_sharded: all-reduce failed: {failure[0]!r}")
    if rc not in (0, 5):
        _check(rc, "tucker_hosvd_fused_sharded")
    return ShardedResult(U, core, S, err, info.as_dict(), rc, exchanges)


def error_fused(grid, kernel, ranks, U, core, ws=None, stream=None) -> torch.Tensor:
    lib = load()
    out = torch.empty(3, dtype=torch.float64, device="cuda")
    ws = ws if ws is not None else workspace_fused(grid, ranks)
    g, k = cgrid(grid), ckernel(kernel)
    _check(lib.tucker_error_fused(ctypes.byref(g), ctypes.byref(k), cranks(ranks), _ptr(U[0]), _ptr(U[1]),
                                  _ptr(U[2]), _ptr(core), _ptr(out), _ptr(ws), ws.numel(), _stream(stream)),
           "tucker_error_fused")
    return out


@dataclass
class HostResult:
    U: list
    core: np.ndarray
    sigma: list
    err: np.ndarray
    info: dict
    rc: int


class HostBuffers:
    """Pinned host output buffers for tucker_approximate."""

    def __init__(self, grid, ranks):
        r = tuple(int(v) for v in ranks)
        self.U = [torch.empty((int(grid.n[m]), r[m]), dtype=torch.float64).pin_memory() for m in range(3)]
        self.sigma = [torch.empty(r[m], dtype=torch.float64).pin_memory() for m in range(3)]
        self.core = torch.empty(r, dtype=torch.float64).pin_memory()
        self.err = torch.empty(3, dtype=torch.float64).pin_memory()

    @property
    def d2h_bytes(self) -> int:
        return 8 * (sum(u.numel() for u in self.U) + sum(s.numel() for s in self.sigma) + self.core.numel() + 3)


def approximate(grid, kernel, ranks, F: torch.Tensor, ws: torch.Tensor, host: HostBuffers, stream=None) -> HostResult:
    """The end-to-end call: fill + HOSVD + error on the device, factors/core/sigma/E to host."""
    lib = load()
    _dev(F, "F")
    g, k = cgrid(grid), ckernel(kernel)
    info = CInfo()
    Uh = (ctypes.c_void_p * 3)(*[u.data_ptr() for u in host.U])
    Sh = (ctypes.c_void_p * 3)(*[s.data_ptr() for s in host.sigma])
    rc = lib.tucker_approximate(ctypes.byref(g), ctypes.byref(k), cranks(ranks), _ptr(F), Uh,
                                ctypes.c_void_p(host.core.data_ptr()), Sh, ctypes.c_void_p(host.err.data_ptr()),
                                _ptr(ws), ws.numel(), _stream(stream), ctypes.byref(info))
    if rc not in (0, 5):
        _check(rc, "tucker_approximate")
    return HostResult([u.numpy() for u in host.U], host.core.numpy(), [s.numpy() for s in host.sigma],
                      host.err.numpy(), info.as_dict(), rc)
