"""CPU FP64 oracle for the Tucker/HOSVD hot path of arXiv 1711.06874 — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this module.  The product package ``paper_1711_06874_b200`` never
imports it, and the two share no code: this file wraps ``oracle/tucker_oracle.c`` (plain C, OpenMP,
Dot2-compensated sums, cyclic Jacobi) with ctypes and numpy arrays.

Citations are to ``/root/reference/PAPER.md`` lines (``P:n``); readings R1..R14 are in DESIGN.md §3.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tucker_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

MATERN, SLATER, MATERN_SPECTRAL = 0, 1, 2
FORCE_GENERAL_BESSEL = 2


def build(force: bool = False) -> str:
    """Compile the oracle (gcc, -O2 -ffp-contract=off, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=gnu11", "-ffp-contract=off", "-mfma", "-fopenmp", "-fPIC",
               "-shared", "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


class OrcGrid(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64 * 3), ("lo", ctypes.c_double * 3), ("hi", ctypes.c_double * 3)]


class OrcKernel(ctypes.Structure):
    _fields_ = [("family", ctypes.c_int32), ("flags", ctypes.c_int32), ("sigma2", ctypes.c_double),
                ("ell", ctypes.c_double), ("nu", ctypes.c_double), ("lam", ctypes.c_double),
                ("p", ctypes.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        d, i64, i32 = ctypes.c_double, ctypes.c_int64, ctypes.c_int
        P = ctypes.POINTER
        pd = P(d)
        pi64 = P(i64)
        sig = {
            "orc_nodes": (None, [i64, d, d, pd]),
            "orc_besselk": (d, [d, d]),
            "orc_besselk_scaled": (d, [d, d]),
            "orc_besselk_series_scaled": (d, [d, d]),
            "orc_besselk_hankel_scaled": (d, [d, d]),
            "orc_besselk_trapz_scaled": (d, [d, d]),
            "orc_kernel_eval": (d, [P(OrcKernel), d, d]),
            "orc_kernel_check": (i32, [P(OrcKernel)]),
            "orc_fill": (i32, [P(OrcGrid), P(OrcKernel), pd]),
            "orc_fill_entry": (d, [P(OrcGrid), P(OrcKernel), i64, i64, i64]),
            "orc_unfold": (None, [pd, pi64, i32, pd]),
            "orc_gram": (None, [pd, i64, i64, pd]),
            "orc_gram_entry_fn": (d, [P(OrcGrid), P(OrcKernel), i32, i64, i64]),
            "orc_row_stats_fn": (None, [P(OrcGrid), P(OrcKernel), i32, i64, pd]),
            "orc_jacobi_eig": (i32, [i64, pd, pd, pd, i32, P(i32)]),
            "orc_sign_fix": (None, [i64, i64, pd, i64]),
            "orc_ttm_core": (None, [pd, pi64, pi64, pd, pd, pd, pd]),
            "orc_reconstruct": (None, [pi64, pi64, pd, pd, pd, pd, pd]),
            "orc_tucker_error": (None, [pd, pi64, pi64, pd, pd, pd, pd, pd]),
            "orc_hosvd": (i32, [pd, pi64, pi64, pd, pd, pd, pd, pd, pd, pd]),
            "orc_hooi": (i32, [pd, pi64, pi64, pd, pd, pd, i32]),
            "orc_tucker_point": (d, [pi64, pd, pd, pd, pd, i64, i64, i64]),
            "orc_num_threads": (i32, []),
            "orc_set_num_threads": (None, [i32]),
        }
        for name, (res, args) in sig.items():
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args
    return _lib


def _pd(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _pi64(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


@dataclass(frozen=True)
class Grid:
    """Axes-parallel box [lo_m, hi_m] with n_m collocation nodes per axis."""
    n: tuple
    lo: tuple
    hi: tuple

    @staticmethod
    def cube(n: int, b: float) -> "Grid":
        return Grid((n, n, n), (-b, -b, -b), (b, b, b))

    def c(self) -> OrcGrid:
        g = OrcGrid()
        for a in range(3):
            g.n[a], g.lo[a], g.hi[a] = int(self.n[a]), float(self.lo[a]), float(self.hi[a])
        return g


@dataclass(frozen=True)
class Kernel:
    """Matérn or p-Slater kernel parameters."""
    family: int = MATERN
    sigma2: float = 1.0
    ell: float = 1.0
    nu: float = 0.5
    lam: float = 1.0
    p: float = 1.0
    flags: int = 0

    @staticmethod
    def matern(nu, ell, sigma2=1.0, flags=0):
        return Kernel(MATERN, sigma2, ell, nu, 1.0, 1.0, flags)

    @staticmethod
    def slater(lam=1.0, p=1.0, sigma2=1.0):
        return Kernel(SLATER, sigma2, 1.0, 0.5, lam, p, 0)

    @staticmethod
    def spectral(alpha, nu, sigma2=1.0):
        """Matérn spectral density C (alpha^2 + rho^2)^{-(nu + 3/2)}, alpha in `lam`."""
        return Kernel(MATERN_SPECTRAL, sigma2, 1.0, nu, alpha, 1.0, 0)

    def c(self) -> OrcKernel:
        return OrcKernel(self.family, self.flags, self.sigma2, self.ell, self.nu, self.lam, self.p)


# ---------------------------------------------------------------------------------------------
def nodes(n: int, lo: float, hi: float) -> np.ndarray:
    x = np.empty(n, dtype=np.float64)
    lib().orc_nodes(n, lo, hi, _pd(x))
    return x


def besselk(nu: float, z: float) -> float:
    return lib().orc_besselk(nu, z)


def besselk_scaled(nu: float, z: float, route: str = "auto") -> float:
    f = {"auto": lib().orc_besselk_scaled, "series": lib().orc_besselk_series_scaled,
         "hankel": lib().orc_besselk_hankel_scaled, "trapz": lib().orc_besselk_trapz_scaled}[route]
    return f(nu, z)


def kernel_eval(k: Kernel, r: float) -> float:
    kc = k.c()
    return lib().orc_kernel_eval(ctypes.byref(kc), float(r), float(r) * float(r))


def fill(g: Grid, k: Kernel) -> np.ndarray:
    F = np.empty(tuple(int(v) for v in g.n), dtype=np.float64)
    gc, kc = g.c(), k.c()
    rc = lib().orc_fill(ctypes.byref(gc), ctypes.byref(kc), _pd(F))
    if rc:
        raise ValueError(f"orc_fill: error {rc}")
    return F


def fill_entry(g: Grid, k: Kernel, i: int, j: int, l: int) -> float:
    gc, kc = g.c(), k.c()
    return lib().orc_fill_entry(ctypes.byref(gc), ctypes.byref(kc), i, j, l)


def unfold(F: np.ndarray, mode: int) -> np.ndarray:
    n = F.shape[mode]
    A = np.empty((n, F.size // n), dtype=np.float64)
    dims, pdims = _pi64(F.shape)
    lib().orc_unfold(_pd(F), pdims, mode, _pd(A))
    return A


def gram(A: np.ndarray) -> np.ndarray:
    A = np.ascontiguousarray(A, dtype=np.float64)
    G = np.empty((A.shape[0], A.shape[0]), dtype=np.float64)
    lib().orc_gram(_pd(A), A.shape[0], A.shape[1], _pd(G))
    return G


def gram_mode(F: np.ndarray, mode: int) -> np.ndarray:
    return gram(unfold(F, mode))


def gram_entry_fn(g: Grid, k: Kernel, mode: int, a: int, b: int) -> float:
    gc, kc = g.c(), k.c()
    return lib().orc_gram_entry_fn(ctypes.byref(gc), ctypes.byref(kc), mode, a, b)


def row_stats_fn(g: Grid, k: Kernel, mode: int, a: int):
    """(max_k |A_(m)[a,k]|, sum_k |A_(m)[a,k]|) of one unfolding row, from the kernel directly."""
    gc, kc = g.c(), k.c()
    out = np.empty(2)
    lib().orc_row_stats_fn(ctypes.byref(gc), ctypes.byref(kc), mode, a, _pd(out))
    return float(out[0]), float(out[1])


def jacobi_eig(G: np.ndarray, max_sweeps: int = 100):
    """Eigenvalues (descending) and sign-fixed eigenvectors (columns) by cyclic Jacobi."""
    G = np.ascontiguousarray(G, dtype=np.float64)
    n = G.shape[0]
    lam = np.empty(n)
    V = np.empty((n, n))
    sw = ctypes.c_int(0)
    rc = lib().orc_jacobi_eig(n, _pd(G), _pd(lam), _pd(V), max_sweeps, ctypes.byref(sw))
    return lam, V, rc, sw.value


def sign_fix(V: np.ndarray) -> np.ndarray:
    V = np.ascontiguousarray(V, dtype=np.float64).copy()
    lib().orc_sign_fix(V.shape[0], V.shape[1], _pd(V), V.shape[1])
    return V


def ttm_core(F, U1, U2, U3) -> np.ndarray:
    r = (U1.shape[1], U2.shape[1], U3.shape[1])
    core = np.empty(r)
    d, pdims = _pi64(F.shape)
    rr, pr = _pi64(r)
    Us = [np.ascontiguousarray(u, dtype=np.float64) for u in (U1, U2, U3)]
    lib().orc_ttm_core(_pd(np.ascontiguousarray(F)), pdims, pr, _pd(Us[0]), _pd(Us[1]), _pd(Us[2]),
                       _pd(core))
    return core


def reconstruct(shape, U1, U2, U3, core) -> np.ndarray:
    Us = [np.ascontiguousarray(u, dtype=np.float64) for u in (U1, U2, U3)]
    r = tuple(u.shape[1] for u in Us)
    Ft = np.empty(tuple(shape))
    d, pdims = _pi64(shape)
    rr, pr = _pi64(r)
    lib().orc_reconstruct(pdims, pr, _pd(Us[0]), _pd(Us[1]), _pd(Us[2]),
                          _pd(np.ascontiguousarray(core, dtype=np.float64)), _pd(Ft))
    return Ft


def tucker_error(F, U1, U2, U3, core):
    """(E, ||F||, ||F - Ft||), eq. (FNorm) P:1016-1025."""
    Us = [np.ascontiguousarray(u, dtype=np.float64) for u in (U1, U2, U3)]
    r = tuple(u.shape[1] for u in Us)
    out = np.empty(3)
    d, pdims = _pi64(F.shape)
    rr, pr = _pi64(r)
    lib().orc_tucker_error(_pd(np.ascontiguousarray(F)), pdims, pr, _pd(Us[0]), _pd(Us[1]),
                           _pd(Us[2]), _pd(np.ascontiguousarray(core, dtype=np.float64)), _pd(out))
    return float(out[0]), float(out[1]), float(out[2])


@dataclass
class Hosvd:
    U: list          # [U1, U2, U3], n_m x r_m
    core: np.ndarray  # r1 x r2 x r3
    lam: list        # full spectra of G_m, descending
    rc: int

    @property
    def sigma(self):
        return [np.sqrt(np.maximum(l[: u.shape[1]], 0.0)) for l, u in zip(self.lam, self.U)]


def hosvd(F: np.ndarray, r) -> Hosvd:
    """Truncated HOSVD with the full eigen-spectra of each G_m."""
    F = np.ascontiguousarray(F, dtype=np.float64)
    r = tuple(int(v) for v in r)
    U = [np.empty((F.shape[m], r[m])) for m in range(3)]
    lam = [np.empty(F.shape[m]) for m in range(3)]
    core = np.empty(r)
    d, pdims = _pi64(F.shape)
    rr, pr = _pi64(r)
    rc = lib().orc_hosvd(_pd(F), pdims, pr, _pd(U[0]), _pd(U[1]), _pd(U[2]), _pd(core),
                         _pd(lam[0]), _pd(lam[1]), _pd(lam[2]))
    return Hosvd(U, core, lam, rc)


def hosvd_svd(F: np.ndarray, r) -> Hosvd:
    """Truncated HOSVD by the SVD of each explicit unfolding, as the paper computes it
    ("SVD of the matrix unfolding A_(l)").  The SVD is LAPACK's (numpy.linalg.svd, a
    library primitive); no Gram is formed, so singular values are resolved down to ~eps sigma_1
    (the reference for NEXT f2).  `lam` holds sigma^2 of the full spectra; U sign-fixed by R6."""
    F = np.ascontiguousarray(F, dtype=np.float64)
    U, lam = [], []
    for m in range(3):
        W, sv, _ = np.linalg.svd(unfold(F, m), full_matrices=False)
        U.append(sign_fix(W[:, : r[m]]))
        lam.append(sv ** 2)
    core = ttm_core(F, *U)
    return Hosvd(U, core, lam, 0)


def hooi(F: np.ndarray, U_init, sweeps: int):
    """Test-only Tucker-ALS sweeps starting from U_init; returns (U, core, rc)."""
    F = np.ascontiguousarray(F, dtype=np.float64)
    U = [np.ascontiguousarray(u, dtype=np.float64).copy() for u in U_init]
    r = tuple(u.shape[1] for u in U)
    d, pdims = _pi64(F.shape)
    rr, pr = _pi64(r)
    rc = lib().orc_hooi(_pd(F), pdims, pr, _pd(U[0]), _pd(U[1]), _pd(U[2]), sweeps)
    core = ttm_core(F, *U)
    return U, core, rc


def tucker_point(U, core, i, j, l) -> float:
    Us = [np.ascontiguousarray(u, dtype=np.float64) for u in U]
    r = tuple(u.shape[1] for u in Us)
    rr, pr = _pi64(r)
    return lib().orc_tucker_point(pr, _pd(Us[0]), _pd(Us[1]), _pd(Us[2]),
                                  _pd(np.ascontiguousarray(core, dtype=np.float64)), i, j, l)


def num_threads() -> int:
    return lib().orc_num_threads()


def set_num_threads(t: int) -> None:
    lib().orc_set_num_threads(int(t))
