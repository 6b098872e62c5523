"""Seeded synthetic workloads shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no kernel evaluation, no grid nodes, no Gram,
no eigensolver): only the problem parameters of BASELINE.json's configs and the counter-based
generator that draws config 4's Matérn settings (reading R10 in DESIGN.md).  The paper's
workloads are analytic functions on grids; there is no dataset to stand in for.
"""
from __future__ import annotations

from dataclasses import dataclass, field

MATERN, SLATER, MATERN_SPECTRAL = 0, 1, 2
SEED_CONFIG4 = 171106874


@dataclass(frozen=True)
class GridSpec:
    n: tuple
    lo: tuple
    hi: tuple

    @staticmethod
    def cube(n: int, b: float = 1.0) -> "GridSpec":
        return GridSpec((n, n, n), (-b, -b, -b), (b, b, b))

    @property
    def points(self) -> int:
        return int(self.n[0]) * int(self.n[1]) * int(self.n[2])


@dataclass(frozen=True)
class KernelSpec:
    family: int = MATERN
    sigma2: float = 1.0
    ell: float = 1.0
    nu: float = 0.5
    lam: float = 1.0
    p: float = 1.0
    flags: int = 0

    @staticmethod
    def matern(nu: float, ell: float, sigma2: float = 1.0, flags: int = 0) -> "KernelSpec":
        return KernelSpec(MATERN, sigma2, ell, nu, 1.0, 1.0, flags)

    @staticmethod
    def slater(lam: float = 1.0, p: float = 1.0, sigma2: float = 1.0) -> "KernelSpec":
        return KernelSpec(SLATER, sigma2, 1.0, 0.5, lam, p, 0)

    @staticmethod
    def spectral(alpha: float, nu: float, sigma2: float = 1.0) -> "KernelSpec":
        """Matérn spectral density sigma2 (alpha^2 + rho^2)^{-(nu + 3/2)} (NEXT f4)."""
        return KernelSpec(MATERN_SPECTRAL, sigma2, 1.0, nu, alpha, 1.0, 0)

    def label(self) -> str:
        if self.family == MATERN_SPECTRAL:
            return f"spectral(alpha={self.lam:g},nu={self.nu:g})"
        if self.family == SLATER:
            return f"slater(lam={self.lam:g},p={self.p:g})"
        return f"matern(nu={self.nu:.6g},ell={self.ell:.6g})"


@dataclass(frozen=True)
class Workload:
    name: str
    grid: GridSpec
    kernels: tuple
    ranks: tuple
    extra: dict = field(default_factory=dict)


class SplitMix64:
    """SplitMix64 (Steele, Lea, Flood 2014); u = (next() >> 11) * 2^-53 in [0, 1)."""

    def __init__(self, seed: int):
        self.state = seed & 0xFFFFFFFFFFFFFFFF

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
        return z ^ (z >> 31)

    def uniform(self) -> float:
        return (self.next() >> 11) * (1.0 / 9007199254740992.0)


def config4_settings(seed: int = SEED_CONFIG4, count: int = 16) -> tuple:
    """BASELINE.json config 4: nu ~ U[0.5, 2.5], ell log-uniform in [0.05, 1] (reading R10)."""
    rng = SplitMix64(seed)
    out = []
    for _ in range(count):
        u0, u1 = rng.uniform(), rng.uniform()
        out.append(KernelSpec.matern(0.5 + 2.0 * u0, 0.05 * 20.0 ** u1))
    return tuple(out)


def config1() -> Workload:
    return Workload("cfg1_32cube_matern_nu0.5", GridSpec.cube(32, 1.0),
                    (KernelSpec.matern(0.5, 0.5),), (8, 8, 8))


def config2() -> Workload:
    ks = tuple(KernelSpec.matern(nu, ell) for nu in (0.5, 1.5, 2.5) for ell in (0.1, 0.5, 1.0))
    return Workload("cfg2_128cube_closed_forms", GridSpec.cube(128, 1.0), ks, (20, 20, 20))


def config3() -> Workload:
    ks = tuple(KernelSpec.matern(nu, 0.5) for nu in (0.3, 0.7, 1.3, 2.1)) + \
        (KernelSpec.slater(1.0), KernelSpec.slater(5.0))
    g = GridSpec((256, 192, 128), (-2.0, -1.5, -1.0), (2.0, 1.5, 1.0))
    return Workload("cfg3_aniso_256x192x128_general_nu", g, ks, (12, 12, 10))


def config4() -> Workload:
    return Workload("cfg4_512cube_batch16", GridSpec.cube(512, 1.0), config4_settings(), (30, 30, 30))


def config5(ranks=(40, 40, 40)) -> Workload:
    return Workload("cfg5_1024cube_matern_nu1.5_ell0.2", GridSpec.cube(1024, 1.0),
                    (KernelSpec.matern(1.5, 0.2),), tuple(ranks))


def table2(n: int) -> Workload:
    """Table 2: Slater e^{-||x||} on a (2k+1)^3 grid; box [-5,5]^3 (reading R1)."""
    return Workload(f"table2_n{n}", GridSpec.cube(n, 5.0), (KernelSpec.slater(1.0, 1.0),), (10, 10, 10))
