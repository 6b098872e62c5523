"""Pins for the oracle's K_nu and kernel families.

Each check is independent of the oracle's own formulas: mpmath's arbitrary-precision besselk,
textbook closed forms of half-integer K_nu, the three-term recurrence, the Wronskian, the small-z
limit, and SPEC.md's worked examples.
"""
import math

import mpmath as mp
import numpy as np
import pytest
import scipy.special as sp

NUS = [0.3, 0.5, 0.7, 0.77, 1.0, 1.3, 1.5, 1.999, 2.1, 2.5]
ZS = np.geomspace(5e-4, 80.0, 41)


@pytest.mark.parametrize("nu", NUS)
def test_besselk_vs_mpmath(orc, nu):
    mp.mp.dps = 40
    worst = 0.0
    for z in ZS:
        ref = mp.besselk(nu, z) * mp.exp(z)
        v = orc.besselk_scaled(nu, float(z))
        worst = max(worst, abs(v - float(ref)) / float(ref))
    assert worst <= 5e-15, worst


def test_besselk_vs_scipy(orc):
    # library routine; scipy's kve itself is only good to ~5e-14 for some (nu, z)
    for nu in NUS:
        for z in ZS:
            ref = sp.kve(nu, z)
            assert abs(orc.besselk_scaled(nu, float(z)) - ref) <= 1e-13 * ref


def test_half_integer_closed_forms(orc):
    # K_{1/2} = sqrt(pi/2z) e^{-z}, K_{3/2} = K_{1/2}(1 + 1/z), K_{5/2} = K_{1/2}(1 + 3/z + 3/z^2)
    for z in ZS:
        base = math.sqrt(math.pi / (2 * z))
        for nu, poly in ((0.5, 1.0), (1.5, 1 + 1 / z), (2.5, 1 + 3 / z + 3 / z ** 2)):
            ref = base * poly
            assert abs(orc.besselk_scaled(nu, float(z)) - ref) <= 4e-15 * ref


def test_recurrence(orc):
    # K_{nu+1}(z) = K_{nu-1}(z) + (2 nu / z) K_nu(z)  (DLMF 10.29.1); all terms positive
    for nu in (1.1, 1.3, 1.5, 1.77):
        for z in ZS:
            z = float(z)
            lhs = orc.besselk_scaled(nu + 1, z)
            rhs = orc.besselk_scaled(nu - 1, z) + 2 * nu / z * orc.besselk_scaled(nu, z)
            assert abs(lhs - rhs) <= 1e-14 * lhs


def test_wronskian(orc):
    # I_nu K_{nu+1} + I_{nu+1} K_nu = 1/z (DLMF 10.28.2), with I from scipy (ive: scaled by e^-z)
    for nu in (0.3, 0.7, 1.3, 2.1):
        for z in np.geomspace(1e-2, 60.0, 25):
            z = float(z)
            w = sp.ive(nu, z) * orc.besselk_scaled(nu + 1, z) + sp.ive(nu + 1, z) * orc.besselk_scaled(nu, z)
            assert abs(w * z - 1.0) <= 1e-13


def test_small_z_limit(orc):
    # z^nu K_nu(z) -> 2^{nu-1} Gamma(nu) as z -> 0 (DLMF 10.30.2); correction O(z^{2 min(nu,1)})
    for nu in (0.7, 1.3, 2.1):
        z = 1e-7
        v = z ** nu * orc.besselk(nu, z)
        ref = 2 ** (nu - 1) * math.gamma(nu)
        assert abs(v - ref) <= 1e-8 * ref


def test_regime_overlap(orc):
    mp.mp.dps = 30
    for nu in (0.3, 1.3, 2.1):
        for z in np.linspace(0.1, 1.0, 10):
            a, b = orc.besselk_scaled(nu, float(z), "series"), orc.besselk_scaled(nu, float(z), "trapz")
            assert abs(a - b) <= 5e-15 * b
        for z in np.linspace(20.0, 80.0, 13):
            a, b = orc.besselk_scaled(nu, float(z), "hankel"), orc.besselk_scaled(nu, float(z), "trapz")
            assert abs(a - b) <= 2e-15 * b


# ------------------------------------------------------------------------------------------
def test_spec_examples(orc):
    K = orc.Kernel
    # S:43  Matern nu=1/2, ell=1, r=1 -> e^-1
    assert orc.kernel_eval(K.matern(0.5, 1.0), 1.0) == pytest.approx(math.exp(-1.0), rel=1e-15)
    # S:44  r = 0 -> sigma^2 for any (nu, ell)
    for nu in (0.3, 0.5, 1.3, 2.5):
        assert orc.kernel_eval(K.matern(nu, 0.7, sigma2=2.5), 0.0) == 2.5
    # S:45  Slater p=2, r=1.5 -> e^{-2.25}
    assert orc.kernel_eval(K.slater(1.0, 2.0), 1.5) == pytest.approx(math.exp(-2.25), rel=1e-15)


def test_exponential_model_1000_points(orc):
    # P:365-366 / S:69: nu = 1/2 is the exponential model, to 1e-12 over r in [0, 10 ell]
    K = orc.Kernel
    ell = 0.37
    for r in np.linspace(0.0, 10 * ell, 1000):
        v = orc.kernel_eval(K.matern(0.5, ell, flags=orc.FORCE_GENERAL_BESSEL), float(r))
        assert abs(v - math.exp(-r / ell)) <= 1e-12


@pytest.mark.parametrize("nu", [0.5, 1.5, 2.5])
def test_closed_forms_vs_general_path(orc, nu):
    # P:356 with half-integer nu: the closed forms and the general K_nu route agree to 1e-14
    K = orc.Kernel
    for ell in (0.05, 0.2, 1.0):
        for r in np.geomspace(1e-4, 1.8, 60):
            a = orc.kernel_eval(K.matern(nu, ell), float(r))
            b = orc.kernel_eval(K.matern(nu, ell, flags=orc.FORCE_GENERAL_BESSEL), float(r))
            assert abs(a - b) <= 1e-14 * abs(a) + 1e-300


def test_matern_vs_mpmath(orc):
    # eq. (Matern) P:356-357 evaluated in 40-digit arithmetic
    mp.mp.dps = 40
    K = orc.Kernel
    for nu in (0.3, 0.7, 1.3, 2.1):
        for ell in (0.05, 0.5):
            for r in np.geomspace(3e-3, 1.8, 15):
                z = mp.sqrt(2 * mp.mpf(nu)) * mp.mpf(float(r)) / mp.mpf(ell)
                ref = 2 ** (1 - mp.mpf(nu)) / mp.gamma(nu) * z ** nu * mp.besselk(nu, z)
                v = orc.kernel_eval(K.matern(nu, ell), float(r))
                assert abs(v - float(ref)) <= 6e-15 * float(ref)
