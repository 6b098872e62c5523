"""Pins for the oracle's grid nodes and collocation fill."""
import math

import mpmath as mp
import numpy as np
import pytest


@pytest.mark.parametrize("n,lo,hi", [(5, -2.0, 2.0), (32, -1.0, 1.0), (129, -5.0, 5.0),
                                     (192, -1.5, 1.5), (7, -0.3, 2.9), (1024, -1.0, 1.0)])
def test_nodes_match_paper_formula(orc, n, lo, hi):
    # x_i = -b + (i-1) h, h = 2b/(n-1) (per axis [lo,hi]); exact-rational reference
    x = orc.nodes(n, lo, hi)
    from fractions import Fraction
    flo, fhi = Fraction(lo), Fraction(hi)
    h = (fhi - flo) / (n - 1)
    for i in range(n):
        ref = float(flo + i * h)
        assert abs(x[i] - ref) <= 2 * np.spacing(max(abs(ref), abs(hi - lo) / (n - 1)))
    assert np.all(np.diff(x) > 0)
    if lo == -hi:  # endpoints exact on centred boxes (c = 0); otherwise within the bound above
        assert x[0] == lo and x[-1] == hi


def test_nodes_mirror_exact(orc):
    for n in (4, 5, 32, 129, 256, 1024):
        x = orc.nodes(n, -1.0, 1.0)
        assert np.array_equal(x, -x[::-1])
    assert list(orc.nodes(5, -2.0, 2.0)) == [-2.0, -1.0, 0.0, 1.0, 2.0]


def test_spec_collocation_examples(orc):
    # 3D Slater e^{-||x||} on n=9, b=1: centre 1.0, corner e^{-sqrt 3}
    F = orc.fill(orc.Grid.cube(9, 1.0), orc.Kernel.slater(1.0, 1.0))
    assert F[4, 4, 4] == 1.0
    assert F[0, 0, 0] == pytest.approx(math.exp(-math.sqrt(3.0)), rel=2e-16)
    # S:111 (1-D example lifted to 3-D): exponential, n=5, b=2, line through the centre
    F = orc.fill(orc.Grid.cube(5, 2.0), orc.Kernel.matern(0.5, 1.0))
    ref = [math.exp(-2), math.exp(-1), 1.0, math.exp(-1), math.exp(-2)]
    assert np.allclose(F[2, 2, :], ref, rtol=2e-16, atol=0)


def test_reflection_symmetry(orc):
    # radial function on a centred grid: reversing any axis leaves F unchanged, bitwise
    g = orc.Grid((12, 9, 10), (-2.0, -1.5, -1.0), (2.0, 1.5, 1.0))
    for k in (orc.Kernel.matern(1.3, 0.5), orc.Kernel.matern(1.5, 0.2), orc.Kernel.slater(5.0)):
        F = orc.fill(g, k)
        for ax in range(3):
            assert np.array_equal(F, np.flip(F, axis=ax))


def test_gaussian_separable(orc):
    # e^{-||x||^2} = prod_m e^{-x_m^2}  (Slater p=2)
    g = orc.Grid((10, 11, 12), (-1.0, -2.0, -0.5), (1.0, 1.5, 3.0))
    F = orc.fill(g, orc.Kernel.slater(1.0, 2.0))
    v = [np.exp(-orc.nodes(g.n[a], g.lo[a], g.hi[a]) ** 2) for a in range(3)]
    ref = np.einsum("i,j,k->ijk", *v)
    assert np.max(np.abs(F - ref) / ref) <= 5e-15


def test_fill_entries_vs_mpmath(orc):
    # random entries of the collocation tensor against eq. (Matern) in 40 digits
    mp.mp.dps = 40
    g = orc.Grid((24, 20, 16), (-2.0, -1.5, -1.0), (2.0, 1.5, 1.0))
    rng = np.random.default_rng(7)
    for nu, ell in ((0.3, 0.5), (1.3, 0.5), (1.5, 0.2), (2.1, 0.05)):
        k = orc.Kernel.matern(nu, ell)
        F = orc.fill(g, k)
        xs = [orc.nodes(g.n[a], g.lo[a], g.hi[a]) for a in range(3)]
        for _ in range(20):
            i, j, l = (int(rng.integers(g.n[a])) for a in range(3))
            r = mp.sqrt(mp.mpf(xs[0][i]) ** 2 + mp.mpf(xs[1][j]) ** 2 + mp.mpf(xs[2][l]) ** 2)
            z = mp.sqrt(2 * mp.mpf(nu)) * r / mp.mpf(ell)
            ref = 2 ** (1 - mp.mpf(nu)) / mp.gamma(nu) * z ** nu * mp.besselk(nu, z)
            # conditioning: rounding r and z to FP64 perturbs e^{-z} by ~z*eps relative
            tol = 6e-15 + 4e-16 * float(z)
            assert abs(F[i, j, l] - float(ref)) <= tol * float(ref)
            assert F[i, j, l] == orc.fill_entry(g, k, i, j, l)


def test_fill_domain_errors(orc):
    g = orc.Grid.cube(4, 1.0)
    for k in (orc.Kernel.matern(0.0, 1.0), orc.Kernel.matern(1.0, -1.0), orc.Kernel.slater(1.0, 2.5),
              orc.Kernel.matern(1.0, 1.0, sigma2=0.0)):
        with pytest.raises(ValueError):
            orc.fill(g, k)


# ------------------------------------------------------------- NEXT f4: Matérn spectral density
def test_spectral_density_exact_values(orc):
    """f(rho) = C (alpha^2 + rho^2)^{-(nu + d/2)}, d = 3, C = sigma^2 (R17).  On the
    n = 3 grid of [-1,1]^3 rho^2 is an integer 0..3; with alpha = 1 the base is 1..4, so the values
    are the rationals 1/(1+rho^2)^s (exact for powers of two, correctly rounded otherwise)."""
    from fractions import Fraction
    g = orc.Grid.cube(3, 1.0)
    for nu, s in ((0.5, 2), (1.5, 3), (2.5, 4)):
        F = orc.fill(g, orc.Kernel.spectral(1.0, nu))
        for i in range(3):
            for j in range(3):
                for k in range(3):
                    rho2 = (i - 1) ** 2 + (j - 1) ** 2 + (k - 1) ** 2
                    ref = Fraction(1, (1 + rho2) ** s)
                    v = F[i, j, k]
                    if (1 + rho2) in (1, 2, 4):
                        assert v == float(ref), (nu, rho2)
                    else:
                        assert abs(Fraction(v) - ref) <= Fraction(np.spacing(float(ref))), (nu, rho2)
    F2 = orc.fill(g, orc.Kernel.spectral(1.0, 0.5, sigma2=2.0))
    assert np.array_equal(F2, 2.0 * orc.fill(g, orc.Kernel.spectral(1.0, 0.5)))


def test_spectral_density_against_mpmath(orc):
    g = orc.Grid((7, 6, 5), (-3.0, -2.0, -1.0), (3.0, 2.5, 1.0))
    x = [orc.nodes(g.n[a], g.lo[a], g.hi[a]) for a in range(3)]
    for alpha, nu in ((0.1, 0.4), (1.7, 1.1), (100.0, 0.4)):
        F = orc.fill(g, orc.Kernel.spectral(alpha, nu))
        for (i, j, k) in ((0, 0, 0), (3, 2, 1), (6, 5, 4), (2, 4, 0)):
            with mp.workdps(40):
                rho2 = mp.mpf(x[0][i]) ** 2 + mp.mpf(x[1][j]) ** 2 + mp.mpf(x[2][k]) ** 2
                # exponent s = fl(nu + 3/2): the method's own double exponent (ln(base) amplifies a
                # 1-ulp exponent difference to ~10 ulp of the result)
                ref = float((mp.mpf(alpha) ** 2 + rho2) ** (-mp.mpf(nu + 1.5)))
            assert abs(F[i, j, k] - ref) <= 4 * np.spacing(ref), (alpha, nu, i, j, k)


def test_spectral_density_rank_depends_on_alpha(orc):
    """the Tucker rank depends strongly on alpha — large alpha makes f nearly constant
    (f ~ alpha^{-2s}(1 - s rho^2/alpha^2), separable to O(alpha^-4)), small alpha a sharp peak."""
    g = orc.Grid.cube(24, 1.0)
    err = {}
    for alpha in (0.1, 100.0):
        F = orc.fill(g, orc.Kernel.spectral(alpha, 0.4))
        h = orc.hosvd(F, (8, 8, 8))
        E = []
        for r in range(1, 9):
            U = [u[:, :r] for u in h.U]
            core = orc.ttm_core(F, *U)
            E.append(orc.tucker_error(F, *U, core)[0])
        assert all(b <= a * (1 + 1e-12) + 1e-15 for a, b in zip(E, E[1:]))
        err[alpha] = E
    assert err[100.0][0] < 1e-8            # alpha = 100: rank 1 already at the Gram route's floor
    assert err[0.1][1] > 1e-2              # alpha = 0.1: many more terms (measured 2.5e-2 at r = 2)
    assert err[0.1][5] > 1e3 * err[100.0][5] and err[0.1][7] > 1e2 * err[100.0][7]
