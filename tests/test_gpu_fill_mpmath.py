"""The GPU's general-nu Matérn fill (Chebyshev tables of z^nu K_nu built on the device from the
trapezoid integral) against mpmath's arbitrary-precision besselk directly — independent of the CPU
oracle's own K_nu (the GPU table and the oracle share the trapezoid device, so the GPU
fill gets its own pin).  eq. (Matern): C(r) = sigma^2 2^(1-nu)/Gamma(nu) z^nu K_nu(z),
z = sqrt(2 nu) r / ell.  Radii span z in [~1e-4, ~80] (the table range and beyond, where the
per-point trapezoid takes over)."""
import mpmath as mp
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from tucker_inputs import GridSpec, KernelSpec  # noqa: E402

mp.mp.dps = 40


@pytest.fixture(scope="module")
def T():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_1711_06874_b200 import tucker
    tucker.load()
    return tucker


def nodes(n, lo, hi):  # the a-1 node formula (R2), in double arithmetic
    c = (lo + hi) * 0.5
    s = (hi - lo) / (2.0 * (n - 1))
    return np.array([c + s * float(2 * i - (n - 1)) for i in range(n)])


def matern_mp(nu, ell, sigma2, r):
    if r == 0:
        return mp.mpf(sigma2)
    nu, ell = mp.mpf(nu), mp.mpf(ell)
    z = mp.sqrt(2 * nu) * mp.mpf(r) / ell
    return mp.mpf(sigma2) * mp.power(2, 1 - nu) / mp.gamma(nu) * mp.power(z, nu) * mp.besselk(nu, z)


@pytest.mark.parametrize("nu,ell", [(0.3, 0.5), (0.77, 0.2), (1.3, 0.5), (1.9999, 0.05), (2.1, 1.0), (4.6, 0.3)])
def test_general_nu_fill_vs_mpmath(T, nu, ell):
    n1 = 192
    g = GridSpec((n1, 2, 2), (1e-5, 0.0, 0.0), (2.0, 1e-9, 1e-9))
    F = T.fill(g, KernelSpec.matern(nu, ell)).cpu().numpy()
    x = nodes(n1, 1e-5, 2.0)
    y = nodes(2, 0.0, 1e-9)
    # bar: 1e-14 (the tables' accuracy, R5) plus the conditioning of C in z (|d ln C / d ln z| <= z
    # for z >> 1): the device forms z = sqrt(2 nu) r / ell in FP64, a few ulps from the exact value
    eps = np.finfo(np.float64).eps
    worst = 0.0
    for i in range(0, n1, 3):
        for j in range(2):
            r = np.sqrt((x[i] * x[i] + y[j] * y[j]) + y[0] * y[0])
            ref = matern_mp(nu, ell, 1.0, float(r))
            rel = abs((mp.mpf(F[i, j, 0]) - ref) / ref)
            z = np.sqrt(2 * nu) * r / ell
            worst = max(worst, float(rel) / (1e-14 + 4 * z * eps))
    assert worst <= 1.0, worst
