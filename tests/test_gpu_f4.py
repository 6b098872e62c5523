"""NEXT f4 on the GPU: the paper's other Tucker workloads.

* Matérn spectral density f = C (alpha^2 + rho^2)^{-(nu + 3/2)} (family
  TUCKER_MATERN_SPECTRAL): fill parity against the oracle (<= 4 ulp: the two libm pow's differ by
  <= 2 ulp each), HOSVD parity (T1-T4) for alpha = 0.1 and 100, nu = 0.4 (the paper's Fig. 12/13
  parameters), and the paper's observation that the rank depends strongly on alpha.
* p-Slater e^{-||x||^p}, p = 0.1, 0.2, 1.9, 2.0 on n = 100 (Fig. 9): HOSVD parity and
  exponentially decaying, non-increasing E(r).
Grids: n = 100 per axis as in P:968; box [-1,1]^3 for the spectral density and [-5,5]^3 (R1) for
p-Slater (the paper states neither, DESIGN R17).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from test_gpu_parity import _compare_hosvd, ogrid, okern  # noqa: E402
from tucker_inputs import GridSpec, KernelSpec  # noqa: E402


@pytest.fixture(scope="module")
def T():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_1711_06874_b200 import tucker
    tucker.load()
    return tucker


SPECTRAL = [KernelSpec.spectral(0.1, 0.4), KernelSpec.spectral(100.0, 0.4), KernelSpec.spectral(1.7, 1.1, 2.0)]
PSLATER = [KernelSpec.slater(1.0, p) for p in (0.1, 0.2, 1.9, 2.0)]


@pytest.mark.parametrize("k", SPECTRAL + PSLATER, ids=lambda k: k.label())
@pytest.mark.parametrize("g", [GridSpec.cube(40, 1.0), GridSpec((24, 20, 13), (-0.5, -2.0, 0.1), (1.5, 1.0, 0.9))],
                         ids=["centred", "offcentre"])
def test_fill_parity_f4(T, orc, g, k):
    F = T.fill(g, k).cpu().numpy()
    R = orc.fill(ogrid(orc, g), okern(orc, k))
    # each libm pow is within ~2 ulp; for p-Slater exp(-lambda r^p) amplifies the argument's
    # relative error by |lambda r^p| = |ln(F / sigma^2)|: bar 4 + 3 |ln(F / sigma^2)| ulp
    amp = np.abs(np.log(R / k.sigma2)) if k.family == 1 else 0.0
    assert np.all(np.abs(F - R) / np.spacing(np.abs(R)) <= 4 + 3 * amp)


@pytest.mark.parametrize("k", [SPECTRAL[0], SPECTRAL[1]], ids=lambda k: k.label())
def test_hosvd_spectral_density(T, orc, k):
    _compare_hosvd(T, orc, GridSpec.cube(100, 1.0), k, (10, 10, 10))


@pytest.mark.parametrize("k", PSLATER, ids=lambda k: k.label())
def test_hosvd_p_slater(T, orc, k):
    _compare_hosvd(T, orc, GridSpec.cube(100, 5.0), k, (10, 10, 10))


def _curve(T, g, k, rmax):
    F = T.fill(g, k)
    h = T.hosvd(g, (rmax,) * 3, F)
    out = []
    for r in range(1, rmax + 1):
        U = [u[:, :r].contiguous() for u in h.U]
        core = T.ttm_core(g, (r, r, r), F, *U)
        out.append(float(T.error(g, (r, r, r), F, U, core)[0]))
    return np.array(out)


def test_rank_curves_f4(T):
    g = GridSpec.cube(100, 1.0)
    e_small = _curve(T, g, SPECTRAL[0], 12)
    e_large = _curve(T, g, SPECTRAL[1], 12)
    assert np.all(np.diff(e_small) <= 1e-15) and np.all(np.diff(e_large) <= 1e-15)
    assert e_large[0] < 1e-8 and e_small[4] > 1e3 * e_large[4]     # rank depends strongly on alpha
    for p in (0.1, 1.9):
        e = _curve(T, GridSpec.cube(100, 5.0), KernelSpec.slater(1.0, p), 12)
        assert np.all(np.diff(e) <= 1e-15)
        big = e[e >= 1e-7]
        if len(big) >= 4:  # log-linear (exponential) decay while above the Gram floor
            x = np.arange(len(big))
            slope, icept = np.polyfit(x, np.log(big), 1)
            resid = np.log(big) - (slope * x + icept)
            assert slope < 0 and 1 - resid.var() / np.log(big).var() >= 0.9
