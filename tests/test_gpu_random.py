"""Seeded randomized parity sweep (a property test of the whole path): random grids (sizes 2..128,
n3 a multiple of 16 half of the time so both INT8 residue layouts run, centred and off-centre
boxes), random kernels (Matérn closed forms and general nu, p-Slater, spectral density) and ranks;
the fill against the oracle element by element and the HOSVD + error under T1–T4, through the
C-ABI.  The inputs come from tucker_inputs' SplitMix64 (no method arithmetic)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from tucker_inputs import GridSpec, KernelSpec, SplitMix64  # noqa: E402
import parity_bars as PB  # noqa: E402


@pytest.fixture(scope="module")
def T():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_1711_06874_b200 import tucker
    tucker.load()
    return tucker


def draw(seed):
    g = SplitMix64(seed)
    u = g.uniform
    n = []
    for a in range(3):
        if a == 2 and u() < 0.5:
            n.append(16 * (1 + int(u() * 8)))
        else:
            n.append(2 + int(u() * 127))
    centred = u() < 0.6
    lo, hi = [], []
    for a in range(3):
        b = 0.5 + 2.5 * u()
        if centred:
            lo.append(-b), hi.append(b)
        else:
            c = (u() - 0.5) * b
            lo.append(c - b * (0.3 + u())), hi.append(c + b * (0.3 + u()))
    fam = int(u() * 5)
    if fam == 0:
        k = KernelSpec.matern([0.5, 1.5, 2.5][int(u() * 3)], 0.05 + 2.0 * u())
    elif fam == 1:
        k = KernelSpec.matern(0.3 + 2.5 * u(), 0.05 + 2.0 * u())
    elif fam == 2:
        k = KernelSpec.slater(0.2 + 5.0 * u(), 0.1 + 1.9 * u())
    elif fam == 3:
        k = KernelSpec.spectral(0.1 + 10.0 * u(), 0.2 + 2.0 * u())
    else:
        k = KernelSpec.slater(1.0 + u(), 2.0)  # Gaussian: rank 1
    r = tuple(max(1, min(n[a], 1 + int(u() * 12))) for a in range(3))
    return GridSpec(tuple(n), tuple(lo), tuple(hi)), k, r


@pytest.mark.parametrize("seed", range(64))
def test_random_case_vs_oracle(T, orc, seed):
    g, k, r = draw(171106874 + 7919 * seed)
    og = orc.Grid(tuple(g.n), tuple(g.lo), tuple(g.hi))
    okk = orc.Kernel(k.family, k.sigma2, k.ell, k.nu, k.lam, k.p, k.flags)
    F = T.fill(g, k)
    Fo = orc.fill(og, okk)
    rel = np.abs(F.cpu().numpy() - Fo) / np.abs(Fo)
    general = k.family == 0 and k.nu not in (0.5, 1.5, 2.5)
    # closed forms / Slater / spectral: a few ulps (p-Slater: exp amplifies pow's ulp by |lam r^p|)
    assert np.max(rel) <= (1e-14 if general else 64 * np.finfo(np.float64).eps), (g, k)
    res = T.hosvd(g, r, F)
    assert res.rc == 0, (g, k, r, res.info)
    e = T.error(g, r, F, res.U, res.core).cpu().numpy()
    h = orc.hosvd(Fo, r)
    E_o = orc.tucker_error(Fo, *h.U, h.core)[0]
    PB.compare(PB.Ref.from_oracle(h, E_o), r, [s.cpu().numpy() for s in res.sigma], [u.cpu().numpy() for u in res.U],
               res.core.cpu().numpy(), float(e[0]))
