"""a-6 error with the reconstruction on the INT8 tensor cores (err_i8.cu, R23) against the oracle.

Under TUCKER_TTM_INT8_ERROR (opt-in) the error pass forms Ft[p, k] = sum_c W[p, c] U3[k, c] (W = U2 X_i, X_i = U1 beta)
from six base-256 digits of rint(W[p, :] 2^(46-E_p)) and rint(U3[k, :] 2^(46-E_k)) (26 digit pairs,
exact int32 groups), then sums (F - Ft)^2 and F^2 in FP64.  Per element
  |dFt[p,k]| <= 2^(E_p-47) sum_c |U3[k,c]| + 2^(E_k-47) sum_c |W[p,c]| + 2^(E_p+E_k-50) r3,
so |E - E_ref| <= ||dFt||_F / ||F|| (+ FP64 summation), E_ref = the oracle's FP64 error of the same
U and core (`orc.tucker_error`).  Grids cover ragged fibre chunks (n1 n2 % 32 != 0), ragged k-tiles
(n3 % 128 != 0) and r3 = 1 .. 40; the DMMA error pass of the same inputs must meet the same bound.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from tucker_inputs import GridSpec, KernelSpec  # noqa: E402
from test_gpu_parity import to_np  # noqa: E402

EPS = np.finfo(np.float64).eps


@pytest.fixture(scope="module")
def T():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_1711_06874_b200 import tucker
    tucker.load()
    return tucker


@pytest.fixture(scope="module")
def orc():
    from oracle import oracle
    return oracle


MATERN32 = KernelSpec.matern(1.5, 0.2)
CASES = [
    (GridSpec.cube(32, 1.0), KernelSpec.matern(0.5, 0.5), (8, 8, 8)),
    (GridSpec((40, 36, 50), (-1.0,) * 3, (1.0,) * 3), MATERN32, (6, 5, 16)),
    (GridSpec((130, 70, 144), (-2.0, -1.0, -1.5), (2.0, 1.0, 1.5)), MATERN32, (10, 12, 40)),
    (GridSpec((64, 64, 256), (-1.0,) * 3, (1.0,) * 3), KernelSpec.matern(2.5, 0.3), (20, 20, 24)),
    (GridSpec((200, 33, 16), (-1.0, -0.5, -1.0), (1.0, 1.5, 1.0)), MATERN32, (5, 7, 1)),
    (GridSpec((96, 80, 208), (-1.0,) * 3, (1.0,) * 3), KernelSpec.slater(1.0, 1.0), (12, 9, 33)),
]


def _dft_norm(F, U1, U2, U3, core):
    W = np.einsum("ia,abc,jb->ijc", U1, core, U2, optimize=True).reshape(-1, U3.shape[1])  # fibre p = (i, j)
    aW = np.abs(W).max(1)
    Ep = np.where(aW > 0, np.frexp(aW)[1], 0).astype(float)
    aU = np.abs(U3).max(1)
    Ek = np.where(aU > 0, np.frexp(aU)[1], 0).astype(float)
    sU = np.abs(U3).sum(1)
    sW = np.abs(W).sum(1)
    R = U3.shape[1]
    b = (2.0 ** (Ep - 47))[:, None] * sU[None, :] + sW[:, None] * (2.0 ** (Ek - 47))[None, :] \
        + R * 2.0 ** (Ep[:, None] + Ek[None, :] - 50)
    return float(np.sqrt(np.sum(b * b)))


@pytest.mark.parametrize("ci", range(len(CASES)))
def test_err_i8_vs_oracle(T, orc, ci):
    g, k, r = CASES[ci]
    F = T.fill(g, k)
    res = T.hosvd(g, r, F)
    ws = T.workspace(g, r)
    try:
        T.set_ttm_engine(T.TTM_INT8_ERROR)
        e8 = to_np(T.error(g, r, F, res.U, res.core, ws))
        T.set_ttm_engine(T.TTM_DMMA)
        ed = to_np(T.error(g, r, F, res.U, res.core, ws))
    finally:
        T.set_ttm_engine(T.TTM_AUTO)
    Fn = to_np(F)
    U = [to_np(u) for u in res.U]
    core = to_np(res.core)
    E_ref, nF_ref = orc.tucker_error(Fn, *U, core)[:2]
    nF = np.linalg.norm(Fn)
    bar = _dft_norm(Fn, *U, core) / nF + 64 * EPS * E_ref + 1e-16
    assert abs(e8[0] - E_ref) <= bar, (ci, e8[0], E_ref, bar)
    assert abs(ed[0] - E_ref) <= bar, (ci, ed[0], E_ref, bar)
    assert abs(e8[1] - nF) <= 1e-14 * nF
    assert bar <= 1e-12  # not vacuous at these sizes (E itself is 1e-9 .. 1e-2)


def test_err_i8_deterministic(T):
    g, k, r = CASES[2]
    F = T.fill(g, k)
    res = T.hosvd(g, r, F)
    T.set_ttm_engine(T.TTM_INT8_ERROR)
    try:
        a = to_np(T.error(g, r, F, res.U, res.core))
        b = to_np(T.error(g, r, F, res.U, res.core))
    finally:
        T.set_ttm_engine(T.TTM_AUTO)
    assert np.array_equal(a, b)
