"""a-5 core with T1 = F x3 U3^T on the INT8 tensor cores (ttm_i8.cu, R22) against the oracle.

On the INT8 hosvd route (TUCKER_TTM_AUTO) the first TTM product runs on tcgen05 kind::i8 by six
balanced base-256 digits per operand: X = rint(F 2^(46-E)) with max|F| < 2^E, Y_c = rint(U3[:, c]
2^(46-E_c)) with max_k |U3[k, c]| < 2^E_c, and the 26 digit pairs of weight >= 256^-6 are summed
exactly in int32.  The core it gives therefore differs from the exact core of the same factors by

  |d beta_abc| <= 2^(E-47) (sum_i |U1_ia|)(sum_j |U2_jb|)(sum_k |U3_kc|)          (F rounding)
               +  2^(E_c-47) sum_ijk |U1_ia| |U2_jb| |F_ijk|                        (U3 rounding)
               +  2^(E+E_c-50) (sum_i |U1_ia|)(sum_j |U2_jb|) n3                  (dropped pairs)
               +  FP64 rounding of the later products (<= 64 eps sum |U1||U2||F||U3|)

element by element, checked here against the oracle's FP64 TTM chain (`orc.ttm_core`) on the GPU's
own factors, on grids that cover ragged fibre tiles (n1 n2 % 128 != 0), a ragged last K-step
(n3 % 32 == 16), a ragged 64-k digit block, n3 = 16 and r3 = 1 / 8 / 16 / 24 / 33 / 40 (digit-block
widths NB = 8 .. 40, with and without the N rounding of the odd digit counts).  The factors do not depend on the TTM engine (bitwise), and the DMMA TTM of the same
factors must agree within the same bound.
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
    (GridSpec((40, 36, 48), (-1.0,) * 3, (1.0,) * 3), MATERN32, (6, 5, 16)),       # ragged tiles and K-step
    (GridSpec((130, 70, 144), (-2.0, -1.0, -1.5), (2.0, 1.0, 1.5)), MATERN32, (10, 12, 40)),  # ragged k block
    (GridSpec((64, 64, 256), (-1.0,) * 3, (1.0,) * 3), KernelSpec.matern(2.5, 0.3), (20, 20, 24)),
    (GridSpec((200, 33, 16), (-1.0, -0.5, -1.0), (1.0, 1.5, 1.0)), MATERN32, (5, 7, 1)),   # n3 = 16, r3 = 1
    (GridSpec((96, 80, 208), (-1.0,) * 3, (1.0,) * 3), KernelSpec.slater(1.0, 1.0), (12, 9, 33)),
]


def _bound(F, U1, U2, U3):
    aF = np.abs(F)
    E = int(np.frexp(aF.max())[1])                                   # max|F| < 2^E
    Ec = np.array([int(np.frexp(np.abs(U3[:, c]).max())[1]) for c in range(U3.shape[1])])
    s1, s2, s3 = np.abs(U1).sum(0), np.abs(U2).sum(0), np.abs(U3).sum(0)
    n3 = F.shape[2]
    bF = 2.0 ** (E - 47) * np.einsum("a,b,c->abc", s1, s2, s3)
    G12 = np.einsum("ijk,ia,jb->ab", aF, np.abs(U1), np.abs(U2), optimize=True)    # sum_ijk |U1||U2||F| (over k)
    bU = np.einsum("ab,c->abc", G12, 2.0 ** (Ec - 47.0))
    bT = np.einsum("a,b,c->abc", s1, s2, 2.0 ** (E + Ec - 50.0) * n3)
    full = np.einsum("ijk,ia,jb,kc->abc", aF, np.abs(U1), np.abs(U2), np.abs(U3), optimize=True)
    return bF + bU + bT + 64 * EPS * full


@pytest.mark.parametrize("ci", range(len(CASES)))
def test_ttm_i8_core_vs_oracle(T, orc, ci):
    g, k, r = CASES[ci]
    F = T.fill(g, k)
    T.set_gram_engine(T.GRAM_INT8)
    try:
        T.set_ttm_engine(T.TTM_AUTO)
        a = T.hosvd(g, r, F)
        T.set_ttm_engine(T.TTM_DMMA)
        d = T.hosvd(g, r, F)
    finally:
        T.set_ttm_engine(T.TTM_AUTO)
        T.set_gram_engine(T.GRAM_AUTO)
    torch.cuda.synchronize()
    U = [to_np(u) for u in a.U]
    for m in range(3):  # the factors do not depend on the TTM engine
        assert np.array_equal(U[m], to_np(d.U[m])), m
    Fn = to_np(F)
    ref = orc.ttm_core(Fn, *U)
    bar = _bound(Fn, *U)
    ci8, cdm = to_np(a.core), to_np(d.core)
    assert np.all(np.abs(ci8 - ref) <= bar), (ci, float(np.max(np.abs(ci8 - ref) / bar)))
    assert np.all(np.abs(cdm - ref) <= bar), (ci, float(np.max(np.abs(cdm - ref) / bar)))
    # the bound is not vacuous: far below the core's scale
    assert np.max(bar) <= 1e-11 * np.max(np.abs(ref)), float(np.max(bar) / np.max(np.abs(ref)))
    # and the INT8 path really ran (its rounding differs from the DMMA product's in the last bits)
    if r[2] >= 8:
        assert not np.array_equal(ci8, cdm)


def test_ttm_engine_flag(T):
    assert T.get_ttm_engine() == T.TTM_AUTO
    T.set_ttm_engine(T.TTM_DMMA)
    assert T.get_ttm_engine() == T.TTM_DMMA
    T.set_ttm_engine(T.TTM_AUTO)
    with pytest.raises(Exception):
        T.set_ttm_engine(7)


def test_hosvd_prepared_twice_same_outputs(T):
    """The INT8 TTM uses the general scratch, not the prepared residue planes: a second
    tucker_hosvd_prepared call on the same prepared workspace gives bitwise the same results."""
    g, k, r = GridSpec.cube(128, 1.0), MATERN32, (12, 12, 12)
    ws = T.workspace(g, r)
    F, ws = T.fill_prepare(g, k, r, ws=ws)
    a = T.hosvd_prepared(g, r, F, ws)
    b = T.hosvd_prepared(g, r, F, ws)
    torch.cuda.synchronize()
    assert np.array_equal(to_np(a.core), to_np(b.core))
    for m in range(3):
        assert np.array_equal(to_np(a.U[m]), to_np(b.U[m]))
