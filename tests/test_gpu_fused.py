"""GPU parity of the a-7 fused generate-and-contract path (F never materialised), through the C-ABI.

* The fused Gram equals the materialised Gram up to summation order (bar DESIGN.md §4: 1e-14
  relative to sqrt(G_aa G_bb) at K <= 65k terms) and the oracle's Gram, on grids that exercise the
  mirrored (centred, n3 % 8 == 0) and the general generator, several chunks (TUCKER_FUSED_CHUNK_KB
  test knob), ragged tiles and the general-nu K_nu table.
* The fused HOSVD / error meet the T1-T4 bars against the oracle (small grids) and against the
  materialised GPU path (256^3, 1024^3).
* 2048^3 (BASELINE config 5f, never materialised): sampled Gram entries against the oracle's
  entry-wise definition (orc_gram_entry_fn), orthonormal factors, the orthogonal-projection
  identity ||F||^2 = ||beta||^2 + (E ||F||)^2, and E(2048) against E(1024) of the same function.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from tucker_inputs import GridSpec, KernelSpec  # noqa: E402
import parity_bars as PB  # noqa: E402


@pytest.fixture(scope="module")
def T():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_1711_06874_b200 import tucker
    tucker.load()
    return tucker


@pytest.fixture
def chunk_kb():
    """Set TUCKER_FUSED_CHUNK_KB for one test (forces many chunks on small grids)."""
    def set_(kb):
        if kb is None:
            os.environ.pop("TUCKER_FUSED_CHUNK_KB", None)
        else:
            os.environ["TUCKER_FUSED_CHUNK_KB"] = str(kb)
    yield set_
    os.environ.pop("TUCKER_FUSED_CHUNK_KB", None)


def ogrid(orc, g):
    return orc.Grid(tuple(g.n), tuple(g.lo), tuple(g.hi))


def okern(orc, k):
    return orc.Kernel(k.family, k.sigma2, k.ell, k.nu, k.lam, k.p, k.flags)


def to_np(t):
    return t.detach().cpu().numpy()


CASES = [
    (GridSpec.cube(128, 1.0), KernelSpec.matern(1.5, 0.2), None),                                  # 1 chunk, 1 tile
    (GridSpec((136, 144, 160), (-2.0, -1.5, -1.0), (2.0, 1.5, 1.0)), KernelSpec.matern(0.7, 0.5), 256),  # K_nu, ragged
    (GridSpec((144, 136, 130), (-0.5, -2.0, 0.1), (1.5, 1.0, 0.9)), KernelSpec.matern(1.5, 0.2), 300),  # general gen
    (GridSpec((130, 129, 136), (-1.0, -1.0, -1.0), (1.0, 1.0, 1.0)), KernelSpec.slater(1.0, 1.0), 200),  # odd n1, n2
]


@pytest.fixture(params=["int8", "dmma"])
def engine(T, request):
    """INT8 fused route (plane chunks -> residues, per-mode row scaling; the materialised reference
    Gram on the same row-scaled layout) and the DMMA route (k_gram_fused: persistent cooperative
    grid, L2-resident ring); restored afterwards."""
    T.set_gram_engine(T.GRAM_INT8_ROWSCALED if request.param == "int8" else T.GRAM_DMMA)
    yield request.param
    T.set_gram_engine(T.GRAM_AUTO)


@pytest.mark.parametrize("ci", range(len(CASES)))
def test_gram_fused_parity(T, orc, chunk_kb, engine, ci):
    g, k, kb = CASES[ci]
    chunk_kb(kb)
    F = T.fill(g, k)
    Fo = orc.fill(ogrid(orc, g), okern(orc, k))
    ws, wsf = T.workspace(g), T.workspace_fused(g)
    for m in range(3):
        Gf = T.gram_fused(g, k, m, wsf)
        G = T.gram(g, m, F, ws)
        assert torch.equal(Gf, Gf.T)
        d = torch.sqrt(torch.diag(G))
        assert ((Gf - G).abs() / torch.outer(d, d)).max().item() <= 1e-14, m
        R = orc.gram_mode(Fo, m)
        dr = np.sqrt(np.diag(R))
        assert np.max(np.abs(to_np(Gf) - R) / np.outer(dr, dr)) <= 1e-14, m
        # deterministic
        assert torch.equal(Gf, T.gram_fused(g, k, m, wsf))


def test_gram_fused_many_chunks_256(T, chunk_kb):
    g, k = GridSpec.cube(256, 1.0), KernelSpec.matern(1.3, 0.3)
    F = T.fill(g, k)
    ws = T.workspace(g)
    for kb in (512, 4096, None):
        chunk_kb(kb)
        wsf = T.workspace_fused(g)
        for m in range(3):
            Gf, G = T.gram_fused(g, k, m, wsf), T.gram(g, m, F, ws)
            d = torch.sqrt(torch.diag(G))
            assert ((Gf - G).abs() / torch.outer(d, d)).max().item() <= 1e-14, (kb, m)


def _bars(lam_ref, lam, U_ref, U, r):
    pos = lam_ref[:r] > 0
    assert np.all(np.abs(lam[pos] - lam_ref[:r][pos]) <= 1e-11 * lam_ref[:r][pos] + 1e-14 * lam_ref[0])
    for c in range(r):
        others = np.delete(lam_ref, c)
        if np.min(np.abs(others - lam_ref[c])) >= 1e-6 * lam_ref[0]:
            assert np.max(np.abs(U[:, c] - U_ref[:, c])) <= 1e-9, c
    assert np.max(np.abs(U.T @ U - np.eye(r))) <= 1e-12


def test_hosvd_fused_vs_oracle(T, orc, chunk_kb, engine):
    g = GridSpec((136, 144, 160), (-2.0, -1.5, -1.0), (2.0, 1.5, 1.0))
    k = KernelSpec.matern(0.7, 0.5)
    r = (12, 10, 9)
    chunk_kb(256)
    res = T.hosvd_fused(g, k, r)
    assert res.rc == 0, res.info
    err = to_np(T.error_fused(g, k, r, res.U, res.core))
    F = orc.fill(ogrid(orc, g), okern(orc, k))
    h = orc.hosvd(F, r)
    E_o = orc.tucker_error(F, *h.U, h.core)[0]
    for m in range(3):
        _bars(h.lam[m], to_np(res.sigma[m]) ** 2, h.U[m], to_np(res.U[m]), r[m])
    blocks = [int(np.sum(h.lam[m][:r[m]] >= 1e-10 * h.lam[m][0])) for m in range(3)]
    a, b, c = blocks
    assert np.linalg.norm(to_np(res.core)[:a, :b, :c] - h.core[:a, :b, :c]) <= 1e-10 * np.linalg.norm(h.core[:a, :b, :c])
    resolved = all(r[m] <= int(np.sum(h.lam[m][:r[m]] >= 1e-12 * h.lam[m][0])) for m in range(3))
    assert abs(err[0] - E_o) <= (1e-12 if resolved else max(1e-12, 1e-15 / E_o)), (err[0], E_o)
    assert abs(err[1] - np.linalg.norm(F)) <= 1e-14 * np.linalg.norm(F)


@pytest.mark.parametrize("n,r,kb", [(256, (20, 20, 20), 2048), (1024, (40, 40, 40), None), (1024, (10, 10, 10), None)])
def test_hosvd_fused_vs_materialised(T, chunk_kb, n, r, kb):
    """Same function tensor through both paths: eigenvalues, gap-separated columns, core, E."""
    chunk_kb(kb)
    g, k = GridSpec.cube(n, 1.0), KernelSpec.matern(1.5, 0.2)
    F = T.fill(g, k)
    ref = T.hosvd(g, r, F)
    e_ref = to_np(T.error(g, r, F, ref.U, ref.core))
    del F
    torch.cuda.empty_cache()
    res = T.hosvd_fused(g, k, r)
    assert res.rc == 0 and ref.rc == 0
    e = to_np(T.error_fused(g, k, r, res.U, res.core))
    for m in range(3):
        lam_ref = to_np(ref.sigma[m]) ** 2
        lam = to_np(res.sigma[m]) ** 2
        lam1 = lam_ref[0]
        assert np.all(np.abs(lam - lam_ref) <= 1e-11 * lam_ref + 1e-14 * lam1), m
        U, Ur = to_np(res.U[m]), to_np(ref.U[m])
        for c in range(r[m]):
            others = np.delete(lam_ref, c)
            if lam_ref[c] >= 1e-6 * lam1 and np.min(np.abs(others - lam_ref[c])) >= 1e-6 * lam1:
                assert np.max(np.abs(U[:, c] - Ur[:, c])) <= 1e-9, (m, c)
        assert np.max(np.abs(U.T @ U - np.eye(r[m]))) <= 1e-12
    nb = np.linalg.norm(to_np(ref.core))
    assert abs(np.linalg.norm(to_np(res.core)) - nb) <= 1e-12 * nb
    assert abs(e[1] - e_ref[1]) <= 1e-13 * e_ref[1]
    assert abs(e[0] - e_ref[0]) <= max(1e-12, 1e-15 / e_ref[0]), (e, e_ref)


def test_fused_2048_config5f(T, orc):
    """BASELINE config 5f: 2048^3 (68.7 GB if stored) through the fused path only."""
    g, k, r = GridSpec.cube(2048, 1.0), KernelSpec.matern(1.5, 0.2), (40, 40, 40)
    wsf = T.workspace_fused(g, r)
    og, ok = ogrid(orc, g), okern(orc, k)
    rng = np.random.default_rng(2048)
    G0 = T.gram_fused(g, k, 0, wsf)
    assert torch.equal(G0, G0.T)
    Gn = to_np(G0)
    # the INT8 route forms X X^T exactly: each sampled entry within the element bound of the fused
    # route's shared layout (R20: one global exponent — max F is C at the centre-most node, from the
    # oracle's kernel evaluation; row 1-norms from orc_row_stats_fn)
    K = 2048 * 2048
    _, bits = T.i8_scheme(K)
    gmax = orc.fill_entry(og, ok, 1023, 1023, 1023)
    for a, b in rng.integers(0, 2048, size=(6, 2)):
        ref = orc.gram_entry_fn(og, ok, 0, int(a), int(b))
        (ma, la), (mb, lb) = orc.row_stats_fn(og, ok, 0, int(a)), orc.row_stats_fn(og, ok, 0, int(b))
        assert max(ma, mb) <= gmax
        assert abs(Gn[a, b] - ref) <= PB.i8_bound_entry(gmax, gmax, la, lb, K, bits, ref), (a, b)
        assert abs(Gn[a, b] - ref) <= 1e-13 * np.sqrt(Gn[a, a] * Gn[b, b]), (a, b)
    del G0
    res = T.hosvd_fused(g, k, r, wsf)
    assert res.rc == 0, res.info
    e = to_np(T.error_fused(g, k, r, res.U, res.core, wsf))
    for m in range(3):
        U = to_np(res.U[m])
        assert np.max(np.abs(U.T @ U - np.eye(r[m]))) <= 1e-12
    nF, nb = e[1], np.linalg.norm(to_np(res.core))
    assert abs(nF ** 2 - (nb ** 2 + e[2] ** 2)) <= 1e-12 * nF ** 2
    # ||F||^2 against the oracle's entry-wise Gram trace sample: G_aa summed over all a is ||F||^2
    assert abs(np.trace(Gn) - nF ** 2) <= 1e-12 * nF ** 2
    # same function, twice the resolution: the relative truncation error is of the same size
    assert 1e-9 < e[0] < 1e-6, e


@pytest.mark.parametrize("g,k,kb", [
    (GridSpec((96, 80, 64), (-0.5, -2.0, 0.1), (1.5, 1.0, 0.9)), KernelSpec.matern(1.5, 0.2), 200),   # off-centre: no mirrors
    (GridSpec((129, 131, 64), (-2.0, -1.5, -1.0), (2.0, 1.5, 1.0)), KernelSpec.matern(0.7, 0.3), 300),  # odd free axes
    (GridSpec((40, 24, 16), (-1.0,) * 3, (1.0,) * 3), KernelSpec.slater(1.0, 0.2), None),               # n3 = 16, 1 chunk
    (GridSpec((2, 3, 32), (-1.0,) * 3, (1.0,) * 3), KernelSpec.spectral(0.1, 0.4), None)])              # tiny axes
def test_gram_fused_shared_bitwise_equals_materialised(T, chunk_kb, g, k, kb):
    """The default fused INT8 route on the shared layout (R20): plane chunks of residues generated
    from the kernel (i-chunks for modes 1, 2; j-chunks for mode 0; mirrored on centred grids, plain
    on off-centre ones) give bitwise the Grams of the materialised shared route on the same values
    (the same global exponent, exact integer sums) — many chunks through the test knob."""
    chunk_kb(kb)
    assert T.i8_layout(g)[0]
    F = T.fill(g, k)
    ws = T.workspace_i8(g)
    wsf = T.workspace_fused(g)
    for m in range(3):
        assert torch.equal(T.gram_fused(g, k, m, wsf), T.gram_i8(g, m, F, ws)), m
