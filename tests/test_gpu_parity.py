"""GPU parity: every stage of the CUDA path (through the C-ABI) against the CPU oracle on the same
seeded synthetic inputs.  Tolerances follow BASELINE.json's north_star as read in DESIGN.md §4
(T1 eigenvalues, T2 factor columns, T3 core, T4 error) and DESIGN.md §4's fill/Gram bounds."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from tucker_inputs import GridSpec, KernelSpec, config1, config3  # noqa: E402

EPS = np.finfo(np.float64).eps


@pytest.fixture(scope="module")
def T():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_1711_06874_b200 import tucker
    tucker.load()
    return tucker


def ogrid(orc, g):
    return orc.Grid(tuple(g.n), tuple(g.lo), tuple(g.hi))


def okern(orc, k):
    return orc.Kernel(k.family, k.sigma2, k.ell, k.nu, k.lam, k.p, k.flags)


def to_np(t):
    return t.detach().cpu().numpy()


# ------------------------------------------------------------------------------------- fill ----
CLOSED = [KernelSpec.matern(0.5, 0.5), KernelSpec.matern(1.5, 0.2), KernelSpec.matern(2.5, 0.05),
          KernelSpec.slater(1.0, 1.0), KernelSpec.slater(5.0, 1.0), KernelSpec.slater(1.0, 2.0)]
GENERAL = [KernelSpec.matern(0.3, 0.5), KernelSpec.matern(0.7, 0.5), KernelSpec.matern(1.3, 0.5),
           KernelSpec.matern(2.1, 0.5), KernelSpec.matern(1.5, 0.2, flags=2), KernelSpec.matern(0.5, 0.5, flags=2),
           KernelSpec.matern(1.9999, 0.05), KernelSpec.matern(0.93, 1.0, sigma2=2.5)]
GRIDS = [GridSpec.cube(32, 1.0), GridSpec((24, 20, 16), (-2.0, -1.5, -1.0), (2.0, 1.5, 1.0)),
         GridSpec((9, 7, 13), (-1.0, -1.0, -1.0), (1.0, 1.0, 1.0)),          # odd sizes: origin node, general path
         GridSpec((12, 10, 8), (-0.5, -2.0, 0.1), (1.5, 1.0, 0.9)),          # off-centre box: general path
         GridSpec((2, 2, 2), (-1.0, -1.0, -1.0), (1.0, 1.0, 1.0))]


@pytest.mark.parametrize("gi", range(len(GRIDS)))
def test_fill_closed_forms_ulp(T, orc, gi):
    g = GRIDS[gi]
    for k in CLOSED:
        F = to_np(T.fill(g, k))
        ref = orc.fill(ogrid(orc, g), okern(orc, k))
        # nodes, radius and z are bitwise identical by construction (R2); exp differs <= 1 ulp per side
        ulp = np.spacing(np.abs(ref))
        assert np.max(np.abs(F - ref) / ulp) <= 4, (g, k)


@pytest.mark.parametrize("gi", range(len(GRIDS)))
def test_fill_general_nu(T, orc, gi):
    g = GRIDS[gi]
    for k in GENERAL:
        F = to_np(T.fill(g, k))
        ref = orc.fill(ogrid(orc, g), okern(orc, k))
        assert np.max(np.abs(F - ref) / np.abs(ref)) <= 1e-14, (g, k)


def test_fill_config3_grid(T, orc):
    w = config3()
    for k in w.kernels:
        F = to_np(T.fill(w.grid, k))
        ref = orc.fill(ogrid(orc, w.grid), okern(orc, k))
        tol = 1e-14 if (k.family == 0 and k.nu not in (0.5, 1.5, 2.5)) else 8 * EPS
        assert np.max(np.abs(F - ref) / np.abs(ref)) <= tol, k


# ------------------------------------------------------------------------------------- Gram ----
GRAM_GRIDS = [GridSpec.cube(32, 1.0),                                        # cp.async path, 1 tile
              GridSpec((40, 36, 33), (-1.0, -1.0, -1.0), (1.0, 1.0, 1.0)),  # odd n3, ragged
              GridSpec.cube(128, 1.0),                                       # TMA path, 1 tile
              GridSpec((136, 144, 160), (-2.0, -1.5, -1.0), (2.0, 1.5, 1.0)),  # TMA, ragged 2x2 tiles
              GridSpec((130, 129, 131), (-1.0, -1.0, -1.0), (1.0, 1.0, 1.0))]  # odd n3 -> cp.async, 2 tiles


@pytest.fixture(params=["int8", "dmma"])
def engine(T, request):
    """Run the test under each Gram engine (the INT8 emulation, R18, and the north_star's FP64
    tensor-core DMMA route: k_gram_tma / k_gram_generic / k_gram_fused); restored afterwards."""
    T.set_gram_engine(T.GRAM_INT8 if request.param == "int8" else T.GRAM_DMMA)
    yield request.param
    T.set_gram_engine(T.GRAM_AUTO)


@pytest.mark.parametrize("gi", range(len(GRAM_GRIDS)))
def test_gram_parity(T, orc, engine, gi):
    g = GRAM_GRIDS[gi]
    k = KernelSpec.matern(1.3, 0.5)
    Fg = T.fill(g, k)
    F = orc.fill(ogrid(orc, g), okern(orc, k))
    ws = T.workspace(g, (8, 8, 8))
    for m in range(3):
        G = to_np(T.gram(g, m, Fg, ws))
        R = orc.gram_mode(F, m)
        d = np.sqrt(np.diag(R))
        assert np.array_equal(G, G.T)
        assert np.max(np.abs(G - R) / np.outer(d, d)) <= 1e-14, m


def test_gram_deterministic(T, engine):
    g = GridSpec((136, 144, 160), (-2.0, -1.5, -1.0), (2.0, 1.5, 1.0))
    F = T.fill(g, KernelSpec.matern(0.7, 0.5))
    ws = T.workspace(g)
    for m in range(3):
        assert torch.equal(T.gram(g, m, F, ws), T.gram(g, m, F, ws))


# -------------------------------------------------------------------------------------- eig ----
def _gap_ok(lam_full, k, rel=1e-6):
    others = np.delete(lam_full, k)
    return np.min(np.abs(others - lam_full[k])) >= rel * lam_full[0]


@pytest.mark.parametrize("n,r,nu,ell", [(32, 8, 0.5, 0.5), (96, 20, 1.3, 0.5), (128, 20, 0.5, 0.1),
                                        (160, 40, 1.5, 0.2), (256, 12, 2.1, 0.5)])
def test_eig_on_oracle_gram(T, orc, n, r, nu, ell):
    g = GridSpec((n, 24, 20), (-1.0, -1.0, -1.0), (1.0, 1.0, 1.0))
    F = orc.fill(ogrid(orc, g), orc.Kernel.matern(nu, ell))
    G = orc.gram_mode(F, 0)
    lam_o, V_o, rc, _ = orc.jacobi_eig(G)
    assert rc == 0
    U, lam, info, rc = T.eig(torch.from_numpy(G).cuda(), r)
    assert rc == 0, info
    U, lam = to_np(U), to_np(lam)
    # T1
    assert np.all(np.abs(lam - lam_o[:r]) <= 1e-11 * np.abs(lam_o[:r]) + 1e-14 * lam_o[0])
    # T2 on gap-separated columns
    for c in range(r):
        if _gap_ok(lam_o, c):
            assert np.max(np.abs(U[:, c] - V_o[:, c])) <= 1e-9, c
    # T2'
    assert np.max(np.abs(U.T @ U - np.eye(r))) <= 1e-12


# ------------------------------------------------------------------------------ core / error ----
def test_ttm_and_error_with_oracle_factors(T, orc):
    g = GridSpec((136, 144, 160), (-2.0, -1.5, -1.0), (2.0, 1.5, 1.0))
    k = KernelSpec.matern(0.7, 0.5)
    F = orc.fill(ogrid(orc, g), okern(orc, k))
    h = orc.hosvd(F, (12, 10, 9))
    Fg = torch.from_numpy(F).cuda()
    Ug = [torch.from_numpy(np.ascontiguousarray(u)).cuda() for u in h.U]
    core = to_np(T.ttm_core(g, (12, 10, 9), Fg, *Ug))
    assert np.linalg.norm(core - h.core) <= 1e-13 * np.linalg.norm(h.core)
    out = to_np(T.error(g, (12, 10, 9), Fg, Ug, torch.from_numpy(h.core).cuda()))
    E, nf, nd = orc.tucker_error(F, *h.U, h.core)
    assert abs(out[0] - E) <= 1e-13 and abs(out[1] - nf) <= 1e-14 * nf
    # odd n3 (cp.async 8-byte path of TTM1) and r3 not a multiple of 8
    g2 = GridSpec((20, 18, 33), (-1.0, -1.0, -1.0), (1.0, 1.0, 1.0))
    F2 = orc.fill(ogrid(orc, g2), orc.Kernel.matern(1.3, 0.5))
    h2 = orc.hosvd(F2, (5, 6, 7))
    U2 = [torch.from_numpy(np.ascontiguousarray(u)).cuda() for u in h2.U]
    c2 = to_np(T.ttm_core(g2, (5, 6, 7), torch.from_numpy(F2).cuda(), *U2))
    assert np.linalg.norm(c2 - h2.core) <= 1e-13 * np.linalg.norm(h2.core)


# ------------------------------------------------------------------------------- full HOSVD ----
def _k_res(lam, r, tau):
    return int(np.sum(lam[:r] >= tau * lam[0]))


def _compare_hosvd(T, orc, g, k, r):
    Fg = T.fill(g, k)
    F = orc.fill(ogrid(orc, g), okern(orc, k))
    res = T.hosvd(g, r, Fg)
    assert res.rc == 0, res.info
    h = orc.hosvd(F, r)
    err = to_np(T.error(g, r, Fg, res.U, res.core))
    E_o = orc.tucker_error(F, *h.U, h.core)[0]
    resolved = True
    blocks = []
    for m in range(3):
        lam_o = h.lam[m]
        lam_g = to_np(res.sigma[m]) ** 2
        rr = r[m]
        # T1 (sigma^2 vs lambda; sigma = sqrt(max(lambda,0)) so compare where lambda > 0)
        pos = lam_o[:rr] > 0
        assert np.all(np.abs(lam_g[pos] - lam_o[:rr][pos]) <= 1e-11 * lam_o[:rr][pos] + 1e-14 * lam_o[0]), m
        U = to_np(res.U[m])
        for c in range(rr):
            if _gap_ok(lam_o, c):
                assert np.max(np.abs(U[:, c] - h.U[m][:, c])) <= 1e-9, (m, c)
        assert np.max(np.abs(U.T @ U - np.eye(rr))) <= 1e-12
        resolved &= rr <= _k_res(lam_o, rr, 1e-12)
        blocks.append(_k_res(lam_o, rr, 1e-10))
    # T3 on the resolved leading block
    a, b, c = blocks
    cg, co = to_np(res.core)[:a, :b, :c], h.core[:a, :b, :c]
    assert np.linalg.norm(cg - co) <= 1e-10 * np.linalg.norm(co)
    assert abs(np.linalg.norm(to_np(res.core)) - np.linalg.norm(h.core)) <= 1e-12 * np.linalg.norm(h.core)
    # T4
    tol = 1e-12 if resolved else max(1e-12, 1e-15 / E_o)
    assert abs(err[0] - E_o) <= tol, (err[0], E_o, resolved)
    return res, err


def test_hosvd_config1(T, orc, engine):
    w = config1()
    res, err = _compare_hosvd(T, orc, w.grid, w.kernels[0], w.ranks)
    assert 9.55e-7 < err[0] < 9.58e-7


@pytest.mark.parametrize("nu,ell", [(0.5, 0.1), (1.5, 0.5), (2.5, 1.0)])
def test_hosvd_config2_kernels(T, orc, engine, nu, ell):
    _compare_hosvd(T, orc, GridSpec.cube(128, 1.0), KernelSpec.matern(nu, ell), (20, 20, 20))


@pytest.mark.parametrize("ki", [0, 2, 4])
def test_hosvd_config3(T, orc, engine, ki):
    w = config3()
    _compare_hosvd(T, orc, w.grid, w.kernels[ki], w.ranks)


def test_hosvd_odd_grid_with_origin(T, orc, engine):
    # Table-2-like grid (n = 2k+1 contains the origin, C(0) = sigma^2); odd n3 -> cp.async paths
    _compare_hosvd(T, orc, GridSpec.cube(129, 5.0), KernelSpec.slater(1.0, 1.0), (10, 10, 10))


def test_hosvd_small_full_rank_and_rank1(T, orc):
    g = GridSpec((6, 5, 4), (-1.0, -1.0, -1.0), (1.0, 1.0, 1.0))
    _compare_hosvd(T, orc, g, KernelSpec.matern(0.7, 0.5), (6, 5, 4))
    g = GridSpec((32, 24, 16), (-2.0, -1.5, -1.0), (2.0, 1.5, 1.0))
    res, err = _compare_hosvd(T, orc, g, KernelSpec.slater(1.0, 2.0), (1, 1, 1))
    assert err[0] <= 1e-14


def test_hosvd_deterministic(T):
    g = GridSpec((136, 144, 160), (-2.0, -1.5, -1.0), (2.0, 1.5, 1.0))
    F = T.fill(g, KernelSpec.matern(1.3, 0.5))
    a = T.hosvd(g, (12, 12, 10), F)
    b = T.hosvd(g, (12, 12, 10), F)
    for m in range(3):
        assert torch.equal(a.U[m], b.U[m])
    assert torch.equal(a.core, b.core)
    assert torch.equal(T.error(g, (12, 12, 10), F, a.U, a.core), T.error(g, (12, 12, 10), F, b.U, b.core))


def test_approximate_host_outputs(T, orc):
    w = config1()
    g, k, r = w.grid, w.kernels[0], w.ranks
    F = torch.empty(tuple(g.n), dtype=torch.float64, device="cuda")
    ws = T.workspace(g, r)
    host = T.HostBuffers(g, r)
    out = T.approximate(g, k, r, F, ws, host)
    assert out.rc == 0
    Fo = orc.fill(ogrid(orc, g), okern(orc, k))
    h = orc.hosvd(Fo, r)
    E_o = orc.tucker_error(Fo, *h.U, h.core)[0]
    assert abs(out.err[0] - E_o) <= 1e-12
    assert T.last_launch_count() > 10


@pytest.mark.parametrize("grid", [GridSpec.cube(256, 1.0), GridSpec((136, 144, 160), (-1.0,) * 3, (1.0,) * 3),
                                  GridSpec((96, 80, 112), (-2.0, -1.0, -0.5), (2.0, 1.5, 1.0))])
def test_approximate_equals_separate_calls(T, grid):
    """tucker_approximate takes the INT8 route's row maxima out of the fill on centred grids (n3 % 8
    == 0); the tensor, factors, core and error are bitwise those of tucker_fill + tucker_hosvd +
    tucker_error (the maxima are the same numbers), also where the fusion does not apply."""
    k, r = KernelSpec.matern(1.5, 0.3), (12, 12, 12)
    F = torch.empty(tuple(grid.n), dtype=torch.float64, device="cuda")
    ws = T.workspace(grid, r)
    host = T.HostBuffers(grid, r)
    out = T.approximate(grid, k, r, F, ws, host)
    F2 = T.fill(grid, k)
    assert torch.equal(F, F2)
    res = T.hosvd(grid, r, F2)
    e = T.error(grid, r, F2, res.U, res.core)
    for m in range(3):
        assert np.array_equal(out.U[m], to_np(res.U[m])), m
        assert np.array_equal(out.sigma[m], to_np(res.sigma[m])), m
    assert np.array_equal(out.core, to_np(res.core))
    assert np.array_equal(out.err, to_np(e))


@pytest.mark.parametrize("g", [GridSpec.cube(256, 1.0), GridSpec((129, 131, 64), (-2.0, -1.5, -1.0), (2.0, 1.5, 1.0))])
def test_fill_rowmax_and_hosvd_rowmax(T, g):
    """tucker_fill_rowmax: the same F as tucker_fill; tucker_hosvd_rowmax with those maxima: bitwise
    tucker_hosvd (they are the row maxima the INT8 route would compute); odd axes (a middle index);
    unsupported grids refuse."""
    k, r = KernelSpec.matern(0.7, 0.3), (16, 16, 16)
    n1, n2, n3 = g.n
    F, mx = T.fill_rowmax(g, k)
    assert torch.equal(F, T.fill(g, k))
    a, b = T.hosvd(g, r, F), T.hosvd(g, r, F, rowmax=mx)
    for m in range(3):
        assert torch.equal(a.U[m], b.U[m]) and torch.equal(a.sigma[m], b.sigma[m])
    assert torch.equal(a.core, b.core)
    # the maxima mirror on a centred grid and bound every |F| row from above in the exponent
    for off, nn in ((0, n1), (n1, n2), (n1 + n2, n3)):
        seg = mx[off:off + nn]
        assert torch.equal(seg, seg.flip(0))
    hw = (F.abs().view(torch.int64) >> 32).to(torch.int32)
    assert torch.equal(mx[:n1], hw.amax(dim=(1, 2)))
    assert torch.equal(mx[n1:n1 + n2], hw.amax(dim=(0, 2)))
    assert torch.equal(mx[n1 + n2:], hw.amax(dim=(0, 1)))
    off_grid = GridSpec((64, 64, 64), (-1.0, -1.0, -0.5), (1.0, 1.0, 1.0))
    with pytest.raises(T.TuckerError) as e:
        T.fill_rowmax(off_grid, k)
    assert e.value.code == 7


@pytest.mark.parametrize("g,k,r", [(GridSpec((2, 3, 16), (-1.0,) * 3, (1.0,) * 3), KernelSpec.matern(1.5, 0.5), (2, 3, 4)),
                                   (GridSpec((5, 7, 32), (-1.0,) * 3, (1.0,) * 3), KernelSpec.matern(0.5, 0.3), (3, 4, 5)),
                                   (GridSpec((33, 17, 48), (-2.0, -0.5, -1.0), (1.0, 1.5, 1.0)), KernelSpec.slater(5.0, 1.0), (6, 5, 7))])
def test_shared_layout_tiny_and_offcentre_vs_oracle(T, orc, g, k, r):
    """The shared INT8 residue layout (n3 % 16 == 0) on tiny and off-centre grids — through
    tucker_fill_prepare where it applies (centred), tucker_hosvd otherwise — against the oracle."""
    assert T.i8_layout(g)[0]
    _compare_hosvd(T, orc, g, k, r)
    centred = all(lo == -hi for lo, hi in zip(g.lo, g.hi))
    if centred:
        F, ws = T.fill_prepare(g, k, r)
        a = T.hosvd_prepared(g, r, F, ws)
        b = T.hosvd(g, r, F)
        assert torch.equal(a.core, b.core)
