"""a-3 on the INT8 tensor cores (tucker_gram_i8, R18) against exact arithmetic and the oracle.

The emulated Gram is G~ = fl(D X X^T D), X = rint(D^-1 F_(m)), D = diag(2^(E_i - b)): X X^T is formed
exactly (residues mod 16 coprime moduli on the int8 tensor cores + CRT), so
  * integer-valued F (|F| < 2^bits, every Gram entry exact in FP64) must give the exact Gram bit for bit;
  * for general F the error is the input rounding only: with m_i = max_k |a_ik| and u = 2^-(b+1)
    (b = 50 at these sizes), |G~_ij - G_ij| <= 2^(E_i-b-1) ||a_j||_1 + 2^(E_j-b-1) ||a_i||_1
    + 3 2^(E_i+E_j-2b-2) K + eps |G_ij|, checked element by element against the oracle's FP64 Gram
    (whose own error, K eps |a_i||a_j|, is added to the bound).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from tucker_inputs import GridSpec, KernelSpec  # noqa: E402
from test_gpu_parity import ogrid, okern, to_np  # noqa: E402

EPS = np.finfo(np.float64).eps


@pytest.fixture(scope="module")
def T():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_1711_06874_b200 import tucker
    tucker.load()
    return tucker


def unfold(F, m):
    return np.moveaxis(F, m, 0).reshape(F.shape[m], -1)


GRIDS = [GridSpec((2, 2, 2), (-1.0,) * 3, (1.0,) * 3),
         GridSpec.cube(32, 1.0),
         GridSpec((40, 36, 33), (-1.0,) * 3, (1.0,) * 3),            # ragged K (not a multiple of 16)
         GridSpec((136, 144, 160), (-2.0, -1.5, -1.0), (2.0, 1.5, 1.0)),
         GridSpec((300, 40, 21), (-1.0,) * 3, (1.0,) * 3),           # 3 row blocks, 2 column blocks
         GridSpec((520, 17, 9), (-1.0,) * 3, (1.0,) * 3)]            # 5 row blocks, 3 column blocks, trimmed N


@pytest.mark.parametrize("gi", [0, 1, 2, 4, 5])
def test_gram_i8_exact_on_integers(T, gi):
    g = GRIDS[gi]
    rng = np.random.default_rng(11 + gi)
    Kmax = max(np.prod(g.n) // g.n[m] for m in range(3))
    bits = min(20, (53 - int(np.ceil(np.log2(Kmax)))) // 2)   # every Gram entry < 2^53: exact in FP64
    F = rng.integers(-(1 << bits), 1 << bits, size=tuple(g.n), dtype=np.int64)
    F[min(1, g.n[0] - 1)] = 0                       # a zero slab: zero rows (mode 0), zero columns
    F[0, 0, :] = rng.integers(-3, 4, size=g.n[2])   # tiny entries next to 2^20 ones
    Fd = torch.from_numpy(F.astype(np.float64)).cuda()
    ws = T.workspace_i8(g)
    for m in range(3):
        A = unfold(F, m)
        assert A.shape[1] * (1 << (2 * bits)) < (1 << 53)
        exact = (A @ A.T).astype(np.float64)
        G = to_np(T.gram_i8(g, m, Fd, ws))
        assert np.array_equal(G, exact), (gi, m, np.max(np.abs(G - exact)))


def _bound(A, b, global_max=None):
    """R18 element bound (per-row exponents), or R20's (global_max given: one exponent for all
    rows, the shared residue layout)."""
    m = np.max(np.abs(A), axis=1)
    if global_max is not None:
        m = np.full_like(m, global_max)
    E = np.where(m > 0, np.frexp(m)[1], 0).astype(np.float64)
    l1 = np.sum(np.abs(A), axis=1)
    s = np.exp2(E - b - 1)
    K = A.shape[1]
    absG = np.abs(A) @ np.abs(A).T
    return np.outer(s, l1) + np.outer(l1, s) + 3 * np.outer(s, s) * K + 2 * K * EPS * absG


@pytest.mark.parametrize("gi", range(len(GRIDS)))
@pytest.mark.parametrize("kern", [KernelSpec.matern(1.3, 0.5), KernelSpec.matern(0.5, 0.1), KernelSpec.slater(1.0, 1.0)])
@pytest.mark.parametrize("layout", ["auto", "rowscaled"])
def test_gram_i8_parity(T, orc, gi, kern, layout):
    """Both residue layouts: per-mode row scaling (R18: element-wise within 1e-14 sqrt(G_aa G_bb))
    and, where it applies (n3 % 16 == 0), the shared layout with one global exponent (R20: within its
    element bound, norm-wise within 2e-15 ||G||_2)."""
    g = GRIDS[gi]
    if layout == "rowscaled":
        T.set_gram_engine(T.GRAM_INT8_ROWSCALED)
    try:
        shared, b = T.i8_layout(g)
        Fg = T.fill(g, kern)
        F = orc.fill(ogrid(orc, g), okern(orc, kern))
        ws = T.workspace_i8(g)
        Gs = [to_np(T.gram_i8(g, m, Fg, ws)) for m in range(3)]
    finally:
        T.set_gram_engine(T.GRAM_AUTO)
    assert shared == (layout == "auto" and g.n[2] % 16 == 0)
    for m in range(3):
        G = Gs[m]
        R = orc.gram_mode(F, m)
        A = unfold(F, m)
        assert np.array_equal(G, G.T)
        if shared:
            assert np.all(np.abs(G - R) <= _bound(A, b, np.max(np.abs(F)))), (gi, m)
            assert np.linalg.norm(G - R, 2) <= 2e-15 * np.linalg.norm(R, 2), (gi, m)
        else:
            assert np.all(np.abs(G - R) <= _bound(A, 50)), (gi, m)
            d = np.sqrt(np.diag(R))
            assert np.max(np.abs(G - R) / np.outer(d, d)) <= 1e-14, (gi, m)


def test_gram_i8_chunks_and_superchunks(T, orc, monkeypatch):
    """K = 2^18: four exact-int32 K-chunks of 2^16; with a 16 MiB residue cap also four
    super-chunks (residues rebuilt per K range, residue sums carried mod p) on the row-scaled layout;
    the shared layout's modes 0 / 1 / 2 (K = 2^18 / 2^15 / 2^15: 4 / 1 / 1 chunks; mode 1 in
    K-blocks per i-slab) within R20's bound."""
    g = GridSpec((64, 512, 512), (-1.0,) * 3, (1.0,) * 3)
    kern = KernelSpec.matern(1.5, 0.3)
    Fg = T.fill(g, kern)
    F = orc.fill(ogrid(orc, g), okern(orc, kern))
    T.set_gram_engine(T.GRAM_INT8_ROWSCALED)
    try:
        R = orc.gram_mode(F, 0)
        A = unfold(F, 0)
        G1 = to_np(T.gram_i8(g, 0, Fg))
        assert np.all(np.abs(G1 - R) <= _bound(A, 50))
        monkeypatch.setenv("TUCKER_I8_RESIDUE_MB", "16")
        G2 = to_np(T.gram_i8(g, 0, Fg))
        assert np.array_equal(G1, G2)  # the result does not depend on how K is split
    finally:
        T.set_gram_engine(T.GRAM_AUTO)
    shared, b = T.i8_layout(g)
    assert shared
    for m in range(3):
        G = to_np(T.gram_i8(g, m, Fg))
        R = orc.gram_mode(F, m)
        assert np.all(np.abs(G - R) <= _bound(unfold(F, m), b, np.max(np.abs(F)))), m


def test_gram_i8_deterministic_and_vs_dmma(T):
    g = GridSpec((136, 144, 160), (-2.0, -1.5, -1.0), (2.0, 1.5, 1.0))
    F = T.fill(g, KernelSpec.matern(0.7, 0.5))
    ws = T.workspace_i8(g)
    for m in range(3):
        G = T.gram_i8(g, m, F, ws)
        assert torch.equal(G, T.gram_i8(g, m, F, ws))
        T.set_gram_engine(T.GRAM_DMMA)
        try:
            D = T.gram(g, m, F, T.workspace(g))  # k_gram_tma (FP64 tensor cores)
        finally:
            T.set_gram_engine(T.GRAM_AUTO)
        d = torch.sqrt(torch.diagonal(D))
        assert float(torch.max(torch.abs(G - D) / torch.outer(d, d))) <= 1e-14


def test_int8_route_lowers_the_noise_floor(T):
    """The emulated Gram has no accumulation error (only the 2^-51 input rounding), the DMMA Gram
    accumulates K = 1M FP64 products: in the noise regime (1024^3, Matérn 3/2, ell = 0.2, r = 40) the
    HOSVD error through the INT8 route is an order of magnitude lower (measured 5.36e-9 vs 6.77e-8)."""
    g, k, rr = GridSpec.cube(1024, 1.0), KernelSpec.matern(1.5, 0.2), (40, 40, 40)
    F = T.fill(g, k)
    E = {}
    for eng in (T.GRAM_INT8, T.GRAM_DMMA):
        T.set_gram_engine(eng)
        try:
            res = T.hosvd(g, rr, F)
            E[eng] = float(T.error(g, rr, F, res.U, res.core)[0])
        finally:
            T.set_gram_engine(T.GRAM_AUTO)
    assert 2 * E[T.GRAM_INT8] < E[T.GRAM_DMMA], E


@pytest.mark.parametrize("g,k,kb,mb", [
    (GridSpec.cube(128, 1.0), KernelSpec.matern(1.5, 0.2), None, None),
    (GridSpec((136, 144, 160), (-2.0, -1.5, -1.0), (2.0, 1.5, 1.0)), KernelSpec.matern(0.7, 0.5), 256, None),
    (GridSpec((144, 136, 130), (-0.5, -2.0, 0.1), (1.5, 1.0, 0.9)), KernelSpec.matern(1.5, 0.2), 300, 1),
    (GridSpec((130, 129, 136), (-1.0,) * 3, (1.0,) * 3), KernelSpec.slater(1.0, 1.0), 200, 2)])
def test_gram_i8_fused_bitwise_equals_materialised(T, monkeypatch, g, k, kb, mb):
    """a-7 through the INT8 Gram: F generated in plane chunks (test knob: chunk KB, residue MB) never
    stored; the residues are of bitwise the same values and the integer products are exact, so the
    fused Gram equals the materialised INT8 Gram bit for bit."""
    if kb:
        monkeypatch.setenv("TUCKER_FUSED_CHUNK_KB", str(kb))
    if mb:
        monkeypatch.setenv("TUCKER_I8_RESIDUE_MB", str(mb))
    F = T.fill(g, k)
    T.set_gram_engine(T.GRAM_INT8_ROWSCALED)  # the fused route's layout (per-mode row scaling)
    try:
        ws = T.workspace_i8(g)
        wsf = T.workspace_fused(g)
        for m in range(3):
            assert torch.equal(T.gram_fused(g, k, m, wsf), T.gram_i8(g, m, F, ws)), m
    finally:
        T.set_gram_engine(T.GRAM_AUTO)


def test_stage_profiler_and_engine_switch(T):
    """tucker_profile_*: per-stage event times on the launching stream; the engine switch routes
    tucker_hosvd through the INT8 Gram (AUTO) or the DMMA Gram, with matching results."""
    g, k, rr = GridSpec.cube(256, 1.0), KernelSpec.matern(1.5, 0.2), (16, 16, 16)
    F = T.fill(g, k)
    T.profile_read()
    T.profile_enable(True)
    try:
        a = T.hosvd(g, rr, F)
        torch.cuda.synchronize()
    finally:
        T.profile_enable(False)
    p = T.profile_read()
    assert p["i8_gemm"][1] == 3 and p["i8_residues"][1] >= 1 and p["i8_rowmax"][1] == 1 and p["eig"][1] >= 3
    assert p["dmma_gram"][1] == 0 and all(v[0] >= 0.0 for v in p.values())
    assert p["i8_gemm"][0] > 0.0
    assert T.profile_read()["i8_gemm"] == (0.0, 0)  # cleared; disabled: nothing recorded
    T.hosvd(g, rr, F)
    assert T.profile_read()["i8_gemm"] == (0.0, 0)
    T.set_gram_engine(T.GRAM_DMMA)
    try:
        T.profile_enable(True)
        b = T.hosvd(g, rr, F)
        torch.cuda.synchronize()
        T.profile_enable(False)
        q = T.profile_read()
    finally:
        T.profile_enable(False)
        T.set_gram_engine(T.GRAM_AUTO)
    assert q["dmma_gram"][1] == 3 and q["i8_gemm"][1] == 0
    for m in range(3):
        la, lb = a.sigma[m] ** 2, b.sigma[m] ** 2
        assert float(torch.max(torch.abs(la - lb) / la[0])) <= 1e-12


def test_gram_i8_2048_materialised_equals_fused(T):
    """Full config-5f size: the materialised INT8 Gram of the stored 2048^3 tensor (68.7 GB) and the
    fused one (F generated chunk by chunk, never stored) are bitwise equal (mode 0: K = 2^22 columns,
    two 8 GiB residue super-chunks, b = 50)."""
    g, k = GridSpec.cube(2048, 1.0), KernelSpec.matern(1.5, 0.2)
    # the row-scaled layout on both sides (at 2048^3 the materialised route cannot hold the shared
    # residues next to F; the default fused route's shared layout is checked in test_gpu_fused.py)
    T.set_gram_engine(T.GRAM_INT8_ROWSCALED)
    try:
        wsf = T.workspace_fused(g)
        Gf = T.gram_fused(g, k, 0, wsf)
        del wsf
        torch.cuda.empty_cache()
        F = T.fill(g, k)
        G = T.gram_i8(g, 0, F)
    finally:
        T.set_gram_engine(T.GRAM_AUTO)
    assert torch.equal(G, Gf)
    d = torch.sqrt(torch.diagonal(G))
    assert bool(torch.all(d > 0)) and torch.equal(G, G.T)


def test_gram_i8_extreme_dynamic_range(T, orc):
    """Row scales far apart: slabs multiplied by 2^e, e in {-1000, -600, 0, 300, 500} (mode-0 rows
    2^-1000 take the two-step scaling, 2^(50+1000) being out of the double exponent range; modes 1
    and 2 mix all scales in every row).  Entries whose exact value underflows are 0 on both sides; the
    rest stay within the R18 bound and no Inf/NaN appears."""
    g = GridSpec((40, 24, 20), (-1.0,) * 3, (1.0,) * 3)
    k = KernelSpec.matern(1.5, 0.3)
    Fo = orc.fill(ogrid(orc, g), okern(orc, k))
    e = np.array([-1000, -600, 0, 300, 500])[np.arange(g.n[0]) % 5]
    F = Fo * np.exp2(e.astype(np.float64))[:, None, None]
    Fd = torch.from_numpy(F).cuda()
    ws = T.workspace_i8(g)
    for m in range(3):
        G = to_np(T.gram_i8(g, m, Fd, ws))
        R = orc.gram_mode(F, m)
        assert np.all(np.isfinite(G)), m
        A = unfold(F, m)
        assert np.all(np.abs(G - R) <= _bound(A, 50) + np.finfo(np.float64).tiny), m


@pytest.mark.parametrize("shape", [(4096, 8, 6), (6, 2048, 16), (3, 5, 2049)])
def test_gram_i8_extreme_aspect(T, orc, shape):
    """Long modes next to tiny ones: 4096 rows with K = 48 (16 x 32 pair tiles, many merged units,
    one K-block), and K = 4 x 2049 columns with 3 rows (one pair tile, ragged K-blocks)."""
    g = GridSpec(shape, (-1.0,) * 3, (1.0,) * 3)
    k = KernelSpec.matern(0.7, 0.4)
    Fg = T.fill(g, k)
    F = orc.fill(ogrid(orc, g), okern(orc, k))
    ws = T.workspace_i8(g)
    for m in range(3):
        G = to_np(T.gram_i8(g, m, Fg, ws))
        R = orc.gram_mode(F, m)
        A = unfold(F, m)
        assert np.array_equal(G, G.T)
        shared, b = T.i8_layout(g)
        gm = np.max(np.abs(F)) if shared else None
        assert np.all(np.abs(G - R) <= _bound(A, b if shared else 50, gm)), (shape, m)


def test_gram_i8_maximum_rows(T, orc):
    """The largest mode the INT8 route takes, n_m = 16384 (64 x 32 pair tiles, K = 12): sampled rows
    of G against the oracle's fill and an FP64 product, within the R18 bound; exact symmetry.  One
    row more (16385) leaves the INT8 route (UNSUPPORTED) and AUTO falls back to the DMMA Gram."""
    g = GridSpec((16384, 4, 3), (-1.0,) * 3, (1.0,) * 3)
    k = KernelSpec.matern(0.7, 0.4)
    Fg = T.fill(g, k)
    A = unfold(orc.fill(ogrid(orc, g), okern(orc, k)), 0)
    G = T.gram_i8(g, 0, Fg, T.workspace_i8(g))
    assert torch.equal(G, G.T)
    rows = np.random.default_rng(16384).choice(16384, 256, replace=False)
    Gs = to_np(G[torch.from_numpy(rows).cuda()])
    m = np.max(np.abs(A), axis=1)
    E = np.where(m > 0, np.frexp(m)[1], 0).astype(np.float64)
    l1 = np.sum(np.abs(A), axis=1)
    s = np.exp2(E - 50 - 1)
    K = A.shape[1]
    bound = (np.outer(s[rows], l1) + np.outer(l1[rows], s) + 3 * np.outer(s[rows], s) * K
             + 2 * K * EPS * (np.abs(A[rows]) @ np.abs(A).T))
    assert np.all(np.abs(Gs - A[rows] @ A.T) <= bound)
    g2 = GridSpec((16385, 4, 3), (-1.0,) * 3, (1.0,) * 3)
    F2 = T.fill(g2, k)
    with pytest.raises(T.TuckerError) as e:
        T.gram_i8(g2, 0, F2, T.workspace_i8(g))
    assert e.value.code in (4, 7)
    G2 = T.gram(g2, 0, F2)  # AUTO engine: the DMMA Gram
    assert torch.equal(G2, G2.T) and G2.shape == (16385, 16385)


@pytest.mark.parametrize("g", [GridSpec((96, 80, 48), (-1.0,) * 3, (1.0,) * 3),
                               GridSpec((136, 144, 160), (-2.0, -1.5, -1.0), (2.0, 1.5, 1.0)),
                               GridSpec((40, 300, 272), (-1.0, -0.5, -1.0), (1.0, 1.5, 0.5))])
def test_gram_i8_shared_layout_exact_on_integers(T, g):
    """The shared residue layout (R20; one residue pass, mode 2 read as MN-major operands, mode 1
    in K-blocks per i-slab with a zero-filled tail when n3 % 128 != 0): on integer-valued F the
    three Grams are the exact integer Grams, bit for bit."""
    shared, b = T.i8_layout(g)
    assert shared
    rng = np.random.default_rng(int(np.prod(g.n)))
    Kmax = max(np.prod(g.n) // g.n[m] for m in range(3))
    bits = min(20, (53 - int(np.ceil(np.log2(Kmax)))) // 2)
    F = rng.integers(-(1 << bits), 1 << bits, size=tuple(g.n), dtype=np.int64)
    F[:, 3, :] = 0
    Fd = torch.from_numpy(F.astype(np.float64)).cuda()
    ws = T.workspace_i8(g)
    for m in range(3):
        A = unfold(F, m)
        exact = (A @ A.T).astype(np.float64)
        G = to_np(T.gram_i8(g, m, Fd, ws))
        assert np.array_equal(G, exact), (m, np.max(np.abs(G - exact)))


@pytest.mark.parametrize("g,k", [(GridSpec.cube(256, 1.0), KernelSpec.matern(1.5, 0.2)),
                                 (GridSpec((129, 131, 64), (-2.0, -1.5, -1.0), (2.0, 1.5, 1.0)), KernelSpec.matern(0.7, 0.3)),
                                 (GridSpec((96, 80, 48), (-1.0,) * 3, (1.0,) * 3), KernelSpec.slater(1.0, 0.2)),
                                 (GridSpec.cube(144, 1.0), KernelSpec.spectral(0.1, 0.4))])
def test_fill_prepare_equals_separate_passes(T, g, k):
    """tucker_fill_prepare (octant fill + shared residues in one pass, the global exponent from the
    smallest radius) gives bitwise the tensor of tucker_fill, and tucker_hosvd_prepared bitwise the
    factors, sigma and core of tucker_hosvd (which takes the exponent from the row maxima and
    re-reads F for the residues); odd axes (middle rows), general nu, p-Slater, spectral density."""
    r = (10, 9, 8)
    F, ws = T.fill_prepare(g, k, r)
    assert torch.equal(F, T.fill(g, k))
    a = T.hosvd_prepared(g, r, F, ws)
    b = T.hosvd(g, r, F)
    assert a.rc == 0 and b.rc == 0
    # the prepared route bounds the unfoldings' row norms and forms the Grams with 14 or 15 moduli
    # where (2^(b-E) max ||a_i|| + sqrt(K)/2)^2 < P_14 / 2 or P_15 / 2 (R21); the plain route always
    # takes 16 — the exact integer Grams, hence every output, are bitwise the same
    assert b.info["moduli"] == [16, 16, 16]
    assert all(x in (14, 15, 16) for x in a.info["moduli"]), a.info["moduli"]
    if tuple(g.n) == (256, 256, 256):
        assert all(x in (14, 15) for x in a.info["moduli"]), a.info["moduli"]
    for m in range(3):
        assert torch.equal(a.U[m], b.U[m]) and torch.equal(a.sigma[m], b.sigma[m]), m
    assert torch.equal(a.core, b.core)
    off = GridSpec((64, 64, 64), (-1.0, -1.0, -0.5), (1.0, 1.0, 1.0))  # not centred: refused
    with pytest.raises(T.TuckerError) as e:
        T.fill_prepare(off, k, (4, 4, 4))
    assert e.value.code == 7


def test_fill_prepare_flat_tensor_keeps_16_moduli(T):
    """R21's bound must fall back to all 16 moduli when the unfolding rows are nearly flat at full
    scale: sigma2 = 1.99 (max F just below 2^1, so |x| reaches ~2^50) and ell = 1000 on 384^3 —
    (2^(b-E) ||a_i||)^2 ~ K 2^100 = 2^117.2 exceeds P_15 / 2 = 2^116.5.  The Grams are still exact
    (bitwise those of the plain route)."""
    g, k, r = GridSpec.cube(384, 1.0), KernelSpec.matern(0.5, 1000.0, 1.99), (4, 4, 4)
    F, ws = T.fill_prepare(g, k, r)
    a = T.hosvd_prepared(g, r, F, ws)
    b = T.hosvd(g, r, F)
    assert a.rc in (0, 5) and b.rc == a.rc  # (5: the noise-level trailing pairs of a near rank-1 G)
    assert a.info["moduli"] == [16, 16, 16]
    for m in range(3):
        assert torch.equal(a.U[m], b.U[m]) and torch.equal(a.sigma[m], b.sigma[m]), m
    assert torch.equal(a.core, b.core)


MODULI = [253, 251, 249, 247, 245, 241, 239, 233, 229, 227, 223, 211, 199, 197, 193, 191]


@pytest.mark.parametrize("g,k", [(GridSpec.cube(256, 1.0), KernelSpec.matern(1.5, 0.2)),
                                 (GridSpec((129, 131, 64), (-2.0, -1.5, -1.0), (2.0, 1.5, 1.0)), KernelSpec.matern(0.7, 0.3)),
                                 (GridSpec((96, 80, 48), (-1.0,) * 3, (1.0,) * 3), KernelSpec.slater(1.0, 0.2)),
                                 (GridSpec.cube(144, 1.0), KernelSpec.spectral(0.1, 0.4)),
                                 (GridSpec.cube(320, 1.0), KernelSpec.matern(0.5, 1000.0, 1.99)),
                                 (GridSpec.cube(384, 1.0), KernelSpec.matern(0.5, 1000.0, 1.99))])
def test_r21_modulus_count_against_true_row_norms(T, g, k):
    """R21 checked against the tensor itself: from the TRUE row norms of every unfolding (numpy on
    the filled tensor), (2^(b-E) max_i ||a_i|| + sqrt(K)/2)^2 is the bound that makes 15 moduli
    exact.  Whenever the prepared route took 15 moduli for a mode, that bound must hold with the
    true norms (the central-row shortcut may only be conservative: it takes 16 at most where the
    true bound is within its 1e-9 margins), and where the true bound holds with room (factor 1.01)
    it must have taken 15."""
    r = (4, 4, 4)
    F, ws = T.fill_prepare(g, k, r)
    a = T.hosvd_prepared(g, r, F, ws)
    assert a.rc in (0, 5)
    A = F.cpu().numpy()
    shared, b = T.i8_layout(g)
    assert shared
    E = int(np.frexp(np.max(np.abs(A)))[1])  # max |a| < 2^E
    P15 = 1
    for p in MODULI[:15]:
        P15 *= p
    for m in range(3):
        U = unfold(A, m)
        K = U.shape[1]
        amax = float(np.sqrt(np.max(np.sum(U * U, axis=1))))
        nx = 2.0 ** (b - E) * amax + 0.5 * np.sqrt(K)
        ok15 = nx * nx < P15 / 2
        got = a.info["moduli"][m]
        assert got in (14, 15, 16), got
        if got == 14:  # the same width b: P_14 / 2 must bound the true S
            P14 = P15 // MODULI[14]
            assert nx * nx < P14 / 2, (m, np.log2(nx * nx), np.log2(P14 / 2))
        elif got == 15:
            assert ok15, (m, np.log2(nx * nx), np.log2(P15 / 2))
        elif nx * nx * 1.01 < P15 / 2:
            pytest.fail(f"mode {m}: 16 moduli although the true bound holds ({np.log2(nx * nx):.3f} < "
                        f"{np.log2(P15 / 2):.3f})")
