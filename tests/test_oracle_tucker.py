"""Pins for the oracle's Gram, Jacobi eigensolver, TTM core, reconstruction error and HOSVD
(P:526-585), and Table 2 through the test-only HOOI sweeps."""
import os

import mpmath as mp
import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


# ---------------------------------------------------------------------------------- Gram ----
def test_gram_exact_on_integers(orc):
    rng = np.random.default_rng(1)
    A = rng.integers(-1000, 1000, size=(17, 301)).astype(np.float64)
    G = orc.gram(A)
    Ai = A.astype(np.int64)
    assert np.array_equal(G, (Ai @ Ai.T).astype(np.float64))


def test_gram_vs_blas(orc):
    rng = np.random.default_rng(2)
    A = rng.standard_normal((40, 5000))
    G = orc.gram(A)
    nrm = np.linalg.norm(A, axis=1)
    assert np.max(np.abs(G - A @ A.T) / np.outer(nrm, nrm)) <= 1e-14


def test_unfold_and_mode_invariants(orc):
    g = orc.Grid.cube(12, 1.0)
    F = orc.fill(g, orc.Kernel.matern(1.3, 0.5))
    nf2 = float(np.sum(F * F))
    Gs = [orc.gram_mode(F, m) for m in range(3)]
    for m in range(3):
        A = orc.unfold(F, m)
        assert np.array_equal(A, np.moveaxis(F, m, 0).reshape(F.shape[m], -1))
        assert abs(np.trace(Gs[m]) - nf2) <= 1e-14 * nf2  # trace G_m = ||F||^2 for every mode
        assert np.array_equal(Gs[m], Gs[m].T)
    # cubic isotropic grid: G_1 == G_2 bitwise (same terms, same order); G_3 to rounding
    assert np.array_equal(Gs[0], Gs[1])
    assert np.max(np.abs(Gs[0] - Gs[2])) <= 1e-15 * np.max(Gs[0])


def test_gram_entry_fn(orc):
    g = orc.Grid((10, 8, 6), (-2.0, -1.5, -1.0), (2.0, 1.5, 1.0))
    k = orc.Kernel.matern(0.7, 0.5)
    F = orc.fill(g, k)
    for m in range(3):
        G = orc.gram_mode(F, m)
        for a, b in ((0, 0), (1, 3), (g.n[m] - 1, 2)):
            assert abs(orc.gram_entry_fn(g, k, m, a, b) - G[a, b]) <= 1e-15 * G[a, a]


def test_row_stats_fn(orc):
    """orc_row_stats_fn (inputs of the R18 element bound) = numpy's max / sum of |row| of the
    filled tensor's unfolding."""
    g = orc.Grid((10, 8, 6), (-2.0, -1.5, -0.5), (2.0, 1.5, 1.0))
    k = orc.Kernel.matern(0.7, 0.5)
    F = orc.fill(g, k)
    for m in range(3):
        A = np.abs(np.moveaxis(F, m, 0).reshape(F.shape[m], -1))
        for a in (0, 3, g.n[m] - 1):
            mx, l1 = orc.row_stats_fn(g, k, m, a)
            assert mx == A[a].max()
            assert abs(l1 - np.sum(A[a])) <= 1e-15 * l1


# ---------------------------------------------------------------------------------- Jacobi --
@pytest.mark.parametrize("n", [1, 2, 3, 7, 16, 33, 64])
def test_jacobi_vs_eigh(orc, n):
    rng = np.random.default_rng(n)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam_true = np.linspace(10.0, 0.5, n)  # separated spectrum (gap >= 0.15)
    G = (Q * lam_true) @ Q.T
    G = 0.5 * (G + G.T)
    lam, V, rc, sweeps = orc.jacobi_eig(G)
    assert rc == 0
    w, Z = np.linalg.eigh(G)
    w, Z = w[::-1], orc.sign_fix(Z[:, ::-1])
    assert np.max(np.abs(lam - w)) <= 1e-13 * w[0]
    assert np.max(np.abs(V - Z)) <= 1e-11  # gaps >= ~0.1: |dv| ~ eps ||G|| / gap
    assert np.max(np.abs(V.T @ V - np.eye(n))) <= 1e-13
    assert np.max(np.abs(G @ V - V * lam)) <= 1e-13 * w[0]


def test_jacobi_2x2_closed_form(orc):
    a, b, c = 3.0, 1.25, -2.0
    lam, V, rc, _ = orc.jacobi_eig(np.array([[a, b], [b, c]]))
    d = np.sqrt((a - c) ** 2 + 4 * b * b)
    assert lam[0] == pytest.approx((a + c + d) / 2, rel=1e-15)
    assert lam[1] == pytest.approx((a + c - d) / 2, rel=1e-15)


def test_jacobi_diagonal_and_ties(orc):
    lam, V, rc, sw = orc.jacobi_eig(np.diag([1.0, 5.0, 5.0, 2.0, 0.0]))
    assert rc == 0 and sw == 1
    assert list(lam) == [5.0, 5.0, 2.0, 1.0, 0.0]
    # ties keep input order (R7): the two 5.0 columns are e_1 then e_2
    assert V[1, 0] == 1.0 and V[2, 1] == 1.0


def test_jacobi_rank_deficient_gram(orc):
    # a numerically rank-deficient PSD Gram (1e16 dynamic range) still converges (R7 floor)
    g = orc.Grid.cube(48, 1.0)
    F = orc.fill(g, orc.Kernel.matern(1.5, 0.2))
    G = orc.gram_mode(F, 0)
    lam, V, rc, sw = orc.jacobi_eig(G)
    assert rc == 0 and sw < 30
    assert np.max(np.abs(V.T @ V - np.eye(48))) <= 1e-13
    s = np.linalg.svd(orc.unfold(F, 0), compute_uv=False)
    k = 6  # resolved part of the spectrum (lambda_k >= 1e-10 lambda_1)
    assert np.all(np.abs(lam[:k] - s[:k] ** 2) <= 1e-12 * s[:k] ** 2 + 1e-14 * s[0] ** 2)


def test_sign_rule(orc):
    V = np.array([[0.1, -0.5], [-0.7, 0.5], [0.7, 0.1]])
    W = orc.sign_fix(V)
    # column 0: first index with |v| >= max/2 is i=1 (-0.7) -> flipped; column 1: i=0 -> flipped
    assert np.array_equal(W, -V)


# ------------------------------------------------------------------------------ TTM / error --
def test_ttm_core_brute_force(orc):
    rng = np.random.default_rng(3)
    F = rng.standard_normal((5, 6, 7))
    U = [np.linalg.qr(rng.standard_normal((n, r)))[0] for n, r in ((5, 2), (6, 3), (7, 4))]
    core = orc.ttm_core(F, *U)
    ref = np.zeros((2, 3, 4))
    for a in range(2):
        for b in range(3):
            for c in range(4):
                ref[a, b, c] = sum(F[i, j, k] * U[0][i, a] * U[1][j, b] * U[2][k, c]
                                   for i in range(5) for j in range(6) for k in range(7))
    assert np.max(np.abs(core - ref)) <= 1e-14 * np.max(np.abs(ref))
    # identity factors select the leading block of F
    I = [np.eye(n)[:, :r] for n, r in ((5, 2), (6, 3), (7, 4))]
    assert np.array_equal(orc.ttm_core(F, *I), F[:2, :3, :4])
    Ft = orc.reconstruct(F.shape, *U, core)
    assert np.allclose(Ft, np.einsum("abc,ia,jb,kc->ijk", core, *U), rtol=0, atol=1e-14)


def test_error_special_cases(orc):
    rng = np.random.default_rng(4)
    F = rng.standard_normal((4, 5, 6))
    I = [np.eye(n) for n in F.shape]
    E, nf, nd = orc.tucker_error(F, *I, F)  # exact representation -> 0
    assert E == 0.0 and nf == pytest.approx(np.linalg.norm(F), rel=1e-15)
    Z = [np.eye(n)[:, :1] for n in F.shape]
    E, nf, nd = orc.tucker_error(F, *Z, np.zeros((1, 1, 1)))  # zero approximation -> 1
    assert E == pytest.approx(1.0, rel=1e-15)


# ---------------------------------------------------------------------------------- HOSVD ----
def test_full_rank_reconstruction(orc):
    rng = np.random.default_rng(5)
    F = rng.standard_normal((6, 7, 8))
    h = orc.hosvd(F, F.shape)
    E = orc.tucker_error(F, *h.U, h.core)[0]
    assert h.rc == 0 and E <= 1e-13


def test_half_rank_reconstruction_on_symmetric_grid(orc):
    # every fibre is even on a centred grid, so rank F_(m) <= ceil(n/2): E(ceil(n/2)) ~ 0
    for n in (4, 5, 8):
        F = orc.fill(orc.Grid.cube(n, 1.0), orc.Kernel.matern(0.5, 0.5))
        r = (n + 1) // 2
        h = orc.hosvd(F, (r, r, r))
        assert orc.tucker_error(F, *h.U, h.core)[0] <= 1e-12


def test_gaussian_rank_one(orc):
    # separable Gaussian -> Tucker rank 1, beta_111 = ||F||, U_m = g_m/||g_m||
    g = orc.Grid((32, 24, 16), (-2.0, -1.5, -1.0), (2.0, 1.5, 1.0))
    F = orc.fill(g, orc.Kernel.slater(1.0, 2.0))
    h = orc.hosvd(F, (1, 1, 1))
    E, nf, _ = orc.tucker_error(F, *h.U, h.core)
    assert E <= 1e-14
    assert abs(h.core[0, 0, 0] - nf) <= 1e-14 * nf
    for a in range(3):
        v = np.exp(-orc.nodes(g.n[a], g.lo[a], g.hi[a]) ** 2)
        assert np.max(np.abs(h.U[a][:, 0] - v / np.linalg.norm(v))) <= 1e-14


def test_two_dimensional_case_is_truncated_svd(orc):
    # for d = 2 the orthogonal Tucker decomposition is the SVD (n3 = 1 embedding)
    rng = np.random.default_rng(6)
    M = rng.standard_normal((20, 15)) @ np.diag(0.5 ** np.arange(15)) @ rng.standard_normal((15, 15))
    F = M[:, :, None].copy()
    r = 5
    h = orc.hosvd(F, (r, r, 1))
    Us, s, Vt = np.linalg.svd(M)
    E = orc.tucker_error(F, *h.U, h.core)[0]
    assert abs(E - np.sqrt(np.sum(s[r:] ** 2)) / np.linalg.norm(M)) <= 1e-13
    assert np.max(np.abs(h.U[0] - orc.sign_fix(Us[:, :r]))) <= 1e-12
    assert np.max(np.abs(h.lam[0][:r] - s[:r] ** 2)) <= 1e-13 * s[0] ** 2


def test_hosvd_vs_unfolding_svd_and_identity(orc):
    F = orc.fill(orc.Grid((20, 16, 12), (-2.0, -1.5, -1.0), (2.0, 1.5, 1.0)), orc.Kernel.matern(0.7, 0.5))
    r = (6, 6, 5)
    h = orc.hosvd(F, r)
    E, nf, nd = orc.tucker_error(F, *h.U, h.core)
    for m in range(3):
        s = np.linalg.svd(orc.unfold(F, m), compute_uv=False)
        k = int(np.sum(s ** 2 >= 1e-10 * s[0] ** 2))
        assert np.all(np.abs(h.lam[m][:k] - s[:k] ** 2) <= 1e-11 * s[:k] ** 2 + 1e-14 * s[0] ** 2)
        assert np.max(np.abs(h.U[m].T @ h.U[m] - np.eye(r[m]))) <= 1e-12  # T2'
    # orthogonal projection: ||F||^2 = ||beta||^2 + (E ||F||)^2
    assert abs(nf ** 2 - (np.sum(h.core ** 2) + nd ** 2)) <= 1e-13 * nf ** 2


def test_n4_brute_force(orc):
    # O8: on a centred n=4 grid each G_m acts on the even subspace span{(1,0,0,1),(0,1,1,0)} only;
    # its two eigenpairs are the closed-form 2x2 ones, computed here in 50-digit arithmetic.
    mp.mp.dps = 50
    ell, nu = mp.mpf("0.5"), mp.mpf("0.5")
    xs = [mp.mpf(-1) + i * mp.mpf(2) / 3 for i in range(4)]
    Fm = [[[mp.exp(-mp.sqrt(xs[i] ** 2 + xs[j] ** 2 + xs[k] ** 2) / ell) for k in range(4)]
           for j in range(4)] for i in range(4)]
    G = [[mp.fsum(Fm[a][j][k] * Fm[b][j][k] for j in range(4) for k in range(4)) for b in range(4)]
         for a in range(4)]
    e = [[1 / mp.sqrt(2), 0, 0, 1 / mp.sqrt(2)], [0, 1 / mp.sqrt(2), 1 / mp.sqrt(2), 0]]
    M = [[mp.fsum(e[p][a] * G[a][b] * e[q][b] for a in range(4) for b in range(4)) for q in range(2)]
         for p in range(2)]
    tr, det = M[0][0] + M[1][1], M[0][0] * M[1][1] - M[0][1] ** 2
    disc = mp.sqrt(tr ** 2 / 4 - det)
    lam1, lam2 = tr / 2 + disc, tr / 2 - disc
    F = orc.fill(orc.Grid.cube(4, 1.0), orc.Kernel.matern(0.5, 0.5))
    assert np.max(np.abs(F - np.array(Fm, dtype=float))) <= 4e-16
    h = orc.hosvd(F, (2, 2, 2))
    for m in range(3):
        assert abs(h.lam[m][0] - float(lam1)) <= 1e-14 * float(lam1)
        assert abs(h.lam[m][1] - float(lam2)) <= 1e-13 * float(lam1)
        assert np.all(np.abs(h.lam[m][2:]) <= 1e-14 * float(lam1))
        # leading eigenvector from the 2x2 problem: w = (M01, lam1 - M00) in the (e1, e2) basis
        w = [M[0][1], lam1 - M[0][0]]
        v = [w[0] * e[0][a] + w[1] * e[1][a] for a in range(4)]
        nv = mp.sqrt(mp.fsum(t * t for t in v))
        v = np.array([float(t / nv) for t in v])
        v = v if v[0] > 0 else -v
        assert np.max(np.abs(h.U[m][:, 0] - v)) <= 1e-14
    assert orc.tucker_error(F, *h.U, h.core)[0] <= 1e-13


def test_error_decays_exponentially_in_rank(orc):
    # E(r) non-increasing for nested truncations, log E ~ linear in r
    F = orc.fill(orc.Grid.cube(40, 1.0), orc.Kernel.matern(0.5, 0.5))
    h = orc.hosvd(F, (12, 12, 12))
    Es = []
    for r in range(1, 13):
        U = [u[:, :r] for u in h.U]
        Es.append(orc.tucker_error(F, *U, orc.ttm_core(F, *U))[0])
    Es = np.array(Es)
    assert np.all(np.diff(Es) <= 1e-15)
    sel = Es >= 1e-7
    x, y = np.arange(1, 13)[sel], np.log(Es[sel])
    slope, icpt = np.polyfit(x, y, 1)
    r2 = 1 - np.sum((y - (slope * x + icpt)) ** 2) / np.sum((y - y.mean()) ** 2)
    assert slope < 0 and r2 >= 0.9


def test_config1_reference_values(orc):
    # BASELINE config 1 (32^3, nu=1/2, ell=0.5, ranks 8): E(8) ~ 9.562e-7, fully resolved
    F = orc.fill(orc.Grid.cube(32, 1.0), orc.Kernel.matern(0.5, 0.5))
    h = orc.hosvd(F, (8, 8, 8))
    E, nf, nd = orc.tucker_error(F, *h.U, h.core)
    assert h.rc == 0
    assert 9.55e-7 < E < 9.58e-7
    for m in range(3):
        assert np.max(np.abs(h.U[m].T @ h.U[m] - np.eye(8))) <= 1e-12


# ---------------------------------------------------------------------------------- Table 2 --
def _table2():
    rows = {}
    with open(os.path.join(HERE, "golden", "table2.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            parts = line.split()
            rows[int(parts[0])] = parts[1:]
    return rows


def _within_last_digit(value, printed):
    s = printed.rstrip("E")
    if "e" in s:
        mant, ex = s.split("e")
        dec = len(mant.split(".")[1]) if "." in mant else 0
        unit = 10.0 ** (int(ex) - dec)
    else:
        dec = len(s.split(".")[1]) if "." in s else 0
        unit = 10.0 ** (-dec)
    return abs(value - float(s)) <= unit * (1 + 1e-9)


@pytest.mark.parametrize("n", [129, 257, pytest.param(513, marks=pytest.mark.slow)])
def test_table2(orc, n):
    """HOSVD + 3 ALS sweeps (R12), box [-5,5]^3 (R1); every cell within one unit
    of its last printed digit; the 'E' cells are compared with E_FN (R13)."""
    printed = _table2()[n]
    F = orc.fill(orc.Grid.cube(n, 5.0), orc.Kernel.slater(1.0, 1.0))
    h = orc.hosvd(F, (10, 10, 10))
    c = (n - 1) // 2
    for r in range(1, 11):
        U, core, rc = orc.hooi(F, [u[:, :r] for u in h.U], 3)
        cell = printed[r - 1]
        if cell.endswith("E"):
            val = orc.tucker_error(F, *U, core)[0]
        else:
            val = abs(1.0 - orc.tucker_point(U, core, c, c, c))
        assert _within_last_digit(val, cell), (n, r, val, cell)


# ------------------------------------------------- NEXT f2 reference: HOSVD by SVD of unfoldings
def test_hosvd_svd_pins(orc):
    """orc.hosvd_svd (LAPACK SVD of the explicit unfoldings) — pinned against the Gram
    route where both are accurate, full-rank exactness, and beating the Gram route's floor."""
    g = orc.Grid((24, 20, 28), (-1.0, -1.0, -1.0), (1.0, 1.0, 1.0))
    F = orc.fill(g, orc.Kernel.matern(1.5, 0.3))
    r = (12, 12, 12)
    hs, hg = orc.hosvd_svd(F, r), orc.hosvd(F, r)
    for m in range(3):
        l_svd, l_gram = hs.lam[m][: r[m]], hg.lam[m][: r[m]]
        big = l_svd >= 1e-12 * l_svd[0]
        # the T1 bar between the two routes (the Gram's eigenvalues carry ~eps lambda_1 absolute)
        assert np.all(np.abs(l_svd - l_gram) <= 1e-11 * l_svd + 1e-14 * l_svd[0])
        U = hs.U[m]
        assert np.max(np.abs(U.T @ U - np.eye(r[m]))) <= 1e-13
        for c in np.nonzero(big)[0]:  # resolved and gap-separated columns agree
            others = np.delete(hs.lam[m], c)
            if np.min(np.abs(others - hs.lam[m][c])) >= 1e-6 * hs.lam[m][0]:
                assert np.max(np.abs(U[:, c] - hg.U[m][:, c])) <= 1e-9
    # full rank: exact reconstruction
    full = orc.hosvd_svd(F, F.shape)
    assert orc.tucker_error(F, *full.U, full.core)[0] <= 1e-14
    # the SVD route keeps decaying where the Gram route plateaus at ~1e-8
    E_svd = [orc.tucker_error(F, *[u[:, :k] for u in hs.U], orc.ttm_core(F, *[u[:, :k] for u in hs.U]))[0]
             for k in range(1, 13)]
    E_gram = orc.tucker_error(F, *hg.U, hg.core)[0]
    assert all(b <= a * (1 + 1e-12) for a, b in zip(E_svd, E_svd[1:]))
    assert E_svd[-1] < 1e-10 and E_svd[-1] < 1e-2 * E_gram, (E_svd[-1], E_gram)
    # Eckart-Young per mode: sum of the discarded sigma^2 of every mode bounds E^2 ||F||^2 from above
    nF2 = np.sum(F * F)
    tail = sum(np.sum(hs.lam[m][r[m]:]) for m in range(3))
    assert E_svd[-1] ** 2 * nF2 <= tail * (1 + 1e-10) + 1e-28 * nF2
