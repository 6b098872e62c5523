"""Edge cases of the CUDA path (through the C-ABI): the smallest grid, the largest supported rank,
nearly-constant functions, and the largest grid both materialised and fused (2048^3: 68.7 GB of F
in HBM against the never-stored path)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from test_gpu_parity import _compare_hosvd, ogrid, okern  # noqa: E402
from tucker_inputs import GridSpec, KernelSpec  # noqa: E402
import parity_bars as PB  # noqa: E402


@pytest.fixture(scope="module")
def T():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_1711_06874_b200 import tucker
    tucker.load()
    return tucker


def to_np(t):
    return t.detach().cpu().numpy()


@pytest.mark.parametrize("r", [(1, 1, 1), (2, 2, 2), (1, 2, 1)])
def test_smallest_grid(T, orc, r):
    _compare_hosvd(T, orc, GridSpec((2, 2, 2), (-1.0, -1.0, -1.0), (1.0, 1.0, 1.0)), KernelSpec.matern(1.5, 0.7), r)


def test_largest_rank_and_beyond(T, orc):
    g = GridSpec((160, 100, 128), (-1.0, -1.0, -1.0), (1.0, 1.0, 1.0))
    _compare_hosvd(T, orc, g, KernelSpec.matern(0.5, 0.05), (56, 56, 56))  # eigensolver block limit
    F = T.fill(g, KernelSpec.matern(0.5, 0.05))
    import ctypes
    lib = T.load()
    U = [torch.empty((g.n[m], 57), dtype=torch.float64, device="cuda") for m in range(3)]
    S = [torch.empty(57, dtype=torch.float64, device="cuda") for _ in range(3)]
    core = torch.empty((57, 57, 57), dtype=torch.float64, device="cuda")
    ws = T.workspace(g, (57, 57, 57))
    rc = lib.tucker_hosvd(ctypes.byref(T.cgrid(g)), T.cranks((57, 57, 57)), T._ptr(F), *[T._ptr(u) for u in U],
                          T._ptr(core), *[T._ptr(s) for s in S], T._ptr(ws), ws.numel(), None, None)
    assert rc == 7  # TUCKER_ERR_UNSUPPORTED, documented in include/tucker.h


def test_nearly_constant_function(T, orc):
    """ell >> box: F ~ sigma^2 (1 - small), numerically rank 1; nothing may break (no NaN, sign rule,
    orthonormal factors) and E(1) is tiny."""
    g, k = GridSpec((40, 36, 32), (-1.0, -1.0, -1.0), (1.0, 1.0, 1.0)), KernelSpec.matern(1.5, 1e4)
    res, err = _compare_hosvd(T, orc, g, k, (3, 3, 3))
    assert np.all(np.isfinite(to_np(res.core))) and err[0] < 1e-6


def test_2048_materialised_vs_fused(T, orc):
    """The largest grid in both forms: F materialised (68.7 GB) against the fused path."""
    g, k, r = GridSpec.cube(2048, 1.0), KernelSpec.matern(1.5, 0.2), (10, 10, 10)
    F = T.fill(g, k)
    og, ok = ogrid(orc, g), okern(orc, k)
    # sampled entries of the materialised fill against the oracle, one by one
    rng = np.random.default_rng(7)
    for i, j, l in rng.integers(0, 2048, size=(8, 3)):
        ref = orc.fill_entry(og, ok, int(i), int(j), int(l))
        assert abs(float(F[i, j, l]) - ref) <= 4 * np.spacing(ref)
    ws = T.workspace(g, r)
    G = T.gram(g, 2, F, ws)
    Gn = to_np(G)
    # INT8 route (R18): sampled entries within the element bound (row maxima and 1-norms from the
    # oracle's kernel evaluation) and within 1e-14 sqrt(G_aa G_bb)
    K = 2048 * 2048
    _, bits = T.i8_scheme(K)
    for a, b in rng.integers(0, 2048, size=(4, 2)):
        ref = orc.gram_entry_fn(og, ok, 2, int(a), int(b))
        (ma, la), (mb, lb) = orc.row_stats_fn(og, ok, 2, int(a)), orc.row_stats_fn(og, ok, 2, int(b))
        assert abs(Gn[a, b] - ref) <= PB.i8_bound_entry(ma, mb, la, lb, K, bits, ref), (a, b)
        assert abs(Gn[a, b] - ref) <= 1e-14 * np.sqrt(Gn[a, a] * Gn[b, b])
    del G
    ref = T.hosvd(g, r, F, ws)
    e_ref = to_np(T.error(g, r, F, ref.U, ref.core, ws))
    del F, ws
    torch.cuda.empty_cache()
    res = T.hosvd_fused(g, k, r)
    e = to_np(T.error_fused(g, k, r, res.U, res.core))
    assert ref.rc == 0 and res.rc == 0
    for m in range(3):
        lr, lam = to_np(ref.sigma[m]) ** 2, to_np(res.sigma[m]) ** 2
        assert np.all(np.abs(lam - lr) <= 1e-11 * lr + 1e-14 * lr[0])
        U, Ur = to_np(res.U[m]), to_np(ref.U[m])
        for c in range(r[m]):
            if lr[c] >= 1e-6 * lr[0] and np.min(np.abs(np.delete(lr, c) - lr[c])) >= 1e-6 * lr[0]:
                assert np.max(np.abs(U[:, c] - Ur[:, c])) <= 1e-9
    assert abs(e[1] - e_ref[1]) <= 1e-13 * e_ref[1]
    assert abs(e[0] - e_ref[0]) <= max(1e-12, 1e-15 / e_ref[0])


def test_config4_batch_512(T, orc):
    """BASELINE config 4: 512^3, the 16 seeded Matérn settings (R10), ranks 30.  Every setting's
    eigensolves converge; sampled entries against the oracle; E(r) non-increasing over r = 10,
    20, 30; the orthogonal-projection identity at r = 30."""
    from tucker_inputs import config4
    w = config4()
    g, r = w.grid, w.ranks
    F = torch.empty(tuple(g.n), dtype=torch.float64, device="cuda")
    ws = T.workspace(g, r)
    rng = np.random.default_rng(4)
    for k in w.kernels:
        T.fill(g, k, F, ws)
        for i, j, l in rng.integers(0, 512, size=(2, 3)):
            ref = orc.fill_entry(ogrid(orc, g), okern(orc, k), int(i), int(j), int(l))
            bound = 4 * np.spacing(ref) if k.nu in (0.5, 1.5, 2.5) else 1e-14 * abs(ref)
            assert abs(float(F[i, j, l]) - ref) <= bound
        res = T.hosvd(g, r, F, ws)
        assert res.rc == 0 and all(res.info["converged"]), (k.label(), res.info)
        es = []
        for rr in (10, 20, 30):
            U = [u[:, :rr].contiguous() for u in res.U]
            core = T.ttm_core(g, (rr,) * 3, F, *U, ws=ws)
            es.append(to_np(T.error(g, (rr,) * 3, F, U, core, ws)))
        assert es[0][0] >= es[1][0] * (1 - 1e-12) >= es[2][0] * (1 - 1e-12) * (1 - 1e-12)
        nb = np.linalg.norm(to_np(core))
        e = es[2]
        assert abs(e[1] ** 2 - nb ** 2 - e[2] ** 2) <= 1e-12 * e[1] ** 2


def test_eig_single_cta_fallback_beyond_cluster(T, orc):
    """n > 2048 exceeds the 16-CTA cluster: tucker_eig falls back to the single-CTA Rayleigh–Ritz
    path.  Against numpy.linalg.eigh (LAPACK) on the oracle's Gram of a 2100 x 8 x 6 tensor."""
    from tucker_inputs import GridSpec, KernelSpec
    g = GridSpec((2100, 8, 6), (-1.0, -1.0, -1.0), (1.0, 1.0, 1.0))
    F = orc.fill(ogrid(orc, g), okern(orc, KernelSpec.matern(0.7, 0.3)))
    G = orc.gram_mode(F, 0)
    lam_ref, V_ref = np.linalg.eigh(G)
    lam_ref, V_ref = lam_ref[::-1], V_ref[:, ::-1]
    r = 12
    U, lam, info, rc = T.eig(torch.from_numpy(G).cuda(), r)
    assert rc == 0, info
    U, lam = to_np(U), to_np(lam)
    assert np.all(np.abs(lam - lam_ref[:r]) <= 1e-11 * np.abs(lam_ref[:r]) + 1e-14 * lam_ref[0])
    assert np.max(np.abs(U.T @ U - np.eye(r))) <= 1e-12
    for c in range(r):
        if np.min(np.abs(np.delete(lam_ref, c) - lam_ref[c])) >= 1e-6 * lam_ref[0]:
            v = V_ref[:, c] * np.sign(V_ref[np.argmax(np.abs(V_ref[:, c]) >= 0.5 * np.max(np.abs(V_ref[:, c]))), c])
            assert np.max(np.abs(U[:, c] - v)) <= 1e-9, c


# ------------------------------------------------------------------------ boundary (round 2) --
def test_hosvd_async_equals_sync_and_graph_capture(T):
    """info == NULL: no host synchronisation; bitwise the synchronous result, and the
    whole HOSVD can be captured in a CUDA Graph and replayed."""
    g, k, r = GridSpec((256, 192, 160), (-1.0,) * 3, (1.0,) * 3), KernelSpec.matern(1.5, 0.3), (20, 16, 12)
    F = T.fill(g, k)
    ws = T.workspace(g, r)
    a = T.hosvd(g, r, F, ws)
    assert a.rc == 0 and min(a.info["k_resolved"]) >= 1
    b = T.hosvd(g, r, F, ws, sync=False)
    torch.cuda.synchronize()
    assert b.rc == 0
    for m in range(3):
        assert torch.equal(a.U[m], b.U[m]) and torch.equal(a.sigma[m], b.sigma[m])
    assert torch.equal(a.core, b.core)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    out = None
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        T.hosvd(g, r, F, ws, stream=s, sync=False)  # warm-up (attributes, side streams)
        s.synchronize()
        with torch.cuda.graph(graph, stream=s):
            out = T.hosvd(g, r, F, ws, stream=s, sync=False)
    graph.replay()
    torch.cuda.synchronize()
    for m in range(3):
        assert torch.equal(out.U[m], a.U[m])
    assert torch.equal(out.core, a.core)


def test_stale_rowmax_is_detected(T):
    """A caller row maximum that does not bound its row: TUCKER_ERR_INPUT (sync), NaN (async)."""
    g, k, r = GridSpec.cube(128, 1.0), KernelSpec.matern(1.5, 0.2), (8, 8, 8)
    F, mx = T.fill_rowmax(g, k)
    good = T.hosvd(g, r, F, rowmax=mx)
    assert good.rc == 0
    stale = mx.clone()
    stale -= 2 << 20  # every row maximum two binades too low (also the global one, R20)
    with pytest.raises(T.TuckerError) as e:
        T.hosvd(g, r, F, rowmax=stale)
    assert e.value.code == 9
    res = T.hosvd(g, r, F, rowmax=stale, sync=False)
    torch.cuda.synchronize()
    assert torch.isnan(res.sigma[0]).any()
    again = T.hosvd(g, r, F, rowmax=mx)  # the flag does not leak into the next call
    assert again.rc == 0 and torch.equal(again.U[0], good.U[0])


def test_nonfinite_input_propagates(T):
    g = GridSpec.cube(64, 1.0)
    F = T.fill(g, KernelSpec.matern(0.5, 0.3))
    F[3, 4, 5] = float("nan")
    for m in range(3):
        assert torch.isnan(T.gram(g, m, F)).all()
    with pytest.raises(T.TuckerError) as e:
        T.hosvd(g, (4, 4, 4), F)
    assert e.value.code in (5, 9)


def test_rank_limits_checked_before_launch(T):
    g = GridSpec((300, 40, 40), (-1.0,) * 3, (1.0,) * 3)
    F = torch.zeros(tuple(g.n), dtype=torch.float64, device="cuda")
    with pytest.raises(T.TuckerError) as e:
        T.hosvd(g, (57, 8, 8), F)
    assert e.value.code == 7
    assert T.last_launch_count() == 0
