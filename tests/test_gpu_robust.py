"""Memory-safety checks of our own (compute-sanitizer is closed on this GPU pool: runs under it
left GPUs needing a reset).  Through the C-ABI on small grids that reach every kernel family:

* guard bands — every output buffer and the workspace sit between canary regions filled with a
  byte pattern; after the call the canaries must be intact (an out-of-bounds store shows here);
* poisoned workspace — the workspace filled with 0xFF bytes (NaN doubles, huge ints) before the call
  must give bitwise the result of a zeroed workspace (a read of scratch the call did not write first
  — what initcheck would report — changes the result);
* repeatability — the same call twice gives bitwise the same outputs (a race between CTAs or a
  missing barrier shows up as run-to-run differences).
"""
import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from tucker_inputs import GridSpec, KernelSpec  # noqa: E402

GUARD = 4096  # bytes of canary on each side
PAT = 0xA5


@pytest.fixture(scope="module")
def T():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_1711_06874_b200 import tucker
    tucker.load()
    return tucker


class Guarded:
    """A device buffer of `nbytes` between two GUARD-byte canaries."""

    def __init__(self, nbytes, fill=0):
        self.n = int(nbytes)
        self.raw = torch.full((self.n + 2 * GUARD,), PAT, dtype=torch.uint8, device="cuda")
        self.raw[GUARD:GUARD + self.n] = fill

    @property
    def ptr(self):
        return ctypes.c_void_p(self.raw.data_ptr() + GUARD)

    def f64(self, shape):
        return self.raw[GUARD:GUARD + self.n].view(torch.float64).view(*shape)

    def intact(self):
        return bool((self.raw[:GUARD] == PAT).all()) and bool((self.raw[GUARD + self.n:] == PAT).all())


def run_hosvd(T, g, r, F, fill, engine=0, info=True):
    lib = T.load()
    T.set_gram_engine(engine)
    try:
        ws = Guarded(T.workspace_bytes(g, r), fill)
        U = [Guarded(8 * g.n[m] * r[m]) for m in range(3)]
        S = [Guarded(8 * r[m]) for m in range(3)]
        core = Guarded(8 * r[0] * r[1] * r[2])
        err = Guarded(24)
        inf = T.CInfo()
        rc = lib.tucker_hosvd(ctypes.byref(T.cgrid(g)), T.cranks(r), T._ptr(F), U[0].ptr, U[1].ptr, U[2].ptr, core.ptr,
                              S[0].ptr, S[1].ptr, S[2].ptr, ws.ptr, ws.n, None, ctypes.byref(inf) if info else None)
        assert rc in (0, 5), rc
        rc = lib.tucker_error(ctypes.byref(T.cgrid(g)), T.cranks(r), T._ptr(F), U[0].ptr, U[1].ptr, U[2].ptr, core.ptr,
                              err.ptr, ws.ptr, ws.n, None)
        assert rc == 0, rc
        torch.cuda.synchronize()
    finally:
        T.set_gram_engine(0)
    bufs = U + S + [core, err, ws]
    assert all(b.intact() for b in bufs), [b.intact() for b in bufs]
    return [u.f64((g.n[m], r[m])).clone() for m, u in enumerate(U)] + [core.f64((r[0] * r[1] * r[2],)).clone(),
                                                                       err.f64((3,)).clone()]


CASES = [(GridSpec.cube(32, 1.0), (8, 8, 8)), (GridSpec.cube(2, 1.0), (2, 2, 2)), (GridSpec.cube(4, 1.0), (2, 2, 2)),
         (GridSpec((40, 36, 33), (-1.0,) * 3, (1.0,) * 3), (6, 5, 4)),
         (GridSpec((136, 144, 160), (-2.0, -1.5, -1.0), (2.0, 1.5, 1.0)), (12, 10, 9)),
         (GridSpec((600, 40, 48), (-1.0,) * 3, (1.0,) * 3), (20, 12, 10))]


@pytest.mark.parametrize("ci", range(len(CASES)))
@pytest.mark.parametrize("engine", [0, 1, 3])  # AUTO (INT8 shared where it applies), DMMA, INT8 row-scaled
def test_hosvd_guards_poison_repeat(T, ci, engine):
    g, r = CASES[ci]
    F = T.fill(g, KernelSpec.matern(0.9, 0.4))
    a = run_hosvd(T, g, r, F, 0x00, engine)
    b = run_hosvd(T, g, r, F, 0xFF, engine)   # poisoned workspace
    c = run_hosvd(T, g, r, F, 0x00, engine, info=False)  # asynchronous variant
    for x, y, z in zip(a, b, c):
        assert torch.equal(x, y) and torch.equal(x, z)


def test_fused_accurate_als_sym_guards(T):
    """The a-7 fused route (INT8 and DMMA k_gram_fused), the SVD-accurate HOSVD (cooperative CGS2,
    cluster SVD), Tucker-ALS and the symmetric path with guarded, poisoned workspaces."""
    lib = T.load()
    g, k, r = GridSpec((136, 144, 160), (-2.0, -1.5, -1.0), (2.0, 1.5, 1.0)), KernelSpec.matern(0.7, 0.5), (12, 10, 9)
    F = T.fill(g, k)

    def outs():
        return [Guarded(8 * g.n[m] * r[m]) for m in range(3)], [Guarded(8 * r[m]) for m in range(3)], \
            Guarded(8 * r[0] * r[1] * r[2])

    results = {}
    for fill in (0x00, 0xFF):
        for eng in (0, 1):
            T.set_gram_engine(eng)
            try:
                ws = Guarded(T.workspace_bytes_fused(g, r), fill)
                U, S, core = outs()
                rc = lib.tucker_hosvd_fused(ctypes.byref(T.cgrid(g)), ctypes.byref(T.ckernel(k)), T.cranks(r),
                                            U[0].ptr, U[1].ptr, U[2].ptr, core.ptr, S[0].ptr, S[1].ptr, S[2].ptr,
                                            ws.ptr, ws.n, None, None)
                torch.cuda.synchronize()
            finally:
                T.set_gram_engine(0)
            assert rc == 0 and all(b.intact() for b in U + S + [core, ws])
            results.setdefault(("fused", eng), []).append(core.f64((r[0] * r[1] * r[2],)).clone())
        ws = Guarded(int(lib.tucker_workspace_size_accurate(ctypes.byref(T.cgrid(g)), T.cranks(r))), fill)
        U, S, core = outs()
        rc = lib.tucker_hosvd_accurate(ctypes.byref(T.cgrid(g)), T.cranks(r), T._ptr(F), U[0].ptr, U[1].ptr, U[2].ptr,
                                       core.ptr, S[0].ptr, S[1].ptr, S[2].ptr, 1, ws.ptr, ws.n, None, None)
        torch.cuda.synchronize()
        assert rc == 0 and all(b.intact() for b in U + S + [core, ws])
        results.setdefault("accurate", []).append(core.f64((r[0] * r[1] * r[2],)).clone())
        h = T.hosvd(g, r, F)
        ws = Guarded(int(lib.tucker_workspace_size_als(ctypes.byref(T.cgrid(g)), T.cranks(r))), fill)
        U, S, core = outs()
        for m in range(3):
            U[m].f64((g.n[m], r[m])).copy_(h.U[m])
        rc = lib.tucker_als(ctypes.byref(T.cgrid(g)), T.cranks(r), T._ptr(F), U[0].ptr, U[1].ptr, U[2].ptr, core.ptr,
                            S[0].ptr, S[1].ptr, S[2].ptr, 2, ws.ptr, ws.n, None, None)
        torch.cuda.synchronize()
        assert rc == 0 and all(b.intact() for b in U + S + [core, ws])
        results.setdefault("als", []).append(core.f64((r[0] * r[1] * r[2],)).clone())
        gs, rs = GridSpec.cube(64, 1.0), (6, 6, 6)
        ws = Guarded(int(lib.tucker_workspace_size_sym(ctypes.byref(T.cgrid(gs)), T.cranks(rs))), fill)
        U = [Guarded(8 * 64 * 6) for _ in range(3)]
        S = [Guarded(8 * 6) for _ in range(3)]
        core, err = Guarded(8 * 216), Guarded(24)
        rc = lib.tucker_hosvd_sym(ctypes.byref(T.cgrid(gs)), ctypes.byref(T.ckernel(k)), T.cranks(rs), U[0].ptr,
                                  U[1].ptr, U[2].ptr, core.ptr, S[0].ptr, S[1].ptr, S[2].ptr, err.ptr, ws.ptr, ws.n,
                                  None, None)
        torch.cuda.synchronize()
        assert rc == 0 and all(b.intact() for b in U + S + [core, err, ws])
        results.setdefault("sym", []).append(core.f64((216,)).clone())
    for key, (z, p) in results.items():
        assert torch.equal(z, p), key
