"""The C-ABI library loads and exports every symbol include/tucker.h declares; host-side
validation returns the documented error codes before any launch (no GPU needed)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1711_06874_b200 import build, tucker
    build.build()
    return tucker.load()


def test_header_symbols_exported(lib):
    hdr = open(os.path.join(ROOT, "include", "tucker.h")).read()
    declared = re.findall(r"TUCKER_API\s+[\w\s\*]+?\b(tucker_\w+)\s*\(", hdr)
    assert len(declared) >= 10
    from paper_1711_06874_b200 import tucker
    assert set(declared) == set(tucker.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
    out = os.popen(f"nm -D {tucker.LIB_PATH}").read()
    for name in declared:
        assert re.search(rf"\bT {name}\b", out), name


def test_library_is_sm100a_only():
    from paper_1711_06874_b200 import tucker
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {tucker.LIB_PATH}").read()
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_sass_uses_dmma_and_tma():
    from paper_1711_06874_b200 import tucker
    sass = os.popen(f"/usr/local/cuda/bin/cuobjdump -sass {tucker.LIB_PATH}").read()
    assert "DMMA.8x8x4" in sass            # FP64 tensor-core MMA (Gram, TTM1, error)
    assert "UTMALDG" in sass               # TMA tile loads (Gram)
    assert "UTCIMMA" in sass               # tcgen05 kind::i8 MMA (INT8-emulated Gram)
    assert "STG.E.ENL2.256" in sass        # 256-bit stores (octant fill)


def test_validation_codes(lib):
    from paper_1711_06874_b200 import tucker as T
    from tucker_inputs import GridSpec, KernelSpec
    g = T.cgrid(GridSpec.cube(8, 1.0))
    k = T.ckernel(KernelSpec.matern(1.5, 0.2))
    dummy = ctypes.c_void_p(1)
    assert lib.tucker_fill(None, ctypes.byref(k), dummy, dummy, 1 << 30, None) == 1
    bad = T.cgrid(GridSpec((1, 8, 8), (-1, -1, -1), (1, 1, 1)))
    assert lib.tucker_fill(ctypes.byref(bad), ctypes.byref(k), dummy, dummy, 1 << 30, None) == 1
    inv = T.cgrid(GridSpec((8, 8, 8), (1, -1, -1), (-1, 1, 1)))
    assert lib.tucker_fill(ctypes.byref(inv), ctypes.byref(k), dummy, dummy, 1 << 30, None) == 1
    for kk in (KernelSpec.matern(0.0, 1.0), KernelSpec.matern(1.0, 0.0), KernelSpec.slater(1.0, 2.5),
               KernelSpec.slater(-1.0, 1.0), KernelSpec.matern(1.0, 1.0, sigma2=-1.0)):
        ck = T.ckernel(kk)
        assert lib.tucker_fill(ctypes.byref(g), ctypes.byref(ck), dummy, dummy, 1 << 30, None) == 2
    assert lib.tucker_fill(ctypes.byref(g), ctypes.byref(k), dummy, dummy, 16, None) == 4  # small ws
    assert lib.tucker_gram(ctypes.byref(g), 3, dummy, dummy, dummy, 1 << 30, None) == 1
    for r in ((0, 2, 2), (9, 2, 2), (2, 2, 0)):
        rc = lib.tucker_hosvd(ctypes.byref(g), T.cranks(r), dummy, dummy, dummy, dummy, dummy, dummy, dummy,
                              dummy, dummy, 1 << 30, None, None)
        assert rc == 3
    assert lib.tucker_eig(8, dummy, 9, dummy, dummy, dummy, 1 << 30, None, None) == 3
    assert lib.tucker_strerror(5).decode().startswith("eigensolver")


def test_workspace_size_monotone(lib):
    from paper_1711_06874_b200 import tucker as T
    from tucker_inputs import GridSpec
    a = T.workspace_bytes(GridSpec.cube(64, 1.0), (8, 8, 8))
    b = T.workspace_bytes(GridSpec.cube(128, 1.0), (8, 8, 8))
    c = T.workspace_bytes(GridSpec.cube(128, 1.0), (40, 40, 40))
    assert 0 < a < b <= c
    T.set_gram_engine(T.GRAM_DMMA)
    try:
        dmma = T.workspace_bytes(GridSpec.cube(1024, 1.0), (40, 40, 40))
    finally:
        T.set_gram_engine(T.GRAM_AUTO)
    assert dmma < 4 * 2 ** 30  # scratch for 1024^3 at ranks 40 stays well inside 180 GB
    # INT8 emulation: residues of up to 16 GiB of the unfolding + partials, still far below 180 GB
    i8 = T.workspace_bytes(GridSpec.cube(1024, 1.0), (40, 40, 40))
    assert dmma < i8 < 20 * 2 ** 30
    assert T.get_gram_engine() == T.GRAM_AUTO
    with pytest.raises(T.TuckerError):
        T.set_gram_engine(7)


def test_validation_codes_next_rows(lib):
    """The fused, symmetric, ALS and SVD-accurate entry points validate before any launch."""
    from paper_1711_06874_b200 import tucker as T
    from tucker_inputs import GridSpec, KernelSpec
    d = ctypes.c_void_p(1)
    g = T.cgrid(GridSpec.cube(16, 1.0))
    k = T.ckernel(KernelSpec.matern(1.5, 0.2))
    bad_k = T.ckernel(KernelSpec.matern(-1.0, 0.2))
    r4, r_bad = T.cranks((4, 4, 4)), T.cranks((17, 4, 4))
    big = 1 << 40
    # fused
    assert lib.tucker_workspace_size_fused(ctypes.byref(g), r4) > 0
    assert lib.tucker_gram_fused(ctypes.byref(g), ctypes.byref(k), 3, d, d, big, None) == 1
    assert lib.tucker_gram_fused(ctypes.byref(g), ctypes.byref(bad_k), 0, d, d, big, None) == 2
    assert lib.tucker_gram_fused(ctypes.byref(g), ctypes.byref(k), 0, d, d, 16, None) == 4
    assert lib.tucker_hosvd_fused(ctypes.byref(g), ctypes.byref(k), r_bad, d, d, d, d, d, d, d, d, big, None,
                                  None) == 3
    assert lib.tucker_error_fused(ctypes.byref(g), ctypes.byref(k), r4, None, d, d, d, d, d, big, None) == 1
    # symmetric: rank above ceil(n/2), off-centre grid
    assert lib.tucker_hosvd_sym(ctypes.byref(g), ctypes.byref(k), T.cranks((9, 4, 4)), d, d, d, d, d, d, d, None, d,
                                big, None, None) == 3
    off = T.cgrid(GridSpec((16, 16, 16), (-1.0, -1.0, -0.5), (1.0, 1.0, 1.0)))
    assert lib.tucker_hosvd_sym(ctypes.byref(off), ctypes.byref(k), r4, d, d, d, d, d, d, d, None, d, big, None,
                                None) == 7
    # ALS: sweeps < 1, rank out of range, workspace too small
    assert lib.tucker_als(ctypes.byref(g), r4, d, d, d, d, d, d, d, d, 0, d, big, None, None) == 1
    assert lib.tucker_als(ctypes.byref(g), r_bad, d, d, d, d, d, d, d, d, 1, d, big, None, None) == 3
    assert lib.tucker_als(ctypes.byref(g), r4, d, d, d, d, d, d, d, d, 1, d, 16, None, None) == 4
    assert lib.tucker_workspace_size_als(ctypes.byref(g), r_bad) == 0
    # SVD-accurate: iters < 1, rank > 56, workspace too small
    assert lib.tucker_hosvd_accurate(ctypes.byref(g), r4, d, d, d, d, d, d, d, d, 0, d, big, None, None) == 1
    g2 = T.cgrid(GridSpec.cube(64, 1.0))
    assert lib.tucker_hosvd_accurate(ctypes.byref(g2), T.cranks((57, 4, 4)), d, d, d, d, d, d, d, d, 1, d, big, None,
                                     None) == 7
    assert lib.tucker_hosvd_accurate(ctypes.byref(g), r4, d, d, d, d, d, d, d, d, 1, d, 16, None, None) == 4
    # row (e) sharded fused HOSVD: shard layout and the callback are validated first
    cb, null_cb = T.ALLREDUCE_FN(lambda *a: 0), T.ALLREDUCE_FN()
    for shard, nsh, fn in ((0, 0, cb), (2, 2, cb), (-1, 2, cb), (0, 2, null_cb)):
        assert lib.tucker_hosvd_fused_sharded(ctypes.byref(g), ctypes.byref(k), r4, shard, nsh, fn, None, d, d, d, d,
                                              d, d, d, None, d, big, None, None) == 1
    assert lib.tucker_hosvd_fused_sharded(ctypes.byref(g), ctypes.byref(k), r_bad, 0, 1, null_cb, None, d, d, d, d,
                                          d, d, d, None, d, big, None, None) == 3
    assert lib.tucker_hosvd_fused_sharded(ctypes.byref(g), ctypes.byref(k), r4, 0, 1, null_cb, None, d, d, d, d,
                                          d, d, d, None, d, 16, None, None) == 4
    assert lib.tucker_strerror(8).decode().startswith("the caller")
    # spectral density domain
    sk = T.ckernel(KernelSpec.spectral(0.0, 0.4))
    assert lib.tucker_fill(ctypes.byref(g), ctypes.byref(sk), d, d, big, None) == 2


def test_host_queries_round2(lib):
    """Host-only queries added in round 2 (no GPU): the INT8 residue layout per grid (R20 shared
    layout where n3 % 16 == 0 and 16 N bytes fit; R18 per-mode otherwise or when forced), the
    fill-only workspace, the multigrid workspace, the new error code."""
    from paper_1711_06874_b200 import tucker as T
    from tucker_inputs import GridSpec
    g = GridSpec.cube(1024, 1.0)
    assert T.i8_layout(g) == (True, 50)
    assert T.i8_layout(GridSpec((40, 36, 33), (-1.0,) * 3, (1.0,) * 3))[0] is False   # n3 % 16 != 0
    assert T.i8_layout(GridSpec.cube(2048, 1.0))[0] is False                            # 137 GB > cap
    T.set_gram_engine(T.GRAM_INT8_ROWSCALED)
    try:
        assert T.i8_layout(g)[0] is False
        assert T.get_gram_engine() == T.GRAM_INT8_ROWSCALED
    finally:
        T.set_gram_engine(T.GRAM_AUTO)
    T.set_gram_engine(T.GRAM_DMMA)
    try:
        with pytest.raises(T.TuckerError):
            T.i8_layout(g)
    finally:
        T.set_gram_engine(T.GRAM_AUTO)
    # fill needs only the nodes and the K_nu table (a few KB), not the HOSVD workspace
    cg = T.cgrid(g)
    nf = lib.tucker_workspace_size_fill(ctypes.byref(cg))
    assert 0 < nf < 64 * 1024 < T.workspace_bytes(g, (40, 40, 40))
    # multigrid: the finest level's ALS workspace dominates; invalid n0 -> 0
    nm = lib.tucker_workspace_size_multigrid(ctypes.byref(cg), T.cranks((40, 40, 40)), 128)
    assert nm > 8 * 512 ** 3
    assert lib.tucker_workspace_size_multigrid(ctypes.byref(cg), T.cranks((40, 40, 40)), 2) == 0
    assert lib.tucker_strerror(9).decode().startswith("input")


def test_multigrid_and_hosvd_validation(lib):
    """tucker_multigrid and tucker_hosvd reject bad arguments before any launch."""
    from paper_1711_06874_b200 import tucker as T
    from tucker_inputs import GridSpec, KernelSpec
    g = T.cgrid(GridSpec.cube(64, 1.0))
    k = T.ckernel(KernelSpec.matern(1.5, 0.2))
    d = ctypes.c_void_p(1)
    # sweeps < 1, n0 < 4, null F
    assert lib.tucker_multigrid(ctypes.byref(g), ctypes.byref(k), T.cranks((4, 4, 4)), 16, 0, d, d, d, d, d, d, d, d,
                                d, 1 << 40, None, None, None) == 1
    assert lib.tucker_multigrid(ctypes.byref(g), ctypes.byref(k), T.cranks((4, 4, 4)), 2, 1, d, d, d, d, d, d, d, d,
                                d, 1 << 40, None, None, None) == 1
    assert lib.tucker_multigrid(ctypes.byref(g), ctypes.byref(k), T.cranks((4, 4, 4)), 16, 1, None, d, d, d, d, d, d,
                                d, d, 1 << 40, None, None, None) == 1
    assert lib.tucker_multigrid(ctypes.byref(g), ctypes.byref(k), T.cranks((65, 4, 4)), 16, 1, d, d, d, d, d, d, d, d,
                                d, 1 << 40, None, None, None) == 3
    # r_m > 56 with n_m > 112: UNSUPPORTED before any launch
    g2 = T.cgrid(GridSpec((300, 64, 64), (-1.0,) * 3, (1.0,) * 3))
    rc = lib.tucker_hosvd(ctypes.byref(g2), T.cranks((57, 8, 8)), d, d, d, d, d, d, d, d, d, 1 << 40, None, None)
    assert rc == 7
    assert lib.tucker_last_launch_count() == 0


def test_ttm_engine_switch_host_only(lib):
    """tucker_set_ttm_engine: per-thread, AUTO / DMMA / INT8_ERROR accepted, anything else rejected
    (host only, no device work)."""
    from paper_1711_06874_b200 import tucker as T
    assert T.get_ttm_engine() == T.TTM_AUTO
    for e in (T.TTM_DMMA, T.TTM_INT8_ERROR, T.TTM_AUTO):
        T.set_ttm_engine(e)
        assert T.get_ttm_engine() == e
    for bad in (-1, 3, 7):
        with pytest.raises(Exception):
            T.set_ttm_engine(bad)
    assert T.get_ttm_engine() == T.TTM_AUTO


def test_sass_uses_int8_tensor_cores_for_ttm():
    """k_ttm1_i8 (R22) and k_err_i8 (R23) are tcgen05 kind::i8 kernels fed by TMA."""
    import subprocess
    from paper_1711_06874_b200 import build
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", build.LIB], capture_output=True, text=True).stdout
    for name in ("9k_ttm1_i8E", "8k_err_i8E"):  # (mangled: the kernels themselves, not k_err_i8_final)
        i = next(k for k, part in enumerate(sass.split("Function : ")) if part.split("\n", 1)[0].find(name) >= 0)
        body = sass.split("Function : ")[i]
        assert "UTCIMMA" in body and "UTMALDG" in body, name
