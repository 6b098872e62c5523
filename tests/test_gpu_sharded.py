"""Row (e) on the GPU: ONE fused HOSVD (+ error) sharded over 2, 3 and 4 ranks
(tucker_hosvd_fused_sharded).  The ranks are processes sharing the test box's one
GPU and exchanging through gloo (a host-staged all-reduce: no kernel waits on another rank —
B200_PROFILING.md); in production the same calls run one process per GPU over NCCL.

Bar: every rank returns the BITWISE result of the single-call tucker_hosvd_fused +
tucker_error_fused — the Gram exchanges are exact integer residue sums, the T2 and error
exchanges add zeros off the owning rank — and all ranks issue the same exchange sequence.
Chunk knobs force several residue super-chunks and slab chunks per mode (uneven over 3 ranks);
the off-centre grid also shards the row-maxima pass (MAX exchange).
"""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from tucker_inputs import GridSpec, KernelSpec  # noqa: E402

CASES = {
    "centred": (GridSpec.cube(128, 1.0), KernelSpec.matern(1.5, 0.3), (10, 10, 10)),
    "offcentre": (GridSpec((96, 80, 112), (-2.0, -1.0, -0.5), (2.0, 1.5, 1.0)), KernelSpec.matern(0.7, 0.5),
                  (8, 9, 10)),
}
KNOBS = {"TUCKER_FUSED_CHUNK_KB": "2048", "TUCKER_I8_RESIDUE_MB": "4"}


def _free_port():
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1711_06874_b200 import tucker as T
        g, k, r = CASES[case]
        res = T.hosvd_fused_sharded(g, k, r, rank, world)
        torch.cuda.synchronize()
        torch.save({"U": [u.cpu() for u in res.U], "core": res.core.cpu(), "S": [s.cpu() for s in res.sigma],
                    "err": res.err.cpu(), "ex": res.exchanges, "rc": res.rc}, f"{out_path}.{rank}")
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def T():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_1711_06874_b200 import tucker
    tucker.load()
    return tucker


@pytest.fixture()
def knobs():
    old = {k: os.environ.get(k) for k in KNOBS}
    os.environ.update(KNOBS)
    yield
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("case", sorted(CASES))
def test_sharded_fused_hosvd_bitwise(T, knobs, tmp_path, case, world):
    import torch.multiprocessing as mp
    g, k, r = CASES[case]
    ref = T.hosvd_fused(g, k, r)
    ref_err = T.error_fused(g, k, r, ref.U, ref.core)
    torch.cuda.synchronize()
    out = str(tmp_path / "shard")
    mp.start_processes(_worker, args=(world, _free_port(), case, out), nprocs=world, join=True, start_method="spawn")
    results = [torch.load(f"{out}.{q}") for q in range(world)]
    # exchanges: per mode the Gram residue sums (3), T2, the error partials; the per-mode row-scaled
    # route (n3 % 16 != 0) adds the row maxima on off-centre grids — the shared route (R20) takes its
    # one exponent from the smallest radius, no exchange
    centred = g.lo[0] == -g.hi[0] and g.lo[1] == -g.hi[1] and g.lo[2] == -g.hi[2]
    n_ex = 5 + (0 if centred or g.n[2] % 16 == 0 else 1)
    for q, res in enumerate(results):
        assert res["rc"] == ref.rc, (q, res["rc"])
        for m in range(3):
            assert torch.equal(res["U"][m], ref.U[m].cpu()), (q, m)
            assert torch.equal(res["S"][m], ref.sigma[m].cpu()), (q, m)
        assert torch.equal(res["core"], ref.core.cpu()), q
        assert torch.equal(res["err"], ref_err.cpu()), (q, res["err"], ref_err)
        assert len(res["ex"]) == n_ex, res["ex"]
        assert res["ex"] == results[0]["ex"]  # same exchange sequence on every rank


def test_sharded_single_rank_equals_fused(T, knobs):
    """nshards = 1: no exchange, the plain fused result."""
    g, k, r = CASES["offcentre"]
    ref = T.hosvd_fused(g, k, r)
    ref_err = T.error_fused(g, k, r, ref.U, ref.core)
    res = T.hosvd_fused_sharded(g, k, r, 0, 1)
    assert res.exchanges == []
    for m in range(3):
        assert torch.equal(res.U[m], ref.U[m])
    assert torch.equal(res.core, ref.core)
    assert torch.equal(res.err, ref_err)


def test_sharded_collective_failure_is_reported(T, knobs):
    """A failing all-reduce stops the call with TUCKER_ERR_COLLECTIVE (no process group here)."""
    g, k, r = CASES["centred"]
    with pytest.raises(T.TuckerError) as e:
        T.hosvd_fused_sharded(g, k, r, 0, 2)
    assert e.value.code == 8


def test_bench_two_ranks_sharded_line(T, tmp_path):
    """bench.py's N > 1 path (torchrun, 2 ranks) in its gloo test mode on the one GPU: the JSON line
    reports n_gpus 2 and the sharded config-5f line (here 256^3) with the same E on both ranks."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TUCKER_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), os.path.join(root, "bench.py"), "--gpus", "2",
           "--steps", "2", "--warmup", "3", "--grid-n", "256", "--fused-n", "256", "--no-e2e", "--no-host-tensor"]
    p = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0
    fs = d["fused_sharded"]
    assert fs["n_shards"] == 2 and fs["rc"] == 0 and fs["E_identical_on_all_ranks"] and fs["exchanges"] == 5
    ref = T.hosvd_fused(GridSpec.cube(256, 1.0), KernelSpec.matern(1.5, 0.2), (40, 40, 40))
    e = T.error_fused(GridSpec.cube(256, 1.0), KernelSpec.matern(1.5, 0.2), (40, 40, 40), ref.U, ref.core)
    assert fs["E"] == float(e[0].item())
