"""Time the CPU oracle, as it stands, on the whole workloads (SURVEY §8(d) "Oracle timing beside
the GPU"; the oracle actually timed on the configs).  Run on the GPU box's host:

    python tools/oracle_timing.py [--skip-1024] [out.json]

For each of BASELINE configs 1-3 (every kernel) and config 5 (1024^3, once): the full oracle step
fill + HOSVD (explicit unfoldings, Dot2 Gram, cyclic Jacobi, naive TTM) + error, wall-clock per
stage, with points/s and FP64 GFLOP/s from the same algorithmic counts bench.py uses (SYRK Gram
N(n_m+1) per mode, TTM 2 N r3, error reconstruction 2 N r3).  Also the 1-thread figure at 128^3
and the host (nproc, CPU model).  Writes profiles/r02_oracle_timing.json by default.
"""
from __future__ import annotations

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

from oracle import oracle as orc  # noqa: E402
from tucker_inputs import GridSpec, KernelSpec, config1, config2, config3  # noqa: E402


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return ""


def step(grid, k, r):
    og = orc.Grid(tuple(grid.n), tuple(grid.lo), tuple(grid.hi))
    ok = orc.Kernel(k.family, k.sigma2, k.ell, k.nu, k.lam, k.p, k.flags)
    t0 = time.perf_counter()
    F = orc.fill(og, ok)
    t1 = time.perf_counter()
    h = orc.hosvd(F, r)
    t2 = time.perf_counter()
    E = orc.tucker_error(F, *h.U, h.core)[0]
    t3 = time.perf_counter()
    n = grid.n
    N = n[0] * n[1] * n[2]
    flops = sum(N * (n[m] + 1) for m in range(3)) + 2.0 * N * r[2] * 2
    sec = t3 - t0
    return {"grid": list(n), "kernel": k.label(), "ranks": list(r), "E": E, "rc": h.rc,
            "seconds": {"fill": t1 - t0, "hosvd": t2 - t1, "error": t3 - t2, "total": sec},
            "points_per_s": N / sec, "gflops_algorithmic": flops / sec / 1e9}


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    out = args[0] if args else os.path.join(ROOT, "profiles", "r02_oracle_timing.json")
    orc.build()
    res = {"host": {"nproc": os.cpu_count(), "model": cpu_model(), "omp_threads": orc.num_threads()},
           "build": "gcc -O2 -std=gnu11 -ffp-contract=off -mfma -fopenmp (oracle/oracle.py)", "runs": []}
    for w in (config1(), config2(), config3()):
        for k in w.kernels:
            x = step(w.grid, k, w.ranks)
            x["workload"] = w.name
            res["runs"].append(x)
            print(json.dumps(x), flush=True)
    nt = orc.num_threads()
    orc.set_num_threads(1)
    x = step(GridSpec.cube(128, 1.0), KernelSpec.matern(1.5, 0.2), (20, 20, 20))
    x["workload"] = "128^3 one thread"
    res["one_thread_128"] = x
    orc.set_num_threads(nt)
    print(json.dumps(x), flush=True)
    if "--skip-1024" not in sys.argv:
        x = step(GridSpec.cube(1024, 1.0), KernelSpec.matern(1.5, 0.2), (40, 40, 40))
        x["workload"] = "cfg5_1024cube_matern_nu1.5_ell0.2"
        res["cfg5_1024"] = x
        print(json.dumps(x), flush=True)
    res["when"] = time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())
    with open(out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
