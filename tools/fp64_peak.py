"""Measure the FP64 peaks the roofline fractions use (VERDICT r1 'measured FP64 peak'):

  * DMMA pipe: mma.sync m8n8k4 f64 (SASS DMMA.8x8x4, 512 flop per warp instruction) in 8
    independent chains per warp, all SMs, best of 5 launches (burst) and back to back for ~4 s
    (sustained);
  * FP64 FMA pipe (DFMA, 2 flop per lane): the same two figures;
  * cuBLAS DGEMM (torch.matmul float64, 8192^3, 2 N^3 flop): burst (best of 10) and sustained (4 s).
Clocks are sampled with nvidia-smi during the sustained runs.  Writes
profiles/fp64_peak_measured.json (or the path given as argv[1]).
"""
from __future__ import annotations

import ctypes
import json
import os
import subprocess
import sys
import threading
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def build():
    so = os.path.join("/tmp", "fp64_peak.so")
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                    "-Xcompiler", "-fPIC", "-o", so, os.path.join(HERE, "fp64_peak.cu")], check=True)
    lib = ctypes.CDLL(so)
    lib.fp64_peak_run.restype = ctypes.c_float
    lib.fp64_peak_run.argtypes = [ctypes.c_int] * 4
    return lib


class Clocks(threading.Thread):
    def __init__(self):
        super().__init__(daemon=True)
        self.samples, self.stop = [], False

    def run(self):
        while not self.stop:
            try:
                o = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                                    "--format=csv,noheader,nounits", "-i", "0"], capture_output=True, text=True,
                                   timeout=5).stdout.strip().split(",")
                self.samples.append((float(o[0]), float(o[1]), o[2].strip()))
            except Exception:
                pass
            time.sleep(0.2)


def pipe(lib, kind, flop_per_iter_per_warp):
    sms = 148
    blocks, threads = sms * 4, 256
    warps = blocks * threads // 32
    iters = 20000
    lib.fp64_peak_run(kind, blocks, threads, 1000)  # warm-up
    ms = [lib.fp64_peak_run(kind, blocks, threads, iters) for _ in range(5)]
    flop = warps * iters * flop_per_iter_per_warp
    burst = flop / (min(ms) * 1e-3) / 1e12
    clk = Clocks()
    clk.start()
    t0, tot_ms, n = time.time(), 0.0, 0
    while time.time() - t0 < 4.0:
        tot_ms += lib.fp64_peak_run(kind, blocks, threads, iters)
        n += 1
    clk.stop = True
    sustained = flop * n / (tot_ms * 1e-3) / 1e12
    sm = sorted(s[0] for s in clk.samples) or [0.0]
    return {"burst_tflops": burst, "sustained_tflops": sustained, "launch_ms_min": min(ms),
            "sm_mhz_median_sustained": sm[len(sm) // 2], "reasons": sorted({s[2] for s in clk.samples})}


def dgemm():
    import torch
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    clk = Clocks()
    clk.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k = max(1, int(4000 / best))
    e0.record()
    for _ in range(k):
        torch.matmul(a, b, out=c)
    e1.record()
    e1.synchronize()
    clk.stop = True
    sm = sorted(s[0] for s in clk.samples) or [0.0]
    fl = 2.0 * n ** 3
    return {"burst_tflops": fl / (best * 1e-3) / 1e12, "sustained_tflops": fl * k / (e0.elapsed_time(e1) * 1e-3) / 1e12,
            "n": n, "sm_mhz_median_sustained": sm[len(sm) // 2], "reasons": sorted({s[2] for s in clk.samples})}


def main():
    lib = build()
    res = {"dmma": pipe(lib, 0, 8 * 512), "dfma": pipe(lib, 1, 8 * 32 * 2), "cublas_dgemm": dgemm(),
           "spec_derived_tflops": 148 * 64 * 2 * 1.965e9 / 1e12,
           "how": "tools/fp64_peak.py: DMMA m8n8k4 / DFMA chains (8 per warp, 148x4 CTAs of 256 threads); "
                  "cuBLAS DGEMM 8192^3 via torch.matmul float64; burst = best launch, sustained = ~4 s back to back",
           "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "fp64_peak_measured.json")
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
