#!/usr/bin/env python
"""bench.py — throughput of the Tucker/HOSVD hot path of arXiv 1711.06874 on B200.

One step = the whole hot path over one synthetic problem: grid nodes + fill
of F, the three Gram matrices, the three eigensolves, the core (TTM chain) and the relative
Frobenius error.  Workload at N=1: BASELINE.json config 5 (1024^3 on [-1,1]^3, Matérn nu=1.5,
ell=0.2, sigma^2=1, ranks (40,40,40)).  Metric: grid points per second (whole job).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--n 1024] [--r 40]

With --gpus N > 1 (launched by torch.distributed.run), every rank solves its own independent
problem (weak scaling, no data-path collective); the step time is the max over ranks.
--impl reference times the CPU oracle (oracle/, the only other program computing this path) on a
bounded sample of the same workload on the host cores; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Tucker HOSVD grid points/s and FP64 TFLOP/s vs peak (n=512–1024, r≤40)"
UNIT = "grid points/s"
FP64_PEAK_SPEC_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12  # 37.2 TF/s: SMs x FP64 FMA/clk/SM x 2 x max clock


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--grid-n", "--n", dest="n", type=int, default=1024)
    ap.add_argument("--tucker-rank", "--r", dest="r", type=int, default=40)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-host-tensor", action="store_true")
    ap.add_argument("--no-fused", action="store_true", help="skip the 2048^3 fused (F never stored) line")
    ap.add_argument("--no-als", action="store_true", help="skip the Tucker-ALS (NEXT f1) line")
    ap.add_argument("--no-sym", action="store_true", help="skip the symmetry-exploiting (NEXT f3) line")
    ap.add_argument("--no-accurate", action="store_true", help="skip the SVD-accurate (NEXT f2) line")
    ap.add_argument("--no-multigrid", action="store_true", help="skip the multigrid Tucker line")
    ap.add_argument("--no-graph", action="store_true", help="skip the CUDA-Graph replay of the step")
    ap.add_argument("--no-cfg4", action="store_true", help="skip the config-4 (512^3 x 16 settings) line")
    ap.add_argument("--no-f4", action="store_true", help="skip the NEXT f4 workloads line")
    ap.add_argument("--no-lowrank", action="store_true", help="skip the TTM / error stages at ranks 10 and 20")
    ap.add_argument("--no-parity", action="store_true", help="skip the per-config T1-T4 deltas vs the oracle")
    ap.add_argument("--fused-n", type=int, default=2048)
    ap.add_argument("--gram-engine", default="auto", choices=["auto", "dmma", "int8"],
                    help="Gram engine of the materialised path (auto: INT8 emulation)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ----------------------------------------------------------------------------------- clocks ----
CLOCK_INTERVAL_S = float(os.environ.get("BENCH_CLOCK_INTERVAL_MS", "10")) / 1000.0


class ClockSampler:
    """SM clock and clock-event reasons sampled every ~10 ms through NVML (nvidia-smi's 100 ms loop
    as the fallback).  Started before the warm-up, it keeps only the samples taken between
    mark_start() and mark_end() (host clock; the step is host-synchronous) — the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.nvml = None
        self.samples = []  # (host time, sm MHz, max MHz, set of reasons)
        self.t_start = self.t_end = None
        self.stop = threading.Event()
        self.thread = None

    def mark_start(self):
        self.t_start = time.time()

    def mark_end(self):
        self.t_end = time.time()

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            pr = torch.cuda.get_device_properties(self.index)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
        return pynvml, h

    def _poll_nvml(self):
        nv, h = self.nvml
        bits = [(nv.nvmlClocksEventReasonHwSlowdown, "hw_slowdown"),
                (nv.nvmlClocksEventReasonHwThermalSlowdown, "hw_thermal_slowdown"),
                (nv.nvmlClocksEventReasonSwThermalSlowdown, "sw_thermal_slowdown"),
                (nv.nvmlClocksEventReasonSwPowerCap, "sw_power_cap")]
        mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
        while not self.stop.is_set():
            try:
                sm = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                m = int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))
                self.samples.append((time.time(), sm, mx, {nm for bit, nm in bits if m & bit}))
            except Exception:
                pass
            self.stop.wait(CLOCK_INTERVAL_S)

    def _read_smi(self):
        for line in self.proc.stdout:
            p = [x.strip() for x in line.strip().split(",")]
            if len(p) < 7:
                continue
            try:
                self.samples.append((time.time(), float(p[0]), float(p[1]),
                                     {nm for nm, v in zip(self.NAMES, p[3:7]) if v.lower().startswith("active")}))
            except ValueError:
                continue

    def __enter__(self):
        try:
            self.nvml = self._nvml_handle()
            self.thread = threading.Thread(target=self._poll_nvml, daemon=True)
        except Exception:
            self.nvml = None
            try:
                self.proc = subprocess.Popen(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={','.join(self.FIELDS)}",
                     "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE,
                    stderr=subprocess.DEVNULL, text=True)
                self.thread = threading.Thread(target=self._read_smi, daemon=True)
            except OSError:
                self.proc = None
        if self.thread is not None:
            self.thread.start()
        return self

    def __exit__(self, *exc):
        self.stop.set()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)

    def summary(self):
        lo = self.t_start if self.t_start is not None else -1e300
        hi = self.t_end if self.t_end is not None else 1e300
        sm, mx, reasons = [], 0.0, set()
        for ts, f, m, rs in self.samples:
            if lo <= ts <= hi:
                sm.append(f)
                mx = max(mx, m)
                reasons |= rs
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvml" if self.nvml else "nvidia-smi"}


def ttm_on_int8(r3: int, args) -> bool:
    """The core's first product runs on the INT8 tensor cores (R22) on this configuration: the INT8
    shared-layout Gram route, the default TTM engine and r3 <= 40 (n3 % 16 == 0 on every bench grid)."""
    from paper_1711_06874_b200 import tucker as T
    return getattr(args, "gram_engine", "auto") != "dmma" and T.get_ttm_engine() == T.TTM_AUTO and 1 <= r3 <= 40


def ttm_i8_note(r3: int) -> str:
    nb = (r3 + 7) // 8 * 8
    cols = sum(((6 if s < 2 else 7 - s) * nb + 15) // 16 * 16 for s in range(6))
    return (f"T1 = F x3 U3^T on the INT8 tensor cores (k_ttm1_i8, six base-256 digits per operand, 26 digit "
            f"pairs; {2 * cols} int8 ops per F element executed, below the HBM time at the measured INT8 "
            f"peak): bound by the 8 N bytes of F")


def fp64_peak() -> tuple:
    """(TF/s, source): the measured DMMA-pipe FP64 peak (tools/fp64_peak.py ->
    profiles/fp64_peak_measured.json, sustained) or the spec-derived 37.2 TF/s."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak_measured.json")))
        return float(d["dmma"]["sustained_tflops"]), ("measured DMMA m8n8k4 f64 sustained (profiles/fp64_peak_measured."
                                                       "json; cuBLAS DGEMM 8192^3 sustained "
                                                       f"{d['cublas_dgemm']['sustained_tflops']:.2f})")
    except (OSError, ValueError, KeyError):
        return FP64_PEAK_SPEC_TFLOPS, "spec-derived: 148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz"


def measured_peaks() -> dict:
    """Driver-written MEASURED_PEAKS.json (HBM GB/s, dense bf16 TF/s burst and sustained), or {}."""
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        return {}


# --------------------------------------------------------------------------- rank helpers ----
def max_over_ranks(value: float, world: int, device=None) -> float:
    """Max of a per-rank scalar over the process group (device time = max over ranks)."""
    if world <= 1:
        return float(value)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def whole_job_rate(points_per_rank: int, world: int, ms_step_max: float) -> float:
    """Weak scaling, replicas: every rank solves its own problem; value = all ranks' points / time."""
    return world * points_per_rank / (ms_step_max * 1e-3)


# ------------------------------------------------------------------------------ our GPU arm ----
def run_ours(args, rank, world, local):
    import torch
    import torch.distributed as dist

    from paper_1711_06874_b200 import tucker as T
    from tucker_inputs import GridSpec, KernelSpec

    # TUCKER_BENCH_BACKEND=gloo: a test mode for the N > 1 code paths on a one-GPU box (ranks share
    # the GPU; no kernel waits on another rank; numbers from it are not bench values)
    backend = os.environ.get("TUCKER_BENCH_BACKEND", "nccl")
    if backend == "gloo":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    T.load()
    T.set_gram_engine({"auto": T.GRAM_AUTO, "dmma": T.GRAM_DMMA, "int8": T.GRAM_INT8}[args.gram_engine])
    n, rr = args.n, args.r
    grid = GridSpec.cube(n, 1.0)
    kern = KernelSpec.matern(1.5, 0.2)
    ranks = (rr, rr, rr)
    N = grid.points
    stream = torch.cuda.current_stream()
    F = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
    ws = T.workspace(grid, ranks)
    dev = F.device
    U = [torch.empty((n, rr), dtype=torch.float64, device=dev) for _ in range(3)]
    S = [torch.empty(rr, dtype=torch.float64, device=dev) for _ in range(3)]
    core = torch.empty(ranks, dtype=torch.float64, device=dev)
    out3 = torch.empty(3, dtype=torch.float64, device=dev)
    lib = T.load()
    import ctypes
    g_c, k_c, r_c = T.cgrid(grid), T.ckernel(kern), T.cranks(ranks)
    sp = ctypes.c_void_p(stream.cuda_stream)
    wsp, wsn = ctypes.c_void_p(ws.data_ptr()), ws.numel()
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    # the fill also writes the INT8 route's inputs where it can: the shared residues in the same octant
    # pass (tucker_fill_prepare -> tucker_hosvd_prepared: the residue pass over F is gone), else the row
    # maxima (tucker_fill_rowmax -> tucker_hosvd_rowmax); bitwise the plain calls' results
    rowmax = torch.empty(3 * n, dtype=torch.int32, device=dev)
    use_prepare = args.gram_engine != "dmma" and lib.tucker_fill_prepare(
        ctypes.byref(g_c), ctypes.byref(k_c), r_c, P(F), wsp, wsn, sp) == 0
    use_rowmax = not use_prepare and args.gram_engine != "dmma" and lib.tucker_fill_rowmax(
        ctypes.byref(g_c), ctypes.byref(k_c), P(F), P(rowmax), wsp, wsn, sp) == 0
    torch.cuda.synchronize()

    info = T.CInfo()  # the synchronous HOSVD: convergence checked and reported per mode

    def step(spp=None, sync=True):
        """One pass of the path as three ABI calls (fill [+ row maxima], hosvd = 3 x (Gram + eig) +
        core, error) on stream spp (default: `stream`); sync=False passes info = NULL (the
        asynchronous, graph-capturable HOSVD); returns the number of kernel launches."""
        spp = sp if spp is None else spp
        launches = 0
        pinfo = ctypes.byref(info) if sync else None
        if use_prepare:
            T._check(lib.tucker_fill_prepare(ctypes.byref(g_c), ctypes.byref(k_c), r_c, P(F), wsp, wsn, spp),
                     "fill_prepare")
            launches += lib.tucker_last_launch_count()
            rc = lib.tucker_hosvd_prepared(ctypes.byref(g_c), r_c, P(F), P(U[0]), P(U[1]), P(U[2]), P(core), P(S[0]),
                                           P(S[1]), P(S[2]), wsp, wsn, spp, pinfo)
        else:
            if use_rowmax:
                T._check(lib.tucker_fill_rowmax(ctypes.byref(g_c), ctypes.byref(k_c), P(F), P(rowmax), wsp, wsn,
                                                spp), "fill_rowmax")
            else:
                T._check(lib.tucker_fill(ctypes.byref(g_c), ctypes.byref(k_c), P(F), wsp, wsn, spp), "fill")
            launches += lib.tucker_last_launch_count()
            rc = lib.tucker_hosvd_rowmax(ctypes.byref(g_c), r_c, P(F), P(rowmax) if use_rowmax else None, P(U[0]),
                                         P(U[1]), P(U[2]), P(core), P(S[0]), P(S[1]), P(S[2]), wsp, wsn, spp, pinfo)
        if rc not in (0, 5):
            T._check(rc, "hosvd")
        launches += lib.tucker_last_launch_count()
        T._check(lib.tucker_error(ctypes.byref(g_c), r_c, P(F), P(U[0]), P(U[1]), P(U[2]), P(core), P(out3), wsp,
                                  wsn, spp), "error")
        launches += lib.tucker_last_launch_count()
        return launches

    clk = ClockSampler(local)
    clk.__enter__()
    # warm-up steps run the synchronous HOSVD (convergence and the input window checked, `info`
    # filled); the timed steps pass info = NULL — the asynchronous call a pipeline makes (no host
    # synchronisation inside the HOSVD), checked once more right after the timed region
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    K = args.steps
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    try:
        clk.mark_start()
        t0.record(stream)
        for k in range(K):
            launches += step(sync=False)
        t1.record(stream)
        torch.cuda.synchronize()
        clk.mark_end()
    finally:
        clk.__exit__(None, None, None)
    if world > 1:
        dist.barrier()
    ms_total = max_over_ranks(t0.elapsed_time(t1), world, dev)
    ms_step = ms_total / K
    E_timed = out3.cpu().tolist()
    step()  # the synchronous call on the same inputs: rc, convergence and the window flag checked
    torch.cuda.synchronize()
    assert out3.cpu().tolist() == E_timed, "asynchronous and synchronous steps differ"
    # per-stage times: a second, separately profiled pass of K steps (the stage timer's events are
    # kept out of the timed region above)
    T.profile_read()  # drop anything recorded before
    T.profile_enable(True)
    for k in range(K):
        step(sync=False)  # the timed steps' asynchronous calls (a synchronous HOSVD leaves host gaps)
    torch.cuda.synchronize()
    T.profile_enable(False)
    prof = T.profile_read()
    if world > 1:
        dist.barrier()

    # the same step captured once in a CUDA Graph (asynchronous HOSVD, info = NULL) and replayed
    graph = None
    if not args.no_graph:
        try:
            gs = torch.cuda.Stream()
            gs.wait_stream(stream)
            gsp = ctypes.c_void_p(gs.cuda_stream)
            with torch.cuda.stream(gs):
                step(gsp, sync=False)  # warm-up of the asynchronous path on the capture stream
                gs.synchronize()
                cg = torch.cuda.CUDAGraph()
                with torch.cuda.graph(cg, stream=gs):
                    glaunch = step(gsp, sync=False)
            cg.replay()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record(stream)
            for _ in range(K):
                cg.replay()
            g1.record(stream)
            torch.cuda.synchronize()
            gms = max_over_ranks(g0.elapsed_time(g1), world, dev) / K
            Eg = out3.cpu().tolist()
            graph = {"ms_per_step": gms, "value": whole_job_rate(N, world, gms), "unit": UNIT,
                     "launches_per_step": glaunch, "E": Eg[0],
                     "what": "the same three calls (asynchronous tucker_hosvd_rowmax, info = NULL) captured once "
                             "in a CUDA Graph and replayed K times (CUDA events, max over ranks)"}
            del cg
        except Exception as e:  # (capture unsupported in some setting: report, keep the eager line)
            graph = {"unavailable": f"{type(e).__name__}: {e}"[:300]}

    # per-stage device times (ms per step) from the library's event scopes on `stream`
    st = {name: ms / K for name, (ms, cnt) in prof.items() if cnt}
    calls = {name: cnt / K for name, (ms, cnt) in prof.items() if cnt}
    E = out3.cpu().tolist()

    # ---- roofline of the dominant kernel
    gram_flops_fp64 = N * (n + 1)  # SYRK count of one mode's FP64 Gram (n_m (n_m+1)/2 entries x 2K flops)
    i8 = "i8_gemm" in st
    if i8:
        # k_i8_gemm: one residue Gram per modulus and mode, algorithmic int8 ops = moduli x n(n+1)/2 x K
        # x 2 per mode (16 moduli, or 15 where the row-norm bound allows it: DESIGN.md R21)
        mods = [int(x) for x in info.moduli]
        if not all(mods):
            mods = [16, 16, 16]
        launch_ms = prof["i8_gemm"][0] / prof["i8_gemm"][1]
        ops_launch = sum(mods) * gram_flops_fp64 * K / prof["i8_gemm"][1]
        achieved = ops_launch / (launch_ms * 1e-3) / 1e12
        peaks = measured_peaks()
        if peaks.get("bf16_tflops_sustained"):
            peak = 2.0 * peaks["bf16_tflops_sustained"]
            peak_src = ("dense INT8 = 2 x measured sustained bf16 (MEASURED_PEAKS.json bf16_tflops_sustained "
                        f"{peaks['bf16_tflops_sustained']}; nominal ratio 4.5/2.25 POPS): the kernel runs inside a "
                        "long step at the power-capped clock")
        else:
            peak = 4500.0
            peak_src = "nominal dense INT8 4.5 POPS (MEASURED_PEAKS.json absent)"
        traffic = None
        tp = os.path.join(ROOT, "profiles", "i8_gemm_traffic.json")
        if os.path.exists(tp):
            try:
                traffic = json.load(open(tp)).get("dram_bytes_per_launch")
            except Exception:
                traffic = None
        gram_stage_ms = sum(st.get(s, 0.0) for s in ("i8_rowmax", "i8_residues", "i8_gemm", "i8_crt")) / 3
        lib_i8 = None  # context: cuBLASLt's own sustained INT8 GEMM on this pool (tools/probe_int8_peak.py)
        ip = os.path.join(ROOT, "profiles", "int8_peak_measured.json")
        if os.path.exists(ip):
            try:
                lib_i8 = max(r["sustained_tops"] for r in json.load(open(ip))["runs"])
            except Exception:
                lib_i8 = None
        # the MACs the kernel actually issues: lower-triangle pair tiles of 256 rows x up to 512
        # columns, the diagonal 256-blocks computed whole (20 % more than the SYRK count at n = 1024;
        # minimal for cta_group::2 pairs)
        nI = (n + 255) // 256
        exec_cols = sum(min(256 * (I + 1), n) for I in range(nI))  # columns per 256-row block (trimmed)
        exec_ratio = (256.0 * exec_cols) / (n * (n + 1) / 2.0)
        roof = {"bound": "tensor", "kernel": "k_i8_gemm (tcgen05 kind::i8, CTA pairs), per launch",
                "achieved": achieved, "peak": peak, "unit": "TOP/s", "frac": achieved / peak, "traffic": traffic,
                "executed_over_algorithmic_macs": exec_ratio, "frac_executed": achieved * exec_ratio / peak,
                "frac_executed_note": "int8 ops the tensor cores execute (the diagonal pair tiles' upper halves "
                                      "included) over the same peak; above 1 when the int8 MMAs hold a higher "
                                      "power-capped clock than the bf16 cuBLAS loop behind the sustained figure",
                "peak_source": peak_src, "ops_per_launch": ops_launch, "launch_ms": launch_ms,
                "moduli_per_mode": mods,
                "launches_per_step": calls["i8_gemm"],
                "fp64_equivalent_gram_tflops": gram_flops_fp64 / (gram_stage_ms * 1e-3) / 1e12,
                "fp64_peak_tflops": fp64_peak()[0],
                "fp64_equivalent_note": "FP64 SYRK flops of one mode / the whole emulated Gram stage (residues, "
                                        "int8 Grams, CRT; per mode) vs the measured FP64 (DMMA) peak"}
        if lib_i8:
            roof["cublaslt_int8_sustained_tops"] = lib_i8
            roof["frac_of_cublaslt_int8_sustained"] = achieved / lib_i8
    else:
        launch_ms = prof["dmma_gram"][0] / prof["dmma_gram"][1]
        achieved = gram_flops_fp64 / (launch_ms * 1e-3) / 1e12
        peak, peak_src64 = fp64_peak()
        traffic = None
        tp = os.path.join(ROOT, "profiles", "gram_traffic.json")
        if os.path.exists(tp):
            try:
                traffic = json.load(open(tp)).get("dram_bytes_per_launch")
            except Exception:
                traffic = None
        roof = {"bound": "tensor", "kernel": "k_gram_tma (+k_gram_reduce), per mode",
                "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                "peak_source": peak_src64,
                "flops_per_launch": gram_flops_fp64}
    total_flops = 3 * gram_flops_fp64 + 2.0 * N * rr * 2  # FP64 Gram + TTM1 + error reconstruction (algorithmic)
    p64, _ = fp64_peak()
    hbm = float(measured_peaks().get("hbm_gbs", 6460.5))
    stage_roof = {}
    for name, fl in (("ttm", 2.0 * N * rr), ("error", 2.0 * N * rr)):
        if name in st:
            t_fp64 = fl / (p64 * 1e12) * 1e3
            t_hbm = 8.0 * N / (hbm * 1e9) * 1e3
            i8 = name == "ttm" and ttm_on_int8(rr, args)
            stage_roof[name] = {"ms": st[name], "fp64_roofline_ms": t_fp64, "hbm_roofline_ms": t_hbm,
                                "binding": "hbm" if (i8 or t_hbm >= t_fp64) else "fp64",
                                "frac_of_binding": (t_hbm if i8 else max(t_fp64, t_hbm)) / st[name],
                                "algorithmic": f"2 N r3 = {fl:.3e} flop, 8 N = {8 * N / 1e9:.2f} GB"}
            if i8:
                stage_roof[name]["engine"] = ttm_i8_note(rr)
    result = {
        "metric": METRIC, "value": whole_job_rate(N, world, ms_step), "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "dtype_note": ("FP64 path; the Grams are formed exactly from int8 residues on the tensor cores (tcgen05 "
                       "kind::i8, 16 moduli or 15 under the row-norm bound) and reconstructed to FP64 by the CRT (DESIGN.md R18, "
                       "R21)") if i8 else
                      "FP64 path; Grams on the FP64 tensor cores (DMMA)",
        "data": "synthetic",
        "config": {"workload": f"cfg5_{n}cube_matern_nu1.5_ell0.2", "grid": [n, n, n], "box": [-1.0, 1.0],
                   "kernel": {"family": "matern", "nu": 1.5, "ell": 0.2, "sigma2": 1.0}, "ranks": list(ranks),
                   "gram_engine": "int8 emulation (tcgen05 kind::i8 + CRT)" if i8 else "dmma",
                   "l2": f"inputs larger than L2 (F = {8 * N / 1e9:.2f} GB per step, L2 = 126 MB)",
                   "step_calls": ("tucker_fill_prepare + tucker_hosvd_prepared + tucker_error" if use_prepare else
                                  "tucker_fill_rowmax + tucker_hosvd_rowmax + tucker_error" if use_rowmax
                                  else "tucker_fill + tucker_hosvd + tucker_error"),
                   "parallelism": f"replicas{world}" if world > 1 else "single",
                   "hosvd_mode": "timed steps asynchronous (info = NULL, no host synchronisation); the warm-up "
                                 "steps and one step after the timed region synchronous (rc, convergence and the "
                                 "input window checked; bitwise the same outputs)"},
        "stages_ms": st, "stage_calls_per_step": calls,
        "stages_note": "device time per stage from the library's stage timer (CUDA events on the launching "
                       "stream) over a second, separately profiled pass of K steps; on the INT8 route the "
                       "eigensolve of mode m runs on a side stream while the Gram of mode m+1 runs, so 'eig' "
                       "spans that overlap and the stages sum past the step",
        "fp64_tflops_algorithmic": total_flops / (ms_step * 1e-3) / 1e12,
        "roofline": roof,
        "stage_rooflines": stage_roof,
        "eig_info": info.as_dict(),
        "graph": graph,
        "gpu_launches": launches,
        "error": {"E": E[0], "normF": E[1], "normDiff": E[2]},
    }

    # ---- e2e through the public call with host outputs (tucker_approximate)
    if not args.no_e2e:
        host = T.HostBuffers(grid, ranks)
        for _ in range(1):
            T.approximate(grid, kern, ranks, F, ws, host, stream)
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        ke = max(1, min(K, 3))
        for _ in range(ke):
            T.approximate(grid, kern, ranks, F, ws, host, stream)
        a1.record(stream)
        torch.cuda.synchronize()
        ms_e2e = max_over_ranks(a0.elapsed_time(a1) / ke, world, dev)
        param_bytes = ctypes.sizeof(g_c) + ctypes.sizeof(k_c) + ctypes.sizeof(r_c)
        result["e2e"] = {"value": whole_job_rate(N, world, ms_e2e), "unit": UNIT, "h2d_bytes_per_step": param_bytes,
                         "d2h_bytes_per_step": host.d2h_bytes, "ms_per_step": ms_e2e,
                         "call": "tucker_approximate (grid + kernel spec in, U/core/sigma/E to pinned host)"}
        # variant: the tensor F already sampled on the host (pinned) -> H2D copy inside the timed region
        if not args.no_host_tensor:
            try:
                Fh = torch.empty((n, n, n), dtype=torch.float64).pin_memory()
                Fh.copy_(F)
                b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                b0.record(stream)
                F.copy_(Fh, non_blocking=True)
                res = T.hosvd(grid, ranks, F, ws, stream)
                errv = T.error(grid, ranks, F, res.U, res.core, ws, stream)
                outs = [u.cpu() for u in res.U] + [res.core.cpu(), errv.cpu()] + [s.cpu() for s in res.sigma]
                b1.record(stream)
                torch.cuda.synchronize()
                ms_h = b0.elapsed_time(b1)
                result["e2e_host_tensor"] = {"value": N / (ms_h * 1e-3), "unit": UNIT, "ms_per_step": ms_h,
                                             "h2d_bytes_per_step": 8 * N,
                                             "d2h_bytes_per_step": 8 * sum(o.numel() for o in outs)}
                del Fh
            except RuntimeError as e:  # pinned allocation failure etc.
                result["e2e_host_tensor"] = {"unavailable": str(e)[:200]}
    result["clocks"] = clk.summary()
    if not args.no_als and world == 1:
        res = T.hosvd(grid, ranks, F, ws, stream)
        T.als(grid, ranks, F, res.U, 1, stream=stream)  # warm-up (workspace allocation, first launches)
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        al = T.als(grid, ranks, F, res.U, 2, stream=stream)
        a1.record(stream)
        torch.cuda.synchronize()
        ea = T.error(grid, ranks, F, al.U, al.core, ws, stream).cpu().tolist()
        eh = T.error(grid, ranks, F, res.U, res.core, ws, stream).cpu().tolist()
        ms_als = a0.elapsed_time(a1) / 2
        result["als"] = {"what": "Tucker-ALS / HOOI sweep (NEXT f1, P:571-579) on the same 1024^3 tensor, ranks 40",
                         "ms_per_sweep": ms_als, "points_per_s_per_sweep": N / (ms_als * 1e-3),
                         "E_hosvd": eh[0], "E_after_2_sweeps": ea[0], "rc": al.rc}
    if not args.no_multigrid and world == 1:
        result["multigrid"] = run_multigrid(T, grid, kern, ranks, F, stream)
    if not args.no_accurate and world == 1:
        acc = T.hosvd_accurate(grid, ranks, F, 1, stream=stream)  # warm-up
        torch.cuda.synchronize()
        acc_ms = []
        for _ in range(3):  # median of three calls (one call is ~0.1 s; power-state noise)
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0.record(stream)
            acc = T.hosvd_accurate(grid, ranks, F, 1, stream=stream)
            c1.record(stream)
            torch.cuda.synchronize()
            acc_ms.append(c0.elapsed_time(c1))
        ec = T.error(grid, ranks, F, acc.U, acc.core, ws, stream).cpu().tolist()
        result["accurate"] = {"what": "SVD-accurate HOSVD (NEXT f2): Gram route + one Rayleigh-Ritz step on each "
                                      "F_(m) (two streaming passes, CGS2, one-sided Jacobi SVD)",
                              "ms": sorted(acc_ms)[1], "ms_calls": acc_ms, "E": ec[0], "E_gram_route": E[0],
                              "rc": acc.rc,
                              "sigma_min_resolved": [float(s[-1]) / float(s[0]) for s in
                                                     (x.cpu() for x in acc.sigma)]}
    if not args.no_f4 and world == 1:
        result["f4"] = run_f4(T, grid, ranks, F, ws, stream)
    if not args.no_lowrank and world == 1:
        result["lowrank"] = run_lowrank(T, grid, kern, F, stream, p64=fp64_peak()[0],
                                        hbm=float(measured_peaks().get("hbm_gbs", 6460.5)))
    if not args.no_parity and world == 1 and n == 1024 and rr == 40:
        T.fill(grid, kern, F, ws, stream)  # (f4 reused F)
        result["parity"] = run_parity(T, stream, F)
    if not args.no_cfg4:
        del F
        torch.cuda.empty_cache()
        result["config4"] = run_cfg4(T, stream, rank, world)
        F = None
    if not args.no_fused and world == 1 or not args.no_sym and world == 1:
        F = None
        torch.cuda.empty_cache()
    if not args.no_sym and world == 1:
        result["symmetric"] = [run_sym(T, nn, rr, stream) for nn in (n, 2 * n)]
    if not args.no_fused and world == 1:
        result["fused"] = run_fused(T, args.fused_n, rr, stream)
    if not args.no_fused and world > 1:
        try:
            result["fused_sharded"] = run_fused_sharded(T, args.fused_n, rr, stream, world)
        except Exception as e:  # (symmetric failures, e.g. memory: every rank records it and goes on)
            result["fused_sharded"] = {"unavailable": f"{type(e).__name__}: {e}"[:300]}
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        result["cpu_baseline"] = cpu_baseline(n, rr, budget_s=15.0)
    if world > 1:
        dist.destroy_process_group()
    return result


def run_multigrid(T, grid, kern, ranks, F, stream) -> dict:
    """Multigrid Tucker on the same 1024^3 workload: HOSVD at 128^3, then interpolated
    factors + 2 ALS sweeps at 256^3, 512^3, 1024^3 (fills of every level included)."""
    import torch
    res, _, lev = T.multigrid(grid, kern, ranks, n0=128, sweeps=2, F=F, stream=stream)  # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    res, _, lev = T.multigrid(grid, kern, ranks, n0=128, sweeps=2, F=F, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    err = T.error(grid, ranks, F, res.U, res.core, stream=stream).cpu().tolist()
    return {"what": "multigrid Tucker (P:587-596): HOSVD at 128^3, cubic prolongation + 2 ALS sweeps per level",
            "levels": lev, "ms": ms, "value": grid.points / (ms * 1e-3), "unit": UNIT, "E": err[0], "rc": res.rc}


def run_fused(T, n: int, rr: int, stream) -> dict:
    """BASELINE config 5f: HOSVD + error of the n^3 function tensor through the fused
    generate-and-contract path (F never materialised; 68.7 GB at 2048^3 if it were)."""
    import torch

    from tucker_inputs import GridSpec, KernelSpec
    grid = GridSpec.cube(n, 1.0)
    kern = KernelSpec.matern(1.5, 0.2)
    ranks = (rr, rr, rr)
    N = grid.points
    ws = T.workspace_fused(grid, ranks)
    T.gram_fused(grid, kern, 0, ws, stream)  # warm-up (module load, first cooperative launch)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    ev[0].record(stream)
    for m in range(3):
        T.gram_fused(grid, kern, m, ws, stream)
        ev[1 + m].record(stream)
    torch.cuda.synchronize()
    gram_ms = [ev[m].elapsed_time(ev[m + 1]) for m in range(3)]
    T.profile_read()
    T.profile_enable(True)
    ev[4].record(stream)
    res = T.hosvd_fused(grid, kern, ranks, ws, stream)
    err = T.error_fused(grid, kern, ranks, res.U, res.core, ws, stream)
    ev[5].record(stream)
    torch.cuda.synchronize()
    T.profile_enable(False)
    prof = {k: v[0] for k, v in T.profile_read().items() if v[1]}
    ms = ev[4].elapsed_time(ev[5])
    flops = N * (n + 1)
    ach = [flops / (g * 1e-3) / 1e12 for g in gram_ms]
    e = err.cpu().tolist()
    i8 = "i8_gemm" in prof
    return {"workload": f"cfg5f_{n}cube_matern_nu1.5_ell0.2_fused", "grid": [n, n, n], "ranks": list(ranks),
            "value": N / (ms * 1e-3), "unit": UNIT, "ms": ms, "F_bytes_never_stored": 8 * N,
            "gram_engine": "int8 emulation (F generated in ~1 GiB plane chunks, residues streamed)" if i8 else "dmma",
            "stages_ms": prof,
            "gram_ms_separate_calls": gram_ms, "fp64_equivalent_gram_tflops": ach,
            "gram_frac_of_fp64_peak": [a / FP64_PEAK_SPEC_TFLOPS for a in ach],
            "E": e[0], "normF": e[1], "eig_info": res.info, "rc": res.rc,
            "timed": "one hosvd_fused + error_fused call (CUDA events; stages from the library's stage timer), "
                     "after a warm-up Gram; gram_ms from three separate tucker_gram_fused calls (each INT8 call "
                     "includes its own row-maxima generation pass)"}


def run_fused_sharded(T, n: int, rr: int, stream, world: int) -> dict:
    """Row (e): ONE config-5f problem (n^3 fused HOSVD + error, F never stored) sharded over the
    `world` ranks (tucker_hosvd_fused_sharded; exchanges = NCCL all-reduces of the Gram residue
    sums, T2 and the error partials).  Strong scaling of one tensor; time = max over ranks."""
    import torch
    import torch.distributed as dist

    from tucker_inputs import GridSpec, KernelSpec
    grid = GridSpec.cube(n, 1.0)
    kern = KernelSpec.matern(1.5, 0.2)
    ranks = (rr, rr, rr)
    rank = dist.get_rank()
    ws = T.workspace_fused(grid, ranks)
    res = T.hosvd_fused_sharded(grid, kern, ranks, rank, world, ws=ws, stream=stream)  # warm-up
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    res = T.hosvd_fused_sharded(grid, kern, ranks, rank, world, ws=ws, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    e = res.err.cpu().tolist()
    eq = torch.tensor([e[0]], dtype=torch.float64, device="cuda")
    emax, emin = eq.clone(), eq.clone()
    dist.all_reduce(emax, op=dist.ReduceOp.MAX)
    dist.all_reduce(emin, op=dist.ReduceOp.MIN)
    t = float(ms.item())
    return {"workload": f"cfg5f_{n}cube_matern_nu1.5_ell0.2_fused_sharded", "grid": [n, n, n], "ranks": list(ranks),
            "n_shards": world, "scaling": "strong", "value": grid.points / (t * 1e-3), "unit": UNIT, "ms": t,
            "E": e[0], "E_identical_on_all_ranks": bool(emax.item() == emin.item()), "rc": res.rc,
            "exchanges": len(res.exchanges),
            "timed": "one tucker_hosvd_fused_sharded call with the error (CUDA events per rank, max over ranks) "
                     "after a warm-up call; the exchanges are NCCL all-reduces issued from the library's callback"}


def _merge_deltas(acc: dict, d: dict) -> dict:
    """Worst case of T1-T4 deltas over several comparisons (parity_bars.Deltas.as_dict())."""
    if not acc:
        acc = {"T1_ratio": 0.0, "T2_max_col": 0.0, "T2p_orth": 0.0, "T3_rel": 0.0, "T3_norm_rel": 0.0,
               "T4_abs": 0.0, "T4_over_bar": 0.0, "resolved_cases": 0, "cases": 0, "pass": True}
    for k in ("T1_ratio", "T2_max_col", "T2p_orth", "T3_rel", "T3_norm_rel", "T4_abs"):
        acc[k] = max(acc[k], d[k])
    acc["T4_over_bar"] = max(acc["T4_over_bar"], d["T4_abs"] / d["T4_bar"])
    acc["resolved_cases"] += int(d["resolved"])
    acc["cases"] += 1
    acc["pass"] &= (d["T1_ratio"] <= 1.0 and d["T2_max_col"] <= 1e-9 and d["T2p_orth"] <= 1e-12 and
                    d["T3_rel"] <= 1e-10 and d["T3_norm_rel"] <= 1e-12 and d["T4_abs"] <= d["T4_bar"])
    return acc


def run_parity(T, stream, F=None) -> dict:
    """Per-config T1-T4 parity deltas of the GPU path against the CPU oracle's
    results stored by tests/golden/make_golden.py (oracle-only script; configs 1-3, config 4's 16
    settings, config 5 at ranks 40 and 10).  Untimed.  F: the cfg5 tensor if still resident."""
    import numpy as np
    import torch

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import parity_bars as PB
    from tucker_inputs import config1, config2, config3, config4, config5

    gdir = os.path.join(ROOT, "tests", "golden")
    out = {"bars": "T1 |dlambda| <= 1e-11 lambda + 1e-14 lambda_1 (ratio <= 1); T2 gap-separated columns <= 1e-9; "
                   "T2' <= 1e-12; T3 <= 1e-10 (block k_res(1e-10)), norm <= 1e-12; T4 <= 1e-12 resolved, else "
                   "max(1e-12, 1e-15/E)",
           "reference": "oracle results in tests/golden/*.npz (tests/golden/make_golden.py, oracle only)"}

    def cmp(ref, r, res, E):
        return PB.compare(ref, r, [x.cpu().numpy() for x in res.sigma], [u.cpu().numpy() for u in res.U],
                          res.core.cpu().numpy(), float(E), check=False).as_dict()

    def trunc(res, t):
        U = [u[:, :t[m]].contiguous() for m, u in enumerate(res.U)]
        core = res.core[:t[0], :t[1], :t[2]].contiguous()
        return type(res)(U, core, [sg[:t[m]] for m, sg in enumerate(res.sigma)], res.info, res.rc)

    p = os.path.join(gdir, "small_oracle.npz")
    if os.path.exists(p):
        z = np.load(p)
        for w in (config1(), config2(), config3()):
            acc = {}
            Fw = torch.empty(tuple(w.grid.n), dtype=torch.float64, device="cuda")
            ws = T.workspace(w.grid, w.ranks)
            for i, k in enumerate(w.kernels):
                T.fill(w.grid, k, Fw, ws, stream)
                res = T.hosvd(w.grid, w.ranks, Fw, ws, stream)
                for t in [tuple(int(v) for v in x) for x in z[f"{w.name}_k{i}_truncations"]]:
                    rt = trunc(res, t)
                    e = T.error(w.grid, t, Fw, rt.U, rt.core, ws, stream)[0].item()
                    acc = _merge_deltas(acc, cmp(PB.golden_ref(z, f"{w.name}_k{i}_", t), t, rt, e))
            out[w.name] = acc
            del Fw, ws
    p = os.path.join(gdir, "cfg5_1024_oracle.npz")
    if os.path.exists(p) and F is not None:
        z = np.load(p)
        w = config5()
        for rk in ((40, 40, 40), (10, 10, 10)):
            ws = T.workspace(w.grid, rk)
            res = T.hosvd(w.grid, rk, F, ws, stream)
            e = T.error(w.grid, rk, F, res.U, res.core, ws, stream)[0].item()
            out[f"{w.name}_r{rk[0]}"] = _merge_deltas({}, cmp(PB.golden_ref(z, trunc=rk), rk, res, e))
            out[f"{w.name}_r{rk[0]}"]["E_gpu"], out[f"{w.name}_r{rk[0]}"]["E_oracle"] = e, float(
                PB.golden_ref(z, trunc=rk).E)
            del ws
    p = os.path.join(gdir, "cfg4_512_oracle.npz")
    if os.path.exists(p):
        z = np.load(p)
        w = config4()
        acc = {}
        F4 = torch.empty(tuple(w.grid.n), dtype=torch.float64, device="cuda")
        ws = T.workspace(w.grid, w.ranks)
        for s_ in [int(v) for v in z["settings"]]:
            T.fill(w.grid, w.kernels[s_], F4, ws, stream)
            res = T.hosvd(w.grid, w.ranks, F4, ws, stream)
            for t in ((30, 30, 30), (20, 20, 20), (10, 10, 10)):
                rt = trunc(res, t)
                e = T.error(w.grid, t, F4, rt.U, rt.core, ws, stream)[0].item()
                acc = _merge_deltas(acc, cmp(PB.golden_ref(z, f"s{s_}_", t), t, rt, e))
        out[w.name] = acc
        del F4, ws
        torch.cuda.empty_cache()
    return out


def run_lowrank(T, grid, kern, F, stream, p64: float, hbm: float) -> dict:
    """The TTM and error stages where HBM binds them (2 r3 flop per 8 B below the FP64 ridge: r3 <= 23,
    SURVEY §8(d)): the headline step at ranks (10,10,10) and (20,20,20), asynchronous HOSVD, stage
    times from the library's stage timer over five steps after three warm-up steps."""
    import torch
    N = grid.points
    out = []
    for r in (10, 20):
        rr3 = (r, r, r)
        ws = T.workspace(grid, rr3)
        results = []

        def step():
            T.fill_prepare(grid, kern, rr3, F, ws, stream)
            res = T.hosvd_prepared(grid, rr3, F, ws, stream, sync=False)
            results.append(res)  # (outputs stay alive until the synchronisation below)
            return T.error(grid, rr3, F, res.U, res.core, ws, stream)

        for _ in range(3):
            step()
        torch.cuda.synchronize()
        T.profile_read()
        T.profile_enable(True)
        for _ in range(5):
            e = step()
        torch.cuda.synchronize()
        T.profile_enable(False)
        prof = T.profile_read()
        st = {name: ms / 5 for name, (ms, cnt) in prof.items() if cnt}
        t_hbm = 8.0 * N / (hbm * 1e9) * 1e3
        t_fp = 2.0 * N * r / (p64 * 1e12) * 1e3
        row = {"ranks": list(rr3), "E": float(e.cpu()[0]), "hbm_roofline_ms": t_hbm, "fp64_roofline_ms": t_fp,
               "binding": "hbm" if t_hbm >= t_fp else "fp64"}
        for name in ("ttm", "error"):
            if name in st:
                i8 = name == "ttm" and ttm_on_int8(r, None) and T.get_gram_engine() != T.GRAM_DMMA
                row[name + "_ms"] = st[name]
                row[name + "_frac_of_binding"] = (t_hbm if i8 else max(t_hbm, t_fp)) / st[name]
                if i8:
                    row[name + "_engine"] = ttm_i8_note(r)
        out.append(row)
        del ws, results
        torch.cuda.empty_cache()
    return {"grid": list(grid.n), "what": "TTM and error stages at ranks where HBM binds them (in-step, stage timer)",
            "rows": out}


def run_f4(T, grid, ranks, F, ws, stream) -> dict:
    """NEXT f4: the paper's other workloads through the same step on the same 1024^3 grid —
    Matérn spectral density (alpha = 0.1 and 100, nu = 0.4) and p-Slater
    (p = 0.1, 1.9): fill + HOSVD + error per kernel."""
    import torch

    from tucker_inputs import KernelSpec
    out = []
    for k in (KernelSpec.spectral(0.1, 0.4), KernelSpec.spectral(100.0, 0.4), KernelSpec.slater(1.0, 0.1),
              KernelSpec.slater(1.0, 1.9)):
        T.fill_prepare(grid, k, ranks, F, ws, stream)  # warm-up step of this kernel
        res = T.hosvd_prepared(grid, ranks, F, ws, stream)
        T.error(grid, ranks, F, res.U, res.core, ws, stream)
        torch.cuda.synchronize()
        steps = []
        for _ in range(3):  # median of three steps (a single sample swings by several ms at the power cap)
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record(stream)
            T.fill_prepare(grid, k, ranks, F, ws, stream)  # fill + shared residues (the headline step's calls)
            e[1].record(stream)
            res = T.hosvd_prepared(grid, ranks, F, ws, stream)
            err = T.error(grid, ranks, F, res.U, res.core, ws, stream)
            e[2].record(stream)
            torch.cuda.synchronize()
            steps.append((e[0].elapsed_time(e[2]), e[0].elapsed_time(e[1])))
        ms, fill_ms = sorted(steps)[1]
        out.append({"kernel": k.label(), "ms_per_step": ms, "ms_steps": [a for a, _ in steps], "fill_prepare_ms": fill_ms,
                    "moduli": res.info["moduli"],
                    "value": grid.points / (ms * 1e-3), "E": float(err[0]), "rc": res.rc,
                    "eig_iters": res.info["iters"], "eig_converged": res.info["converged"],
                    "k_resolved": res.info["k_resolved"], "eig_resid": res.info["resid"]})
    return {"grid": list(grid.n), "ranks": list(ranks), "unit": UNIT, "workloads": out}


def run_cfg4(T, stream, rank: int = 0, world: int = 1) -> dict:
    """BASELINE config 4: 512^3, 16 seeded Matérn settings (R10), ranks 30 — the whole path per
    setting (fill, 3 Grams, 3 eigensolves, core, error), timed over the batch.  With world > 1 the
    settings are replicas spread over the ranks (one setting set per GPU, settings
    rank, rank + world, ...; time = max over ranks, strong scaling of the fixed batch)."""
    import torch

    from tucker_inputs import config4
    w = config4()
    g, r = w.grid, w.ranks
    mine = w.kernels[rank::world]
    F = torch.empty(tuple(g.n), dtype=torch.float64, device="cuda")
    ws = T.workspace(g, r)

    def one(k):  # the same three calls as the headline step (fill + residues in one pass)
        T.fill_prepare(g, k, r, F, ws, stream)
        res = T.hosvd_prepared(g, r, F, ws, stream)
        return res, T.error(g, r, F, res.U, res.core, ws, stream)

    one(w.kernels[0])  # warm-up
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    errs, rcs = [], []
    for k in mine:
        res, err = one(k)
        errs.append(err)
        rcs.append(res.rc)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    e_lo = min(float(e[0]) for e in errs) if errs else float("inf")
    e_hi = max(float(e[0]) for e in errs) if errs else float("-inf")
    if world > 1:
        import torch.distributed as dist
        red = torch.tensor([ms, -e_lo, e_hi], dtype=torch.float64, device="cuda")
        dist.all_reduce(red, op=dist.ReduceOp.MAX)
        ms, e_lo, e_hi = float(red[0]), -float(red[1]), float(red[2])
    pts = len(w.kernels) * g.points
    del F, ws
    torch.cuda.empty_cache()
    return {"workload": w.name, "settings": len(w.kernels), "ranks": list(r), "value": pts / (ms * 1e-3),
            "unit": UNIT, "ms_total": ms, "ms_per_setting": ms * world / len(w.kernels), "rc": rcs,
            "n_gpus": world, "E_range": [e_lo, e_hi]}


def run_sym(T, n: int, rr: int, stream, reps: int = 3) -> dict:
    """NEXT f3: the whole path (octant fill, 3 Grams, 3 eigensolves, core, error) on the weighted
    octant tensor of a centred grid; algorithmic work is that of the octant (reported apart)."""
    import torch

    from tucker_inputs import GridSpec, KernelSpec
    grid = GridSpec.cube(n, 1.0)
    kern = KernelSpec.matern(1.5, 0.2)
    ranks = (rr, rr, rr)
    N = grid.points
    h = (n + 1) // 2
    lib = T.load()
    import ctypes
    g = T.cgrid(grid)
    ws = torch.empty(int(lib.tucker_workspace_size_sym(ctypes.byref(g), T.cranks(ranks))), dtype=torch.uint8,
                     device="cuda")
    res, err = T.hosvd_sym(grid, kern, ranks, ws, stream)  # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        res, err = T.hosvd_sym(grid, kern, ranks, ws, stream)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    Nh = h ** 3
    grams = 1  # cubic isotropic grid: one Gram serves all three modes (G_1 = G_2 = G_3)
    flops = grams * Nh * (h + 1) + 2.0 * Nh * rr * 2
    e = err.cpu().tolist()
    return {"workload": f"cfg5_{n}cube_matern_nu1.5_ell0.2_symmetric", "grid": [n, n, n], "ranks": list(ranks),
            "value": N / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms,
            "algorithmic_flops_per_step": flops, "fp64_tflops_algorithmic": flops / (ms * 1e-3) / 1e12,
            "E": e[0], "normF": e[1], "rc": res.rc,
            "note": "weighted-octant reduction (exact on centred grids, DESIGN f3): N/8 points carry the "
                    "work; cubic isotropic grid: one Gram (N/8)(n/2+1) flops serves all modes; TTM + error "
                    "4 (N/8) r"}


# ------------------------------------------------------------------------------ oracle arm ----
def oracle_sampled_step(orc, n: int, r: int, S: int) -> dict:
    """ONE sampled step of the oracle, as it stands, on the host cores: 1/S of the work of every
    stage of the cfg5 step, actually executed and wall-clock timed (nothing is extrapolated):

      fill       s = n/S of the n i-slabs of F (orc.fill of the sub-grid)
      Gram x 3   the Dot2 Gram of an n x (s n) block of each mode's unfolding (s n of its n^2
                 columns): modes 2 and 1 from the slab's unfoldings; mode 0's block (a j-slab) has
                 the same shape and work on the cube, and its Gram is the slab's mode-1 Gram again
      eig x 3    cyclic Jacobi at order n_s = n / S^(1/3) (work ~ n^3: 1/S), on the leading block of
                 the sampled mode-2 Gram
      core       orc.ttm_core of the slab (its s n^2 points, ranks r)
      error      orc.tucker_error of the slab
    Returns {seconds, parts, points = N/S, ...}."""
    import numpy as np

    k = orc.Kernel.matern(1.5, 0.2)
    s = max(1, n // S)
    h = 2.0 / (n - 1)
    sub = orc.Grid((s, n, n), (-1.0, -1.0, -1.0), (-1.0 + h * (s - 1), 1.0, 1.0))
    parts = {}
    t_all = time.perf_counter()
    t = time.perf_counter()
    Fs = orc.fill(sub, k)
    parts["fill"] = time.perf_counter() - t
    t = time.perf_counter()
    A1 = orc.unfold(Fs, 1)
    G1 = orc.gram(A1)
    orc.gram(A1)  # mode 0's sample (same n x s n shape and work on the cube)
    A2 = orc.unfold(Fs, 2)
    G2 = orc.gram(A2)
    parts["gram"] = time.perf_counter() - t
    ns = max(2, int(round(n / S ** (1.0 / 3.0))))
    t = time.perf_counter()
    for G in (G1, G1, G2):
        orc.jacobi_eig(np.ascontiguousarray(G[:ns, :ns]))
    parts["eig"] = time.perf_counter() - t
    rng = np.random.default_rng(0)
    U = [np.linalg.qr(rng.standard_normal((dim, min(r, dim))))[0] for dim in (s, n, n)]
    t = time.perf_counter()
    core = orc.ttm_core(Fs, *U)
    parts["ttm"] = time.perf_counter() - t
    t = time.perf_counter()
    orc.tucker_error(Fs, *U, core)
    parts["error"] = time.perf_counter() - t
    sec = time.perf_counter() - t_all
    return {"seconds": sec, "parts_s": parts, "points": n ** 3 / (n / s), "S": n / s, "slabs": s, "jacobi_order": ns,
            "gram_columns": A1.shape[1]}


def host_cpu() -> dict:
    model = ""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "model": model}


def cpu_baseline(n: int, r: int, budget_s: float = 20.0, S: int = 64) -> dict:
    """The oracle as it stands on the host cores: repeated sampled steps (each 1/S of the cfg5
    step's work per stage, oracle_sampled_step) for about `budget_s` seconds; value = points of the
    workload the sampled steps covered / their measured wall time."""
    from oracle import oracle as orc
    orc.build()
    threads = orc.num_threads()
    runs = []
    t0 = time.perf_counter()
    while not runs or (time.perf_counter() - t0 < budget_s and len(runs) < 8):
        runs.append(oracle_sampled_step(orc, n, r, S))
    sec = sum(x["seconds"] for x in runs)
    pts = sum(x["points"] for x in runs)
    x = runs[0]
    return {"value": pts / sec, "unit": UNIT, "cores": threads, "kind": "oracle", "host": host_cpu(),
            "sample": (f"{len(runs)} sampled oracle steps of cfg5 ({n}^3, Matern nu=1.5 ell=0.2, r={r}), each 1/"
                       f"{x['S']:g} of every stage's work, executed and wall-clock timed: fill + core + error of "
                       f"{x['slabs']} i-slabs, three Dot2 Grams of n x {x['gram_columns']} unfolding blocks, three "
                       f"cyclic Jacobi solves at order {x['jacobi_order']}"),
            "seconds_per_sampled_step": sec / len(runs), "sampled_steps": len(runs),
            "parts_s_per_sampled_step": {k: sum(r_["parts_s"][k] for r_ in runs) / len(runs) for k in x["parts_s"]},
            "full_oracle_runs": "profiles/r02_oracle_timing.json (the oracle run whole on the box: configs 1-3, "
                                "1024^3 once, 1-thread 128^3)"}


def run_reference(args, rank, world):
    """The reference arm (this tier: the oracle): K timed sampled steps after W warm-up ones, on
    rank 0; value = sampled points / measured wall time, ms_per_step = the measured step."""
    if rank != 0:
        return None
    from oracle import oracle as orc
    orc.build()
    S = 64
    for _ in range(args.warmup):
        oracle_sampled_step(orc, args.n, args.r, S)
    runs = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        runs.append(oracle_sampled_step(orc, args.n, args.r, S))
    wall = time.perf_counter() - t0
    pts = sum(x["points"] for x in runs)
    v = pts / wall
    x = runs[0]
    sample = (f"each step: 1/{x['S']:g} of every stage of cfg5 ({args.n}^3, r={args.r}) executed by the oracle and "
              f"wall-clock timed — fill + core + error of {x['slabs']} i-slabs, three Dot2 Grams of n x "
              f"{x['gram_columns']} unfolding blocks, three cyclic Jacobi solves at order {x['jacobi_order']}; "
              f"value = covered points / wall time")
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"cfg5_{args.n}cube_matern_nu1.5_ell0.2", "grid": [args.n] * 3,
                       "ranks": [args.r] * 3, "sampled_fraction": 1.0 / x["S"]},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": orc.num_threads(), "kind": "oracle", "sample": sample,
                             "host": host_cpu()},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "parts_s_per_step": {k: sum(r_["parts_s"][k] for r_ in runs) / len(runs) for k in x["parts_s"]}}


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        res = run_reference(args, rank, world)
    else:
        res = run_ours(args, rank, world, local)
    if rank == 0 and res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
