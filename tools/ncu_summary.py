"""Summarise ncu outputs (launch list CSV and --set full reports) into profiles/.

    python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/r01_launches.md
    python tools/ncu_summary.py report gpurun_out/prof_gram.ncu-rep > profiles/r01_gram_full.md
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__average_warp_latency_issue_stalled_barrier", "sm__cycles_elapsed.avg",
        "sm__cycles_elapsed.avg.per_second", "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "l1tex__m_xbar2l1tex_read_bytes.sum"]


def to_us(v, unit):
    v = float(v.replace(",", ""))
    return v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
                "second": 1e6, "s": 1e6}.get(unit, 1.0)


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg, cnt, tot = collections.OrderedDict(), collections.Counter(), 0.0
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = to_us(r[vi], r[ui])
        name = r[ki].split("(")[0]
        agg[name] = agg.get(name, 0.0) + v
        cnt[name] += 1
        tot += v
    print(f"# ncu launch list ({path}) — cold-cache, serialised; compare shares, not absolutes\n")
    print("| kernel | launches | total ms | mean us | share |\n|---|---:|---:|---:|---:|")
    for k, v in sorted(agg.items(), key=lambda x: -x[1]):
        print(f"| `{k}` | {cnt[k]} | {v / 1e3:.3f} | {v / cnt[k]:.1f} | {100 * v / tot:.1f}% |")
    print(f"\nTotal: {tot / 1e3:.3f} ms over {sum(cnt.values())} launches.")


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    print(f"# ncu --set full summary ({path})\n")
    for r in rows[2:]:
        name = r[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print(f"## `{name.split('(')[0]}` (ID {r[h.index('ID')]})\n")
        print("| metric | value | unit |\n|---|---:|---|")
        for k in KEYS:
            # raw-page columns may carry a section prefix ("TPC.TriageCompute.<metric>")
            idx = [i for i, c in enumerate(h) if c == k or c.endswith("." + k)]
            if idx:
                i = idx[0]
                print(f"| {k} | {r[i]} | {units[i]} |")
        print()


if __name__ == "__main__":
    {"launches": launches, "report": report}[sys.argv[1]](sys.argv[2])
