"""Aggregate an ncu source-page metric (default: warp-stall samples) per CUDA source line.

    python tools/ncu_lines.py report.ncu-rep [top] [metric column] [kernel regex]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
metric = sys.argv[3] if len(sys.argv) > 3 else "Warp Stall Sampling (All Samples)"
kernel = sys.argv[4] if len(sys.argv) > 4 else None
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if kernel:
    cmd += ["-k", kernel]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
col = None
path = None
agg = {}
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if len(r) >= 8 and r[0] == "Line No":
        col = r.index(metric)
        continue
    if len(r) < 8 or r[0] == "" or col is None:
        continue
    try:
        samples = float(r[col] or 0)
    except ValueError:
        continue
    key = (path, int(r[0]))
    agg[key] = (agg.get(key, (0.0, ""))[0] + samples, r[1])
tot = sum(v[0] for v in agg.values()) or 1
for (f, ln), (s, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{s / tot * 100:5.1f}%  {f}:{ln}  {src.strip()[:100]}")
