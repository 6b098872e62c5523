"""Aggregate ncu source-page warp-stall samples per CUDA source line.

    python tools/ncu_lines.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
path = None
agg = {}
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] == "Line No" or r[0] == "":
        continue
    try:
        samples = float(r[4] or 0)
    except ValueError:
        continue
    agg[(path, int(r[0]))] = (samples, r[1])
tot = sum(v[0] for v in agg.values()) or 1
for (f, ln), (s, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{s / tot * 100:5.1f}%  {f}:{ln}  {src.strip()[:100]}")
