"""Probe: time the a-4 eigensolver alone on the config-5 mode-0 Gram (n=1024, r=40) through the
C-ABI; prints per-call ms and the solver report.  Used with ncu for per-kernel launch times."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1711_06874_b200 import tucker as T  # noqa: E402
from tucker_inputs import GridSpec, config5  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
w = config5()
g = w.grid
g = GridSpec((n, n, n), g.lo, g.hi)
F = T.fill(g, w.kernels[0])
G = T.gram(g, 0, F)
ws = T.workspace(g, w.ranks)
for rep in range(reps):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    U, lam, info, rc = T.eig(G, w.ranks[0], ws=ws)
    e1.record()
    torch.cuda.synchronize()
    print(f"n={n} eig {e0.elapsed_time(e1):.3f} ms  info={info}")
