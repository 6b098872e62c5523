"""Probe: one tucker_gram_fused call (n^3 cube, Matérn nu=1.5 ell=0.2) for ncu captures.

    python tools/probe_fused_gram.py [n] [mode]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1711_06874_b200 import tucker as T  # noqa: E402
from tucker_inputs import GridSpec, KernelSpec  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 2
g, k = GridSpec.cube(n, 1.0), KernelSpec.matern(1.5, 0.2)
ws = T.workspace_fused(g)
torch.cuda.synchronize()
t = time.time()
G = T.gram_fused(g, k, mode, ws)
torch.cuda.synchronize()
print(f"n={n} mode={mode} {1e3 * (time.time() - t):.1f} ms")
