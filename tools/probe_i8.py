"""Time the INT8-emulated Gram (tucker_gram_i8) against the DMMA Gram at 1024^3 (bench workload)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_1711_06874_b200 import tucker as T
from tucker_inputs import GridSpec, KernelSpec
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
g = GridSpec.cube(n, 1.0)
F = T.fill(g, KernelSpec.matern(1.5, 0.2))
ws8 = T.workspace_i8(g)
ws = T.workspace(g, (40, 40, 40))
print("ws_i8 GB", ws8.numel() / 1e9, flush=True)
for m in range(3):
    for name, fn in (("i8", lambda: T.gram_i8(g, m, F, ws8)), ("dmma", lambda: T.gram(g, m, F, ws))):
        G = fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(3):
            e0.record(); G = fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        if name == "i8":
            Gi = G
        else:
            d = torch.sqrt(torch.diagonal(G))
            rel = float(torch.max(torch.abs(Gi - G) / torch.outer(d, d)))
        print(m, name, ["%.2f" % t for t in ts], flush=True)
    print(m, "max |Gi8-Gdmma|/sqrt(GiiGjj) = %.3e" % rel, flush=True)
