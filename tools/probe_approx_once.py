import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1711_06874_b200 import tucker as T
from tucker_inputs import GridSpec, KernelSpec
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
g, k, r = GridSpec.cube(n, 1.0), KernelSpec.matern(1.5, 0.2), (40, 40, 40)
F = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
ws = T.workspace(g, r)
host = T.HostBuffers(g, r)
for _ in range(2):
    out = T.approximate(g, k, r, F, ws, host)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    out = T.approximate(g, k, r, F, ws, host)
e1.record(); torch.cuda.synchronize()
print("approximate ms %.2f" % (e0.elapsed_time(e1) / 5), out.err[0])
