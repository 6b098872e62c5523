"""Time tucker_hosvd at 1024^3 on the INT8 Gram route, with the library's per-stage device times."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1711_06874_b200 import tucker as T
from tucker_inputs import GridSpec, KernelSpec
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
g = GridSpec.cube(n, 1.0)
F = T.fill(g, KernelSpec.matern(1.5, 0.2))
ws = T.workspace(g, (40, 40, 40))
for _ in range(2):
    T.hosvd(g, (40, 40, 40), F, ws)
torch.cuda.synchronize()
T.profile_read(); T.profile_enable(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    T.hosvd(g, (40, 40, 40), F, ws)
e1.record(); torch.cuda.synchronize()
T.profile_enable(False)
p = T.profile_read()
print("hosvd ms %.2f" % (e0.elapsed_time(e1) / 3),
      {k: round(v[0] / 3, 2) for k, v in p.items() if v[1]}, flush=True)
