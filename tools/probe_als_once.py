import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1711_06874_b200 import tucker as T
from tucker_inputs import GridSpec, KernelSpec
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
g = GridSpec.cube(n, 1.0)
F = T.fill(g, KernelSpec.matern(1.5, 0.2))
res = T.hosvd(g, (40, 40, 40), F)
torch.cuda.synchronize()
out = T.als(g, (40, 40, 40), F, res.U, sweeps=1)
torch.cuda.synchronize()
