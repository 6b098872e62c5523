import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1711_06874_b200 import tucker as T
from tucker_inputs import GridSpec, KernelSpec
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
g = GridSpec.cube(n, 1.0)
F = T.fill(g, KernelSpec.matern(1.5, 0.2))
G = T.gram(g, 0, F)
del F
torch.cuda.synchronize()
U, lam = T.eig(G, 40)
torch.cuda.synchronize()
print(lam[:3])
