import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_1711_06874_b200 import tucker as T
from tucker_inputs import GridSpec, KernelSpec
for n, nu, ell, r in [(512, 0.5, 0.05, 40), (512, 0.5, 0.05, 56), (256, 0.3, 0.05, 56), (1024, 0.5, 0.05, 40), (200, 0.5, 0.02, 56)]:
    g = GridSpec.cube(n, 1.0); k = KernelSpec.matern(nu, ell)
    F = T.fill(g, k)
    torch.cuda.synchronize(); t = time.time()
    res = T.hosvd(g, (r, r, r), F)
    torch.cuda.synchronize()
    print(n, nu, ell, r, res.rc, res.info['iters'], [f"{x:.1e}" for x in res.info['resid']], f"{1e3*(time.time()-t):.0f} ms", flush=True)
    del F; torch.cuda.empty_cache()
