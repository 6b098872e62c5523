import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1711_06874_b200 import tucker as T
from tucker_inputs import GridSpec, KernelSpec
g, k = GridSpec.cube(1024, 1.0), KernelSpec.matern(1.5, 0.2)
for eng in (T.GRAM_AUTO, T.GRAM_DMMA):
    T.set_gram_engine(eng)
    for r in (10, 40):
        rr = (r, r, r)
        F = T.fill(g, k)
        ref = T.hosvd(g, rr, F)
        e_ref = T.error(g, rr, F, ref.U, ref.core).cpu().numpy()
        del F; torch.cuda.empty_cache()
        res, err = T.hosvd_sym(g, k, rr)
        print("engine", eng, "r", r, "E_gen %.6e E_sym %.6e" % (e_ref[0], err.cpu().numpy()[0]), flush=True)
