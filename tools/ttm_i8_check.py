"""Core of the INT8-TTM hosvd against the DMMA-TTM core on the same factors, prepared and plain calls."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1711_06874_b200 import tucker as T  # noqa: E402
from tucker_inputs import GridSpec, KernelSpec, config4_settings  # noqa: E402

T.load()
cases = [(GridSpec.cube(1024, 1.0), KernelSpec.matern(1.5, 0.2), (10, 10, 10)),
         (GridSpec.cube(512, 1.0), config4_settings()[0], (30, 30, 30)),
         (GridSpec.cube(256, 1.0), KernelSpec.matern(1.5, 0.2), (10, 10, 10))]
for g, k, r in cases:
    F = T.fill(g, k)
    for eng in (T.TTM_AUTO, T.TTM_DMMA):
        T.set_ttm_engine(eng)
        a = T.hosvd(g, r, F)
        c = a.core.cpu().numpy()
        if eng == T.TTM_AUTO:
            c0, U0 = c, [u.cpu().numpy() for u in a.U]
        else:
            same = all(np.array_equal(U0[m], a.U[m].cpu().numpy()) for m in range(3))
            d = np.abs(c0 - c)
            print(g.n, r, "U same", same, "max|dcore|/max|core|", d.max() / np.abs(c).max(),
                  "argmax", np.unravel_index(d.argmax(), d.shape), "norms", np.linalg.norm(c0), np.linalg.norm(c))
    T.set_ttm_engine(T.TTM_AUTO)
    ws = T.workspace(g, r)
    for eng in (T.TTM_AUTO, T.TTM_DMMA):
        T.set_ttm_engine(eng)
        T.fill_prepare(g, k, r, F, ws)
        a = T.hosvd_prepared(g, r, F, ws)
        c = a.core.cpu().numpy()
        if eng == T.TTM_AUTO:
            c1 = c
        else:
            print("  prepared: max|dcore|/max|core|", np.abs(c1 - c).max() / np.abs(c).max())
    T.set_ttm_engine(T.TTM_AUTO)
    del F, ws
    torch.cuda.empty_cache()
