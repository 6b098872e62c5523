"""One hosvd call (argv: n r prepared) with the INT8 TTM, printing rc and the core norm against DMMA."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1711_06874_b200 import tucker as T  # noqa: E402
from tucker_inputs import GridSpec, KernelSpec  # noqa: E402

n, r, prep = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3] == "1"
T.load()
g, k, rr = GridSpec.cube(n, 1.0), KernelSpec.matern(1.5, 0.2), (r, r, r)
F = T.fill(g, k)
out = []
for eng in (T.TTM_AUTO, T.TTM_DMMA):
    T.set_ttm_engine(eng)
    if prep:
        ws = T.workspace(g, rr)
        T.fill_prepare(g, k, rr, F, ws)
        a = T.hosvd_prepared(g, rr, F, ws)
    else:
        a = T.hosvd(g, rr, F)
    torch.cuda.synchronize()
    out.append(a.core.cpu().numpy())
print(n, r, prep, "ok", np.abs(out[0] - out[1]).max() / np.abs(out[1]).max())
