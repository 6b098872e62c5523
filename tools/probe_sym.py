"""Probe: one tucker_hosvd_sym call at n^3 (config 5 function, ranks 40) for ncu launch lists."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1711_06874_b200 import tucker as T  # noqa: E402
from tucker_inputs import GridSpec, KernelSpec  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
g, k, r = GridSpec.cube(n, 1.0), KernelSpec.matern(1.5, 0.2), (40, 40, 40)
res, err = T.hosvd_sym(g, k, r)
torch.cuda.synchronize()
print("rc", res.rc, float(err[0]))
