"""Stage breakdown of hosvd_fused + error_fused at n^3 (INT8 route) with the library's stage timer."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1711_06874_b200 import tucker as T
from tucker_inputs import GridSpec, KernelSpec
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
g, k, r = GridSpec.cube(n, 1.0), KernelSpec.matern(1.5, 0.2), (40, 40, 40)
ws = T.workspace_fused(g, r)
T.gram_fused(g, k, 0, ws)
torch.cuda.synchronize()
T.profile_read(); T.profile_enable(True)
e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
e0.record()
res = T.hosvd_fused(g, k, r, ws)
e1.record()
err = T.error_fused(g, k, r, res.U, res.core, ws)
e2.record(); torch.cuda.synchronize()
T.profile_enable(False)
print("hosvd %.1f ms, error %.1f ms" % (e0.elapsed_time(e1), e1.elapsed_time(e2)),
      {kk: round(v[0], 1) for kk, v in T.profile_read().items() if v[1]}, float(err[0]), flush=True)
