"""Probe: BASELINE config 4 (512^3, 16 seeded Matérn settings, ranks 30) through the C-ABI —
eigensolver iterations/convergence, E at r = 10, 20, 30, time per setting."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1711_06874_b200 import tucker as T  # noqa: E402
from tucker_inputs import config4  # noqa: E402

w = config4()
g, r = w.grid, w.ranks
F = torch.empty(tuple(g.n), dtype=torch.float64, device="cuda")
ws = T.workspace(g, r)
for s, k in enumerate(w.kernels):
    torch.cuda.synchronize()
    t = time.time()
    T.fill(g, k, F, ws)
    res = T.hosvd(g, r, F, ws)
    es = []
    for rr in (10, 20, 30):
        U = [u[:, :rr].contiguous() for u in res.U]
        core = T.ttm_core(g, (rr,) * 3, F, *U, ws=ws)
        es.append(float(T.error(g, (rr,) * 3, F, U, core, ws)[0]))
    torch.cuda.synchronize()
    print(f"{s:2d} {k.label():32s} rc={res.rc} iters={res.info['iters']} resid={[f'{x:.1e}' for x in res.info['resid']]} "
          f"E(10,20,30)={[f'{e:.2e}' for e in es]} {1e3 * (time.time() - t):.0f} ms", flush=True)
