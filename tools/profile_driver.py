"""One small driver for the ncu captures under profiles/ (run under ncu on the GPU box):

    python tools/profile_driver.py step [n] [r]        fill_prepare + hosvd_prepared + error (the bench step)
    python tools/profile_driver.py fill NU [n]          the general-nu K_nu fill (Chebyshev table route)
    python tools/profile_driver.py als [n] [r]          HOSVD + one Tucker-ALS sweep
    python tools/profile_driver.py accurate [n] [r]     the SVD-accurate HOSVD (f2)
    python tools/profile_driver.py fused [n] [r]        fused (F never stored) HOSVD + error

Each does one warm-up call first (so `ncu --launch-skip` can skip it) unless WARM=0.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1711_06874_b200 import tucker as T  # noqa: E402
from tucker_inputs import GridSpec, KernelSpec  # noqa: E402


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "step"
    args = [float(a) for a in sys.argv[2:]]
    warm = os.environ.get("WARM", "1") != "0"
    T.load()
    if what == "fill":
        nu = args[0] if args else 1.3
        n = int(args[1]) if len(args) > 1 else 1024
        g, k = GridSpec.cube(n, 1.0), KernelSpec.matern(nu, 0.5)
        F = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
        for _ in range(2 if warm else 1):
            T.fill(g, k, F)
        torch.cuda.synchronize()
        return
    n = int(args[0]) if args else 1024
    r = int(args[1]) if len(args) > 1 else 40
    g, k, rr = GridSpec.cube(n, 1.0), KernelSpec.matern(1.5, 0.2), (r, r, r)
    if what == "fused":
        ws = T.workspace_fused(g, rr)
        for _ in range(2 if warm else 1):
            res = T.hosvd_fused(g, k, rr, ws)
            T.error_fused(g, k, rr, res.U, res.core, ws)
        torch.cuda.synchronize()
        return
    F, mx = T.fill_rowmax(g, k)
    ws = T.workspace(g, rr)
    for _ in range(2 if warm else 1):
        if what == "step":  # the bench step: fill + shared residues, prepared HOSVD, error
            T.fill_prepare(g, k, rr, F, ws)
            res = T.hosvd_prepared(g, rr, F, ws)
            T.error(g, rr, F, res.U, res.core, ws)
        elif what == "als":
            res = T.hosvd(g, rr, F, ws)
            T.als(g, rr, F, res.U, 1)
        elif what == "accurate":
            T.hosvd_accurate(g, rr, F)
        else:
            raise SystemExit(f"unknown: {what}")
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
