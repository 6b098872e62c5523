"""TTM and error stage times at ranks where they are HBM-bound (2 r3 flop per 8 B below the ridge):
1024^3, r = 10 and 20, the bench step's calls, library stage timer."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1711_06874_b200 import tucker as T  # noqa: E402
from tucker_inputs import GridSpec, KernelSpec  # noqa: E402


def main():
    T.load()
    n = 1024
    g, k = GridSpec.cube(n, 1.0), KernelSpec.matern(1.5, 0.2)
    F = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
    out = {}
    for r in (10, 20, 30, 40):
        rr = (r, r, r)
        ws = T.workspace(g, rr)

        def step():
            T.fill_prepare(g, k, rr, F, ws)
            res = T.hosvd_prepared(g, rr, F, ws, sync=False)
            return T.error(g, rr, F, res.U, res.core, ws)

        for _ in range(3):
            step()
        torch.cuda.synchronize()
        T.profile_read()
        T.profile_enable(True)
        for _ in range(5):
            step()
        torch.cuda.synchronize()
        T.profile_enable(False)
        prof = T.profile_read()
        out[r] = {s: v[0] / 5 for s, v in prof.items() if v[1]}
        del ws
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
