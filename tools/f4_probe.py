"""Stage times and eigensolver report of the bench step for the f4 workloads (spectral density
alpha = 0.1 / 100, p-Slater) against the headline Matern kernel at 1024^3, ranks 40."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1711_06874_b200 import tucker as T  # noqa: E402
from tucker_inputs import GridSpec, KernelSpec  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    T.load()
    g, rr = GridSpec.cube(n, 1.0), (40, 40, 40)
    F = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
    ws = T.workspace(g, rr)
    out = {}
    for name, k in (("matern1.5", KernelSpec.matern(1.5, 0.2)), ("spectral0.1", KernelSpec.spectral(0.1, 0.4)),
                    ("spectral100", KernelSpec.spectral(100.0, 0.4))):
        def step():
            T.fill_prepare(g, k, rr, F, ws)
            res = T.hosvd_prepared(g, rr, F, ws)
            return res, T.error(g, rr, F, res.U, res.core, ws)
        for _ in range(2):
            res, e = step()
        torch.cuda.synchronize()
        T.profile_read()
        T.profile_enable(True)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            res, e = step()
        b.record()
        torch.cuda.synchronize()
        T.profile_enable(False)
        prof = T.profile_read()
        out[name] = {"ms": a.elapsed_time(b) / 3, "stages": {s: v[0] / 3 for s, v in prof.items() if v[1]},
                     "info": res.info, "E": float(e[0])}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
