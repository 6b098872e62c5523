"""Eigensolver iteration counts (synchronous HOSVD, info) over the BASELINE configs and the f4
workloads: the evidence for the asynchronous iteration budget (kMaxItersAsync in eig.cu)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1711_06874_b200 import tucker as T  # noqa: E402
from tucker_inputs import GridSpec, KernelSpec, config1, config2, config3, config4  # noqa: E402


def main():
    T.load()
    out = []
    cases = []
    for w in (config1(), config2(), config3(), config4()):
        for k in w.kernels:
            cases.append((w.name, w.grid, k, w.ranks))
    for k in (KernelSpec.spectral(0.1, 0.4), KernelSpec.spectral(100.0, 0.4), KernelSpec.slater(1.0, 0.1),
              KernelSpec.slater(1.0, 1.9), KernelSpec.matern(1.5, 0.2), KernelSpec.matern(0.5, 0.05),
              KernelSpec.matern(2.5, 1.0)):
        cases.append(("f4/1024", GridSpec.cube(1024, 1.0), k, (40, 40, 40)))
    for n in (129, 257):
        cases.append(("table2", GridSpec.cube(n, 5.0), KernelSpec.slater(1.0, 1.0), (10, 10, 10)))
    worst = 0
    for name, g, k, r in cases:
        F = T.fill(g, k)
        res = T.hosvd(g, r, F)
        it = res.info["iters"]
        worst = max(worst, max(it))
        out.append({"case": name, "n": list(g.n), "kernel": k.label(), "r": list(r), "iters": it,
                    "converged": res.info["converged"], "rc": res.rc})
        del F
        torch.cuda.empty_cache()
    print(json.dumps({"max_iters": worst, "cases": out}))


if __name__ == "__main__":
    main()
