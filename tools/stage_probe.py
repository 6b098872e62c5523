"""Times the bench step's stages (profile counters) and the whole step (CUDA events) at 1024^3,
ranks 40: used for A/B runs of environment knobs (e.g. TUCKER_I8_UNIT_KB, the int8 Gram's unit length)."""
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
    g, k, rr = GridSpec.cube(n, 1.0), KernelSpec.matern(1.5, 0.2), (40, 40, 40)
    F = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
    ws = T.workspace(g, rr)

    def step():
        T.fill_prepare(g, k, rr, F, ws)
        res = T.hosvd_prepared(g, rr, F, ws)
        return T.error(g, rr, F, res.U, res.core, ws)

    for _ in range(3):
        e = step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(5):
        a.record()
        e = step()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    T.profile_read()
    T.profile_enable(True)
    for _ in range(2):
        step()
    torch.cuda.synchronize()
    T.profile_enable(False)
    p = T.profile_read()
    print(json.dumps({"unit_kb": os.environ.get("TUCKER_I8_UNIT_KB", "auto"), "step_ms": sorted(ts),
                      "E": float(e[0]), "stages": {s: v[0] / max(1, v[1]) * (v[1] / 2) for s, v in p.items() if v[1]}}))


if __name__ == "__main__":
    main()
