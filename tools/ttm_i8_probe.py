"""TTM stage of the bench step at 1024^3 under both TTM engines (TUCKER_TTM_AUTO: T1 on the INT8
tensor cores, R22; TUCKER_TTM_DMMA), ranks from argv (default 10 40): library stage timer, and a
launch list under ncu when run with PROBE_ONCE=1 (one step per engine)."""
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
    once = os.environ.get("PROBE_ONCE") == "1"
    ranks = [int(a) for a in sys.argv[1:]] or [10, 40]
    g, k = GridSpec.cube(n, 1.0), KernelSpec.matern(1.5, 0.2)
    F = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
    out = {}
    for r in ranks:
        rr = (r, r, r)
        ws = T.workspace(g, rr)
        for eng in (T.TTM_AUTO, T.TTM_DMMA) + ((T.TTM_INT8_ERROR,) if os.environ.get("PROBE_ERR_I8") else ()):
            T.set_ttm_engine(eng)

            def step():
                T.fill_prepare(g, k, rr, F, ws)
                res = T.hosvd_prepared(g, rr, F, ws, sync=False)
                return res, T.error(g, rr, F, res.U, res.core, ws)

            for _ in range(1 if once else 3):
                res, e = step()
            torch.cuda.synchronize()
            if once:
                continue
            T.profile_read()
            T.profile_enable(True)
            for _ in range(5):
                step()
            torch.cuda.synchronize()
            T.profile_enable(False)
            prof = T.profile_read()
            out[f"r{r}_{ {T.TTM_AUTO: 'int8', T.TTM_DMMA: 'dmma'}.get(eng, 'int8_err')}"] = {
                "stages_ms": {s: v[0] / 5 for s, v in prof.items() if v[1]}, "E": float(e[0])}
        T.set_ttm_engine(T.TTM_AUTO)
        del ws
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
