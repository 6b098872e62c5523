"""Stage breakdown of the config-4 batch (512^3, 16 Matérn settings, ranks 30): per-setting time,
the library's stage timer, and the same batch through the asynchronous HOSVD (info = NULL)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1711_06874_b200 import tucker as T  # noqa: E402
from tucker_inputs import config4  # noqa: E402


def main():
    T.load()
    w = config4()
    g, r = w.grid, w.ranks
    F = torch.empty(tuple(g.n), dtype=torch.float64, device="cuda")
    ws = T.workspace(g, r)
    out = {}
    for sync in (True, False):
        def one(k):
            T.fill_prepare(g, k, r, F, ws)
            res = T.hosvd_prepared(g, r, F, ws, sync=sync)
            return T.error(g, r, F, res.U, res.core, ws)
        one(w.kernels[0])
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for k in w.kernels:
            one(k)
        b.record()
        torch.cuda.synchronize()
        T.profile_read()
        T.profile_enable(True)
        for k in w.kernels:
            one(k)
        torch.cuda.synchronize()
        T.profile_enable(False)
        p = T.profile_read()
        out["sync" if sync else "async"] = {"ms_per_setting": a.elapsed_time(b) / 16,
                                            "stages_per_setting": {s: v[0] / 16 for s, v in p.items() if v[1]}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
