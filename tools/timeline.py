"""Device timeline of a few steps (torch.profiler / CUPTI: every kernel of the process, all streams):
busy time (union of kernel intervals), idle gaps on the device, and the longest gaps with the kernels
around them.

    python tools/timeline.py step [n] [r]     fill_prepare + hosvd_prepared + error (the bench step)
    python tools/timeline.py cfg4             config 4 (512^3, 16 Matérn settings, ranks 30)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1711_06874_b200 import tucker as T  # noqa: E402
from tucker_inputs import GridSpec, KernelSpec, config4  # noqa: E402


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "step"
    T.load()
    if what == "cfg4":
        w = config4()
        g, rr = w.grid, w.ranks
        kernels = w.kernels
    else:
        n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
        r = int(sys.argv[3]) if len(sys.argv) > 3 else 40
        g, rr = GridSpec.cube(n, 1.0), (r, r, r)
        kernels = [KernelSpec.matern(1.5, 0.2)] * 3
    F = torch.empty(tuple(g.n), dtype=torch.float64, device="cuda")
    ws = T.workspace(g, rr)

    def one(k):
        T.fill_prepare(g, k, rr, F, ws)
        res = T.hosvd_prepared(g, rr, F, ws, sync=os.environ.get("TIMELINE_ASYNC") is None)
        return T.error(g, rr, F, res.U, res.core, ws)

    for k in kernels[:2]:
        one(k)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for k in kernels:
            one(k)
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    iv = sorted((e.time_range.start, e.time_range.end, e.name) for e in ev)
    if not iv:
        print(json.dumps({"error": "no CUDA events"}))
        return
    t0, t1 = iv[0][0], max(e for _, e, _ in iv)
    busy, cur_s, cur_e, gaps = 0.0, iv[0][0], iv[0][1], []
    last_name = iv[0][2]
    for s, e, nm in iv[1:]:
        if s > cur_e:
            busy += cur_e - cur_s
            gaps.append((s - cur_e, last_name, nm))
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
        if e >= cur_e:
            last_name = nm
    busy += cur_e - cur_s
    gaps.sort(reverse=True)
    per = {}
    for s, e, nm in iv:
        per[nm] = per.get(nm, 0.0) + (e - s)
    out = {"what": what, "items": len(kernels), "span_ms": (t1 - t0) / 1e3, "busy_ms": busy / 1e3,
           "idle_ms": (t1 - t0 - busy) / 1e3, "per_item_ms": (t1 - t0) / 1e3 / len(kernels),
           "gaps_top": [(round(gp / 1e3, 4), a[:60], b[:60]) for gp, a, b in gaps[:15]],
           "gap_count_over_20us": sum(1 for gp, _, _ in gaps if gp > 20),
           "kernels_ms": {k[:70]: round(v / 1e3, 3) for k, v in sorted(per.items(), key=lambda x: -x[1])[:20]}}
    dump = os.environ.get("TIMELINE_DUMP")
    if dump:  # every kernel of the run: (start us, end us, stream, name)
        rows = sorted((e.time_range.start - t0, e.time_range.end - t0, getattr(e, "device_resource_id", -1), e.name[:48])
                      for e in ev)
        with open(dump, "w") as fh:
            json.dump(rows, fh)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
