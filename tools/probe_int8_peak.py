"""Measured dense INT8 tensor throughput on this GPU through torch._int_mm (cuBLASLt int8 x int8 ->
int32), burst (short loop) and sustained (~10 s loop), for the INT8 roofline denominator."""
import json
import sys
import time

import torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda").t().contiguous().t()
for _ in range(3):
    torch._int_mm(a, b)
torch.cuda.synchronize()
out = {}
for name, secs in (("burst", 0.3), ("sustained", 10.0)):
    # calibrate the loop length, then time it with events
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch._int_mm(a, b)
    e1.record()
    torch.cuda.synchronize()
    per = e0.elapsed_time(e1) * 1e-3
    it = max(3, int(secs / per))
    e0.record()
    for _ in range(it):
        torch._int_mm(a, b)
    e1.record()
    torch.cuda.synchronize()
    dt = e0.elapsed_time(e1) * 1e-3
    out[name + "_tops"] = 2.0 * n ** 3 * it / dt / 1e12
    out[name + "_iters"] = it
bf = torch.randn(n, n, dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    bf @ bf
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
it = 400
e0.record()
for _ in range(it):
    bf @ bf
e1.record()
torch.cuda.synchronize()
out["bf16_same_run_tflops"] = 2.0 * n ** 3 * it / (e0.elapsed_time(e1) * 1e-3) / 1e12
out["n"] = n
print(json.dumps(out))
