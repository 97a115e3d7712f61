#!/usr/bin/env python
"""Dense e4m3 GEMM peak with the protocol of MEASURED_PEAKS.json (BASELINE.md §2 leaves the fp8 peak to the builder):
torch._scaled_mm 8192^3 (cuBLASLt fp8, fp32 accumulate, bf16 out), best of 10 (burst) and back to back for 4 s
(sustained). Writes profiles/fp8_peak.json, which bench.py --dtype fp8 uses as the roofline denominator."""
import json
import os
import time

import torch

dev = torch.device("cuda", 0)
n = 8192
a = torch.randn((n, n), device=dev).to(torch.float8_e4m3fn)
b = torch.randn((n, n), device=dev).to(torch.float8_e4m3fn).t()  # column-major second operand, as cuBLASLt fp8 requires
one = torch.ones((), device=dev)


def mm():
    return torch._scaled_mm(a, b, scale_a=one, scale_b=one, out_dtype=torch.bfloat16)


for _ in range(5):
    mm()
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); mm(); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
flop = 2.0 * n ** 3
burst = flop / best / 1e9
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.time(); reps = 0
e0.record()
while time.time() - t0 < 4.0:
    for _ in range(20):
        mm()
    reps += 20
    torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize()
sustained = flop * reps / e0.elapsed_time(e1) / 1e9
out = {"fp8_tflops": round(burst, 1), "fp8_tflops_sustained": round(sustained, 1), "gpu_name": torch.cuda.get_device_name(0),
       "how": "torch._scaled_mm e4m3 8192^3 (2*N^3), bf16 out: best of 10 (burst) and back to back for 4 s (sustained)"}
print(json.dumps(out))
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.makedirs(os.path.join(root, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(root, "gpurun_out", "fp8_peak.json"), "w"), indent=1)
