"""Measured dense TF32 tensor-core peak on this B200 (the conv roofline's
denominator): cuBLAS TF32 GEMM 8192^3 (torch.matmul, allow_tf32), best of 10
back-to-back (burst) and sustained for ~3 s, CUDA events.
Usage: measure_tf32_peak.py [json_out]"""
import json
import sys
import time

import torch

torch.backends.cuda.matmul.allow_tf32 = True
n = 8192
a = torch.randn(n, n, device="cuda")
b = torch.randn(n, n, device="cuda")
for _ in range(3):
    a @ b
torch.cuda.synchronize()
flops = 2.0 * n ** 3
best = 0.0
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    a @ b
    e1.record()
    torch.cuda.synchronize()
    best = max(best, flops / (e0.elapsed_time(e1) * 1e-3) / 1e12)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
iters = 0
t0 = time.time()
e0.record()
while time.time() - t0 < 3.0:
    for _ in range(10):
        a @ b
    iters += 10
    torch.cuda.synchronize()
e1.record()
torch.cuda.synchronize()
sustained = iters * flops / (e0.elapsed_time(e1) * 1e-3) / 1e12
res = {"tf32_tflops": round(best, 1), "tf32_tflops_sustained": round(sustained, 1),
       "how": "cuBLAS TF32 GEMM 8192^3 via torch.matmul(allow_tf32): best of 10 (burst) and "
              "back to back for ~3 s (sustained), CUDA events",
       "gpu": torch.cuda.get_device_name()}
print(json.dumps(res))
if len(sys.argv) > 1:
    json.dump(res, open(sys.argv[1], "w"), indent=1)
