"""Measured compute peaks that MEASURED_PEAKS.json does not carry (tools only):
cuBLAS TF32 8192^3 burst (best of 10) and sustained (back to back for 4 s),
the denominator of the tcgen05 3xTF32 GEMM roofline.  Prints one JSON line."""

import json
import time

import torch

n = 8192
a = torch.rand(n, n, device="cuda")
b = torch.rand(n, n, device="cuda")
torch.backends.cuda.matmul.allow_tf32 = True
torch.backends.cuda.matmul.fp32_precision = "tf32"
for _ in range(3):
    torch.matmul(a, b)
torch.cuda.synchronize()
best = 1e30
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch.matmul(a, b)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
flops = 2 * n ** 3
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.time()
iters = 0
e0.record()
while time.time() - t0 < 4.0:
    for _ in range(10):
        torch.matmul(a, b)
    iters += 10
    torch.cuda.synchronize()
e1.record()
torch.cuda.synchronize()
sust = e0.elapsed_time(e1) / iters
torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cuda.matmul.fp32_precision = "ieee"
torch.matmul(a, b)
torch.cuda.synchronize()
e0.record()
for _ in range(3):
    torch.matmul(a, b)
e1.record()
torch.cuda.synchronize()
sgemm = e0.elapsed_time(e1) / 3
print(json.dumps({"tf32_tflops": round(flops / best / 1e9, 1), "tf32_tflops_sustained": round(flops / sust / 1e9, 1),
                  "fp32_sgemm_tflops": round(flops / sgemm / 1e9, 1), "n": n,
                  "how": "torch.matmul fp32 inputs with TF32 allowed, 8192^3: best of 10 (burst) and back to back "
                         "for 4 s (sustained); cuBLAS SGEMM (TF32 off) for reference",
                  "gpu": torch.cuda.get_device_name()}))
