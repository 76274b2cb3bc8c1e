"""cuBLAS FP64 GEMM throughput on this GPU (torch.matmul on float64 -> cuBLAS DGEMM): the practical
FP64 tensor ceiling next to tools/fp64_peak.cu's register-only DMMA loop.  usage: python tools/dgemm_peak.py"""
import json

import torch

res = {}
for n in (4096, 8192, 16384):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        torch.matmul(a, b)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    res[n] = round(2.0 * n ** 3 / (ms * 1e-3) / 1e12, 2)
print(json.dumps({"cublas_dgemm_tflops": res}))
