"""Measured FP64 peak of this B200 (cuBLAS DGEMM via torch.matmul, 8192^3,
2 N^3 flops, CUDA events, best of 10 after warm-up) -- the denominator for
the FP64 build kernels (K0 Cholesky / inverse tiles).  Writes one JSON line."""
import json
import sys

import torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(3):
    c = a @ b
torch.cuda.synchronize()
best = 1e30
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    c = a @ b
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
tf = 2 * n ** 3 / (best * 1e-3) / 1e12
print(json.dumps({"what": "cuBLAS DGEMM (torch.matmul fp64)", "n": n, "ms": best, "tflops_fp64": tf,
                  "device": torch.cuda.get_device_name()}))
