"""Read-only HBM bandwidth of this B200 (torch.sum over 8 GiB of fp64, CUDA
events, best of 10) next to the copy figure of MEASURED_PEAKS.json: the level-1
sweeps read 12 GB and write 0.24 GB per apply."""
import json

import torch

n = 1 << 30  # 8 GiB of doubles
a = torch.rand(n, dtype=torch.float64, device="cuda")
for _ in range(3):
    s = a.sum()
torch.cuda.synchronize()
best = 1e30
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s = a.sum()
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
print(json.dumps({"what": "torch.sum fp64 read-only", "bytes": n * 8, "ms": best, "read_gbs": n * 8 / (best * 1e-3) / 1e9}))
