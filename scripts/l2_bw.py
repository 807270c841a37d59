"""Device copy bandwidth vs working-set size (L2-resident vs HBM) on one GPU."""
import json
import torch

dev = torch.device("cuda", 0)
res = {}
for mb in (4, 16, 32, 48, 64, 96, 128, 256, 1024):
    n = mb * 1024 * 1024 // 2
    x = torch.randn(n, device=dev, dtype=torch.bfloat16)
    y = torch.empty_like(x)
    for _ in range(5):
        y.copy_(x)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 50
    a.record()
    for _ in range(reps):
        y.copy_(x)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    res[mb] = round(2 * mb * 1.048576e6 / (ms * 1e-3) / 1e9, 1)
print(json.dumps({"copy_GBps_by_MB": res}))
