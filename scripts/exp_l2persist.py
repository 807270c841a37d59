"""Experiment: effect of the device's persisting-L2 carve-out (cudaLimitPersistingL2CacheSize)
on the forward, whose workspace stores carry an evict_last policy."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2602_12271_b200 import ops  # noqa: E402

rt = ctypes.CDLL("libcudart.so.12")
cfg = sys.argv[1] if len(sys.argv) > 1 else "sf"
wl = bench.workload(cfg, 1)
dev = torch.device("cuda", 0)
q = torch.randn(wl["B"], wl["H"], wl["nq"], wl["d"], device=dev, dtype=torch.bfloat16)
k = torch.randn(wl["B"], wl["H"], wl["nk"], wl["d"], device=dev, dtype=torch.bfloat16)
v = torch.randn(wl["B"], wl["H"], wl["nk"], wl["dv"], device=dev, dtype=torch.bfloat16)
out = torch.empty_like(q)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for mb in (0, 32, 64, 96, 0):
    torch.cuda.synchronize()
    err = rt.cudaDeviceSetLimit(ctypes.c_int(0x06), ctypes.c_size_t(mb << 20))
    got = ctypes.c_size_t(0)
    rt.cudaDeviceGetLimit(ctypes.byref(got), ctypes.c_int(0x06))
    ts = []
    for it in range(30):
        flush.fill_(it & 255)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ops.forward(q, k, v, wl["low"], 1, out=out)
        b.record()
        torch.cuda.synchronize()
        if it >= 5:
            ts.append(a.elapsed_time(b))
    ts.sort()
    print(f"{cfg} persist_limit={mb}MB (err {err}, got {got.value >> 20} MB) median_ms={ts[len(ts) // 2]:.4f}", flush=True)
