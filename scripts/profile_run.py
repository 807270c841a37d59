"""Minimal driver for ncu: W warm-up + a few forwards of a bench config."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2602_12271_b200 import ops  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "sf"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 1
wl = bench.workload(cfg, iters)
dev = torch.device("cuda", 0)
dt = torch.bfloat16 if wl["dtype"] == "bf16" else torch.float32
q = torch.randn(wl["B"], wl["H"], wl["nq"], wl["d"], device=dev, dtype=dt)
k = torch.randn(wl["B"], wl["H"], wl["nk"], wl["d"], device=dev, dtype=dt)
v = torch.randn(wl["B"], wl["H"], wl["nk"], wl["dv"], device=dev, dtype=dt)
for _ in range(reps):
    ops.forward(q, k, v, wl["low"], iters)
torch.cuda.synchronize()
print("ok")
