"""Experiment: one forward over all (b,h) vs the same work split into head chunks
(row -> column per chunk), with L2 flushed before each timed step."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2602_12271_b200 import ops  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "sf"
wl = bench.workload(cfg, 1)
dev = torch.device("cuda", 0)
q = torch.randn(wl["B"], wl["H"], wl["nq"], wl["d"], device=dev, dtype=torch.bfloat16)
k = torch.randn(wl["B"], wl["H"], wl["nk"], wl["d"], device=dev, dtype=torch.bfloat16)
v = torch.randn(wl["B"], wl["H"], wl["nk"], wl["dv"], device=dev, dtype=torch.bfloat16)
out = torch.empty_like(q)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
H = wl["H"]
for nch in (1, 2, 3, 4, 6):
    hs = H // nch
    chunks = [(q[:, i * hs:(i + 1) * hs].contiguous(), k[:, i * hs:(i + 1) * hs].contiguous(),
               v[:, i * hs:(i + 1) * hs].contiguous(), out[:, i * hs:(i + 1) * hs].contiguous()) for i in range(nch)]
    print(ops.selected_path(*chunks[0][:3], wl["low"], 1))
    ts = []
    for it in range(25):
        flush.fill_(it & 255)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for qc, kc, vc, oc in chunks:
            ops.forward(qc, kc, vc, wl["low"], 1, out=oc)
        b.record()
        torch.cuda.synchronize()
        if it >= 5:
            ts.append(a.elapsed_time(b))
    ts.sort()
    print(f"{cfg} chunks={nch} median_ms={ts[len(ts) // 2]:.4f} min_ms={ts[0]:.4f}", flush=True)
