"""Experiment: one forward over all heads vs head halves on two concurrent streams."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2602_12271_b200 import ops  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "sf"
wl = bench.workload(cfg, 1)
dev = torch.device("cuda", 0)
q, k, v = (torch.randn(wl["B"], wl["H"], wl["nq"] if i == 0 else wl["nk"], wl["d"], device=dev,
                       dtype=torch.bfloat16) for i in range(3))
out = torch.empty(q.shape, dtype=q.dtype, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
H = wl["H"]
streams = [torch.cuda.Stream() for _ in range(4)]


def run(nsplit):
    main = torch.cuda.current_stream()
    if nsplit == 1:
        ops.forward(q, k, v, wl["low"], 1, out=out)
        return
    hs = H // nsplit
    for i in range(nsplit):
        st = streams[i]
        st.wait_stream(main)
        with torch.cuda.stream(st):
            sl = slice(i * hs, (i + 1) * hs)
            ops.forward(q[:, sl], k[:, sl], v[:, sl], wl["low"], 1, out=out[:, sl])
    for i in range(nsplit):
        main.wait_stream(streams[i])


graphs = {}
for n in (1, 2, 3, 4):
    run(n)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        run(n)
    graphs[n] = gr
for n in (1, 2, 3, 4, 1):
    ts = []
    for it in range(25):
        flush.fill_(it & 255)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        graphs[n].replay()
        b.record()
        torch.cuda.synchronize()
        if it >= 5:
            ts.append(a.elapsed_time(b))
    ts.sort()
    print(f"{cfg} graph streams={n} median_ms={ts[len(ts) // 2]:.4f}", flush=True)
