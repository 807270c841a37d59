"""Experiment: end-to-end host-buffer forward at C2 -- transfer floors vs the pipelined host API."""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2602_12271_b200 as pk  # noqa: E402

wl = bench.workload("sf", 1)
dev = torch.device("cuda", 0)
q, k, v = (torch.randn(wl["B"], wl["H"], wl["nq"], wl["d"]).to(torch.bfloat16).pin_memory() for _ in range(3))
out_h = torch.empty_like(q).pin_memory()
qd, kd, vd = (torch.empty(x.shape, dtype=x.dtype, device=dev) for x in (q, k, v))
od = torch.empty_like(qd)


def t(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def h2d():
    qd.copy_(q, non_blocking=True); kd.copy_(k, non_blocking=True); vd.copy_(v, non_blocking=True)


def d2h():
    out_h.copy_(od, non_blocking=True)


def seq():
    h2d()
    o = pk.monarch_attention(qd, kd, vd, wl["plan"])
    out_h.copy_(o, non_blocking=True)


print("h2d 43MB", round(t(h2d), 4))
print("d2h 14MB", round(t(d2h), 4))
print("sequential e2e", round(t(seq), 4))
for c in (1, 2, 3, 4):
    print("host api chunks", c, round(t(lambda: pk.monarch_attention_host(q, k, v, wl["plan"], out=out_h, chunks=c)), 4))
t0 = time.perf_counter()
for _ in range(20):
    pk.monarch_attention_host(q, k, v, wl["plan"], out=out_h, chunks=6)
torch.cuda.synchronize()
print("host api chunks 6 wall ms/call", round((time.perf_counter() - t0) / 20 * 1e3, 4))
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        h2d()
    with torch.cuda.stream(s2):
        d2h()
    cur.wait_stream(s1)
    cur.wait_stream(s2)


print("h2d || d2h concurrent", round(t(both), 4))
