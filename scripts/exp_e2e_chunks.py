"""e2e (host buffers) at C2 vs the number of (b,h) chunks of monarch_attention_host,
timed like bench.py's e2e (per-step CUDA events on the current stream, L2 flushed between)."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2602_12271_b200 as pk  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "sf"
wl = bench.workload(cfg, 1)
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
pin = [torch.randn(wl["B"], wl["H"], n, wl["d"]).to(torch.bfloat16).pin_memory() for n in (wl["nq"], wl["nk"], wl["nk"])]
out_h = torch.empty(wl["B"], wl["H"], wl["nq"], wl["dv"], dtype=torch.bfloat16).pin_memory()
flush_buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
stream = torch.cuda.current_stream(dev)
kvf = wl["fkv"] if wl["fq"] != wl["fkv"] else None
ref = None
for ch in (1, 2, 3, 4, 6, 12):
    def step():
        pk.monarch_attention_host(pin[0], pin[1], pin[2], wl["plan"], iterations=wl["T"], kv_frames=kvf, out=out_h,
                                  chunks=ch)
    ms = bench.time_steps(step, 20, 3, flush_buf.zero_, stream) / 20
    torch.cuda.synchronize()
    if ref is None:
        ref = out_h.clone()
    print(f"chunks {ch}: {ms:.4f} ms  equal={torch.equal(out_h, ref)}", flush=True)
