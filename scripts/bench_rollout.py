"""Self-Forcing rollout timing: 21 latent frames of 30x52 decoded in 7 chunks of 3
frames, every chunk attending to all cached frames (B=1, H=12, d=128, bf16), through
paper_2602_12271_b200.rollout (frame KV cache + chunked-KV operator), against the same
block-causal loop on dense cuDNN SDPA.  Device time per whole rollout (CUDA events,
L2 flushed before each rollout).  Prints one JSON line per plan.

    python scripts/bench_rollout.py [--steps 10] [--warmup 3]
"""
import argparse
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_12271_b200 import rollout  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    B, H, F, h, w, d, cf = 1, 12, 21, 30, 52, 128, 3
    hw = h * w
    g = torch.Generator(device="cpu").manual_seed(0)
    q, k, v = (torch.randn(B, H, F * hw, d, generator=g).to(dev, torch.bfloat16) for _ in range(3))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def timed(fn):
        for _ in range(a.warmup):
            fn()
        ts = []
        for i in range(a.steps):
            flush.fill_(i & 255)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        return ts[len(ts) // 2]

    def dense():
        from torch.nn.attention import SDPBackend, sdpa_kernel

        with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
            for c in range(F // cf):
                sl = slice(c * cf * hw, (c + 1) * cf * hw)
                torch.nn.functional.scaled_dot_product_attention(q[:, :, sl], k[:, :, :(c + 1) * cf * hw],
                                                                 v[:, :, :(c + 1) * cf * hw])

    dense_ms = timed(dense)
    for name, tile in (("(h,w)", (1, h, w)), ("(3h,w)", (3, h, w))):
        cache = rollout.FrameKVCache(B, H, F, h, w, d, device=dev)
        ro = rollout.Rollout(h, w, cache, tile)

        def run():
            cache.reset()
            for c in range(F // cf):
                sl = slice(c * cf * hw, (c + 1) * cf * hw)
                ro.step(q[:, :, sl], k[:, :, sl], v[:, :, sl])

        ms = timed(run)
        # the same rollout captured once as a CUDA graph (host descriptor setup and
        # launch overhead of the 7 steps leave the timed path)
        run()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            run()
        graph_ms = timed(graph.replay)
        print(json.dumps({"workload": f"Self-Forcing rollout, 21 frames 30x52 in 7 chunks of 3, B=1 H=12 d=128, "
                                      f"plan {name}, T=1, bf16", "unit": "ms/rollout", "ours_ms": round(ms, 4), "ours_cuda_graph_ms": round(graph_ms, 4),
                          "dense_cudnn_block_causal_ms": round(dense_ms, 4), "speedup": round(dense_ms / ms, 3), "speedup_graph": round(dense_ms / graph_ms, 3),
                          "includes": "K/V cache appends (copy) + 7 chunked-KV forwards", "l2": "flushed per rollout",
                          "steps": a.steps, "warmup": a.warmup}))


if __name__ == "__main__":
    main()
