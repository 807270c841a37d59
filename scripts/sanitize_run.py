"""Small forwards that launch every kernel family once (for compute-sanitizer runs):
    compute-sanitizer --tool memcheck|racecheck|synccheck python scripts/sanitize_run.py
tcgen05 kernels: tc_row_pair, tc_row_stage, tc_row_flash, tc_column_stage (modes 0, 1, 2),
tc_column_wide, tc_alpha_r_stage (+ export mode); SIMT forward / apply; backward."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2602_12271_b200 as pk  # noqa: E402
from paper_2602_12271_b200 import _lib, ops  # noqa: E402

dev = torch.device("cuda", 0)
torch.manual_seed(0)


def run(frames, h, w, nb, H=2, T=1, q_frames=None, factors=False, dtype=torch.bfloat16, pair=-1, note=""):
    shape = pk.VideoShape(frames, h, w)
    plan = pk.make_tile_plan(shape, pk.aligned_config(shape, ("f", "h")), nb)
    low = pk.lower_square(plan) if q_frames is None else pk.lower_chunked(plan, q_frames)
    q = torch.randn(1, H, low.n_q, 128, device=dev, dtype=dtype)
    k = torch.randn(1, H, shape.n, 128, device=dev, dtype=dtype)
    v = torch.randn(1, H, shape.n, 128, device=dev, dtype=dtype)
    prev = _lib.set_option("MBX_PAIR", pair)
    try:
        r = ops.forward(q, k, v, low, T, return_factors=factors)
    finally:
        _lib.set_option("MBX_PAIR", prev)
    torch.cuda.synchronize()
    print("ok", note, flush=True)
    return r


run(3, 6, 52, (1, 6, 52), pair=1, note="pair (h,w) small")
run(3, 6, 52, (1, 6, 52), pair=0, note="classic row stage")
run(2, 6, 52, (2, 6, 52), note="pair G_q=1 + wide column stage (s1 = 12 > ... )")
run(3, 6, 52, (1, 6, 52), T=2, note="T=2 fused hand-off (mode 2)")
run(9, 6, 52, (1, 6, 52), T=2, note="T=2 stats + alpha stage (multi-chunk)")
run(3, 6, 52, (1, 6, 52), factors=True, note="factor export (stats + alpha export)")
run(3, 4, 80, (1, 4, 80), note="flash row stage (s2 = 80)")
run(3, 4, 80, (1, 4, 80), T=2, note="flash row stage T=2")
run(6, 6, 52, (1, 6, 52), q_frames=3, note="chunked KV")
run(3, 6, 52, (3, 6, 52), note="(3h,w): s1 = 18")
run(3, 12, 52, (3, 12, 52), note="wide column stage (s1 = 36)")
run(2, 4, 8, (1, 4, 8), dtype=torch.float32, T=2, factors=True, note="SIMT fp32 + factors")
# backward (fp32 SIMT chain)
shape = pk.VideoShape(2, 4, 8)
plan = pk.make_tile_plan(shape, pk.aligned_config(shape, ("f", "h")), (1, 4, 8))
low = pk.lower_square(plan)
q, k, v, do = (torch.randn(1, 1, shape.n, 32, device=dev) for _ in range(4))
ops.backward(q, k, v, do, low, 2)
torch.cuda.synchronize()
print("ok backward", flush=True)
print("all ok")
