"""Per-contraction times of one bf16 backward at C2 (B=1, H=12), averaged over REPS calls:
python scripts/bwd_profile.py [reps]  (MBX_BWD_CUBLAS=name,... routes contractions to cuBLAS)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2602_12271_b200 as pk  # noqa: E402
from paper_2602_12271_b200 import ops, _lib  # noqa: E402
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
s = pk.VideoShape(3, 30, 52)
plan = pk.make_tile_plan(s, pk.aligned_config(s, ("f", "h")), (1, 30, 52))
low = pk.lower_square(plan)
dev = torch.device("cuda", 0)
q, k, v, do = (torch.randn(1, 12, 4680, 128, device=dev).to(torch.bfloat16) for _ in range(4))
for _ in range(3):
    ops.backward(q, k, v, do, low, 1)
torch.cuda.synchronize()
lib = _lib.load()
tot = {}
for _ in range(reps):
    lib.mbx_profile_enable(1)
    ops.backward(q, k, v, do, low, 1)
    torch.cuda.synchronize()
    lib.mbx_profile_enable(0)
    for nm, st, ms in _lib.profile_collect_ex():
        tot[nm] = tot.get(nm, 0) + ms / reps
for nm, ms in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{nm:28s} {ms*1000:8.1f} us")
print("sum", round(sum(tot.values()) * 1000, 1))
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    ops.backward(q, k, v, do, low, 1)
b.record()
torch.cuda.synchronize()
print("backward ms/call (10 calls, unprofiled)", round(a.elapsed_time(b) / 10, 4))
