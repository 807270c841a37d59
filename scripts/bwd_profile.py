import sys, torch
sys.path.insert(0, ".")
import paper_2602_12271_b200 as pk
from paper_2602_12271_b200 import ops, _lib
s = pk.VideoShape(3, 30, 52)
plan = pk.make_tile_plan(s, pk.aligned_config(s, ("f", "h")), (1, 30, 52))
low = pk.lower_square(plan)
dev = torch.device("cuda", 0)
q, k, v, do = (torch.randn(1, 12, 4680, 128, device=dev).to(torch.bfloat16) for _ in range(4))
for _ in range(3):
    ops.backward(q, k, v, do, low, 1)
torch.cuda.synchronize()
lib = _lib.load()
lib.mbx_profile_enable(1)
ops.backward(q, k, v, do, low, 1)
torch.cuda.synchronize()
lib.mbx_profile_enable(0)
recs = _lib.profile_collect_ex()
tot = {}
for nm, st, ms in recs:
    tot[nm] = tot.get(nm, 0) + ms
for nm, ms in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{nm:28s} {ms*1000:8.1f} us")
print("sum", sum(tot.values()) * 1000)
