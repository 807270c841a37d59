import sys, torch
sys.path.insert(0, ".")
import paper_2602_12271_b200 as pk
from paper_2602_12271_b200 import ops
dev = torch.device("cuda", 0)
shape = pk.VideoShape(21, 30, 52)
q = torch.empty(1, 1, shape.n, 128, device=dev, dtype=torch.bfloat16)
for cfg in pk.enumerate_aligned_configs(shape):
    low = pk.lower_square(cfg)
    for T in (1, 2):
        print(cfg.g1, cfg.g2, cfg.b1, cfg.b2, "T", T, "s1", low.s1, "s2", low.s2, ops.selected_path(q, q, q, low, T))
