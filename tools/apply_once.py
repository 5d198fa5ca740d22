"""One warm-up apply + N timed-free applies of a config (for ncu captures).
usage: python tools/apply_once.py [CFG] [DEGREE] [N]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import cutgen
import paper_2404_07911_b200 as cf

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
deg = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "-" else None
n = int(sys.argv[3]) if len(sys.argv) > 3 else 2
P = cutgen.config(cfg, degree=deg)
op = cf.CutFEM(P)
u = torch.from_numpy(P.seeded_u(0)).cuda()
v = torch.empty_like(u)
for _ in range(n):
    op.apply(u, v)
torch.cuda.synchronize()
print(op.stats())
