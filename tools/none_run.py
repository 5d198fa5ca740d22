import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, cutgen, paper_2404_07911_b200 as cf
P = cutgen.config("C2")
u = torch.from_numpy(P.seeded_u(0)).cuda(); v = torch.empty_like(u)
op = cf.CutFEM(P, term_mask=int(os.environ.get("MASK", "16")))
for _ in range(5):
    op.apply_kernel(0, u, v); op.apply_kernel(1, u, v)
torch.cuda.synchronize(); print("ok")
