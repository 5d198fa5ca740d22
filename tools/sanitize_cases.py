"""Small applies through every kernel family, for compute-sanitizer (racecheck /
synccheck / memcheck): p = 1, 2 (k_cut1, k_cell), p = 3 (k_cutp<4>, k_tile2,
k_uncw<4>), p = 4..8 (k_cut, k_uncw), the H1 gather / scatter and a Jacobi-PCG step.
usage: python tools/sanitize_cases.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import cutgen  # noqa: E402
import paper_2404_07911_b200 as cf  # noqa: E402

for p, N in ((1, 6), (2, 6), (3, 8), (4, 5), (5, 5), (6, 4), (7, 5), (8, 4)):
    P = cutgen.generate(cutgen.SPHERE, N, -1.0, 1.0, p)
    op = cf.CutFEM(P)
    u = torch.from_numpy(P.seeded_u(1)).cuda()
    v = op.apply(u)
    torch.cuda.synchronize()
    print(f"p={p} N={N} n_cut={P.n_cut} n_uncut={P.n_active - P.n_cut} |v|={float(v.norm()):.6e}", flush=True)
P = cutgen.config("C1")
h1 = cf.CutFEMH1(P)
x = torch.ones(h1.n_dofs, dtype=torch.float64, device="cuda")
y = h1.apply(x)
op = cf.CutFEM(P)
b = op.rhs_const(1.0)
xs, hist = op.cg(b, iters=3, precond="jacobi")
torch.cuda.synchronize()
print("h1", float(y.norm()), "pcg", hist.tolist(), flush=True)
