"""The CG energy functional along the C5 solve (BASELINE configs[4]: 50 unpreconditioned CG
iterations on f = 1): CG minimises J(x) = 1/2 x.Ax - b.x over growing Krylov spaces, so
J(x_k) must fall monotonically even where ||r_k|| grows (ill-conditioned A, DESIGN A18).
Each x_k is recomputed by a fresh k-iteration solve from 0 (the library's CG is
deterministic), J evaluated with the library's apply.
usage: python tools/cg_energy.py [CFG] [K_MAX] [STEP]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import cutgen  # noqa: E402
import paper_2404_07911_b200 as cf  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
kmax = int(sys.argv[2]) if len(sys.argv) > 2 else 50
step = int(sys.argv[3]) if len(sys.argv) > 3 else 5
P = cutgen.config(cfg)
op = cf.CutFEM(P)
b = op.rhs_const(1.0)
rows = []
for k in range(0, kmax + 1, step):
    x, hist = op.cg(b, iters=k)
    Ax = op.apply(x)
    J = 0.5 * float(torch.dot(x, Ax)) - float(torch.dot(b, x))
    rows.append({"iters": k, "J": J, "res": float(hist[-1]), "rel_res": float(hist[-1] / hist[0])})
mono = all(rows[i + 1]["J"] <= rows[i]["J"] for i in range(len(rows) - 1))
print(json.dumps({"config": cfg, "n_dofs": P.n_dofs, "energy_monotone": mono, "rows": rows}))
