"""Solver benchmark: time to a relative residual of
1e-8 for f = 1 with (a) Jacobi-PCG, (b) Chebyshev(block-Jacobi)-PCG on one level, (c)
p-multigrid PCG (levels p -> ... -> 1 by halving, Chebyshev smoothing with the cell-block
inner preconditioner).  Setup (level handles, probing, inversion, Lanczos) timed apart.
usage: python tools/mg_bench.py [C2] [maxit]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import cutgen
import paper_2404_07911_b200 as cf

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
maxit = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
P = cutgen.config(name)
pf = P.degree
degs = [pf]
while degs[0] > 1:
    degs.insert(0, max(1, degs[0] // 2))
kw = dict(sipg_gamma=10.0 * pf ** 2, nitsche_tau=10.0 * pf ** 2)
t0 = time.time()
probs = [cutgen.generate(P.level_set, P.n_cells, P.lower, [P.lower[i] + P.h * P.n_cells[i] for i in range(3)], p,
                         name=f"{name}p{p}", **kw) for p in degs]
tgen = time.time() - t0
ops = [cf.CutFEM(Q) for Q in probs]
b = ops[-1].rhs_const(1.0)
bn = float(b.norm())


def run(label, fn):
    torch.cuda.synchronize()
    t = time.time()
    x, h = fn()
    torch.cuda.synchronize()
    dt = time.time() - t
    r = float((b - ops[-1].apply(x)).norm()) / bn
    return {"solver": label, "iters": len(h) - 1, "s": dt, "ms_per_iter": 1e3 * dt / max(len(h) - 1, 1),
            "rel_res": h[-1] / bn, "true_rel_res": r}


out = {"config": name, "degree": pf, "levels": degs, "n_dofs": P.n_dofs, "gen_s": tgen, "runs": []}
ops[-1].cg(b, iters=1, precond="jacobi")  # probe the diagonal outside the timing
out["runs"].append(run("jacobi-pcg", lambda: ops[-1].cg(b, iters=maxit, tol=1e-8, precond="jacobi")))
out["runs"].append(run("cg", lambda: ops[-1].cg(b, iters=maxit, tol=1e-8)))
inners = os.environ.get("MG_INNER", "block,jacobi").split(",")
for label, lv, inner in (("chebyshev-block-pcg", ops[-1:], "block"), ("pmg-block-pcg", ops, "block"),
                         ("chebyshev-jacobi-pcg", ops[-1:], "jacobi"), ("pmg-jacobi-pcg", ops, "jacobi")):
    if inner not in inners:
        continue
    torch.cuda.synchronize()
    t = time.time()
    mg = cf.CutFEMMG(lv, inner=inner, smooth_degree=3, coarse_degree=16, eig_iters=20)
    torch.cuda.synchronize()
    ts = time.time() - t
    rec = run(label, lambda: mg.pcg(b, iters=maxit, tol=1e-8))
    rec["setup_s"] = ts
    rec["lambdas"] = mg.lambdas().tolist()
    out["runs"].append(rec)
    del mg
print(json.dumps(out))


def ev_ms(fn, reps=10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


if len(sys.argv) > 3 and sys.argv[3] == "grid":
    mg = cf.CutFEMMG(ops, inner="block", eig_iters=20)
    lam = mg.lambdas()
    r = torch.rand(P.n_dofs, dtype=torch.float64, device="cuda")
    z = torch.empty_like(r)
    parts = {"apply_fine_ms": ev_ms(lambda: ops[-1].apply(r, z)),
             "apply_coarse_ms": ev_ms(lambda: ops[0].apply(torch.zeros(ops[0].n_dofs, dtype=torch.float64,
                                                                       device="cuda"))),
             "block_step_fine_ms": ev_ms(lambda: mg.smooth(len(ops) - 1, r, z, 1, lam[-1], lam[-1] / 15)),
             "vcycle_ms": ev_ms(lambda: mg.vcycle(r, z))}
    grid = []
    for sd in (2, 3, 5):
        for cdg in (4, 8, 16):
            mg = cf.CutFEMMG(ops, inner="block", smooth_degree=sd, coarse_degree=cdg, eig_iters=20)
            rec = run(f"pmg-block sd={sd} cd={cdg}", lambda: mg.pcg(b, iters=maxit, tol=1e-8))
            grid.append(rec)
            del mg
    print(json.dumps({"parts": parts, "grid": grid}))
