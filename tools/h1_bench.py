"""H1 (continuous Galerkin) operator throughput and the Jacobi-PCG solve (SURVEY
§8(f) f2, f4): CUDA events on the stream, L2 flushed before every apply.
usage: python tools/h1_bench.py [CFG|C3:p ...]   (one JSON line per config; NO_CG=1: apply only)"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import cutgen  # noqa: E402
import paper_2404_07911_b200 as cf  # noqa: E402


def timed(fn, K=20):
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    for _ in range(3):
        fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for a, b in ev:
        flush.zero_()
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ev]))


for cfg in (sys.argv[1:] or ["C2", "C5"]):
    name, _, deg = cfg.partition(":")  # "C3:p" = the degree sweep mesh of degree p
    P = cutgen.config(name, degree=int(deg) if deg else None)
    t0 = time.time()
    h1 = cf.CutFEMH1(P)
    t_setup = time.time() - t0
    u = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, h1.n_dofs)).cuda()
    v = torch.empty_like(u)
    ms = timed(lambda: h1.apply(u, v))
    dg = cf.CutFEM(P)
    ud = torch.from_numpy(P.seeded_u(0)).cuda()
    vd = torch.empty_like(ud)
    ms_dg = timed(lambda: dg.apply(ud, vd))
    out = {"config": cfg, "degree": P.degree, "h1_dofs": h1.n_dofs, "dg_dofs": P.n_dofs,
           "h1_apply_ms": ms, "h1_gdofs": h1.n_dofs / ms / 1e6, "dg_apply_ms": ms_dg,
           "dg_gdofs": P.n_dofs / ms_dg / 1e6, "h1_setup_s": round(t_setup, 2),
           "what": "H1 apply = gather + block kernels without SIPG + fixed-order scatter"}
    # PCG: iterations to ||r|| <= 1e-6 ||b|| (DG), plain vs Jacobi
    b = dg.rhs_const(1.0)
    for pc in (() if os.environ.get("NO_CG") else ("none", "jacobi")):
        torch.cuda.synchronize()
        t0 = time.time()
        x, hist = dg.cg(b, iters=3000, tol=1e-6, precond=pc)
        torch.cuda.synchronize()
        out[f"dg_cg_{pc}"] = {"iters": len(hist) - 1, "s": round(time.time() - t0, 3),
                              "rel_res": float(hist[-1] / float(b.norm()))}
    print(json.dumps(out), flush=True)
    del h1, dg
    torch.cuda.empty_cache()
