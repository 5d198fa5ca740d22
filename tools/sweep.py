"""Degree sweep (C3) and large configs: apply time, DoF/s, roofline fraction, parity spot check.
usage: python tools/sweep.py [C3:1,C3:2,...,C4,C5]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import cutgen
import paper_2404_07911_b200 as cf
from paper_2404_07911_b200 import costmodel

specs = (sys.argv[1] if len(sys.argv) > 1 else ",".join(f"C3:{p}" for p in range(1, 9))).split(",")
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for spec in specs:
    name, _, deg = spec.partition(":")
    t0 = time.time()
    P = cutgen.config(name, degree=int(deg) if deg else None)
    tg = time.time() - t0
    op = cf.CutFEM(P)
    st = op.stats()
    u = torch.from_numpy(P.seeded_u(0)).cuda()
    v = torch.empty_like(u)
    for _ in range(3):
        op.apply(u, v)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
    for a, b in ev:
        flush.zero_()
        a.record()
        op.apply(u, v)
        b.record()
    torch.cuda.synchronize()
    ms = float(np.median([a.elapsed_time(b) for a, b in ev]))
    kms = {}
    for which, kn in ((0, "structured"), (1, "unstructured")):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(5)]
        for a, b in evs:
            flush.zero_()
            a.record()
            op.apply_kernel(which, u, v)
            b.record()
        torch.cuda.synchronize()
        kms[kn] = float(np.median([a.elapsed_time(b) for a, b in evs]))
    w = costmodel.apply_work(st, costmodel.face_classes(P))
    troof = max(w["F_total"] / (costmodel.fp64_peak_tflops() * 1e12), w["B_total"] / 6539.2e9)
    print(json.dumps({"config": P.name, "degree": P.degree, "n_dofs": P.n_dofs, "n_cut": P.n_cut,
                      "gen_s": round(tg, 1), "ms": ms, "gdofs": P.n_dofs / ms / 1e6,
                      "frac": troof / (ms * 1e-3), "flop_per_dof": w["F_total"] / P.n_dofs,
                      "kernel_ms": kms}), flush=True)
    del op, u, v
    torch.cuda.empty_cache()
