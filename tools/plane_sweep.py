"""SURVEY §8(f) f1 / PAPER §5.2 "Plane benchmark": operator-apply
throughput against the ratio of cut cells to physical cells, controlled by the
position of a (slightly tilted) plane  n.x < offset  in a box of (L+2) x NY x NY
cubic cells, NY chosen so that every case has ~230k physical cells (the GPU equally
busy).  The plane sits in the middle of layer L, so 1/(L+1) of the physical cells
are cut (L = 0, 1, 9, 99), plus the plane outside the box (ratio 0).
The bounds of the paper's envelope are added: the whole box through the
structured path (no cut cells) and through the unstructured path (every cell
"cut" with its tensor rule).
usage: python tools/plane_sweep.py [degrees, default 1,3]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import cutgen
import paper_2404_07911_b200 as cf
from paper_2404_07911_b200 import costmodel

degrees = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,3").split(",")]
CELLS = 230400                      # physical cells per case


def box(L):
    ny = int(round(np.sqrt(CELLS / (L + 1))))
    h = 1.0 / ny
    nrm = np.array([1.0, 0.3 / ny, 0.15 / ny])  # tilt: ~0.45 cells of x-shift across the box
    return [L + 2, ny, ny], [0.0, 0.0, 0.0], [(L + 2) * h, 1.0, 1.0], h, nrm / np.linalg.norm(nrm)


flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")


def timed(op, u, v, K=10):
    for _ in range(3):
        op.apply(u, v)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for a, b in ev:
        flush.zero_()
        a.record()
        op.apply(u, v)
        b.record()
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ev]))


def run(name, P):
    op = cf.CutFEM(P)
    st = op.stats()
    u = torch.from_numpy(P.seeded_u(0)).cuda()
    v = torch.empty_like(u)
    ms = timed(op, u, v)
    w = costmodel.apply_work(st, costmodel.face_classes(P))
    troof = max(w["F_total"] / (costmodel.fp64_peak_tflops() * 1e12), w["B_total"] / 6539.2e9)
    print(json.dumps({"case": name, "degree": P.degree, "n_dofs": P.n_dofs, "n_active": P.n_active,
                      "n_cut": P.n_cut, "cut_ratio": P.n_cut / max(P.n_active, 1), "ms": ms,
                      "gdofs": P.n_dofs / ms / 1e6, "frac": troof / (ms * 1e-3)}), flush=True)
    del op, u, v
    torch.cuda.empty_cache()


for p in degrees:
    for L in (0, 1, 9, 99):
        nc, lo, up, h, nrm = box(L)
        off = float(nrm @ np.array([(L + 0.5) * h, 0.5, 0.5]))
        run(f"plane L={L}", cutgen.generate({"type": "plane", "normal": list(nrm), "offset": off}, nc, lo, up, p))
    nc, lo, up, h, nrm = box(99)
    far = {"type": "plane", "normal": list(nrm), "offset": float(nrm @ np.array([1e3, 0.5, 0.5]))}
    run("plane outside (ratio 0, all structured)", cutgen.generate(far, nc, lo, up, p))
    run("all cells through the unstructured path (tensor rules, P:850)",
        cutgen.generate(far, nc, lo, up, p, force_cut_cells=True, force_cut_faces=True))
