"""Per-kernel, per-term timing on a config (CUDA events, L2 flushed)."""
import json
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import cutgen
import paper_2404_07911_b200 as cf

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
deg = int(sys.argv[2]) if len(sys.argv) > 2 else None
P = cutgen.config(cfg, degree=deg)
u = torch.from_numpy(P.seeded_u(0)).cuda()
v = torch.empty_like(u)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
flush2 = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
MODE = os.environ.get("FLUSH", "write")


def do_flush():
    if MODE in ("write", "writeread"):
        flush.zero_()
    if MODE == "writeread":
        flush2.sum()


def t(fn, K=20):
    for _ in range(3):
        fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for a, b in ev:
        do_flush()
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ev])) * 1e3


res = {"cfg": cfg, "n_dofs": P.n_dofs, "flush": MODE, "lib": os.environ.get("CUTFEM_LIB", "default")}
ALL = ((15, "all"), (1, "cell"), (2, "sipg"), (4, "nitsche"), (8, "gp"), (0x10 | 0, "none"))
want = os.environ.get("MASKS")
for mask, name in ALL:
    if want and name not in want.split(","):
        continue
    m = mask if mask != 0x10 else 0x10
    try:
        op = cf.CutFEM(P, term_mask=m)
    except Exception as e:
        continue
    row = {"apply_us": t(lambda: op.apply(u, v))}
    for which, kn in ((0, "structured"), (1, "unstructured")):
        row[kn + "_us"] = t(lambda: op.apply_kernel(which, u, v))
    res[name] = row
    del op
print(json.dumps(res))
