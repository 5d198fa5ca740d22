"""Kernel timeline of one apply (first CTA start / last CTA end per kernel family),
with a library built with -DCUTFEM_TIMELINE:
  python tools/build_variant.py tl -DCUTFEM_TIMELINE
  CUTFEM_LIB=build/variants/libcutfem_tl.so python tools/timeline.py [CFG]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import cutgen
import paper_2404_07911_b200 as cf

P = cutgen.config(sys.argv[1] if len(sys.argv) > 1 else "C2")
op = cf.CutFEM(P)
L = op._L
L.cutfem_debug_timeline.argtypes = [ctypes.c_int, ctypes.c_void_p]
u = torch.from_numpy(P.seeded_u(0)).cuda()
v = torch.empty_like(u)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
names = {0: "k_cutp", 1: "k_tile2", 2: "k_uncw"}
ALONE = os.environ.get("ALONE")  # "1": the cut-cell kernel alone (cutfem_apply_kernel 1)
for rep in range(4):
    flush.zero_()
    torch.cuda.synchronize()
    assert L.cutfem_debug_timeline(1, None) == 0
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    if ALONE:
        op.apply_kernel(int(ALONE), u, v)
    else:
        op.apply(u, v)
    b.record()
    torch.cuda.synchronize()
    out = (ctypes.c_ulonglong * (16 + 3 * 8192))()
    L.cutfem_debug_timeline(0, ctypes.addressof(out))
    t0 = min(out[2 * k] for k in names if out[2 * k] != 2 ** 64 - 1)
    row = {names[k]: (round((out[2 * k] - t0) / 1e3, 1), round((out[2 * k + 1] - t0) / 1e3, 1)) for k in names
           if out[2 * k] != 2 ** 64 - 1}
    print(f"apply {a.elapsed_time(b) * 1e3:.1f} us  (start, end) us: {row}")
    raw = np.ctypeslib.as_array(out)[16:].reshape(3, 8192).astype(np.float64)
    ok = raw[0] > 0
    if ok.any() and os.environ.get("WARPS"):
        end, beg, sm = (raw[0][ok] - t0) / 1e3, (raw[1][ok] - t0) / 1e3, raw[2][ok].astype(int)
        dur = end - beg
        np.save(os.environ["WARPS"] + f"_{rep}.npy", np.stack([np.nonzero(ok)[0], beg, end, sm]))
        smend = np.array([end[sm == k].max() for k in np.unique(sm)])
        smsum = np.array([dur[sm == k].sum() for k in np.unique(sm)])
        print("  warp start pct 0/50/100:", np.round(np.percentile(beg, [0, 50, 100]), 1).tolist(),
              " duration pct 0/10/50/90/99/100:", np.round(np.percentile(dur, [0, 10, 50, 90, 99, 100]), 1).tolist())
        print("  per-SM last end pct 0/50/90/100:", np.round(np.percentile(smend, [0, 50, 90, 100]), 1).tolist(),
              " per-SM summed warp time pct 0/50/90/100:", np.round(np.percentile(smsum, [0, 50, 90, 100]), 1).tolist())
        slow = np.argsort(-end)[:12]
        print("  slowest warps (gw, sm, start, end):", [(int(np.nonzero(ok)[0][i]), int(sm[i]), round(beg[i], 1),
                                                        round(end[i], 1)) for i in slow])
    we = np.array([out[16 + i] for i in range(8192)], dtype=np.float64)
    we = (we[we > 0] - t0) / 1e3
    if we.size:
        print("  k_cutp warp end times (us) pct 0/10/25/50/75/90/99/100:",
              np.round(np.percentile(we, [0, 10, 25, 50, 75, 90, 99, 100]), 1).tolist(), "n", we.size)
