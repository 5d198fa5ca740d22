"""Executed FP64 work (ncu: 2 dfma + dadd + dmul, thread level) per kernel against
the algorithmic FLOPs of costmodel.apply_work, per config.
Input: the output of, per config,
  python tools/apply_once.py CFG DEG 1        (prints the stats dict)
  ncu --metrics smsp__sass_thread_inst_executed_op_{dfma,dadd,dmul}_pred_on.sum,gpu__time_duration.sum --csv ...
usage: python tools/flops_check.py FLOPS.csv"""
import ast
import collections
import csv
import io
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_07911_b200 import costmodel  # noqa: E402

lines = open(sys.argv[1]).read().splitlines()
blocks, cur = [], None
for ln in lines:
    if ln.startswith("{"):
        cur = {"stats": ast.literal_eval(ln), "rows": []}
        blocks.append(cur)
    elif ln.startswith('"') and cur is not None and not ln.startswith('"ID"'):
        cur["rows"].append(next(csv.reader(io.StringIO(ln))))
print(f"{'config':>10} {'kernel':>16} {'time us':>9} {'exec GFLOP':>11} {'alg GFLOP':>10} {'exec/alg':>9} {'exec TF/s':>10}")
for b in blocks:
    st = b["stats"]
    w = costmodel.apply_work(st, costmodel.face_classes(P))
    k = collections.defaultdict(lambda: collections.defaultdict(float))
    for r in b["rows"]:
        name = r[4].split("(")[0].replace("void ", "")
        k[name][r[12]] += float(r[14].replace(",", ""))  # launches of one kernel summed
    cfg = f"p={st['degree']} {st['n_dofs'] / 1e6:.1f}M"
    for name, m in k.items():
        ex = 2 * m.get("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", 0) + \
            m.get("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", 0) + \
            m.get("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", 0)
        t = m.get("gpu__time_duration.sum", 0) * 1e-9
        fam = "F_cut" if ("cutp" in name or "k_cut<" in name or "k_cut1" in name) else "F_uncut"
        alg = w[fam]
        print(f"{cfg:>10} {name:>16} {t * 1e6:9.1f} {ex / 1e9:11.3f} {alg / 1e9:10.3f} {ex / alg:9.2f} {ex / t / 1e12 if t else 0:10.2f}")
