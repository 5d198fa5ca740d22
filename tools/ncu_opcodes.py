"""Histogram of executed SASS opcodes (warp-level) for one kernel of an ncu report."""
import csv
import subprocess
import sys
from collections import Counter

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = None
cnt = Counter()
samp = Counter()
for row in r:
    if row and row[0] == "Address":
        h = row
        continue
    if h is None or len(row) < len(h):
        continue
    src = row[1].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    try:
        cnt[op] += int(row[h.index("Instructions Executed")])
        samp[op] += int(row[h.index("Warp Stall Sampling (All Samples)")])
    except ValueError:
        pass
tot = sum(cnt.values())
ts = sum(samp.values()) or 1
print(f"total warp instructions {tot}")
for op, c in cnt.most_common(25):
    print(f"{op:10s} {c:12d} {100*c/tot:5.1f}%  stall-samples {100*samp[op]/ts:5.1f}%")
