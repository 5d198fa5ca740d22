"""Aggregate ncu source-page warp-stall samples per CUDA source line.
usage: python tools/ncu_lines.py report.ncu-rep kernel_regex [top]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
rows, h, fname = [], None, ""
for row in r:
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        h = row
        continue
    if h is None or not row[0]:
        continue
    si = 4
    try:
        s = int(row[si])
    except Exception:
        continue
    cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    st = sorted(((int(row[i] or 0) if row[i] not in ("-", "") else 0, h[i][6:]) for i in cols), reverse=True)[:3]
    ie = row[7]
    rows.append((s, f"{fname}:{row[0]}", row[1].strip()[:80], st, ie))
tot = sum(x[0] for x in rows) or 1
rows.sort(reverse=True)
print("total samples", tot)
for s, l, src, st, ie in rows[:top]:
    print(f"{s:7d} {100*s/tot:5.1f}% {l:>16}: {src:80s} inst={ie} {[(b, a) for a, b in st if a]}")
