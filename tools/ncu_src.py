"""Per-CUDA-line samples/instructions for one function of an ncu report.
usage: ncu_src.py report substring_of_function_name [top]"""
import csv, subprocess, sys
rep, fsub = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = None; fname = ""; fn = ""; rows = {}
for row in r:
    if not row: continue
    if row[0] == "File Path": fname = row[1].split("/")[-1]; continue
    if row[0] == "Function Name": fn = row[1]; continue
    if row[0] == "Line No": h = row; continue
    if h is None or not row[0] or fsub not in fn: continue
    try: ie = int(row[7]); s = int(row[4])
    except Exception: continue
    key = f"{fname}:{row[0]}"
    a = rows.setdefault(key, [0, 0, row[1].strip()[:90]])
    a[0] += s; a[1] += ie
tot = sum(v[1] for v in rows.values()) or 1; ts = sum(v[0] for v in rows.values()) or 1
print("instructions", tot, "samples", ts)
for k, (s, ie, src) in sorted(rows.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*s/ts:5.1f}% inst {100*ie/tot:5.1f}% {k:>24}: {src}")
