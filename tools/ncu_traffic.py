"""Write profiles/ncu_traffic.json from an ncu --set full report: DRAM bytes
(read + write) per launch of each kernel, keyed by config and the bench's
kernel name.  usage: python tools/ncu_traffic.py REPORT CFG NAME=regex [...]"""
import csv
import json
import os
import re
import subprocess
import sys

rep, cfg = sys.argv[1], sys.argv[2]
pairs = [a.split("=", 1) for a in sys.argv[3:]]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units, data = rows[0], rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
db = json.load(open(path)) if os.path.exists(path) else {}
for name, rx in pairs:
    vals = []
    for d in data:
        if re.search(rx, d[ix["Kernel Name"]]):
            b = 0.0
            for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                b += float(d[ix[m]]) * scale.get(units[ix[m]], 1)
            vals.append(b)
    if vals:
        db.setdefault(cfg, {})[name] = sum(vals) / len(vals)
        print(name, sum(vals) / len(vals))
json.dump(db, open(path, "w"), indent=1, sort_keys=True)
