"""Summarise an ncu --set full report into JSON (per kernel: duration, DRAM bytes,
pipe / issue / occupancy metrics, top stall reasons).
usage: python tools/ncu_summary.py REPORT OUT.json"""
import csv
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
     "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
     "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
     "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
     "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum",
     "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct"]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, data = rows[0], rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
res = {}
for d in data:
    name = d[ix["Kernel Name"]].split("(")[0].replace("void ", "").strip()
    e = {m: f"{d[ix[m]]} {units[ix[m]]}".strip() for m in M if m in ix}
    st = {h.split("smsp__pcsamp_warps_issue_stalled_")[1]: float(d[ix[h]] or 0) for h in hdr
          if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")}
    e["top_stalls"] = dict(sorted(st.items(), key=lambda kv: -kv[1])[:6])
    res[name] = e
json.dump(res, open(out, "w"), indent=1)
print(json.dumps({k: v["gpu__time_duration.sum"] for k, v in res.items()}))
