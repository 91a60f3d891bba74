"""Summarise one `ncu --set full` capture of k_energy (the full-system
energy pass at 1M) into OUT_DIR/energy_ncu.md and a JSON line (stdout) that
bench.py's full_system_energy block reads as profiles/energy_ncu.json.
usage: python tools/ncu_energy.py REPORT.ncu-rep OUT_DIR"""
import csv
import io
import json
import os
import subprocess
import sys

rep, out_dir = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                     check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
data = [r for r in rows[2:] if any("k_energy" in c for c in r)]
r = data[0]
want = {"duration_us": "gpu__time_duration.sum", "dram_read": "dram__bytes_read.sum",
        "dram_write": "dram__bytes_write.sum",
        "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l2_hit_pct": "lts__t_sector_hit_rate.pct", "registers": "launch__registers_per_thread"}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "us": 1,
         "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3, "ns": 1e-3}
got, table = {}, []
for k, m in want.items():
    if m in hdr:
        i = hdr.index(m)
        v = float(r[i].replace(",", ""))
        got[k] = v * scale.get(units[i], 1.0)
        table.append((m, r[i], units[i]))
os.makedirs(out_dir, exist_ok=True)
with open(os.path.join(out_dir, "energy_ncu.md"), "w") as f:
    f.write("k_energy at 1M (random start, rho 0.67), ncu --set full --clock-control none\n\n"
            "| metric | value | unit |\n|---|---|---|\n")
    for m, v, u in table:
        f.write(f"| {m} | {v} | {u} |\n")
res = {"source": f"{os.path.relpath(out_dir)}/energy_ncu.md",
       "duration_us": got.get("duration_us"),
       "dram_bytes": got.get("dram_read", 0) + got.get("dram_write", 0),
       "issue_active_pct": got.get("issue_active_pct"), "fp64_pipe_pct": got.get("fp64_pipe_pct"),
       "warps_active_pct": got.get("warps_active_pct"), "l2_hit_pct": got.get("l2_hit_pct")}
print(json.dumps(res))
