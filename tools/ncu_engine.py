"""Summarise one `ncu --set full` capture of k_engine2 (taken in bench.py's
timed window) into profiles/engine_ncu.json, the file bench.py's roofline
`traffic` and latency block read, plus a markdown table beside it.

usage: python tools/ncu_engine.py REPORT.ncu-rep MOVES_PER_LAUNCH OUT_DIR "how it was captured"
"""
import csv
import io
import json
import os
import subprocess
import sys

rep, moves, out_dir, how = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
data = [r for r in rows[2:] if any("k_engine2" in c for c in r)]
if not data:
    raise SystemExit("no k_engine2 launch in the report")
r = data[0]
ix = {h: i for i, h in enumerate(hdr)}


def val(name):
    v = r[ix[name]].replace(",", "")
    u = units[ix[name]]
    x = float(v)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1e-3, "us": 1e-6,
             "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "nsecond": 1e-9, "s": 1, "second": 1}
    return x * scale.get(u, 1.0), u


want = {
    "duration_s": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "warp_latency_per_inst": "smsp__average_warp_latency_per_inst_issued.ratio",
}
got, table = {}, []
for k, m in want.items():
    if m in ix:
        x, u = val(m)
        got[k] = x
        table.append((m, r[ix[m]], u))
dram = got.get("dram_read", 0.0) + got.get("dram_write", 0.0)
res = {
    "source": f"{os.path.relpath(out_dir)}/engine_ncu.md: {how}",
    "moves_per_launch": moves,
    "duration_ms": 1e3 * got["duration_s"],
    "dram_bytes_per_launch": dram,
    "dram_bytes_per_move": dram / moves,
    "moves_per_s_under_ncu": moves / got["duration_s"],
}
for k in ("l2_hit_pct", "issue_active_pct", "fp64_pipe_pct", "warps_active_pct",
          "warp_latency_per_inst"):
    if k in got:
        res[k] = got[k]
os.makedirs(out_dir, exist_ok=True)
with open(os.path.join(out_dir, "engine_ncu.md"), "w") as f:
    f.write(f"k_engine2, {how}\n\n| metric | value | unit |\n|---|---|---|\n")
    for m, v, u in table:
        f.write(f"| {m} | {v} | {u} |\n")
    f.write(f"\nDRAM bytes per move: {dram / moves:.1f}\n")
print(json.dumps(res, indent=1))
