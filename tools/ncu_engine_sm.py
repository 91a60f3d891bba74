"""Summarise one `ncu --set full` capture of k_engine_sm (the 148-chain sweep
launch) into OUT_DIR/engine_sm_ncu.md and a JSON line (stdout).
usage: python tools/ncu_engine_sm.py REPORT.ncu-rep OUT_DIR MOVES NOTE"""
import csv
import io
import json
import os
import subprocess
import sys

rep, out_dir, moves, note = sys.argv[1], sys.argv[2], float(sys.argv[3]), sys.argv[4]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                     check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
r = [x for x in rows[2:] if any("k_engine_sm" in c for c in x)][0]
want = {"duration_us": "gpu__time_duration.sum", "dram_read": "dram__bytes_read.sum",
        "dram_write": "dram__bytes_write.sum",
        "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l2_hit_pct": "lts__t_sector_hit_rate.pct", "registers": "launch__registers_per_thread",
        "grid": "launch__grid_size", "smem_per_block": "launch__shared_mem_per_block_dynamic"}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "us": 1,
         "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3, "ns": 1e-3, "second": 1e6}
got, table = {}, []
for k, m in want.items():
    if m in hdr:
        i = hdr.index(m)
        v = float(r[i].replace(",", ""))
        got[k] = v * scale.get(units[i], 1.0)
        table.append((m, r[i], units[i]))
os.makedirs(out_dir, exist_ok=True)
dram = got.get("dram_read", 0) + got.get("dram_write", 0)
with open(os.path.join(out_dir, "engine_sm_ncu.md"), "w") as f:
    f.write(f"k_engine_sm, {note}, ncu --set full --clock-control none\n\n"
            "| metric | value | unit |\n|---|---|---|\n")
    for m, v, u in table:
        f.write(f"| {m} | {v} | {u} |\n")
    f.write(f"\nDRAM bytes per move: {dram / moves:.1f} ({moves:.0f} moves in the launch)\n")
print(json.dumps({"source": f"{os.path.relpath(out_dir)}/engine_sm_ncu.md", "note": note,
                  "duration_us": got.get("duration_us"), "moves": moves,
                  "dram_bytes_per_move": dram / moves,
                  "issue_active_pct": got.get("issue_active_pct"),
                  "fp64_pipe_pct": got.get("fp64_pipe_pct"),
                  "warps_active_pct": got.get("warps_active_pct"), "l2_hit_pct": got.get("l2_hit_pct")}))
