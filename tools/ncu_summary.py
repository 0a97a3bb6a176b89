"""Dev tool: one-screen summary of an ncu report (per kernel launch).
usage: python tools/ncu_summary.py report.ncu-rep [name-regex] > profiles/xxx.txt"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active", "tensor inst %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
head, units = rows[0], rows[1]
for r in rows[2:]:
    d = dict(zip(head, r))
    u = dict(zip(head, units))
    name = d.get("Kernel Name", "")
    if pat and not pat.search(name):
        continue
    print(f"== {name[:110]}")
    for key, label in METRICS:
        if key in d and d[key] not in ("", "n/a"):
            print(f"   {label:20s} {d[key]} {u.get(key, '')}")
    stalls = {k: d[k] for k in head if k.startswith("smsp__average_warp_latency_issue_stalled") and
              k.endswith(".ratio") and d[k] not in ("", "n/a")}
    top = sorted(stalls.items(), key=lambda kv: -float(kv[1]))[:5]
    if top:
        print("   top stalls (cycles/issue): " + ", ".join(
            f"{k.split('stalled_')[1].split('.')[0]}={float(v):.2f}" for k, v in top))
