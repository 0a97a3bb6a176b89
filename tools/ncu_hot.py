"""Dev tool: stall-sample hot spots of one kernel in an ncu report (source page).
usage: python tools/ncu_hot.py report.ncu-rep kernel-regex [min-samples]"""
import collections
import csv
import io
import subprocess
import sys

rep, pat = sys.argv[1], sys.argv[2]
thr = int(sys.argv[3]) if len(sys.argv) > 3 else 400
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{pat}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
head = rows[1]
ia, isamp, iex = head.index("Source"), head.index("# Samples"), head.index("Instructions Executed")
stall = [(i, h) for i, h in enumerate(head) if h.startswith("stall_") and "Not Issued" not in h]
data = [r for r in rows[2:] if len(r) > isamp and r[isamp].isdigit()]
tot = sum(int(r[isamp]) for r in data)
agg = collections.Counter()
for r in data:
    for i, h in stall:
        if r[i].isdigit():
            agg[h] += int(r[i])
print("total samples", tot, "instructions", len(data))
print("stalls:", ", ".join(f"{h[6:]}={100 * v / tot:.1f}%" for h, v in agg.most_common(8)))
for n, r in enumerate(data):
    if int(r[isamp]) >= thr:
        top = sorted(((int(r[i]), h[6:]) for i, h in stall if r[i].isdigit()), reverse=True)[:2]
        print(f"{n:5d} {int(r[isamp]):6d} {100 * int(r[isamp]) / tot:4.1f}% x{r[iex]:>9s} "
              f"{r[ia].strip()[:70]:70s} {top}")
