"""Dev tool: per-launch durations of the SYRK kernel in one CRT Gram (normal
run, CUPTI via torch.profiler) against the tasks each launch holds, to read
tail losses; samples SM clocks while it runs.
usage: python tools/syrk_launches.py [slices] [rows] [n]"""
import ctypes as C

import numpy as np
import os
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1907_05884_b200 as F
from paper_1907_05884_b200._lib import Err, check, lib

ns = int(sys.argv[1]) if len(sys.argv) > 1 else 4
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 262144
n = int(sys.argv[3]) if len(sys.argv) > 3 else 32768
a = torch.randn(n, rows, dtype=torch.float64, device="cuda")
g = torch.zeros(n * n, dtype=torch.float64, device="cuda")
stream = torch.cuda.current_stream().cuda_stream


def run():
    err = Err()
    check(lib().fstk_gpu_gram_device(a.data_ptr(), rows, rows, n, g.data_ptr(), ns, 0, stream,
                                     C.byref(err)), err)


run()
torch.cuda.synchronize()
clk = []
stop = False


def sample():
    while not stop:
        o = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active",
                            "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout.strip()
        clk.append(o)
        time.sleep(0.02)


th = threading.Thread(target=sample)
th.start()
from torch.profiler import ProfilerActivity, profile

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    run()
    torch.cuda.synchronize()
stop = True
th.join()
ev = [e for e in prof.events() if e.device_type.name == "CUDA" and ("syrk" in e.name or "cutlass" in e.name)]
d = [e.device_time_total / 1e3 for e in ev]
print(f"{F.gram_engine()}: {len(d)} launches, total {sum(d):.1f} ms")
grp = 9 if F.gram_engine() == "cublaslt" else 1  # one launch per modulus vs all moduli
blocks = [sum(d[i:i + grp]) for i in range(0, len(d), grp)]
per = len(blocks) // max(1, rows // 32768)
print("  per column block (first segment):", " ".join(f"{b:.2f}" for b in blocks[:per]))
busy = [c for c in clk if not c.startswith("1965")]
mhz = [float(c.split(",")[0]) for c in busy]
pw = [float(c.split(",")[1]) for c in busy]
print(f"busy samples {len(busy)}: median SM clock {np.median(mhz) if mhz else 0:.0f} MHz, "
      f"median power {np.median(pw) if pw else 0:.0f} W, reasons {sorted(set(c.split(',')[2].strip() for c in busy))}")
