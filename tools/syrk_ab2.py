"""Dev tool: A/B/C of Gram variants (env per variant is read once, so each
variant runs in its own subprocess, interleaved, cooled); reports the summed
device time of the Gram's kernels (CUPTI), not wall time (which includes the
scratch allocations of the standalone Gram entry point).
usage: python tools/syrk_ab2.py reps 'NAME:ENV=V,ENV=V' ..."""
import os
import statistics
import subprocess
import sys
import time

reps = int(sys.argv[1])
variants = sys.argv[2:]
code = r'''
import ctypes as C, os, sys, time, torch
sys.path.insert(0, os.getcwd())
import paper_1907_05884_b200 as F
from paper_1907_05884_b200._lib import Err, check, lib
rows, n = 262144, 32768
torch.manual_seed(0)
a = torch.randn(n, rows, dtype=torch.float64, device="cuda")
g = torch.zeros(n * n, dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
def run():
    err = Err(); torch.cuda.synchronize(); t0 = time.perf_counter()
    check(lib().fstk_gpu_gram_device(a.data_ptr(), rows, rows, n, g.data_ptr(), 4, 0, s, C.byref(err)), err)
    torch.cuda.synchronize(); return time.perf_counter() - t0
run(); time.sleep(2)
from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    wall = run()
kern = sum(e.device_time_total for e in prof.events() if e.device_type.name == "CUDA") / 1e6
print(wall, kern)
'''
res = {v: [] for v in variants}
for _ in range(reps):
    for v in variants:
        name, _, envs = v.partition(":")
        env = dict(os.environ)
        for kv in filter(None, envs.split(",")):
            k, _, val = kv.partition("=")
            env[k] = val
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        try:
            w, k = out.stdout.strip().splitlines()[-1].split()
            res[v].append(float(k))
        except Exception:
            print(v, "failed:", out.stderr[-500:])
        time.sleep(2)
for v, ts in res.items():
    if ts:
        print(f"{v.partition(':')[0]:12s} median {statistics.median(ts):.3f} s  ({' '.join(f'{t:.3f}' for t in ts)})")
