"""Dev tool: bench-style C2 refits with nvidia-smi sampled every 50 ms, to
correlate slow stages with SM clock / power / throttle reasons.
usage: FSTK_DEBUG_TIMING=1 python tools/refit_clocks.py [runs] [config] > gpurun_out/refit_clocks.log"""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1907_05884_b200 as F
from bench import workload
from paper_1907_05884_b200.dist import refine_distributed

FIELDS = ("timestamp,clocks.sm,clocks.mem,power.draw,temperature.gpu,memory.used,"
          "clocks_event_reasons.active")
log = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out",
                   f"smi_refit_{os.getpid()}.csv")
smi = subprocess.Popen(["nvidia-smi", f"--query-gpu={FIELDS}", "--format=csv,noheader",
                        "-lms", "50"], stdout=open(log, "w"), stderr=subprocess.DEVNULL)
CFG = sys.argv[2] if len(sys.argv) > 2 else "C2"
model, pts, vals, c = workload(CFG, 0, 0)
R = int(np.prod(model.ranks))
t_origin = time.time()


def mark(tag):
    print(f"  [{time.time() - t_origin:8.3f}] {tag}", flush=True)


for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    mark(f"run {i} begin")
    s = F.RefitSession(model, pts, vals, seed=0, sample_rows=c["m_factor"] * R)
    mark("begin done")
    g = torch.empty(R * R, dtype=torch.float64, device="cuda")
    rhs = torch.empty(R, dtype=torch.float64, device="cuda")
    s.normal_equations(g, rhs)
    torch.cuda.synchronize()
    mark("gram done")
    x = refine_distributed(s, g, rhs)
    torch.cuda.synchronize()
    mark("refine done")
    s.finish(x)
    t4 = time.perf_counter()
    info = s.info_dict()
    tm = info["timings"]
    print(f"run {i}: total {t4 - t0:.3f} | prepare {tm['prepare_s']:.3f} sketch {tm['sketch_s']:.3f} "
          f"gram {tm['gram_s']:.3f} solve {tm['solve_s']:.3f} steps {info['refine_steps']} "
          f"slices {info['gram_slices']} free {torch.cuda.mem_get_info()[0] / 1e9:.1f} GB",
          flush=True)
    s.close()
    del g
smi.terminate()
print("origin", t_origin)
