"""Dev tool: sketch-stage time at C2 (RefitSession begin only), profiling off.
usage: python tools/sketch_time.py [runs]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1907_05884_b200 as F
from bench import workload

model, pts, vals, c = workload("C2", 0, 0)
R = int(np.prod(model.ranks))
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    s = F.RefitSession(model, pts, vals, seed=0, sample_rows=c["m_factor"] * R)
    t = s.info_dict()["timings"]
    print(f"prefetch={os.environ.get('FSTK_SKETCH_PREFETCH', '1')} prepare {t['prepare_s']:.3f} "
          f"sketch {t['sketch_s']:.3f} alloc {t['alloc_s']:.3f}", flush=True)
    s.close()
