"""Dev tool: per-rank sketch time of shard 0 of G at C2, row vs column layout
(what each rank of a G-GPU refit does before the exchange / Gram).
usage: python tools/shard_sketch_time.py [G ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1907_05884_b200 as F
from bench import workload

model, pts, vals, c = workload("C2", 0, 0)
R = int(np.prod(model.ranks))
S = c["m_factor"] * R
s = F.RefitSession(model, pts, vals, seed=0, sample_rows=S)  # warm-up
s.close()
for G in [int(a) for a in sys.argv[1:]] or [1, 2, 4, 8]:
    for layout in ("rows", "columns"):
        s = F.RefitSession(model, pts, vals, seed=0, sample_rows=S, shard=0, shards=G, layout=layout)
        t = s.info_dict()["timings"]
        print(f"G={G} {layout:7s} prepare {t['prepare_s']:.3f} sketch {t['sketch_s']:.3f} s", flush=True)
        s.close()
