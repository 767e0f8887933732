"""Stage times (CUDA events on the launching stream) of one BASELINE config:
python tools/time_cpqr.py cfg2 [reps] [cpqr_mode]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2105_07076_b200 as idk  # noqa: E402
from paper_2105_07076_b200.configs import CONFIGS, make_torch  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
mode = int(sys.argv[3]) if len(sys.argv) > 3 else 0
cfg = CONFIGS[name]
a = make_torch(name, seed=20260601)
ctx = idk.context(0)
ctx.set_cpqr_mode(mode)
ctx.set_profiling(True)
rows = []
for it in range(reps + 3):
    if cfg.randomized:
        idk.id_auto(a, cfg.k, idk.RANDOMIZED, seed=1, p=cfg.p)
    else:
        idk.id_auto(a, cfg.k, idk.DETERMINISTIC)
    if it >= 3:
        rows.append([ctx.stage_times()[kk] for kk in ("prep", "sketch", "cpqr", "solve", "gather")])
r = np.array(rows)
print(name, "mode", mode, "median ms:", dict(zip(("prep", "sketch", "cpqr", "solve", "gather"), np.round(np.median(r, 0), 4))),
      "total", round(float(np.median(r.sum(1))), 4))
