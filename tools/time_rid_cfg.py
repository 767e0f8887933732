"""optim_rid (the reference's column-sampling RID) at the BASELINE shapes with
frac = p/k: python tools/time_rid_cfg.py cfg2|cfg4|cfg5"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2105_07076_b200 as idk  # noqa: E402
from paper_2105_07076_b200.configs import CONFIGS, make_torch  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = CONFIGS[name]
a = make_torch(name, seed=3)
ctx = idk.context(0)
ctx.set_profiling(True)
frac = cfg.p / cfg.k
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = idk.id_auto(a, cfg.k, idk.SAMPLED, seed=9, oversampling_fraction=frac)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
print(name, f"optim_rid (frac {frac:.4f}): {dt * 1e3:.2f} ms", {k: round(v, 3) for k, v in ctx.stage_times().items()},
      "plan", ctx.cpqr_plan(min(cfg.m, cfg.n), cfg.k + int(frac * cfg.k), cfg.k)["kind"])
