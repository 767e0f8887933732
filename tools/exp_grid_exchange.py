"""A/B of the grid-exchange layout knobs of the resident CPQR (cfg4 by default):
record stride (IDK_REC_STRIDE), copies of the published column
(IDK_COL_COPIES), poll back-off (IDK_POLL_SLEEP).  One process, variants
interleaved over several rounds; prints the median CPQR stage time per variant.
python tools/exp_grid_exchange.py [cfg4] [rounds]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2105_07076_b200 as idk  # noqa: E402
from paper_2105_07076_b200.configs import CONFIGS, make_torch  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 6
cfg = CONFIGS[name]
a = make_torch(name, seed=20260601)
ctx = idk.context(0)
ctx.set_profiling(True)
variants = [dict(IDK_REC_STRIDE="4", IDK_COL_COPIES="1"), dict(IDK_COL_COPIES="2"), dict(IDK_COL_COPIES="3"),
            dict(IDK_COL_COPIES="4"), dict(IDK_COL_COPIES="6"), dict(IDK_REC_STRIDE="8", IDK_COL_COPIES="4"),
            dict(IDK_REC_STRIDE="16", IDK_COL_COPIES="4"), dict(IDK_REC_STRIDE="16", IDK_COL_COPIES="3")]
if len(sys.argv) > 3:
    variants = [dict(x.split("=") for x in v.split(",") if x) for v in sys.argv[3:]]
keys = ["IDK_REC_STRIDE", "IDK_COL_COPIES", "IDK_POLL_SLEEP"]
ref = idk.id_auto(a, cfg.k, idk.RANDOMIZED, seed=1, p=cfg.p)
times = {i: [] for i in range(len(variants))}
for r in range(rounds):
    for i, v in enumerate(variants):
        for kk in keys:
            os.environ.pop(kk, None)
        os.environ.update(v)
        for _ in range(3):
            res = idk.id_auto(a, cfg.k, idk.RANDOMIZED, seed=1, p=cfg.p)
            times[i].append(ctx.stage_times()["cpqr"])
        assert torch.equal(res.cols, ref.cols) and torch.equal(res.z, ref.z)
for i, v in enumerate(variants):
    t = np.array(times[i])
    print(f"{str(v):80s} cpqr median {np.median(t):.4f} ms  ({1e3 * np.median(t) / cfg.k:.2f} us/step)  min {t.min():.4f}")
