"""Run a few IDs of one BASELINE config (for ncu captures): python tools/prof_id.py cfg2 [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2105_07076_b200 as idk  # noqa: E402
from paper_2105_07076_b200.configs import CONFIGS, make_torch  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = CONFIGS[name]
a = make_torch(name, seed=20260601)
torch.cuda.synchronize()
for _ in range(reps):
    if name == "cfg3":
        idk.optim_id_batched(a, cfg.k)
    elif cfg.randomized:
        idk.id_auto(a, cfg.k, idk.RANDOMIZED, seed=1, p=cfg.p)
    else:
        idk.id_auto(a, cfg.k, idk.DETERMINISTIC)
torch.cuda.synchronize()
print("ok", name, idk.context(0).kernel_launches)
