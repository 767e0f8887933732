"""One warm cfg5 ID (profiling target): python tools/one_cfg5.py"""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2105_07076_b200 as idk  # noqa: E402
from paper_2105_07076_b200.configs import make_torch  # noqa: E402
a = make_torch("cfg5", seed=1)
for _ in range(2):
    idk.id_auto(a, 64, idk.RANDOMIZED, seed=1, p=8)
torch.cuda.synchronize()
