"""One warm cfg2 ID (profiling target): python tools/one_cfg2.py"""
import sys
import torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2105_07076_b200 as idk  # noqa: E402
from paper_2105_07076_b200.configs import make_torch  # noqa: E402
a = make_torch("cfg2", seed=1)
for _ in range(2):
    idk.id_auto(a, 100, idk.RANDOMIZED, seed=1, p=10)
torch.cuda.synchronize()
