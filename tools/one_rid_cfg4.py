import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2105_07076_b200 as idk
from paper_2105_07076_b200.configs import CONFIGS, make_torch
cfg = CONFIGS["cfg4"]
a = make_torch("cfg4", seed=3)
for _ in range(2):
    idk.id_auto(a, cfg.k, idk.SAMPLED, seed=9, oversampling_fraction=cfg.p / cfg.k)
torch.cuda.synchronize()
