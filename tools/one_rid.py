"""One optim_rid call on 16384^2, k=256, 5 % sample (profiling target)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2105_07076_b200 as idk
g = torch.Generator(device="cuda"); g.manual_seed(1)
a = torch.randn((16384, 16384), generator=g, device="cuda", dtype=torch.float64).t()
for _ in range(2):
    idk.optim_rid(a, 256, 0.05, 3)
torch.cuda.synchronize()
