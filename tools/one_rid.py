import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2105_07076_b200 as idk
a = torch.randn(1000, 784, dtype=torch.float64, device="cuda").t()
for _ in range(2):
    idk.optim_rid(a, 190, 0.2, 7)
torch.cuda.synchronize()
