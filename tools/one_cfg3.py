import sys, torch
sys.path.insert(0, '/root/repo')
import paper_2105_07076_b200 as idk
from paper_2105_07076_b200.configs import make_torch
a = make_torch("cfg3", seed=1)
for _ in range(2):
    idk.optim_id_batched(a, 16)
torch.cuda.synchronize()
