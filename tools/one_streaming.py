"""One streaming CPQR launch (profiling target): python tools/one_streaming.py [n] [k]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2105_07076_b200 as idk  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 16
g = torch.Generator(device="cuda")
g.manual_seed(3)
a = torch.randn((n, n), generator=g, device="cuda", dtype=torch.float64).t()
for _ in range(2):
    idk.optim_id(a, k)
torch.cuda.synchronize()
