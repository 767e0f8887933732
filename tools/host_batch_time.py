import os, sys, time
sys.path.insert(0, os.getcwd())
import torch, paper_2105_07076_b200 as idk
from paper_2105_07076_b200.configs import make_torch
mats = [make_torch("cfg2", seed=s) for s in range(8)]
for it in range(5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    idk.id_auto_batch(mats, 100, idk.RANDOMIZED, seeds=list(range(8)), p=10, lanes=8)
    torch.cuda.synchronize(); print(f"batch of 8: {(time.perf_counter()-t0)*1e3:.3f} ms wall", file=sys.stderr)
idk.context(0).set_profiling(True)
for it in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    idk.id_auto_batch(mats, 100, idk.RANDOMIZED, seeds=list(range(8)), p=10, lanes=8)
    torch.cuda.synchronize(); print(f"batch of 8 (profiling on): {(time.perf_counter()-t0)*1e3:.3f} ms wall", file=sys.stderr)
