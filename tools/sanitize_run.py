"""Small runs of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2105_07076_b200 as idk  # noqa: E402

rng = np.random.default_rng(1)
def dev(a):
    return torch.from_numpy(np.asfortranarray(a)).cuda()
a = dev(rng.standard_normal((110, 600)))
ctx = idk.context(0)
for mode in (0, 1, 2, 3):
    ctx.set_cpqr_mode(mode)
    idk.optim_id(a, 20)
    idk.sketch_rid(dev(rng.standard_normal((300, 800))), 30, 5, seed=3)
ctx.set_cpqr_mode(0)
idk.optim_rid(dev(rng.standard_normal((2000, 300))), 20, 0.5, 4)   # CholeskyQR3 path
idk.optim_rid(dev(rng.standard_normal((100, 300))), 40, 0.2, 4)     # direct path
b = torch.from_numpy(rng.standard_normal((20, 256, 64))).cuda()
idk.optim_id_batched(b, 16)
ctx.set_batched_exact(True)
idk.optim_id_batched(b, 16)
ctx.set_batched_exact(False)
idk.id_auto_batch([dev(rng.standard_normal((60, 90))) for _ in range(5)], 8, idk.RANDOMIZED, p=3, lanes=3)
# TMA sketch (both layouts, partial boxes), DMMA Z solves (k <= 128 and 128 < k <= 256), both gathers,
# the pipelined host entries
idk.sketch_rid(dev(rng.standard_normal((900, 150))), 20, 6, seed=5)            # dual: TMA with A transposed
idk.sketch_rid(dev(rng.standard_normal((170, 1100))), 150, 10, seed=6)         # k in (128, 256]
idk.optim_id(dev(rng.standard_normal((140, 333))), 100)
idk.select_columns(dev(rng.standard_normal((64, 300))), torch.arange(0, 40, 3).cuda())
idk.select_columns(dev(rng.standard_normal((301, 77))), torch.arange(0, 40, 3).cuda(), rows_of_a=True)
idk.id_auto_many([np.asfortranarray(rng.standard_normal((60, 90))) for _ in range(5)], 8, idk.RANDOMIZED, p=3)
idk.optim_id_batched(rng.standard_normal((300, 256, 64)), 16)
torch.cuda.synchronize()
print("sanitize run ok")
