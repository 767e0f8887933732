"""Stage times of optim_rid vs optim_id (acceptance criterion 7 shape: 784 x 1000, k = 190)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2105_07076_b200 as idk  # noqa: E402

m, n, k = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (784, 1000, 190)))
a = torch.randn(n, m, dtype=torch.float64, device="cuda").t()
ctx = idk.context(0)
ctx.set_profiling(True)
for name, fn in [("optim_id", lambda: idk.optim_id(a, k)), ("optim_rid", lambda: idk.optim_rid(a, k, 0.2, 7))]:
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    print(name, f"{(time.perf_counter() - t0) / 10 * 1e3:.3f} ms/call", {kk: round(v, 4) for kk, v in ctx.stage_times().items()})
print("plan id", ctx.cpqr_plan(m, n, k), "\nplan rid", ctx.cpqr_plan(m, int(k * 1.2), k))
