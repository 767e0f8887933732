"""Streaming CPQR (cpqr.cu) on matrices that do not fit on chip: time per pivot step against the
algorithmic HBM traffic of a rank-1 trailing update (one read + one write of the active part of
the matrix per step; the axpy's re-read hits L2).
python tools/time_streaming.py [n] [k] [m]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2105_07076_b200 as idk  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 16
g = torch.Generator(device="cuda")
g.manual_seed(3)
m = int(sys.argv[3]) if len(sys.argv) > 3 else n
a = torch.randn((n, m), generator=g, device="cuda", dtype=torch.float64).t()  # m x n, column-major
ctx = idk.context(0)
print("plan", ctx.cpqr_plan(m, n, k))
for reps in range(3):
    ctx.set_profiling(True)
    idk.optim_id(a, k)
    st = ctx.stage_times()
    cp = st["cpqr"]
    # active part at step s: (m - s) rows x (n - s - 1) columns, read once and written once
    alg = sum(16.0 * (m - s) * (n - s - 1) for s in range(k))
    print(f"m={m} n={n} k={k}: cpqr {cp:.2f} ms = {cp / k * 1e3:.1f} us/step; algorithmic {alg / 1e9:.2f} GB "
          f"-> {alg / 1e9 / (cp / 1e3):.0f} GB/s; stages {st}")
