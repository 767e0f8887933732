"""Wall times (CUDA events around the call) of the entry points outside the headline path, on large inputs:
where is a secondary kernel far from its bound?  python tools/time_secondary.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2105_07076_b200 as idk  # noqa: E402


def timed(name, fn, reps=3, bytes_alg=None):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        t0 = time.perf_counter()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    extra = f"  {bytes_alg / 1e9 / (best / 1e3):.0f} GB/s of {bytes_alg / 1e9:.2f} GB" if bytes_alg else ""
    print(f"{name:58s} {best:9.3f} ms{extra}", flush=True)


g = torch.Generator(device="cuda")
g.manual_seed(1)
ctx = idk.context(0)


def randn(m, n):  # m x n column-major
    return torch.randn((n, m), generator=g, device="cuda", dtype=torch.float64).t()


a = randn(65536, 4096)
timed("optim_id 65536x4096 k=64 (dual: transpose + CPQR)", lambda: idk.optim_id(a, 64))
ctx.set_profiling(True)
idk.optim_id(a, 64)
print("   stages", {k: round(v, 3) for k, v in ctx.stage_times().items()})
ctx.set_profiling(False)
timed("sketch_rid 65536x4096 k=64 p=8 (cfg5 shape)", lambda: idk.sketch_rid(a, 64, 8, seed=1))
cols = torch.arange(0, 64 * 50, 50, device="cuda")
timed("select_columns rows_of_a 65536x4096 -> 64 rows", lambda: idk.select_columns(a, cols, rows_of_a=True),
      bytes_alg=16.0 * 4096 * 64)
del a
b = randn(16384, 16384)
r = idk.sketch_rid(b, 256, 16, seed=1)
timed("diagnostics 16384^2 k=256 (C Z GEMM + fused residual)", lambda: idk.diagnostics(b, r))
timed("optim_rid 16384^2 k=64 frac 0.02", lambda: idk.optim_rid(b, 64, 0.02, 3))
timed("select_columns 16384^2 -> 256 columns", lambda: idk.select_columns(b, r.cols), bytes_alg=16.0 * 16384 * 256)
del b, r
c = randn(100000, 50)
timed("qr_column_pivoted 100000x50 steps=50 (Q, R, perm)", lambda: idk.qr_column_pivoted(c, 50))
d = randn(4000, 100000)
timed("optim_id 4000x100000 k=32 (wide, streaming)", lambda: idk.optim_id(d, 32))
