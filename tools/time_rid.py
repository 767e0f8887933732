"""optim_rid (the reference's column-sampling RID) on large inputs: python tools/time_rid.py"""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2105_07076_b200 as idk
g = torch.Generator(device="cuda"); g.manual_seed(1)
def t(fn, reps=3):
    fn(); torch.cuda.synchronize(); best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    return best
for (m, n, k, frac) in ((65536, 4096, 64, 0.1), (16384, 16384, 64, 0.02), (16384, 16384, 256, 0.05), (4096, 65536, 64, 0.01)):
    a = torch.randn((n, m), generator=g, device="cuda", dtype=torch.float64).t()
    ms = t(lambda: idk.optim_rid(a, k, frac, 3))
    p = max(k, int(round(frac * n)))
    flop = 2.0 * k * m * n  # C^T A
    print(f"{m}x{n} k={k} sample~{p}: optim_rid {ms:.2f} ms (C^T A alone: {flop / 33e12 * 1e3:.2f} ms at 33 TFLOP/s)", flush=True)
    del a
