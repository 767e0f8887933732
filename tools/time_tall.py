"""Tall-skinny shapes through the streaming kernel: python tools/time_tall.py"""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2105_07076_b200 as idk
g = torch.Generator(device="cuda"); g.manual_seed(1)
ctx = idk.context(0)
def t(fn, reps=3):
    fn(); torch.cuda.synchronize(); best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    return best
for (m, n, k) in ((100000, 50, 50), (100000, 50, 20), (200000, 100, 50), (50000, 500, 50)):
    c = torch.randn((n, m), generator=g, device="cuda", dtype=torch.float64).t()
    a = t(lambda: idk.qr_column_pivoted(c, k))
    ctx.set_profiling(True); idk.optim_id(c, min(k, n - 1)); st = ctx.stage_times(); ctx.set_profiling(False)
    b = t(lambda: idk.optim_id(c, min(k, n - 1)))
    print(f"{m}x{n} k={k}: qr_column_pivoted {a:.2f} ms, optim_id {b:.2f} ms, cpqr stage {st['cpqr']:.2f} ms ({st['cpqr']/min(k,n-1)*1e3:.0f} us/step)", flush=True)
