"""Per-phase breakdown of the resident CPQR kernel from %globaltimer marks of
every CTA.  The marks exist only in the debug library:
  python -m paper_2105_07076_b200.build --trace
  IDK_LIB_PATH=paper_2105_07076_b200/libidkit_b200_trace.so python tools/trace_cpqr.py cfg2 [mode]

Marks per step s: 0 top, 1 trailing update (cluster: dot + downdate) done,
2 CTA argmax done, 3 candidate + record published (cluster: by the publishing
warp), 4 all records read (after the barrier / polling), 5 winner selected,
6 reflector in place (= next step's top), 7 cluster: tid 0's deferred axpy done."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2105_07076_b200 as idk  # noqa: E402
from paper_2105_07076_b200.configs import CONFIGS, make_torch  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = CONFIGS[name]
a = make_torch(name, seed=20260601)
ctx = idk.context(0)
ctx.set_cpqr_mode(mode)
mm = cfg.l if cfg.randomized else min(cfg.m, cfg.n)
nn = max(cfg.m, cfg.n) if cfg.randomized else cfg.n
plan = ctx.cpqr_plan(mm, nn, cfg.k)
G, k = plan["ctas"], cfg.k
buf = torch.zeros(G * (k + 1) * 16, dtype=torch.int64, device="cuda")
for it in range(3):
    ctx.lib.idk_debug_cpqr_trace(ctx.h, C.c_void_p(buf.data_ptr()) if it == 2 else None)
    if cfg.randomized:
        idk.id_auto(a, cfg.k, idk.RANDOMIZED, seed=1, p=cfg.p)
    else:
        idk.id_auto(a, cfg.k, idk.DETERMINISTIC)
ctx.lib.idk_debug_cpqr_trace(ctx.h, None)
tt = buf.cpu().numpy().reshape(G, k + 1, 16)
smid = tt[:, k, 15].copy()
t = tt.astype(np.float64)[:, :k, :]
steps = k - 1
print(name, "mode", mode, "plan", plan)
print(f"{'phase':24s} {'cta0 ns':>9s} {'mean ns':>9s} {'max ns':>9s}")
names = ["trailing update", "CTA argmax", "publish cand+record", "wait + read records", "select (CTA sync)",
         "copy winner column"]
for i, nm in enumerate(names):
    d = t[:, :steps, i + 1] - t[:, :steps, i]
    print(f"{nm:24s} {d[0].mean():9.0f} {d.mean():9.0f} {d.max(axis=0).mean():9.0f}")
d = t[:, 1:steps + 1, 0] - t[:, :steps, 6]
print(f"{'-> next top':24s} {d[0].mean():9.0f} {d.mean():9.0f} {d.max(axis=0).mean():9.0f}")
arr = t[:, :steps, 3]
print(f"arrival skew (max-min over CTAs of 'record written'): {(arr.max(0) - arr.min(0)).mean():.0f} ns")
rel = t[:, :steps, 4]
print(f"release skew (max-min of 'records read'): {(rel.max(0) - rel.min(0)).mean():.0f} ns; "
      f"last arrival -> first release: {(rel.min(0) - t[:, :steps, 3].max(0)).mean():.0f} ns")
tot = (t[0, 1:steps + 1, 0] - t[0, :steps, 0])
print(f"step (cta0): mean {tot.mean():.0f} ns  first {tot[0]:.0f}  last {tot[-1]:.0f}")
if t[:, :steps, 7].max() > 0:
    d = t[:, :steps, 7] - t[:, :steps, 2]
    print(f"{'(tid0 deferred axpy)':24s} {d[0].mean():9.0f} {d.mean():9.0f} {d.max(axis=0).mean():9.0f}")
def recorded(*marks):
    """A phase is printed only when every CTA recorded both of its marks in every
    step (grid mode never records the cluster-only marks 9-12)."""
    return all((t[:, :steps, mk] > 0).all() for mk in marks)


# cluster publish path of the winner warp (marks 2 -> 8..12 -> 3)
pw = [("winner rows staged", 2, 8), ("pending update + norm", 8, 9), ("reflector scalars", 9, 10),
      ("scaled v + header", 10, 11), ("fence.proxy.async", 11, 12), ("bulk pushes issued", 12, 3)]
for nm, a0, a1 in pw:
    if recorded(a0, a1) and recorded(12):
        d = t[:, :steps, a1] - t[:, :steps, a0]
        print(f"  {nm:22s} {d[0].mean():9.0f} {d.mean():9.0f} {d.max(axis=0).mean():9.0f}")
# grid publish path of the publishing warp (marks 2 -> 8 -> 9 -> 10 -> 11 -> 3)
if recorded(8, 9, 10, 11) and not recorded(12):
    for nm, a0, a1 in [("rows staged", 2, 8), ("column to L2 + norm", 8, 9), ("reflector + header", 9, 10),
                       ("release fence", 10, 11), ("ready flags", 11, 3)]:
        d = t[:, :steps, a1] - t[:, :steps, a0]
        print(f"  {nm:22s} {d[0].mean():9.0f} {d.mean():9.0f} {d.max(axis=0).mean():9.0f}")
if recorded(4, 13, 14, 5):  # grid select: records -> vmax -> winner (before the tie pass) -> done
    for nm, a0, a1 in [("  records -> vmax", 4, 13), ("  vmax -> winner", 13, 14), ("  tie pass / rest", 14, 5)]:
        d = t[:, :steps, a1] - t[:, :steps, a0]
        print(f"  {nm:22s} {d[0].mean():9.0f} {d.mean():9.0f} {d.max(axis=0).mean():9.0f}")
# per-CTA lateness: when each CTA saw the exchange complete (mark 4) and published (mark 3),
# relative to the earliest CTA of the same step, by SM id
rel4 = (t[:, :steps, 4] - t[:, :steps, 4].min(axis=0)).mean(axis=1)
rel3 = (t[:, :steps, 3] - t[:, :steps, 3].min(axis=0)).mean(axis=1)
order = np.argsort(smid)
print("per-CTA mean lateness (ns) of 'records read' / 'published', by SM id:")
print("  " + " ".join(f"{int(smid[g])}:{rel4[g]:.0f}/{rel3[g]:.0f}" for g in order))
# the same by CTA (block) index, with each CTA's own phase durations: is a late CTA slow in its own
# update / argmax (marks 0 -> 2), or does it start late (mark 0 relative to the earliest CTA)?
rel0 = (t[:, :steps, 0] - t[:, :steps, 0].min(axis=0)).mean(axis=1)
upd = (t[:, :steps, 2] - t[:, :steps, 0]).mean(axis=1)
pub = (t[:, :steps, 3] - t[:, :steps, 2]).mean(axis=1)
print("per-CTA by block index: sm | start lateness | update+argmax | publish | 'published' lateness")
for g in range(G):
    print(f"  cta {g:3d} sm {int(smid[g]):3d}  {rel0[g]:6.0f} {upd[g]:6.0f} {pub[g]:6.0f} {rel3[g]:6.0f}")
for lo, hi in [(0, 10), (k // 2 - 5, k // 2 + 5), (steps - 10, steps)]:
    dd = [(t[:, lo:hi, i + 1] - t[:, lo:hi, i]).mean() for i in range(6)]
    print(f"  steps {lo:3d}-{hi:3d}: " + " ".join(f"{x:7.0f}" for x in dd))
