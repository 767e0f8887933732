"""Sketch GEMM time vs split-K count (IDK_GEMM_SPLITS, read per call):
python tools/time_sketch_splits.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2105_07076_b200 as idk  # noqa: E402

def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps

shapes = [("cfg2", 110, 2000, 4000, False), ("cfg4", 272, 16384, 16384, False), ("cfg5", 72, 4096, 65536, True)]
for name, l, m, n, trans in shapes:
    om = idk.sketch_omega(l, m, 7)
    a = torch.randn(n, m, dtype=torch.float64, device="cuda").t() if not trans else \
        torch.randn(m, n, dtype=torch.float64, device="cuda").t()
    # a: column-major m x n (not trans) / n x m storage read transposed (trans)
    for sp in ["auto", "1", "2", "3", "4", "5", "6", "8", "12"]:
        if sp == "auto":
            os.environ.pop("IDK_GEMM_SPLITS", None)
        else:
            os.environ["IDK_GEMM_SPLITS"] = sp
        for wm in (["auto"] if name != "cfg4" else ["auto", "5", "6", "7"]):
            if wm == "auto":
                os.environ.pop("IDK_GEMM_WM", None)
            else:
                os.environ["IDK_GEMM_WM"] = wm
            ms = timed(lambda: idk.sketch(om, a, transposed=trans))
            print(f"{name} splits={sp:4s} wm={wm:4s} {ms:.3f} ms  {2*l*m*n/ms/1e9:.1f} TFLOP/s", flush=True)
    os.environ.pop("IDK_GEMM_WM", None)
