"""cuBLAS DGEMM (torch.matmul, fp64) on the sketch shapes, as a yardstick for
sketch_gemm_kernel: python tools/time_dgemm_ref.py"""
import torch

def t(fn, reps=10):
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

for name, l, m, n, trans in [("cfg2", 110, 2000, 4000, False), ("cfg4", 272, 16384, 16384, False),
                             ("cfg5", 72, 4096, 65536, True)]:
    om = torch.randn(l, m, dtype=torch.float64, device="cuda")
    a = torch.randn(m, n, dtype=torch.float64, device="cuda") if not trans else \
        torch.randn(n, m, dtype=torch.float64, device="cuda")
    # column-major A (m x n) == row-major A^T; Y = Om @ A
    if trans:
        fn = lambda: om @ a.t()
    else:
        fn = lambda: om @ a
    ms = t(fn)
    print(f"{name}: cuBLAS DGEMM {l}x{m} @ {m}x{n}: {ms:.3f} ms  {2*l*m*n/ms/1e9:.1f} TFLOP/s")
