# TMA-fed sketch GEMM (default) vs the cp.async kernel (IDK_GEMM_TMA=0), same box
python -m pytest tests -x -q -m gpu > gpurun_out/t_all.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/t_all.log
for r in 1 2; do for t in 0 1; do
  IDK_GEMM_TMA=$t python - <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2105_07076_b200 as idk
def timed(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps
out = []
for name, l, m, n, trans in [("cfg2", 110, 2000, 4000, False), ("cfg4", 272, 16384, 16384, False), ("cfg5", 72, 4096, 65536, True)]:
    om = idk.sketch_omega(l, m, 7)
    a = torch.randn(n, m, dtype=torch.float64, device="cuda").t() if not trans else torch.randn(m, n, dtype=torch.float64, device="cuda").t()
    y = idk.sketch(om, a, transposed=trans)
    ref = om @ (a.t() if trans else a)
    err = ((y - ref).norm() / ref.norm()).item()
    ms = timed(lambda: idk.sketch(om, a, transposed=trans))
    out.append(f"{name} {2*l*m*n/ms/1e9:.2f} TF ({err:.0e})")
print("TMA=" + os.environ["IDK_GEMM_TMA"], " | ".join(out), flush=True)
PY
done; done
for c in cfg4 cfg5; do for t in 0 1; do IDK_GEMM_TMA=$t python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('TMA=$t $c', round(d['value'],2), d['ms_per_step'])"; done; done
