# dual (cfg5) sketch: TMA (IDK_GEMM_TMA=2) vs cp.async (default for the dual), same box
for r in 1 2; do for t in 1 2; do
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
l, m, n = 72, 4096, 65536
om = idk.sketch_omega(l, m, 7)
a = torch.randn(m, n, dtype=torch.float64, device="cuda").t()
ms = timed(lambda: idk.sketch(om, a, transposed=True))
print("TMA=" + os.environ["IDK_GEMM_TMA"], f"cfg5 {2*l*m*n/ms/1e9:.2f} TF", flush=True)
PY
done; done
for t in 1 2; do IDK_GEMM_TMA=$t python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('TMA=$t cfg5 bench', round(d['value'],1))"; done
python -m pytest tests -x -q -m gpu > gpurun_out/t_all.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/t_all.log
python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4 bench', round(d['value'],1), d['roofline']['frac'])"
