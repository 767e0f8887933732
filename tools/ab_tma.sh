# same-box A/B of two TMA sketch builds (ab/A.so, ab/B.so): sketch alone + cfg2 headline + cfg4
IDK_LIB_PATH=paper_2105_07076_b200/ab/B.so python -m pytest tests -x -q -m gpu -k "sketch or rid or config or approx or diag" 2>&1 | tail -1; IDK_GEMM_TMA=2 IDK_LIB_PATH=paper_2105_07076_b200/ab/B.so python -m pytest tests -x -q -m gpu -k "sketch or rid or config or dual or tall" 2>&1 | tail -1
for r in 1 2; do for v in A B C; do
  IDK_LIB_PATH=paper_2105_07076_b200/ab/$v.so python - <<'PY'
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
for name, l, m, n in [("cfg2", 110, 2000, 4000), ("cfg4", 272, 16384, 16384)]:
    om = idk.sketch_omega(l, m, 7)
    a = torch.randn(n, m, dtype=torch.float64, device="cuda").t()
    ms = timed(lambda: idk.sketch(om, a))
    out.append(f"{name} {2*l*m*n/ms/1e9:.2f}")
print(os.environ["IDK_LIB_PATH"].split("/")[-1], " | ".join(out), flush=True)
PY
  IDK_LIB_PATH=paper_2105_07076_b200/ab/$v.so python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v bench', round(d['value'],1))"
done; done
