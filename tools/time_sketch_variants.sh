# sketch GEMM with pipeline variants (IDK_LIB_PATH = a variant build of the library)
for v in default paper_2105_07076_b200/variants/lib_bk16_s3.so paper_2105_07076_b200/variants/lib_bk16_s4.so paper_2105_07076_b200/variants/lib_bk32_s2.so paper_2105_07076_b200/variants/lib_bk8_s4.so; do
  echo "== $v"
  if [ "$v" = default ]; then unset IDK_LIB_PATH; else export IDK_LIB_PATH=$v; fi
  for sp in auto 2 8; do
    if [ $sp = auto ]; then unset IDK_GEMM_SPLITS; else export IDK_GEMM_SPLITS=$sp; fi
    python - <<'PY'
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
    ms = timed(lambda: idk.sketch(om, a, transposed=trans))
    out.append(f"{name} {ms:.3f} ms {2*l*m*n/ms/1e9:.1f} TF")
print("  splits", os.environ.get("IDK_GEMM_SPLITS", "auto"), " | ".join(out), flush=True)
PY
  done
done
