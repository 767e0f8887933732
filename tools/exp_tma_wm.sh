# cfg2 headline vs the sketch M tile with the TMA kernel (same box)
for r in 1 2; do for wm in 7 4 5; do IDK_GEMM_WM=$wm python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('wm $wm', round(d['value'],1))"; done; done
