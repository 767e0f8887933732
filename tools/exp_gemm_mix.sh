# cfg2 throughput (48 in flight) vs the sketch tile (IDK_GEMM_WM) and split-K
for wm in 7 4 5; do for sp in 4 8; do IDK_GEMM_WM=$wm IDK_GEMM_SPLITS=$sp python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('wm $wm splits $sp', round(d['value'],1), round(d['ms_per_step'],3))"; done; done
