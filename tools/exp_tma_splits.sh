# cfg2 headline vs sketch split-K with the TMA kernel (same box)
for r in 1 2; do for sp in 2 4 8; do IDK_GEMM_SPLITS=$sp python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('splits $sp', round(d['value'],1))"; done; done
for sp in 2 4 8; do IDK_GEMM_SPLITS=$sp python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4 splits $sp', round(d['value'],2))"; done
for sp in 1 2 4; do IDK_GEMM_SPLITS=$sp python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5 splits $sp', round(d['value'],2))"; done
python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5 auto', round(d['value'],2))"
