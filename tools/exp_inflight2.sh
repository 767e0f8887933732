# cfg2 headline: 48 vs 64 IDs in flight, same box, alternating
for r in 1 2 3; do for b in 48 64; do python bench.py --batch $b --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('batch $b', round(d['value'],1))"; done; done
