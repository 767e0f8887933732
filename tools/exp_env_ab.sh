# same-box A/B of runtime knobs on the cfg2 headline: lane stream priority, IDs in flight
for r in 1 2; do
  for v in "X=0" "IDK_LANE_PRIO=0"; do env $v python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1))"; done
  for b in 48 64; do python bench.py --batch $b --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('batch $b', round(d['value'],1))"; done
done
