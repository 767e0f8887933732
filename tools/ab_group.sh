# A/B of the cfg3 kernels on one box: IDK_BATCHED_GROUP = 0 (one thread per column), 2, 4.
# usage: bash tools/ab_group.sh [variants...]   (tests run on every non-zero variant first)
V="${*:-0 2 4}"
for v in $V; do
  if [ "$v" != "0" ]; then
    echo "tests group=$v"
    IDK_BATCHED_GROUP=$v timeout 900 python -m pytest tests/test_gpu_id.py tests/test_gpu_configs.py tests/test_gpu_edges.py tests/test_gpu_fullsize.py -x -q -k "batch or cfg3" 2>&1 | tail -2
  fi
done
for r in 1 2 3; do for v in $V; do
  IDK_BATCHED_GROUP=$v python bench.py --config cfg3 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('group=$v', round(d['value'],1), round(d['ms_per_step'],4))"
done; done
