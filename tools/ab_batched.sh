# A/B of library builds on the same box (IDK_LIB_PATH), alternating: cfg3 batched bench
# usage: bash tools/ab_batched.sh A B [C ...]  (builds in paper_2105_07076_b200/ab/<name>.so; tests run on the last)
V="${*:-A B}"
LAST="${@: -1}"; LAST="${LAST:-B}"
IDK_LIB_PATH=paper_2105_07076_b200/ab/$LAST.so python -m pytest tests/test_gpu_id.py tests/test_gpu_configs.py tests/test_gpu_edges.py -x -q -k "batch or cfg3" 2>&1 | tail -1
for r in 1 2 3; do for v in $V; do
  IDK_LIB_PATH=paper_2105_07076_b200/ab/$v.so python bench.py --config cfg3 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), round(d['ms_per_step'],4))"
done; done
