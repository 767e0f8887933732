# A/B of two library builds on the same box (IDK_LIB_PATH), alternating: cfg2 headline bench
# (build paper_2105_07076_b200/ab/A.so and B.so first)
IDK_LIB_PATH=paper_2105_07076_b200/ab/B.so python -m pytest tests/test_gpu_edges.py tests/test_gpu_id.py tests/test_gpu_configs.py -x -q 2>&1 | tail -1
for r in 1 2 3; do for v in A B; do
  IDK_LIB_PATH=paper_2105_07076_b200/ab/$v.so python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), round(d['ms_per_step'],3), {k: round(v,4) for k,v in d['stages_ms_per_step'].items()})"
done; done
