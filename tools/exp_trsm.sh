python -m pytest tests/test_gpu_edges.py -x -q > gpurun_out/t_edges.log 2>&1; echo edges rc=$?; tail -3 gpurun_out/t_edges.log
python -m pytest tests -x -q -m gpu > gpurun_out/t_all.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/t_all.log
for T in 1 0; do IDK_TRSM_DMMA=$T python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('dmma=$T cfg4', round(d['value'],1), d['ms_per_step'], {k: round(v,4) for k,v in d['stages_ms_per_step'].items()})"; done
python tools/prof_id.py cfg4 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:trsm -c 1 python tools/prof_id.py cfg4 1 2>&1 | grep -E "trsm|duration" | head -4
