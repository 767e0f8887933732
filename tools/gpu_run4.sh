timeout 600 python -m pytest tests/test_gpu_id.py -q -x --timeout 300 -k "batched" > gpurun_out/pytest_b.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_b.log
timeout 600 python bench.py --config cfg3 --steps 10 --no-cpu-baseline > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; echo cfg3 rc=$?; tail -2 gpurun_out/bench_cfg3.err
