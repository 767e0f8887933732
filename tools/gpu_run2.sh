# round-1 measurement script: GPU tests, then each config's bench line
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo cfg2 rc=$?
for c in cfg1 cfg3 cfg4 cfg5; do timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c rc=$?; done
