timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu.log
for c in cfg4 cfg5; do timeout 600 python bench.py --config $c --steps 5 --shard --no-cpu-baseline > gpurun_out/bench_${c}_shard.json 2> gpurun_out/bench_${c}_shard.err; echo $c shard rc=$?; tail -2 gpurun_out/bench_${c}_shard.err; done
