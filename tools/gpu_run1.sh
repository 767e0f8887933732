set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo rc=$?
for c in cfg1 cfg3 cfg4 cfg5; do timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c rc=$?; done
