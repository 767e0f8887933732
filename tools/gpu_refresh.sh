# Round-end evidence: GPU tests, one bench line per config + the reference arm, ncu launch list and captures.
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gpu_tests.log
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc=$?
bash tools/gpu_bench_all.sh
bash tools/gpu_profiles.sh > gpurun_out/profiles.log 2>&1; echo profiles rc=$?
python tools/trace_cpqr.py cfg2 > gpurun_out/trace2c.txt 2>&1
python tools/trace_cpqr.py cfg1 > gpurun_out/trace1c.txt 2>&1
python tools/trace_cpqr.py cfg4 > gpurun_out/trace4c.txt 2>&1
du -sh gpurun_out
