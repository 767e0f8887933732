python -m pytest tests -x -q -m gpu -k "qr or id or rid or config" > gpurun_out/t_cpqr.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/t_cpqr.log
python tools/trace_cpqr.py cfg2 > gpurun_out/trace2c.txt 2>&1
python tools/trace_cpqr.py cfg1 > gpurun_out/trace1c.txt 2>&1
python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['ms_per_step'], {k: round(v,4) for k,v in d['stages_ms_per_step'].items()})"
