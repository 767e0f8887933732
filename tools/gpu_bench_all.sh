# One bench line per BASELINE config (N=1), plus the reference arm for cfg2.
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
  python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c rc=$?
done
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
