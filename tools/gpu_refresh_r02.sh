# Round-2 measurement refresh on one B200 (run under gpurun):
#   bench lines per config (ours + reference arm), ncu launch list of the default
#   command (our kernels + the L2 flush), ncu --set full of the cfg4 kernels.
set -u
out=gpurun_out/r02
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/gpu.txt
for c in cfg4 cfg1 cfg2 cfg3 cfg5; do
  python bench.py --config $c --steps 20 --warmup 5 > $out/bench_$c.json 2> $out/bench_$c.err
  python bench.py --config $c --impl reference --steps 5 --warmup 1 > $out/ref_$c.json 2> $out/ref_$c.err
done
KR='regex:^(sketch_tma|splitk_reduce|omega_philox|cpqr_resident|gather_r11|id_trsm|gather_columns|gather_rows|vectorized_elementwise)'
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base function -k "$KR" -c 400 --csv \
    --log-file $out/launches_cfg4.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base function \
    -k 'regex:^(sketch_tma|cpqr_resident|id_trsm|splitk_reduce|gather_columns)' -s 8 -c 5 \
    -o $out/ncu_full_cfg4 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_full.log 2>&1
echo done
