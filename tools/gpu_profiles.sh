# ncu evidence for profiles/ (one GPU).  Each plain command must exit 0 before
# its ncu pass.  Kernel filter = our kernels only (input generation excluded).
set -x
KF='regex:"sketch_gemm|sketch_tma|splitk|omega|cpqr|invert_positions|extract_r|form_q|gather|trsm|batched|transpose|resid|z_stats|ldlt|map_cols|copy_pivots"'
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_plain.log 2>&1 && \
eval ncu --metrics gpu__time_duration.sum --clock-control none -k $KF --csv --log-file gpurun_out/launches_cfg2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
python tools/prof_id.py cfg2 3 > gpurun_out/p2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"cpqr_resident|sketch_gemm|sketch_tma|trsm|gather_r11|gather_columns|omega" -s 6 -c 6 \
    -o gpurun_out/full_cfg2 -f python tools/prof_id.py cfg2 3 > gpurun_out/ncu_full2.log 2>&1; echo full2 rc=$?
python tools/prof_id.py cfg4 2 > gpurun_out/p4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"sketch_gemm|sketch_tma|cpqr_resident|trsm|gather_columns|gather_rows" -s 4 -c 4 \
    -o gpurun_out/full_cfg4 -f python tools/prof_id.py cfg4 2 > gpurun_out/ncu_full4.log 2>&1; echo full4 rc=$?
python tools/prof_id.py cfg3 2 > gpurun_out/p3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:batched -s 1 -c 1 \
    -o gpurun_out/full_cfg3 -f python tools/prof_id.py cfg3 2 > gpurun_out/ncu_full3.log 2>&1; echo full3 rc=$?
python tools/prof_id.py cfg5 2 > gpurun_out/p5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"sketch_gemm|sketch_tma|cpqr_resident|trsm|gather_columns|gather_rows" -s 4 -c 4 \
    -o gpurun_out/full_cfg5 -f python tools/prof_id.py cfg5 2 > gpurun_out/ncu_full5.log 2>&1; echo full5 rc=$?
for c in 2 3 4 5; do ncu -i gpurun_out/full_cfg$c.ncu-rep --page raw --csv > gpurun_out/full_cfg${c}_raw.csv 2>/dev/null; done
ls -la gpurun_out/
# keep gpurun_out under the 64 MiB copy-back limit: raw CSVs suffice for 3/4/5
ncu -i gpurun_out/full_cfg2.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/full_cfg2_src.csv 2>/dev/null
rm -f gpurun_out/full_cfg3.ncu-rep gpurun_out/full_cfg4.ncu-rep gpurun_out/full_cfg5.ncu-rep
du -sh gpurun_out
