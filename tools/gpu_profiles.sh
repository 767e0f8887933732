# Round-1 ncu evidence (one GPU).  Plain runs first (must exit 0), then ncu.
set -x
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg2.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
python tools/prof_id.py cfg2 3 > gpurun_out/p2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"cpqr_resident|sketch_gemm|trsm_warp|gather_r11|gather_columns|omega" -s 6 -c 6 \
    -o gpurun_out/full_cfg2 -f python tools/prof_id.py cfg2 3 > gpurun_out/ncu_full2.log 2>&1; echo full2 rc=$?
python tools/prof_id.py cfg4 2 > gpurun_out/p4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"sketch_gemm|cpqr_resident|trsm_warp" -s 3 -c 3 \
    -o gpurun_out/full_cfg4 -f python tools/prof_id.py cfg4 2 > gpurun_out/ncu_full4.log 2>&1; echo full4 rc=$?
python tools/prof_id.py cfg3 2 > gpurun_out/p3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:batched -s 1 -c 1 \
    -o gpurun_out/full_cfg3 -f python tools/prof_id.py cfg3 2 > gpurun_out/ncu_full3.log 2>&1; echo full3 rc=$?
