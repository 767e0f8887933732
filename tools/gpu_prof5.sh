python tools/prof_id.py cfg3 2 > gpurun_out/prof_plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:batched -s 1 -c 1 -o gpurun_out/prof_batched_cfg3 -f python tools/prof_id.py cfg3 2 > gpurun_out/ncu_b3.log 2>&1; echo ncu rc=$?
