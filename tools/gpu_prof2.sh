python tools/prof_id.py cfg2 3 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:cpqr_resident -s 1 -c 1 -o gpurun_out/prof_cpqr_cfg2 -f python tools/prof_id.py cfg2 3 > gpurun_out/ncu_cpqr.log 2>&1; echo ncu1 rc=$?
