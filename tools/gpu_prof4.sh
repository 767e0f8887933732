python tools/prof_id.py cfg2 3 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"id_trsm|gather_r11" -s 2 -c 2 -o gpurun_out/prof_trsm_cfg2 -f python tools/prof_id.py cfg2 3 > gpurun_out/ncu_trsm.log 2>&1; echo ncu1 rc=$?
python tools/prof_id.py cfg4 2 > gpurun_out/prof_plain4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"id_trsm|gather_r11" -s 2 -c 2 -o gpurun_out/prof_trsm_cfg4 -f python tools/prof_id.py cfg4 2 > gpurun_out/ncu_trsm4.log 2>&1; echo ncu2 rc=$?
