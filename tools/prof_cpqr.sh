# CPQR phase traces (cfg1, cfg2, cfg4) + an ncu source-level capture of the cfg2 CPQR kernel
for c in cfg2 cfg1 cfg4; do python tools/trace_cpqr.py $c > gpurun_out/trace_$c.txt 2>&1; echo trace $c rc=$?; done
python tools/prof_id.py cfg2 2 > gpurun_out/p2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:cpqr_resident -s 1 -c 1 \
    -o gpurun_out/full_cpqr2 -f python tools/prof_id.py cfg2 2 > gpurun_out/ncu_cpqr2.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/full_cpqr2.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_cpqr2.csv 2>/dev/null
ncu -i gpurun_out/full_cpqr2.ncu-rep --page details > gpurun_out/det_cpqr2.txt 2>/dev/null
rm -f gpurun_out/full_cpqr2.ncu-rep
