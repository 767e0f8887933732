# ncu --set full of the cfg4 (or $1) resident CPQR launch: per-line stall / instruction tops, opcode histogram
cfg=${1:-cfg4}
ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:cpqr_resident -s 1 -c 1 -o gpurun_out/ncu_cpqr_$cfg python tools/one_$cfg.py > gpurun_out/ncu_cpqr_$cfg.log 2>&1
ncu -i gpurun_out/ncu_cpqr_$cfg.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncu_cpqr_${cfg}_source.csv 2>/dev/null
ncu -i gpurun_out/ncu_cpqr_$cfg.ncu-rep --page raw --csv > gpurun_out/ncu_cpqr_${cfg}_raw.csv
python tools/ncu_line_top.py gpurun_out/ncu_cpqr_${cfg}_source.csv 45 | cut -c1-160
python tools/ncu_opcode_hist.py gpurun_out/ncu_cpqr_${cfg}_source.csv > gpurun_out/ncu_cpqr_${cfg}_ops.txt 2>&1; head -22 gpurun_out/ncu_cpqr_${cfg}_ops.txt
