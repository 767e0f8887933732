# ncu --set full of one cfg3 launch with IDK_BATCHED_GROUP=$1; per-line stall/instruction tops + key metrics
g=${1:-2}
export IDK_BATCHED_GROUP=$g
ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:batched_ -s 1 -c 1 -o gpurun_out/ncu_group$g python tools/one_cfg3.py > gpurun_out/ncu_group$g.log 2>&1
ncu -i gpurun_out/ncu_group$g.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncu_group${g}_source.csv 2>/dev/null
ncu -i gpurun_out/ncu_group$g.ncu-rep --page raw --csv > gpurun_out/ncu_group${g}_raw.csv
python tools/ncu_line_top.py gpurun_out/ncu_group${g}_source.csv 28 | cut -c1-150
python - <<PY
import csv
rows=list(csv.reader(open('gpurun_out/ncu_group${g}_raw.csv')))
hdr=rows[0]; vals=rows[2]
for h,v in zip(hdr,vals):
    if any(k in h for k in ['gpu__time_duration.sum','smsp__issue_active.avg.pct','_per_issue','pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active','smsp__inst_executed.sum']):
        if 'not_issued' in h: continue
        try:
            if '_per_issue' in h and float(v) < 0.3: continue
        except ValueError: pass
        print(h.replace('smsp__average_warps_issue_stalled_','stall '), v)
PY
