# ncu --set full of the two kernels outside the cfg4 path that changed in round 2:
# batched_group_kernel (cfg3) and cpqr_persistent_kernel (streaming CPQR, 20000^2, k=16).
ncu --set full --clock-control none --kernel-name-base function -k regex:batched_group -s 1 -c 1 -o gpurun_out/ncu_x_cfg3 python tools/one_cfg3.py > /dev/null 2>&1
ncu --set full --clock-control none --kernel-name-base function -k regex:cpqr_persistent -s 1 -c 1 -o gpurun_out/ncu_x_stream python tools/one_streaming.py 20000 16 > /dev/null 2>&1
for f in cfg3 stream; do ncu -i gpurun_out/ncu_x_$f.ncu-rep --page raw --csv > gpurun_out/ncu_x_$f.csv; done
python - <<'PY'
import csv, json
keys = {"gpu__time_duration.sum": "duration_ns", "dram__bytes_read.sum": "dram_read_bytes", "dram__bytes_write.sum": "dram_write_bytes",
        "lts__t_bytes.sum": "l2_bytes", "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct", "launch__registers_per_thread": "registers",
        "launch__grid_size": "grid", "launch__block_size": "block", "smsp__inst_executed.sum": "warp_instructions",
        "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_cycles_pct"}
out = {}
for f, name in (("cfg3", "batched_group_kernel<64,2,16> (cfg3, 4096 x 64x256, k=16)"), ("stream", "cpqr_persistent_kernel (20000^2, k=16)")):
    rows = list(csv.reader(open(f"gpurun_out/ncu_x_{f}.csv")))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for h, u, v in zip(hdr, units, vals):
        if h in keys:
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                continue
            scale = {"usecond": 1e3, "msecond": 1e6, "ms": 1e6, "us": 1e3, "second": 1e9, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0)
            d[keys[h]] = x * scale
    out[name] = d
json.dump(out, open("gpurun_out/ncu_extra_r02.json", "w"), indent=1)
print(json.dumps(out, indent=1))
PY
