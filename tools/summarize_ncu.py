"""Summarise ncu --set full captures into profiles/ (per-kernel duration, DRAM
bytes, throughput %, FP64/tensor pipe activity, occupancy)."""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_inst_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_cycles_pct",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct",
    "SM_C.TriageCompute.smsp__pipe_tensor_subpipe_dmma_cycles_active.avg": "dmma_subpipe_cycles_per_smsp",
    "TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "fp64_pipe_realtime_pct",
    "smsp__cycles_active.avg": "smsp_cycles_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active": "shared_pipe_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "lts__t_bytes.sum": "l2_bytes",
}


def summarize(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    unit_of = dict(zip(hdr, units))
    scale = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "ns": 1.0, "us": 1e3, "ms": 1e6, "s": 1e9,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1.0, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    res = []
    for r in data:
        d = dict(zip(hdr, r))
        item = {"kernel": d.get("Kernel Name", "")[:120]}
        for k, nm in KEYS.items():
            if k in d:
                try:
                    item[nm] = float(d[k].replace(",", "")) * scale.get(unit_of.get(k, ""), 1.0)
                except ValueError:
                    item[nm] = d[k]
        if "dram_read_bytes" in item and "dram_write_bytes" in item:
            item["dram_bytes"] = item["dram_read_bytes"] + item["dram_write_bytes"]
        res.append(item)
    return res


if __name__ == "__main__":
    allres = {}
    for rep in sys.argv[1:]:
        allres[rep.split("/")[-1]] = summarize(rep)
    print(json.dumps(allres, indent=1))
