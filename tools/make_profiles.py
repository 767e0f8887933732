"""Turn the ncu captures of tools/gpu_profiles.sh (in gpurun_out/) into the
tracked summaries under profiles/ for round `tag`:

  launches_cfg2_<tag>.csv / .txt   per-launch list and per-kernel shares
  ncu_full_<tag>.json / .txt       --set full metrics per kernel and config
  ncu_summary_<tag>.json           dram bytes per launch of each stage (bench.py reads it)

python tools/make_profiles.py r01
"""
import csv
import io
import json
import os
import re
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"

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
    "launch__cluster_dim_x": "cluster_x",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_inst_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_cycles_pct",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active": "shared_pipe_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active": "dmma_inst_pct",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct",
    "TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "fp64_pipe_realtime_pct",
}
SCALE = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "ns": 1.0, "us": 1e3, "ms": 1e6, "s": 1e9,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1.0, "KB": 1e3, "MB": 1e6, "GB": 1e9}
STAGE = [("sketch_gemm", "sketch"), ("sketch_tma", "sketch"), ("splitk", "sketch"), ("cpqr", "cpqr"), ("trsm", "solve"),
         ("gather_r11", "solve"), ("gather_columns", "gather"), ("omega", "prep"), ("batched", "batched")]


def short(name):
    name = re.sub(r"\(.*", "", name)
    return name.replace("void ", "").replace("unnamed>::", "").replace("idk::", "").strip()


def stage_of(name):
    for key, st in STAGE:
        if key in name:
            return st
    return None


def launches():
    src = os.path.join(OUT, "launches_cfg2.csv")
    text = open(src).read()
    body = text[text.index('"ID"'):]
    rows = list(csv.DictReader(io.StringIO(body)))
    shutil.copy(src, os.path.join(PROF, f"launches_cfg2_{tag}.csv"))
    agg = {}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = short(r["Kernel Name"])
        v = float(r["Metric Value"].replace(",", "")) * SCALE.get(r.get("Metric Unit", "ns"), 1.0)
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    lines = ["ncu launch list (gpu__time_duration.sum, --clock-control none, serialised by ncu) of "
             "`python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e` (cfg2, 64 IDs per step), "
             "our kernels only (-k filter in tools/gpu_profiles.sh):",
             f"{'kernel':58s} {'launches':>8s} {'total us':>10s} {'avg us':>9s} {'share':>6s}"]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{k[:58]:58s} {n:8d} {t / 1e3:10.1f} {t / n / 1e3:9.1f} {100 * t / tot:5.1f}%")
    open(os.path.join(PROF, f"launches_cfg2_{tag}.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full():
    allres, summary, table = {}, {}, []
    for c in ("cfg2", "cfg3", "cfg4", "cfg5"):
        path = os.path.join(OUT, f"full_{c}_raw.csv")
        if not os.path.exists(path):
            continue
        rows = list(csv.reader(open(path)))
        hdr, units, data = rows[0], rows[1], rows[2:]
        unit_of = dict(zip(hdr, units))
        res = []
        for r in data:
            d = dict(zip(hdr, r))
            item = {"kernel": short(d.get("Kernel Name", ""))}
            for k, nm in KEYS.items():
                if k in d:
                    try:
                        item[nm] = float(d[k].replace(",", "")) * SCALE.get(unit_of.get(k, ""), 1.0)
                    except ValueError:
                        item[nm] = d[k]
            if "dram_read_bytes" in item and "dram_write_bytes" in item:
                item["dram_bytes"] = item["dram_read_bytes"] + item["dram_write_bytes"]
            res.append(item)
        allres[c] = res
        per = {}
        for it in res:
            st = stage_of(it["kernel"])
            if st and "dram_bytes" in it:
                per.setdefault(st, []).append(it["dram_bytes"])
        summary[c] = {st: {"dram_bytes_per_launch": sum(v) / len(v)} for st, v in per.items()}
        def nv(it, key):
            v = it.get(key, 0)
            return v if isinstance(v, float) else 0.0

        for it in res:
            table.append(f"{c:5s} {it['kernel'][:44]:44s} {nv(it, 'duration_ns') / 1e3:9.1f} us  "
                         f"dram {nv(it, 'dram_bytes') / 1e6:9.2f} MB ({nv(it, 'dram_pct_of_peak'):5.1f}% peak)  "
                         f"sm {nv(it, 'sm_throughput_pct'):5.1f}%  fp64pipe {nv(it, 'fp64_pipe_cycles_pct'):5.1f}%  "
                         f"tensor(DMMA) {nv(it, 'tensor_pipe_pct'):5.1f}%  "
                         f"shared {nv(it, 'shared_pipe_pct'):5.1f}%  occ {nv(it, 'achieved_occupancy_pct'):5.1f}%")
    summary["source"] = f"profiles/ncu_full_{tag}.json (ncu --set full --clock-control none, tools/gpu_profiles.sh)"
    json.dump(allres, open(os.path.join(PROF, f"ncu_full_{tag}.json"), "w"), indent=1)
    json.dump(summary, open(os.path.join(PROF, f"ncu_summary_{tag}.json"), "w"), indent=1)
    hdr = ("ncu --set full --clock-control none captures (cold-cache, serialised; durations are per launch "
           "under the profiler, not bench values):")
    open(os.path.join(PROF, f"ncu_full_{tag}.txt"), "w").write(hdr + "\n" + "\n".join(table) + "\n")
    print(hdr)
    print("\n".join(table))


if __name__ == "__main__":
    launches()
    full()
