"""Turn the output of tools/gpu_refresh_r02.sh (gpurun_out/r02/) into the
tracked round-2 profiles:

  bench_<cfg>_r02.json / bench_ref_<cfg>_r02.json   the bench lines (ours / reference arm)
  launches_cfg4_r02.csv / .txt                       ncu launch list of the default command + shares
  ncu_full_r02.json                                  --set full metrics per cfg4 kernel
  ncu_summary_r02.json                               DRAM bytes + duration per launch of each stage
                                                     (bench.py reads it for roofline.traffic)
  parity_r02.json                                    the GPU parity records of the same call

python tools/make_profiles_r02.py
"""
import csv
import io
import json
import os
import re
import shutil
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out", "r02")
PROF = os.path.join(ROOT, "profiles")
NCU = "/usr/local/cuda/bin/ncu"

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
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "lts__t_bytes.sum": "l2_bytes",
}
SCALE = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "ns": 1.0, "us": 1e3, "ms": 1e6,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
STAGE = [("sketch_tma", "sketch"), ("sketch_gemm", "sketch"), ("splitk", "splitk_reduce"), ("cpqr", "cpqr"),
         ("trsm", "solve"), ("gather_r11", "solve_prep"), ("gather_columns", "gather"), ("gather_rows", "gather"),
         ("omega", "prep")]


def short(name):
    name = re.sub(r"\(.*", "", name)
    return name.replace("void ", "").replace("idk::", "").replace("(anonymous namespace)::", "") \
        .replace("<unnamed>::", "").strip()


def stage_of(name):
    for key, st in STAGE:
        if key in name:
            return st
    return None


def last_json(path):
    lines = [ln for ln in open(path).read().splitlines() if ln.strip().startswith("{")]
    return json.loads(lines[-1])


def bench_lines():
    for c in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5"):
        for src, dst in ((f"bench_{c}.json", f"bench_{c}_r02.json"), (f"ref_{c}.json", f"bench_ref_{c}_r02.json")):
            p = os.path.join(OUT, src)
            if os.path.exists(p):
                d = last_json(p)
                open(os.path.join(PROF, dst), "w").write(json.dumps(d) + "\n")
                print(f"{dst:26s} {d.get('value'):.6g} {d.get('unit')}")


def launches():
    src = os.path.join(OUT, "launches_cfg4.csv")
    text = open(src).read()
    body = text[text.index('"ID"'):]
    rows = list(csv.DictReader(io.StringIO(body)))
    shutil.copy(src, os.path.join(PROF, "launches_cfg4_r02.csv"))
    agg, order = {}, []
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = short(r["Kernel Name"])
        v = float(r["Metric Value"].replace(",", "")) * SCALE.get(r.get("Metric Unit", "ns"), 1.0)
        if k not in agg:
            order.append(k)
            agg[k] = [0, 0.0]
        agg[k][0] += 1
        agg[k][1] += v
    ours = {k: v for k, v in agg.items() if "at::" not in k}
    tot = sum(v[1] for v in agg.values())
    n_ids = max(v[0] for v in ours.values())
    lines = ["ncu --metrics gpu__time_duration.sum --clock-control none (kernel filter: the library's kernels + the "
             "L2-flush memset)",
             "of `python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e` (cfg4: 16384^2, k=256, p=16), "
             "tools/gpu_refresh_r02.sh",
             "per-launch times are cold-cache and serialised (ncu replays each kernel); the SHARE of the step is what "
             "matches the bench", ""]
    for k in order:
        n, t = agg[k]
        lines.append(f"{k[:64]:64s} launches {n:3d}  mean {t / n / 1e3:10.1f} us  share {t / tot:.3f}")
    per_id = sum(v[1] for v in ours.values()) / n_ids / 1e6
    bench = os.path.join(OUT, "bench_cfg4.json")
    ms = last_json(bench)["ms_per_step"] if os.path.exists(bench) else float("nan")
    lines += ["", f"per ID (library kernels): {per_id:.3f} ms  (bench.py ms_per_step in the same call: {ms:.3f})"]
    open(os.path.join(PROF, "launches_cfg4_r02.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full():
    rep = os.path.join(OUT, "ncu_full_cfg4.ncu-rep")
    raw = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
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
    json.dump({"cfg4": res, "source": "ncu --set full --clock-control none --import-source on, bench.py default "
               "(cfg4), tools/gpu_refresh_r02.sh", "units": "duration_ns in ns, bytes in bytes, the rest as ncu "
               "reports"}, open(os.path.join(PROF, "ncu_full_r02.json"), "w"), indent=1)
    old = json.load(open(os.path.join(PROF, "ncu_summary_r02.json")))
    per = {}
    for it in res:
        st = stage_of(it["kernel"])
        if st and "dram_bytes" in it:
            per.setdefault(st, []).append((it["dram_bytes"], it.get("duration_ns", 0.0)))
    old["cfg4"] = {st: {"dram_bytes_per_launch": sum(b for b, _ in v) / len(v),
                        "duration_ns": sum(t for _, t in v) / len(v)} for st, v in per.items()}
    old["source"] = ("cfg4: profiles/ncu_full_r02.json (final round-2 kernels); cfg2/cfg3/cfg5: "
                     "profiles/ncu_full_r01.json (kernels unchanged for the traffic figure, except the grid CPQR "
                     "of cfg5)")
    json.dump(old, open(os.path.join(PROF, "ncu_summary_r02.json"), "w"), indent=1)
    for st, v in old["cfg4"].items():
        print(f"{st:14s} dram {v['dram_bytes_per_launch'] / 1e6:10.1f} MB  {v['duration_ns'] / 1e3:9.1f} us")


def parity():
    p = os.path.join(OUT, "parity_r02.json")
    if os.path.exists(p):
        shutil.copy(p, os.path.join(PROF, "parity_r02.json"))


if __name__ == "__main__":
    bench_lines()
    launches()
    full()
    parity()
