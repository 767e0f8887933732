#!/usr/bin/env python
"""bench.py -- throughput of the B200 ID path on BASELINE.json's workload.

Default workload (N=1): the largest single-GPU configuration, BASELINE
configs[3] ("cfg4"): Gaussian-sketch RID of a 16384 x 16384 fp64
A = U diag(sigma) V^T (sigma_i = 1 for i < 128, (i-127)^-2 after), k = 256,
p = 16, Omega from the on-device Philox generator.  A "step" is one full ID
(Omega -> sketch Y = Omega A -> CPQR(Y) -> Z -> C) through the C ABI
(idk_id_auto), input resident in HBM; A (2 GiB) is larger than L2 and L2 is
also flushed with a 256 MiB memset between timed steps (outside the events).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg1..cfg5]
  python bench.py --impl reference ...   # the reference's CPU path (oracle/_ref)

--gpus N > 1 without a launcher re-executes itself under torch.distributed.run
(one rank per GPU, NCCL).  cfg4/cfg5 are column-sharded;
cfg3 partitions the batch by matrix; cfg1/cfg2 run as independent replicas
("replicas only").  Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "IDs/sec & achieved HBM GB/s / FP64 TFLOPS at 1/2/4/8 B200 vs CPU ref"
UNIT = "IDs/s"
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FP64_PEAK_FILE = os.path.join(ROOT, "profiles", "fp64_peak.json")
NCU_SUMMARY = os.path.join(ROOT, "profiles", "ncu_summary_r02.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="cfg4", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--seed", type=int, default=20260601)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=20.0,
                    help="cfg1-3: time budget of the 1-thread cpu_baseline repeats (cfg4/cfg5: one full run)")
    ap.add_argument("--shard", action="store_true", help="cfg4/cfg5: use the sharded layer even at N=1")
    ap.add_argument("--batch", type=int, default=None,
                    help="cfg1/cfg2: distinct matrices per step, run concurrently through idk_id_auto_batch "
                         "(default 64, the lane limit of idk_set_concurrency -- throughput rises with IDs in flight: 48 -> 7.25k, 64 -> 7.36k IDs/s at cfg2, profiles/inflight_r01.txt; 1 = one ID per step through idk_id_auto)")
    return ap.parse_args()


def load_json(path):
    try:
        with open(path) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


def workload_desc(cfg):
    if cfg.name == "cfg3":
        return f"{cfg.name}: batched deterministic ID, {cfg.batch} x {cfg.m}x{cfg.n} fp64, k={cfg.k}"
    if cfg.randomized:
        return (f"{cfg.name}: Gaussian-sketch RID {cfg.m}x{cfg.n} fp64, k={cfg.k}, p={cfg.p}, "
                f"Omega on device (Philox)" + (" , id_auto dual (m > n)" if cfg.m > cfg.n else ""))
    return f"{cfg.name}: deterministic ID {cfg.m}x{cfg.n} fp64, k={cfg.k}"


def ids_per_step(cfg, batch=1):
    return cfg.batch if cfg.name == "cfg3" else batch


# ---------------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)
# ---------------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        loaded = [s for s in sm if smax and s >= 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------
def stage_work(cfg, n_local):
    """Algorithmic bytes / flops per launch of each stage; DESIGN.md states them."""
    m, n, k = cfg.m, n_local, cfg.k
    if cfg.m > cfg.n:  # dual: the ID runs on A^T (n x m)
        m, n = cfg.n, cfg.m
    l = cfg.l if cfg.randomized else m
    return {
        "sketch": {"flops": 2.0 * l * m * n, "bytes": 8.0 * (m * n + l * m + l * n)},
        "cpqr": {"bytes": 8.0 * 2 * l * n, "flops": sum(4.0 * (l - s) * (n - s - 1) for s in range(k))},
        "solve": {"bytes": 8.0 * 2 * k * n, "flops": float(k) * k * (n - k)},
        "gather": {"bytes": 8.0 * 2 * m * k},
        "prep": {"bytes": 8.0 * l * m if cfg.randomized else 8.0 * 2 * m * n},
    }


def stage_rooflines(cfg, stage_avg, peaks, fp64_peak):
    """Every stage against its own bound (sketch and Z solve: DMMA TFLOP/s; the
    rest: HBM GB/s on algorithmic bytes).  With several IDs in flight the stage
    times are per-launch durations under co-running kernels, so these fractions
    are lower bounds of the kernels' own rates (DESIGN.md section 3 has the
    stand-alone ncu numbers)."""
    work = stage_work(cfg, cfg.n)
    out = {"_note": "per-launch durations measured on each ID's lane stream while the other IDs in flight share "
                    "the GPU: lower bounds of each kernel's own rate (stand-alone rates: profiles/ncu_full_r02.json, launches_cfg4_r02.txt)"}
    for st, ms in stage_avg.items():
        if ms <= 0 or st not in work:
            continue
        w = work[st]
        if st in ("sketch", "solve") and "flops" in w:
            tf = w["flops"] / (ms / 1e3) / 1e12
            out[st] = {"bound": "tensor", "achieved": tf, "peak": fp64_peak["tflops"], "unit": "TFLOP/s",
                       "frac": tf / fp64_peak["tflops"], "avg_launch_ms": ms}
        else:
            gb = w["bytes"] / (ms / 1e3) / 1e9
            out[st] = {"bound": "hbm" if st != "cpqr" else "latency (k dependent steps)", "achieved": gb,
                       "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": gb / peaks["hbm_gbs"], "avg_launch_ms": ms}
            if st == "cpqr":
                out[st]["per_pivot_step_us"] = 1e3 * ms / cfg.k
        out[st]["kernel"] = stage_kernels(cfg, cpqr_plan_for(cfg)).get(st, st)
    return out


def stage_kernels(cfg, plan=None):
    """The kernels each stage launches for this config (what actually runs:
    the dispatch of id_solve_z in csrc/trsm.cu and, for the CPQR, the plan the
    library reports through idk_cpqr_plan)."""
    tall = cfg.m > cfg.n
    k = cfg.k
    nblk = (k + 31) // 32
    if k <= 128:
        trsm = f"id_trsm_dmma_kernel<{nblk}, 1>"
    elif k <= 256:
        trsm = f"invert_diag_blocks_kernel + id_trsm_dinv_kernel<{nblk}, 64, 256>"
    else:
        trsm = "id_trsm_rl_kernel"
    kind = (plan or {}).get("kind")
    if kind == "resident-grid":
        cpqr = (f"cpqr_resident_kernel (grid exchange: {plan['ctas']} CTAs, one per SM, tagged L2 records; "
                f"{plan['cols_per_cta']} columns x {plan['threads_per_col']} threads per CTA)")
    elif kind in ("cluster", "cluster-pull"):
        cpqr = (f"cpqr_resident_kernel (one {plan['ctas']}-CTA cluster, DSMEM exchange; "
                f"{plan['cols_per_cta']} columns x {plan['threads_per_col']} threads per CTA)")
    elif kind == "streaming":
        cpqr = "cpqr_kernel (streaming, matrix in HBM)"
    else:
        cpqr = "cpqr_resident_kernel"
    return {
        "prep": "omega_philox_kernel" if cfg.randomized else ("transpose_kernel" if tall else "cudaMemcpy2DAsync"),
        "sketch": f"sketch_tma_kernel<WM, {'true' if tall else 'false'}> + splitk_reduce_kernel (TMA-fed DMMA m8n8k4)",
        "cpqr": cpqr,
        "solve": "gather_r11_kernel + " + trsm,
        "gather": "gather_rows_kernel<2>" if tall else "gather_columns_vec_kernel",
        "batched": "batched_group_kernel<64, 2, 16>",
    }


_PLAN = {}


def cpqr_plan_for(cfg):
    """idk_cpqr_plan of the CPQR this config runs (Y: l x n, or the dual's l x m)."""
    if cfg.name not in _PLAN:
        try:
            import paper_2105_07076_b200 as idk
            m, n = (cfg.n, cfg.m) if cfg.m > cfg.n else (cfg.m, cfg.n)
            rows = cfg.l if cfg.randomized else m
            _PLAN[cfg.name] = idk.context(0).cpqr_plan(rows, n, cfg.k)
        except Exception:  # noqa: BLE001 - labels only
            _PLAN[cfg.name] = None
    return _PLAN[cfg.name]


def roofline_for(stage, work, avg_ms, peaks, fp64_peak, traffic, cfg):
    secs = avg_ms / 1e3
    kern = stage_kernels(cfg, cpqr_plan_for(cfg)).get(stage, stage)
    if stage in ("sketch", "solve") and "flops" in work:
        achieved = work["flops"] / secs / 1e12
        return {"kernel": kern, "bound": "tensor", "achieved": achieved,
                "peak": fp64_peak["tflops"], "unit": "TFLOP/s", "frac": achieved / fp64_peak["tflops"],
                "peak_source": fp64_peak["source"], "traffic": traffic, "avg_launch_ms": avg_ms,
                "algorithmic_per_launch": work["flops"]}
    achieved = work["bytes"] / secs / 1e9
    return {"kernel": kern, "bound": "latency" if stage == "cpqr" else "hbm", "achieved": achieved,
            "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)", "traffic": traffic, "avg_launch_ms": avg_ms,
            "algorithmic_per_launch": work["bytes"]}


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2105_07076_b200 as idk
    from paper_2105_07076_b200 import sharded
    from paper_2105_07076_b200.configs import CONFIGS, make_torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # IDK_BENCH_BACKEND=gloo + more ranks than GPUs: plumbing check of the N > 1
    # path on a one-GPU box (ranks share a device; not a measurement)
    backend = os.environ.get("IDK_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    cfg = CONFIGS[args.config]
    dev = torch.device("cuda", local)
    k, p = cfg.k, max(cfg.p, 0)
    replicas = cfg.name in ("cfg1", "cfg2")       # too small to shard -> replicas only
    use_sharded = (not replicas) and (world > 1 or args.shard) and cfg.name in ("cfg4", "cfg5")

    # ---- inputs (harness; not timed) ----
    seed = args.seed + (rank if replicas else 0)
    a = make_torch(cfg.name, seed=seed, device=f"cuda:{local}")
    nb = (args.batch if args.batch is not None else 64) if replicas else 1
    # a stream of distinct IDs: B different matrices of the same construction
    mats = [a] + [make_torch(cfg.name, seed=seed + 1000 * j, device=f"cuda:{local}") for j in range(1, nb)]
    tall = cfg.m > cfg.n
    n_dec = cfg.m if tall else cfg.n               # columns of the decomposed matrix M
    begin, end = sharded.column_range(n_dec, world, rank) if use_sharded else (0, n_dec)
    if cfg.name == "cfg3" and world > 1:           # partition by matrix, no collective
        b3, e3 = sharded.batched_partition(cfg.batch, world, rank)
        a = a[b3:e3].contiguous()
    elif use_sharded:                              # this rank's block, stored contiguously
        a = (a[begin:end, :] if tall else a[:, begin:end]).t().contiguous().t()
    nccl_path = use_sharded and backend == "nccl"  # the C-ABI entry idk_id_sharded over its own NCCL communicator
    if nccl_path:
        try:
            sharded.nccl_setup(local)
        except Exception as exc:  # noqa: BLE001 -- keep the run alive on the torch.distributed path
            print(f"bench.py: C-ABI NCCL setup failed ({exc}); sharded path via torch.distributed", file=sys.stderr)
            nccl_path = False
    torch.cuda.empty_cache()
    ctx = idk.context(local)
    ctx.set_profiling(False)  # per-stage events cost ~35% with 8 IDs in flight: a separate pass records them
    stream = torch.cuda.current_stream(dev)

    method = idk.RANDOMIZED if cfg.randomized else idk.DETERMINISTIC
    if nb > 1:
        zc_ = max(cfg.m, cfg.n)
        crow_ = cfg.n if tall else cfg.m
        bout = ([torch.empty(k, dtype=torch.int64, device=dev) for _ in range(nb)],
                [idk.idkit.empty_f(k, zc_, dev) for _ in range(nb)],
                [idk.idkit.empty_f(crow_, k, dev) for _ in range(nb)])
        bseeds = [args.seed + j for j in range(nb)]

    def step():
        if nb > 1:
            return idk.id_auto_batch(mats, k, method, seeds=bseeds, p=p, out=bout, lanes=nb)
        if cfg.name == "cfg3":
            return idk.optim_id_batched(a, k)
        if nccl_path:
            return sharded.id_sharded_nccl(a, n_dec, k, p, seed=args.seed, transposed=tall)
        if use_sharded:
            return sharded.sketch_rid_sharded(a, n_dec, k, p, seed=args.seed, transposed=tall)
        if cfg.randomized:
            return idk.id_auto(a, k, idk.RANDOMIZED, seed=args.seed, p=p)
        return idk.id_auto(a, k, idk.DETERMINISTIC)

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)
    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize(dev)

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.1)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    stage_tot = {}
    launches0 = ctx.kernel_launches
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    for i in range(args.steps):
        flush.zero_()
        starts[i].record(stream)
        step()
        ends[i].record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    launches = ctx.kernel_launches - launches0
    total_ms = sum(s_.elapsed_time(e_) for s_, e_ in zip(starts, ends))
    clocks = sampler.stop()

    # ---- stage breakdown: a second timed pass with per-stage CUDA events on
    # each ID's launching stream (idk_stage_times); feeds `roofline` ----
    n_stage = 0
    if cfg.name != "cfg3" and not use_sharded:
        ctx.set_profiling(True)
        n_stage = max(1, min(args.steps, 10))
        for _ in range(n_stage):
            flush.zero_()
            step()
            for kname, v in ctx.stage_times().items():
                stage_tot[kname] = stage_tot.get(kname, 0.0) + v
        torch.cuda.synchronize(dev)
        ctx.set_profiling(False)

    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    if replicas:
        total_ids, scaling = world * nb * args.steps, "weak"  # N independent replicas, nb IDs per step
    elif cfg.name == "cfg3":
        total_ids, scaling = cfg.batch * args.steps, "strong"  # the 4096-matrix batch split over N
    else:
        total_ids, scaling = args.steps, "strong"            # one sharded ID over N GPUs
    value = total_ids / (max_ms / 1e3)

    # ---- e2e through the public host-buffer API (H2D + compute + D2H each step) ----
    e2e = None
    if not args.no_e2e and cfg.name == "cfg3":
        # idk_optim_id_batched_host: the whole (rank's) batch from pinned host memory,
        # chunks uploaded / factored / downloaded in a pipeline, outputs to pinned memory
        B3, n3, m3 = a.shape
        ah3 = torch.empty(a.shape, dtype=torch.float64).pin_memory()
        ah3.copy_(a.cpu())
        oc3 = torch.empty((B3, k), dtype=torch.int64).pin_memory()
        oz3 = torch.empty((B3, n3, k), dtype=torch.float64).pin_memory()
        occ3 = torch.empty((B3, k, m3), dtype=torch.float64).pin_memory()
        ctx.bind_stream()

        def e2e3():
            ctx.check(ctx.lib.idk_optim_id_batched_host(ctx.h, ah3.data_ptr(), B3, m3, n3, k, oc3.data_ptr(),
                                                        oz3.data_ptr(), occ3.data_ptr()))
        e2e3()
        reps3 = max(3, min(args.steps, 10))
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        flush.zero_()
        ev0.record(stream)
        for _ in range(reps3):
            e2e3()
        ev1.record(stream)
        torch.cuda.synchronize(dev)
        e_ms = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        e2e_val = cfg.batch * reps3 / (float(e_ms.item()) / 1e3)
        h2d3 = 8 * B3 * m3 * n3
        e2e = {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d3,
               "d2h_bytes_per_step": 8 * B3 * (k + k * n3 + k * m3),
               "h2d_gbs": h2d3 * reps3 / (float(e_ms.item()) / 1e3) / 1e9 / max(world, 1),
               "h2d_peak_gbs": 55.1, "h2d_peak_source": "profiles/probe_h2d_r01.txt (pinned H2D, measured)",
               "api": "idk_optim_id_batched_host (include/idkit_b200.h): pinned host buffers, chunks of 2 x SMs "
                      "matrices pipelined (upload / factor / download)"}
    if not args.no_e2e and cfg.name != "cfg3":
        pinned = torch.empty((a.shape[1], a.shape[0]), dtype=torch.float64).pin_memory()
        pinned.copy_(a.t().cpu())
        ha = pinned.numpy().T  # column-major view of pinned memory
        assert ha.flags["F_CONTIGUOUS"]
        method = idk.RANDOMIZED if cfg.randomized else idk.DETERMINISTIC
        zc = max(cfg.m, cfg.n)
        crow = cfg.n if tall else cfg.m

        ke = max(1, min(max(args.steps, 20), 40))  # pipeline fill amortised over >= 20 IDs
        if not use_sharded:
            # pinned outputs so the downloads are asynchronous too
            def pinned_f(rows, cols_):
                return torch.empty((cols_, rows), dtype=torch.float64).pin_memory().numpy().T
            outs = ([torch.empty(k, dtype=torch.int64).pin_memory().numpy() for _ in range(ke)],
                    [pinned_f(k, zc) for _ in range(ke)], [pinned_f(crow, k) for _ in range(ke)])

        def e2e_step():
            if use_sharded:  # this rank's shard in from pinned memory, its Z block and C out
                da = torch.empty_like(a)
                da.copy_(pinned.t(), non_blocking=True)
                if nccl_path:
                    cols, zl, c = sharded.id_sharded_nccl(da, n_dec, k, p, seed=args.seed, transposed=tall)
                else:
                    cols, zl, c = sharded.sketch_rid_sharded(da, n_dec, k, p, seed=args.seed, transposed=tall)
                cols.cpu(), zl.cpu(), c.cpu()
                return
            idk.id_auto(ha, k, method, seed=args.seed, p=p)

        def e2e_run():
            """ke steps; the pipelined host entry overlaps step i+1's upload and
            step i-1's download with step i's compute."""
            if use_sharded:
                for _ in range(ke):
                    e2e_step()
            else:
                idk.id_auto_many([ha] * ke, k, method, seed=args.seed, p=p, out=outs)

        e2e_run()
        torch.cuda.synchronize(dev)
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        flush.zero_()
        ev0.record(stream)
        e2e_run()
        ev1.record(stream)
        torch.cuda.synchronize(dev)
        e_ms = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        ids = (world if replicas else 1) * ke
        if use_sharded:
            h2d = 8 * a.numel()
            d2h = 8 * k + 8 * k * (end - begin) + 8 * crow * k
        else:
            h2d = 8 * cfg.m * cfg.n
            d2h = 8 * k + 8 * k * zc + 8 * crow * k
        e2e_val = ids / (float(e_ms.item()) / 1e3)
        e2e = {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "h2d_gbs": e2e_val / max(ids / ke, 1) * h2d / 1e9,
               "h2d_peak_gbs": 55.1, "h2d_peak_source": "profiles/probe_h2d_r01.txt (pinned H2D, measured)",
               "api": ("idk_id_sharded via sharded.id_sharded_nccl (per-rank shard from pinned host)" if nccl_path else
                       "paper_2105_07076_b200.sharded.sketch_rid_sharded (per-rank shard, pinned host)" if use_sharded
                       else "idk_id_auto_host_many (include/idkit_b200.h): pinned host buffers, upload/compute/"
                            "download overlapped across steps")}

    # ---- roofline of the dominant kernel ----
    peaks = load_json(PEAKS_FILE) or {"hbm_gbs": 6650.0, "_fallback": True}
    fp64 = load_json(FP64_PEAK_FILE) or {"tflops": 37.15, "source": "fallback: tools/probe_fp64.cu DMMA loop"}
    fp64.setdefault("source", "tools/probe_fp64.cu")
    ncu = load_json(NCU_SUMMARY) or {}
    roofline = None
    stage_avg = {}
    if stage_tot:
        stage_avg = {s_: v / n_stage for s_, v in stage_tot.items()}
        dom = max(stage_avg, key=stage_avg.get)
        nc = ncu.get(cfg.name) or {}
        traffic = nc.get(dom, {}).get("dram_bytes_per_launch")
        if dom == "sketch" and traffic is not None and "splitk_reduce" in nc:
            traffic += nc["splitk_reduce"]["dram_bytes_per_launch"]  # the stage's two kernels, as timed
        roofline = roofline_for(dom, stage_work(cfg, cfg.n)[dom], stage_avg[dom], peaks, fp64, traffic, cfg)
        # share of the device time per ID (with nb IDs in flight, per-launch times include co-running kernels)
        roofline["step_share"] = stage_avg[dom] / sum(stage_avg.values())
        if dom == "cpqr":  # k dependent pivot steps: latency-bound, report the per-step time
            roofline["per_pivot_step_us"] = 1e3 * stage_avg[dom] / cfg.k
            roofline["latency_note"] = ("CPQR is a chain of k dependent pivot steps (global argmax each); its HBM "
                                        "fraction is low by construction -- the matrix is read once into "
                                        "registers/shared memory and written once")
        if nb > 1:
            roofline["note"] = (f"{nb} IDs in flight on {nb} streams: avg_launch_ms is the launch duration measured "
                                f"by CUDA events on its lane stream in {n_stage} extra timed steps (co-running kernels "
                                f"included; the events are left out of the headline steps, where they cost ~35%); "
                                f"step_share = share of the per-ID stage times")
    elif cfg.name == "cfg3":
        per = a.shape[0]
        bytes_ = 8.0 * per * (cfg.m * cfg.n + cfg.k * cfg.n + cfg.m * cfg.k) + 8.0 * per * cfg.k
        traffic = (ncu.get(cfg.name) or {}).get("batched", {}).get("dram_bytes_per_launch")
        roofline = roofline_for("batched", {"bytes": bytes_}, total_ms / args.steps, peaks, fp64, traffic, cfg)
    if peaks.get("_fallback") and roofline:
        roofline["peak_source"] = "fallback 6.65 TB/s (B200_PROFILING.md)"

    # ---- cpu baseline (rank 0, N=1, bounded sample) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, a, args)

    if rank == 0:
        if replicas:
            par = f"replicas x{world}"
        elif cfg.name == "cfg3":
            par = f"partition-by-matrix x{world}" if world > 1 else "single GPU (whole batch)"
        elif use_sharded:
            par = f"column-sharded x{world}: local sketch, all_gather_into_tensor(Y), replicated CPQR, local Z"
        else:
            par = "single GPU (no sharding)"
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded BASELINE construction (" + cfg.name + "), generated on device",
            "config": {"workload": workload_desc(cfg), "m": cfg.m, "n": cfg.n, "k": cfg.k, "p": cfg.p,
                       "batch": cfg.batch if cfg.name == "cfg3" else nb,
                       "ids_in_flight": nb if replicas else None,
                       "api": ("idk_id_auto_batch (one lane stream per ID in flight)" if nb > 1 else
                               "idk_optim_id_batched" if cfg.name == "cfg3" else
                               "idk_id_sharded (NCCL inside the C ABI)" if nccl_path else
                               "sharded.sketch_rid_sharded" if use_sharded else "idk_id_auto"),
                       "parallelism": par,
                       "l2": "flushed between timed steps (256 MiB memset, outside the events)",
                       "inputs": "resident in HBM"},
            "stages_ms_per_step": stage_avg or None,
            "stage_rooflines": stage_rooflines(cfg, stage_avg, peaks, fp64) if stage_avg else None,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------------
# reference CPU path (oracle/_ref = the reference sources compiled in place)
# ---------------------------------------------------------------------------------
def host_info():
    """nproc and CPU model of this host (BASELINE.md section 2 asks for both)."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    return {"nproc": threads, "cpu_model": model}


def _ref_lib():
    from oracle import Oracle, Reference
    if Reference.available():
        return Reference(), "reference"
    return Oracle(), "port"


def _ref_inputs(cfg, seed, a_dev=None):
    """Host inputs of the workload.  cfg4/cfg5 (2 GiB) are built on the GPU when
    one is present (harness construction only, make_torch) and copied to the
    host; otherwise numpy builds them (slow)."""
    import numpy as np
    from paper_2105_07076_b200.configs import make_np, make_torch
    if a_dev is not None:
        return a_dev.cpu().numpy() if cfg.name == "cfg3" else np.asfortranarray(a_dev.cpu().numpy())
    if cfg.name in ("cfg4", "cfg5"):
        try:
            import torch
            if torch.cuda.is_available():
                t = make_torch(cfg.name, seed=seed)
                out = np.asfortranarray(t.cpu().numpy())
                del t
                torch.cuda.empty_cache()
                return out
        except Exception:  # noqa: BLE001 -- fall back to the host construction
            pass
    return make_np(cfg.name, seed=seed)


class RefPath:
    """The reference's CPU implementation of the path on `threads` host threads.

    cfg1 / cfg3: idkit::optim_id (id.cpp:29-45; cfg3: the 4096 independent calls
    spread over the threads).  cfg2 / cfg4 / cfg5: the composed
    sketch path generate(gaussian) -> matmul -> qr_column_pivoted ->
    solve_triangular -> select_columns (the reference has no sketch RID; SURVEY.md
    section 8(c)); with several threads matmul and solve_triangular are split by
    column blocks, which is bit-identical to the single call (ref_sketch_id_mt).
    cfg1 / cfg2 are too small to split: one ID per thread, `threads` IDs per step.
    """

    def __init__(self, cfg, a, threads, seed):
        self.cfg, self.a, self.threads, self.seed = cfg, a, threads, seed
        self.lib, self.kind = _ref_lib()
        self.stage_s = None

    @property
    def ids_per_call(self):
        if self.cfg.name == "cfg3":
            return self.a.shape[0]
        return self.threads if self.cfg.name in ("cfg1", "cfg2") else 1

    def _one(self):
        cfg, a = self.cfg, self.a
        if cfg.name == "cfg1":
            if self.kind == "reference":
                self.lib.optim_id(a, cfg.k)
            else:
                self.lib.optim_id(a, cfg.k, want_approx=True)
        elif self.kind == "reference":
            _, _, _, self.stage_s = self.lib.sketch_id_mt(a, cfg.k, None, l=cfg.l, seed=self.seed,
                                                          transposed=cfg.m > cfg.n, threads=1)
        else:
            om = self.lib.generate(1, cfg.l, a.shape[1] if cfg.m > cfg.n else a.shape[0], self.seed)
            self.lib.interp_decomp(np.asfortranarray(a.T) if cfg.m > cfg.n else a, cfg.k, om)

    def call(self):
        """One step; returns wall seconds."""
        cfg = self.cfg
        t0 = time.perf_counter()
        if cfg.name == "cfg3":
            if self.kind == "reference":
                self.lib.optim_id_batch_mt(self.a, cfg.k, threads=self.threads)
            else:
                for b in range(self.a.shape[0]):
                    self.lib.optim_id(np.asfortranarray(self.a[b].T), cfg.k, want_approx=True)
        elif cfg.name in ("cfg1", "cfg2"):
            errs = []

            def work():
                try:
                    self._one()
                except Exception as e:  # noqa: BLE001
                    errs.append(e)
            ts = [threading.Thread(target=work) for _ in range(self.threads)]
            for t in ts:
                t.start()
            for t in ts:
                t.join()
            if errs:
                raise errs[0]
        elif self.kind == "reference":
            _, _, _, self.stage_s = self.lib.sketch_id_mt(self.a, cfg.k, None, l=cfg.l, seed=self.seed,
                                                          transposed=cfg.m > cfg.n, threads=self.threads)
        else:
            self._one()
        return time.perf_counter() - t0

    def describe(self):
        cfg = self.cfg
        if cfg.name == "cfg3":
            what = f"the full batch of {self.a.shape[0]} {cfg.m}x{cfg.n} matrices through optim_id"
        elif cfg.name == "cfg1":
            what = f"{self.threads} concurrent optim_id calls (one per thread) on {cfg.m}x{cfg.n}"
        elif cfg.name == "cfg2":
            what = (f"{self.threads} concurrent composed sketch IDs (one per thread): generate(gaussian) -> "
                    "matmul -> qr_column_pivoted -> solve_triangular -> select_columns")
        else:
            what = ("one full composed sketch ID: generate(gaussian) -> " +
                    ("transpose(A rows) -> " if cfg.m > cfg.n else "") +
                    "matmul -> qr_column_pivoted -> solve_triangular -> select_columns"
                    + (", matmul / solve_triangular split by column blocks over the threads (bit-identical)"
                       if self.threads > 1 else ""))
        return what


import numpy as np  # noqa: E402  (used by RefPath; bench's GPU arm imports lazily)


def cpu_baseline(cfg, a_dev, args):
    """The reference's CPU path on this host, 1 thread (the reference is
    single-threaded), a full ID (cfg3: the full batch) -- no extrapolation."""
    a = _ref_inputs(cfg, args.seed, a_dev)
    rp = RefPath(cfg, a, 1, args.seed)
    budget = args.cpu_seconds
    dt = rp.call()  # cfg4 / cfg5: the one measured run (minutes on one core)
    reps, total = 1, dt
    if cfg.name not in ("cfg4", "cfg5"):  # warm-up done: time the median of up to 5 runs within the budget
        times = []
        while len(times) < 5 and (sum(times) < budget or len(times) < 1):
            times.append(rp.call())
        reps, total = len(times), statistics.median(times) * len(times)
    out = {"value": reps * rp.ids_per_call / total, "unit": UNIT, "cores": 1, "kind": rp.kind,
           "sample": f"{reps} x [{rp.describe()}] on 1 thread; " +
                     (f"median of {reps} after a warm-up run" if reps > 1 else f"single run, {total:.1f} s"),
           **host_info()}
    if rp.stage_s:
        out["stage_seconds"] = rp.stage_s
    return out


def run_reference(args):
    from paper_2105_07076_b200.configs import CONFIGS
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:  # the ranks meet once (gloo), then rank 0 alone runs the CPU reference
        import torch.distributed as dist
        dist.init_process_group("gloo")
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    info = host_info()
    threads = info["nproc"]
    base = {"impl": "reference", "metric": METRIC, "unit": UNIT, "n_gpus": world, "higher_is_better": True,
            "scaling": "weak" if cfg.name in ("cfg1", "cfg2") else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded BASELINE construction (" + cfg.name + ")",
            "config": {"workload": workload_desc(cfg), "m": cfg.m, "n": cfg.n, "k": cfg.k, "p": cfg.p,
                       "batch": cfg.batch}}
    a = _ref_inputs(cfg, args.seed)
    rp = RefPath(cfg, a, threads, args.seed)
    t_w = 0.0
    warm = max(0, min(args.warmup, 1))
    for _ in range(warm):
        t_w = rp.call()
    budget = 150.0
    steps = args.steps if t_w <= 0 else max(1, min(args.steps, int(budget / t_w)))
    times = [rp.call() for _ in range(steps)]
    total = sum(times)
    value = steps * rp.ids_per_call / total
    sample = (f"each step: {rp.describe()}; {threads} threads; {steps} timed steps (requested {args.steps}, "
              f"capped to ~{budget:.0f} s), {warm} warm-up")
    base.update({"value": value, "steps": steps, "warmup": warm, "ms_per_step": 1e3 * total / steps,
                 "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": rp.kind, "sample": sample,
                                  **info},
                 "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})
    if rp.stage_s:
        base["stage_seconds_last_step"] = rp.stage_s
    print(json.dumps(base), flush=True)


def spawn_ranks(args):
    """--gpus N > 1 without a launcher: re-exec this script under
    torch.distributed.run, one rank per GPU (NCCL's INIT log stays on so the
    communicator size can be checked)."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd, env=env).returncode


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus != world:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; the launcher's world size wins", file=sys.stderr)
    if args.warmup < 3 and args.impl == "ours":
        print("bench.py: --warmup raised to 3 (timing rules)", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
