"""Benchmark of the hot path (BASELINE.json metric: trees/s and predictions/s; CV-study wall
time vs the CPU oracle), one JSON line.

Headline (top-level value): the full paper-shaped CV study, configs[1]:
10 datasets = 5 GPUs of Table 3 x {time (n=189, LOG, paper custom split), power (n=168, plain
k-fold)}, 30 repeats x 10-fold CV, grid ntree {128,256,512,1024} (prefixes of 1024-tree
forests) x mtry {12 (max), 3 (sqrt), 3 (log2)}: 6,144,000 distinct trees per step.  Every step
runs the whole hot path: validation + quantisation + presort (a1, a3), folds (a2), bootstrap /
feature draws / split search / partition / leaves (a4-a8), CV scoring (a10); N > 1 adds the
cross-rank gather of the fold-MAPE tables (a11).

Multi-GPU (--scaling strong, the default): the FIXED study's 3,000 (dataset, rep, fold) tasks
are cut into contiguous rank ranges (SURVEY 8(e) "shard whole (dataset, rep, fold) tasks"),
so its wall time drops with N; --scaling weak: every rank runs its own 30-repeat study.  value
= trees grown by all ranks / max over ranks of the device time.

Per-config objects ("configs": C1, C3, C4, C5 of BASELINE.json, measured on rank 0 at N = 1):
value / unit / ms, roofline of the dominant kernel, cpu_baseline (oracle, 1 core and N pinned
cores), e2e through the host-pointer C ABI, clocks during the timed region.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--scaling strong|weak]
                  [--configs c1,c3,c4,c5 | --no-configs] [--no-cpu-baseline] [--no-e2e]
                  [--split exact|extra] [--criterion mse|mae] [--streams S]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402

METRIC = "trees trained/sec (full paper-shaped CV study)"
UNIT = "trees/s"
K_FOLDS, REPS = 10, 30
NTREES = [128, 256, 512, 1024]
MTRYS = [12, 3, 3]
SEED = 7104
DISTINCT_MTRY = 2

# fp64 arithmetic per evaluated candidate split: 2 squares + 2 divisions + 1 add
FLOPS_PER_CANDIDATE = 5
# measured on the B200 (profiles/micro/microbench.cu, profiles/rd2_02_micro.txt): DFMA 17.12 T
# ops/s = 34.2 TFLOP/s counting 2 flops per FMA (DMUL 17.2 T, DADD 18.6 T ops/s)
FP64_PEAK_TFLOPS = 34.23
FP64_PEAK_SOURCE = "measured: profiles/rd2_02_micro.txt (DFMA 17.12 Tops/s x 2 flops, 148 SMs, 1965 MHz)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--configs", default="c1,c3,c4,c5")
    ap.add_argument("--no-configs", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--criterion", default="mse", choices=["mse", "mae"],
                    help="mse (north_star, default) or mae (the criterion of the paper's best models, "
                         "T4/T5 P:858-861; R32)")
    ap.add_argument("--streams", type=int, default=10,
                    help="CUDA streams the datasets of a step are spread over (1 = one after another)")
    ap.add_argument("--split", default="exact", choices=["exact", "extra"],
                    help="exact: bootstrap + exhaustive CART (north_star, default); extra: the paper's "
                         "ExtraTrees learner without bootstrap (P:468-469, R29)")
    return ap.parse_args()


def split_kw(args):
    kw = {"split_mode": 2, "bootstrap": False} if args.split == "extra" else {}
    if getattr(args, "criterion", "mse") == "mae":
        kw["criterion"] = 1
    return kw


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy bandwidth, burst)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "B200_PROFILING.md fallback (MEASURED_PEAKS.json absent)"


# ------------------------------------------------------------ clocks -------
REASONS = ["gpu_idle", "applications_clocks_setting", "sw_power_cap", "hw_slowdown", "sync_boost",
           "sw_thermal_slowdown", "hw_thermal_slowdown", "hw_power_brake_slowdown", "display_clock_setting"]


class ClockSampler:
    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 3:
                continue
            try:
                s, m = float(parts[0]), float(parts[1])
                act = int(parts[2], 16)
            except ValueError:
                continue
            sm.append(s)
            mx = max(mx, m)
            for bit, name in enumerate(REASONS):
                if act & (1 << bit) and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------- CPU oracle baselines -----
def host_info():
    model, gov = None, None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        gov = open("/sys/devices/system/cpu/cpu0/cpufreq/scaling_governor").read().strip()
    except OSError:
        gov = "n/a (no cpufreq interface)"
    return {"cpu_model": model, "governor": gov}


def _pinned_worker(core, fn, arg, q):
    try:
        os.sched_setaffinity(0, {core})
    except OSError:
        pass
    t0 = time.perf_counter()
    units = fn(arg)
    q.put((core, units, time.perf_counter() - t0))


def run_on_cores(fn, args_per_core):
    """SURVEY 8(d) protocol (ii): one oracle process pinned per host core over disjoint
    units; returns (units done, wall seconds, cores)."""
    import multiprocessing as mp
    cores = sorted(os.sched_getaffinity(0))[:len(args_per_core)]
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    t0 = time.perf_counter()
    ps = [ctx.Process(target=_pinned_worker, args=(c, fn, a, q)) for c, a in zip(cores, args_per_core)]
    for p in ps:
        p.start()
    res = [q.get() for _ in ps]
    for p in ps:
        p.join()
    wall = time.perf_counter() - t0
    return sum(r[1] for r in res), wall, len(ps)


def ncores():
    return len(os.sched_getaffinity(0))


def _oracle():
    import oracle
    oracle.build()
    return oracle


def _cv_trees(a):
    """Oracle CV of dataset a['ds'] over tasks [lo, hi) of repeat block a['reps']: trees grown."""
    oracle = _oracle()
    d = datagen.study(datagen.SEED)[a["ds"]]
    custom = d["target"] == "time"
    folds = oracle.make_folds(d["y"], K_FOLDS, a["reps"], seed=SEED + a["ds"], custom=custom)
    oracle.cv_grid(d["X"], d["y"], K_FOLDS, a["reps"], a.get("ntrees", NTREES), a.get("mtrys", [12, 3]),
                   fold_ids=folds, target=1 if custom else 0, seed=SEED + a["ds"], task_begin=a["lo"],
                   task_end=a["hi"], **a.get("skw", {}))
    return (a["hi"] - a["lo"]) * len(a.get("mtrys", [12, 3])) * max(a.get("ntrees", NTREES))


def cpu_baseline_c2(skw):
    """1 core: K20/time repeat 0, 10 folds, mtry {12, 3} x 1024 trees (20,480 trees); N cores:
    every core runs the same block of a different (dataset, repeat)."""
    tasks = 1 if skw.get("criterion") else 10
    t0 = time.perf_counter()
    trees = _cv_trees(dict(ds=0, reps=1, lo=0, hi=tasks, skw=skw))
    one = trees / (time.perf_counter() - t0)
    n = ncores()
    args = [dict(ds=i % 10, reps=1 + i // 10, lo=(i // 10) * K_FOLDS, hi=(i // 10) * K_FOLDS + tasks, skw=skw)
            for i in range(n)]
    tot, wall, used = run_on_cores(_cv_trees, args)
    return {"value": one, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{trees} trees: K20/time dataset, repeat 0 (folds 0-{tasks - 1}), ntree<=1024 x mtry {{12,3}}",
            "n_cores": {"value": tot / wall, "unit": UNIT, "cores": used,
                        "sample": f"{used} processes pinned one per core, each {trees} trees of a different "
                                  f"(dataset, repeat) block; {tot} trees in {wall:.1f} s wall"},
            **host_info()}


# ------------------------------------------------------- reference arm ------
def study_config(args, world):
    """The workload both arms report (the reference arm times a bounded sample of it)."""
    strong = getattr(args, "scaling", "strong") == "strong"
    reps = REPS if strong else REPS * world
    return {"workload": "full study (configs[1]): 5 GPUs x {time n=189, power n=168} x 12 features, "
                        f"{reps}x10-fold CV, ntree {{128,256,512,1024}} x mtry {{12,3,3}}",
            "trees_per_step": len(datagen.GPU_NAMES) * 2 * reps * K_FOLDS * DISTINCT_MTRY * max(NTREES),
            "nominal_grid_trees_per_step": len(datagen.GPU_NAMES) * 2 * reps * K_FOLDS * len(MTRYS) * sum(NTREES),
            "l2": "flushed between timed steps (256 MB write)",
            "split": ("ExtraTrees, no bootstrap (P:468-469)" if args.split == "extra"
                      else "bootstrap + exact CART (north_star)"),
            "criterion": getattr(args, "criterion", "mse"),
            "tie_break": "lowest feature, then lowest threshold (north_star; R9)",
            "parallelism": f"{'task' if strong else 'repeat'}-sharded x{world} "
                           f"({'strong: one fixed study' if strong else 'weak: a study per rank'})",
            "cuda_streams": getattr(args, "streams", 1)}


def run_reference(args):
    """The oracle (plain single-threaded C), timed as it stands on the host."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    oracle = _oracle()
    ds = datagen.study(datagen.SEED)[0]  # K20 / time
    folds = oracle.make_folds(ds["y"], K_FOLDS, 1, seed=SEED, custom=True)
    # bounded sample: repeat 0, tasks (folds) 0..3 of one dataset, full grid (~3 s per step;
    # one task under MAE, whose oracle is ~10x slower per tree)
    sample_tasks = 1 if getattr(args, "criterion", "mse") == "mae" else 4

    def step():
        t0 = time.perf_counter()
        oracle.cv_grid(ds["X"], ds["y"], K_FOLDS, 1, NTREES, [12, 3], fold_ids=folds, target=1, seed=SEED,
                       task_begin=0, task_end=sample_tasks, **split_kw(args))
        return time.perf_counter() - t0

    for _ in range(args.warmup):
        step()
    ts = [step() for _ in range(args.steps)]
    trees = sample_tasks * DISTINCT_MTRY * max(NTREES)
    value = trees * len(ts) / sum(ts)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(ts) / len(ts),
        "higher_is_better": True, "scaling": "strong" if args.scaling == "strong" else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(study_config(args, 1), reference_sample=f"per step: K20/time, repeat 0, folds "
                       f"0-{sample_tasks - 1}, ntree {{128..1024}} x mtry {{12,3}} = {trees} trees"),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"{trees} trees ({sample_tasks} CV tasks x 2 mtry x 1024) of the K20 time dataset per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# --------------------------------------------------------------- our arm ----
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2001_07104_b200 as rfg
    from paper_2001_07104_b200.dist import cv_study_sharded, gather_task_tables

    rank, world, local = dist_env()
    # test hooks of the multi-rank driver on a one-GPU box (tests/test_gpu_dist.py): gloo instead of
    # NCCL and every rank on cuda:0 -- a functional check of this path, never a measurement
    backend = os.environ.get("RF_BENCH_BACKEND", "nccl")
    if os.environ.get("RF_BENCH_SAME_GPU") == "1":
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    def all_reduce_(t, op=dist.ReduceOp.SUM):  # gloo: through the host
        if backend == "nccl":
            dist.all_reduce(t, op=op)
        else:
            c = t.cpu()
            dist.all_reduce(c, op=op)
            t.copy_(c)
    rfg.lib()
    stream = torch.cuda.current_stream()
    ds = datagen.study(datagen.SEED)
    strong = args.scaling == "strong"
    reps_total = REPS if strong else REPS * world
    dX = [torch.as_tensor(d["X"], device=dev) for d in ds]
    dy = [torch.as_tensor(d["y"], device=dev) for d in ds]
    folds = [torch.empty((reps_total, d["X"].shape[0]), dtype=torch.int32, device=dev) for d in ds]
    out = [torch.empty((len(MTRYS), len(NTREES), reps_total, K_FOLDS), dtype=torch.float64, device=dev) for _ in ds]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > L2 (126 MB)
    skw = split_kw(args)
    datasets = [dict(X=dX[i], y=dy[i], target=1 if d["target"] == "time" else 0, seed=SEED + i)
                for i, d in enumerate(ds)]
    # one CUDA stream per dataset: the launches of a step overlap, so each launch's last partial
    # wave of CTAs is filled by the next dataset's work (--streams 1: serial)
    streams = [torch.cuda.Stream(device=dev) for _ in ds] if args.streams > 1 else None
    task_lo, task_hi = rank * REPS * K_FOLDS, (rank + 1) * REPS * K_FOLDS  # weak scaling

    def step():
        for i, d in enumerate(ds):
            rfg.make_folds(dy[i], K_FOLDS, reps_total, seed=SEED + i, custom=d["target"] == "time", out=folds[i])
        if strong:
            cv_study_sharded(datasets, K_FOLDS, reps_total, NTREES, MTRYS, folds=folds, outs=out, streams=streams,
                             **skw)
            return
        main = torch.cuda.current_stream()
        for i, d in enumerate(ds):
            st = streams[i % len(streams)] if streams else main
            st.wait_stream(main)
            with torch.cuda.stream(st):
                rfg.cross_validate_grid(dX[i], dy[i], K_FOLDS, reps_total, NTREES, MTRYS, fold_ids=folds[i],
                                        target=datasets[i]["target"], seed=SEED + i, task_begin=task_lo,
                                        task_end=task_hi, out=out[i], **skw)
        for st in streams or []:
            main.wait_stream(st)
        if world > 1:  # a11: fold-MAPE tables of all ranks, in task order
            for i in range(len(ds)):
                mine = out[i].reshape(len(MTRYS), len(NTREES), -1)[:, :, task_lo:task_hi]
                out[i].copy_(gather_task_tables(mine, reps_total * K_FOLDS).reshape(out[i].shape))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    rfg.set_profiling(True)
    start = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    stop = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0, cands0 = rfg.counters()  # cumulative since process start (incl. warm-up)
    with ClockSampler(local) as clk:
        wall0 = time.perf_counter()
        for s in range(args.steps):
            flush.zero_()  # L2 flush between timed iterations (outside the events)
            start[s].record(stream)
            step()
            stop[s].record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
    launches1, cands1 = rfg.counters()
    launches, cands = launches1 - launches0, cands1 - cands0
    if world > 1:
        dist.barrier()
    dev_ms = sum(a.elapsed_time(b) for a, b in zip(start, stop))
    prof = rfg.last_profile()
    rfg.set_profiling(False)
    t = torch.tensor([dev_ms], dtype=torch.float64, device=dev)
    if world > 1:
        all_reduce_(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item()) / args.steps
    trees_per_step = len(ds) * reps_total * K_FOLDS * DISTINCT_MTRY * max(NTREES)
    value = trees_per_step / (ms_per_step / 1e3)
    # candidates of all ranks (each rank counts its own)
    ct = torch.tensor([float(cands)], dtype=torch.float64, device=dev)
    if world > 1:
        all_reduce_(ct)
    cands_all = float(ct.item())

    # dominant kernel: the small-tree kernel, plain fp64/integer ALU bound
    kern_ms, kern_n = prof.get("small_tree", (0.0, 0))
    roofline = None
    if kern_n:
        # overlapping per-dataset streams: the kernel's busy time is bounded by the step's device time
        kern_busy_ms = min(kern_ms, dev_ms)
        achieved = cands * FLOPS_PER_CANDIDATE / (kern_busy_ms / 1e3) / 1e12
        roofline = {"bound": "alu", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s (fp64)",
                    "frac": achieved / FP64_PEAK_TFLOPS, "traffic": SMALL_TREE_DRAM_BYTES_PER_LAUNCH,
                    "traffic_source": "ncu --set full of one launch (one dataset): dram read + write bytes; the "
                                      "working set is on chip (profiles/README.md)",
                    "kernel": "small_tree_kernel",
                    "flops_per_candidate": FLOPS_PER_CANDIDATE,
                    "flops_definition": "SURVEY 8(d) C2: per evaluated candidate split 2 fp64 divisions + 2 squares "
                                        "+ 1 add (algorithmic, not the kernel's instruction count)",
                    "candidates_per_step": cands / args.steps,
                    "kernel_ms_per_step": kern_busy_ms / args.steps, "launches_per_step": kern_n / args.steps,
                    "kernel_share_of_step": kern_busy_ms / max(dev_ms, 1e-9),
                    "peak_source": FP64_PEAK_SOURCE,
                    "bound_context": "issue/latency bound, not fp64 bound: ncu shows ~12 warp instructions per "
                                     "candidate (profiles/README.md); the fraction is low by construction"}

    e2e = None
    if not args.no_e2e and world == 1:
        e2e = measure_e2e(rfg, ds, args, skw)
    elif not args.no_e2e and strong:
        e2e = measure_e2e_dist(rfg, ds, args, skw, rank, world, all_reduce_)
    configs = None
    if rank == 0 and world == 1 and not args.no_configs:
        configs = run_configs(rfg, torch, args, dev, flush)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": study_config(args, world),
            "study_wall_s": ms_per_step / 1e3,
            "roofline": roofline,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "wall_s_timed": wall,
            "candidates_per_step_all_ranks": cands_all / args.steps,
            "kernels_ms_per_step": {k: v[0] / args.steps for k, v in prof.items()},
        }
        if e2e:
            line["e2e"] = e2e
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline_c2(skw)
        if configs:
            line["configs"] = configs
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def measure_e2e(rfg, ds, args, skw):
    """Same study through the host-pointer C ABI (rf_make_folds + rf_cross_validate_grid) with
    the inputs in pinned host memory: H2D of X, y and the fold ids and D2H of fold ids and fold
    MAPEs inside the timed region.  The ten datasets are issued from ten host threads (the
    host API runs each thread's calls on its own CUDA stream), as a user of the library would."""
    import concurrent.futures as cf

    import torch

    def pinned(a):
        t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
        t.numpy()[...] = a
        return t.numpy()

    Xs = [pinned(d["X"]) for d in ds]
    ys = [pinned(d["y"]) for d in ds]
    h2d = d2h = 0

    def one(i):
        d = ds[i]
        custom = d["target"] == "time"
        f = rfg.make_folds(ys[i], K_FOLDS, REPS, seed=SEED + i, custom=custom)
        fm = rfg.cross_validate_grid(Xs[i], ys[i], K_FOLDS, REPS, NTREES, MTRYS, fold_ids=f,
                                     target=1 if custom else 0, seed=SEED + i, **skw)
        # bytes copied: y (folds), X + y + fold ids (CV) in; fold ids and fold MAPEs out
        return ys[i].nbytes + Xs[i].nbytes + ys[i].nbytes + f.nbytes, f.nbytes + fm.nbytes

    pool = cf.ThreadPoolExecutor(max_workers=len(ds))

    def step():
        nonlocal h2d, d2h
        res = list(pool.map(one, range(len(ds))))
        h2d = sum(r[0] for r in res)
        d2h = sum(r[1] for r in res)
    step()
    t0 = time.perf_counter()
    n = max(1, min(args.steps, 3))
    for _ in range(n):
        step()
    dt = (time.perf_counter() - t0) / n
    pool.shutdown()
    trees = len(ds) * REPS * K_FOLDS * DISTINCT_MTRY * max(NTREES)
    return {"value": trees / dt, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": dt * 1e3, "host_threads": len(ds),
            "api": "rf_make_folds + rf_cross_validate_grid (host pointers, pinned inputs)"}


def measure_e2e_dist(rfg, ds, args, skw, rank, world, all_reduce_):
    """e2e at N > 1 (strong scaling): each rank runs its (dataset, task) units of the fixed study
    (dist.study_units, as the device-timed step) through the host-pointer C ABI from pinned host
    memory, one host thread per unit, then the owned fold-MAPE columns of all ranks are
    all-gathered on the host -- every rank ends with the full tables.  Per step: barrier, the
    rank's wall time, max over ranks; bytes summed over ranks."""
    import concurrent.futures as cf

    import torch
    import torch.distributed as dist

    from paper_2001_07104_b200.dist import study_units

    def pinned(a):
        t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
        t.numpy()[...] = a
        return t.numpy()

    Xs = [pinned(d["X"]) for d in ds]
    ys = [pinned(d["y"]) for d in ds]
    units = study_units([REPS * K_FOLDS] * len(ds), rank, world)
    G = len(MTRYS) * len(NTREES)

    def one(u):
        d, lo, hi = u
        custom = ds[d]["target"] == "time"
        f = rfg.make_folds(ys[d], K_FOLDS, REPS, seed=SEED + d, custom=custom)
        fm = rfg.cross_validate_grid(Xs[d], ys[d], K_FOLDS, REPS, NTREES, MTRYS, fold_ids=f,
                                     target=1 if custom else 0, seed=SEED + d, task_begin=lo, task_end=hi, **skw)
        cols = fm.reshape(G, -1)[:, lo:hi]
        return cols, ys[d].nbytes + Xs[d].nbytes + ys[d].nbytes + f.nbytes, f.nbytes + fm.nbytes

    pool = cf.ThreadPoolExecutor(max_workers=max(1, len(units)))
    io = [0, 0]

    def step():
        res = list(pool.map(one, units))
        tables = [None] * world
        dist.all_gather_object(tables, [r[0] for r in res])  # the full study's tables on every rank
        io[0], io[1] = sum(r[1] for r in res), sum(r[2] for r in res)
        return tables

    step()
    n = max(1, min(args.steps, 3))
    dts = []
    for _ in range(n):
        dist.barrier()
        t0 = time.perf_counter()
        step()
        dts.append(time.perf_counter() - t0)
    pool.shutdown()
    t = torch.tensor([sum(dts) / n], dtype=torch.float64, device="cuda")
    all_reduce_(t, op=dist.ReduceOp.MAX)
    b = torch.tensor([float(io[0]), float(io[1])], dtype=torch.float64, device="cuda")
    all_reduce_(b)
    dt = float(t.item())
    trees = len(ds) * REPS * K_FOLDS * DISTINCT_MTRY * max(NTREES)
    return {"value": trees / dt, "unit": UNIT, "h2d_bytes_per_step": int(b[0].item()),
            "d2h_bytes_per_step": int(b[1].item()), "ms_per_step": dt * 1e3, "host_threads_per_rank": len(units),
            "api": "rf_make_folds + rf_cross_validate_grid (host pointers, pinned inputs, task ranges per rank), "
                   "tables all-gathered on the host; max over ranks"}


# dram__bytes_read.sum + dram__bytes_write.sum of one small_tree_kernel launch (one dataset of the
# study), ncu --set full (profiles/README.md)
SMALL_TREE_DRAM_BYTES_PER_LAUNCH = 2.25e6

from bench_configs import run_configs  # noqa: E402  (C1, C3, C4, C5 objects)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    run_ours(args)


if __name__ == "__main__":
    main()
