"""Benchmark: the paper-shaped full CV study (BASELINE.json configs[1]).

Workload of one step ("full study"): 10 datasets = 5 GPUs
of Table 3 x {time (n=189, LOG, paper custom split), power (n=168, plain
k-fold)}, 30 repeats x 10-fold CV, grid ntree {128,256,512,1024} (prefixes of
1024-tree forests) x mtry {12 (max), 3 (sqrt), 3 (log2)}.  Distinct trees
grown per step per rank: 10 x 300 tasks x 2 distinct mtry x 1024 = 6,144,000.
Every step runs the whole hot path: validation + quantisation + presort
(a1, a3), folds (a2), bootstrap / feature draws / split search / partition /
leaves (a4-a8) in the small-tree kernel, CV scoring (a10); N>1 adds the
cross-rank gather of the fold-MAPE tables (a11).

Multi-GPU (weak scaling): rank r runs repeats [30 r, 30 r + 30) of a
30 N-repeat study (task sharding, no data-path collective besides the final
all_gather of MAPE tables).  value = trees grown by all ranks / max over
ranks of the device time.  Within a rank the ten datasets run on ten CUDA
streams (--streams 1: one after another).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--split exact|extra]
                  [--streams S] [--no-cpu-baseline] [--no-e2e]
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
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


# -------------------------------------------------------------- data -------
def study_config(args, world):
    """The workload both arms report (the reference arm times a bounded sample of it)."""
    return {"workload": "full study (configs[1]): 5 GPUs x {time n=189, power n=168} x 12 features, "
                        "30x10-fold CV per rank, ntree {128,256,512,1024} x mtry {12,3,3}",
            "trees_per_step": len(datagen.GPU_NAMES) * 2 * REPS * K_FOLDS * DISTINCT_MTRY * max(NTREES) * world,
            "nominal_grid_trees_per_step": len(datagen.GPU_NAMES) * 2 * REPS * K_FOLDS * len(MTRYS) * sum(NTREES)
            * world,
            "l2": "flushed between timed steps (256 MB write)",
            "split": ("ExtraTrees, no bootstrap (P:468-469)" if args.split == "extra"
                      else "bootstrap + exact CART (north_star)"),
            "criterion": getattr(args, "criterion", "mse"),
            "parallelism": f"task-sharded x{world}",
            "cuda_streams": getattr(args, "streams", 1)}


def study_inputs():
    return datagen.study(datagen.SEED)


# ------------------------------------------------------- reference arm ------
def run_reference(args):
    """The oracle (plain single-threaded C), timed as it stands on the host."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle
    oracle.build()
    ds = study_inputs()[0]  # K20 / time
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
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": dict(study_config(args, 1), reference_sample=f"per step: K20/time, repeat 0, folds "
                       f"0-{sample_tasks - 1}, ntree {{128..1024}} x mtry {{12,3}} = {trees} trees"),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"{trees} trees ({sample_tasks} CV tasks x 2 mtry x 1024) of the K20 time dataset per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def cpu_baseline_sample(skw):
    import oracle
    oracle.build()
    ds = study_inputs()[0]
    folds = oracle.make_folds(ds["y"], K_FOLDS, 1, seed=SEED, custom=True)
    tasks = 1 if skw.get("criterion") else 10  # one repeat of 10-fold CV: ~8 s on one host core (MAE: one fold)
    t0 = time.perf_counter()
    oracle.cv_grid(ds["X"], ds["y"], K_FOLDS, 1, NTREES, [12, 3], fold_ids=folds, target=1, seed=SEED,
                   task_begin=0, task_end=tasks, **skw)
    dt = time.perf_counter() - t0
    trees = tasks * DISTINCT_MTRY * max(NTREES)
    return {"value": trees / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{trees} trees: K20/time dataset, repeat 0 (folds 0-{tasks - 1}), ntree<=1024 x mtry {{12,3}} "
                      f"({dt:.1f} s on 1 host core)"}


# --------------------------------------------------------------- our arm ----
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2001_07104_b200 as rfg
    from paper_2001_07104_b200.dist import gather_task_tables

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    rfg.lib()
    stream = torch.cuda.current_stream()
    ds = study_inputs()
    reps_total = REPS * world
    task_lo, task_hi = rank * REPS * K_FOLDS, (rank + 1) * REPS * K_FOLDS
    dX = [torch.as_tensor(d["X"], device=dev) for d in ds]
    dy = [torch.as_tensor(d["y"], device=dev) for d in ds]
    folds = [torch.empty((reps_total, d["X"].shape[0]), dtype=torch.int32, device=dev) for d in ds]
    out = [torch.empty((len(MTRYS), len(NTREES), reps_total, K_FOLDS), dtype=torch.float64, device=dev) for _ in ds]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > L2 (126 MB)
    skw = split_kw(args)

    # one CUDA stream per dataset: the ten CV launches of a step overlap, so each launch's
    # last partial wave of CTAs is filled by the next dataset's work (--streams 1: serial)
    streams = [torch.cuda.Stream(device=dev) for _ in ds] if args.streams > 1 else None

    def one(i, d):
        custom = d["target"] == "time"
        rfg.make_folds(dy[i], K_FOLDS, reps_total, seed=SEED + i, custom=custom, out=folds[i])
        rfg.cross_validate_grid(dX[i], dy[i], K_FOLDS, reps_total, NTREES, MTRYS, fold_ids=folds[i],
                                target=1 if custom else 0, seed=SEED + i, task_begin=task_lo,
                                task_end=task_hi, out=out[i], **skw)

    def step():
        if streams is None:
            for i, d in enumerate(ds):
                one(i, d)
        else:
            main = torch.cuda.current_stream()
            for i, d in enumerate(ds):
                st = streams[i % len(streams)]
                st.wait_stream(main)
                with torch.cuda.stream(st):
                    one(i, d)
            for st in streams:
                main.wait_stream(st)
        if world > 1:  # a11: fold-MAPE tables of all ranks, in task order (NCCL all_gather)
            for i in range(len(ds)):
                mine = out[i].reshape(len(MTRYS), len(NTREES), -1)[:, :, task_lo:task_hi]
                out[i].copy_(gather_task_tables(mine, reps_total * K_FOLDS).reshape(out[i].shape))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # profile pass (per-kernel events) outside the timed loop is not used for the roofline;
    # the roofline uses events recorded inside the timed steps.
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
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item()) / args.steps
    trees_per_step_rank = len(ds) * REPS * K_FOLDS * DISTINCT_MTRY * max(NTREES)
    value = trees_per_step_rank * world / (ms_per_step / 1e3)

    # dominant kernel roofline: the small-tree kernel is ALU (fp64 + integer/SMEM issue) bound
    kern_ms, kern_n = prof.get("small_tree", (0.0, 0))
    roofline = None
    if kern_n:
        ops_per_cand = FP64_OPS_PER_CANDIDATE
        # with overlapping per-dataset streams the per-launch event spans overlap, so the kernel's
        # busy time is bounded by the step's device time
        kern_busy_ms = min(kern_ms, dev_ms)
        achieved = cands * ops_per_cand / (kern_busy_ms / 1e3) / 1e12
        peak = FP64_PEAK_TOPS
        roofline = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s (fp64 pipe ops)",
                    "frac": achieved / peak, "traffic": SMALL_TREE_DRAM_BYTES_PER_LAUNCH,
                    "traffic_source": "ncu --set full, one launch (one dataset, 614,400 trees): dram read + write "
                                      "bytes (profiles/r02i_small_tree_ncu.txt); the working set is on chip",
                    "kernel": "small_tree_kernel",
                    "ncu_context": {"ipc": 2.55, "issue_slots_busy_pct": 63.8, "warps_per_sm": 16,
                                    "top_stalls": "wait 37 %, short_scoreboard 17 %",
                                    "source": "profiles/r02i_small_tree_ncu.txt (latency-bound: the fp64 "
                                              "pipe fraction is low because each candidate also costs "
                                              "shared-memory scans and per-level node work)"},
                    "kernel_ms_per_step": kern_busy_ms / args.steps, "launches_per_step": kern_n / args.steps,
                    "kernel_share_of_step": kern_busy_ms / max(dev_ms, 1e-9),
                    "kernel_launch_spans_ms_per_step": kern_ms / args.steps,
                    "streams": args.streams,
                    "candidates_per_step": cands / args.steps, "fp64_ops_per_candidate": ops_per_cand,
                    "peak_source": "DESIGN.md sec. 6: 148 SM x 64 fp64 lanes x 1965 MHz (guide unit counts)"}

    e2e = None
    if not args.no_e2e and rank == 0 and world == 1:
        e2e = measure_e2e(rfg, ds, args, skw)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": study_config(args, world),
            "roofline": roofline,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "wall_s_timed": wall,
            "kernels_ms_per_step": {k: v[0] / args.steps for k, v in prof.items()},
        }
        if e2e:
            line["e2e"] = e2e
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline_sample(skw)
        print(json.dumps(line))
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


# fp64 arithmetic per evaluated candidate split: 2 squares (DMUL),
# 2 correctly rounded divisions by W <= 255 as DMUL + 2 DFMA each (Markstein), 1 DADD
FP64_OPS_PER_CANDIDATE = 9
# dram__bytes_read.sum + dram__bytes_write.sum of one small_tree_kernel launch (1.75 MB + 0.50 MB),
# from the round-1 final ncu --set full capture (profiles/r02i_small_tree_ncu.txt)
SMALL_TREE_DRAM_BYTES_PER_LAUNCH = 2.25e6
FP64_PEAK_TOPS = 148 * 64 * 1.965e9 / 1e12


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    run_ours(args)


if __name__ == "__main__":
    main()
