"""Per-config measurements of BASELINE.json's other configurations, used by
bench.py for the "configs" object of its JSON line (and runnable alone):

  C1  paper-shaped CV: 189 x 12, K20 time, 100 trees, mtry 12, 10-fold    (trees/s)
  C3  100k x 64 exact presorted, mtry 21, 500 trees (+ predict 100k rows)   (trees/s)
  C4  10M x 64, 256-bin histograms, mtry 21, depth 12, 1000 trees           (trees/s)
  C5  100M query rows through the C4 forest + single-query latency          (predictions/s)

Each object: value / unit / ms (CUDA events on the launching stream, L2 flushed or inputs
larger than L2), the roofline of the dominant kernel (algorithmic bytes or flops per DESIGN.md
sec. 6), cpu_baseline (the oracle as it stands: 1 core and N pinned cores, bounded samples,
extrapolations labelled), e2e through the host-pointer C ABI (copies inside the timed region)
and the SM clocks sampled during the timed region.

  python bench_configs.py [--configs c1,c3,c4,c5] [--no-cpu-baseline] [--no-e2e]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402

C4_ROWS, C4_TREES, C5_ROWS = 10_000_000, 1000, 100_000_000


def _bench():
    import bench
    return bench


def _timed(torch, fn, steps, warmup, flush=None, clock_index=0):
    """warmup untimed calls, then `steps` calls each bracketed by CUDA events on the current
    stream (L2 flushed before each when `flush` is given); clocks sampled over the timed part."""
    B = _bench()
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    with B.ClockSampler(clock_index) as clk:
        for a, b in ev:
            if flush is not None:
                flush.zero_()
            a.record(st)
            fn()
            b.record(st)
        torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in ev]
    return float(np.mean(ms)), clk.summary()


def _pinned(torch, a):
    t = torch.empty(a.shape, dtype=torch.float64 if a.dtype == np.float64 else torch.int32, pin_memory=True)
    t.numpy()[...] = a
    return t.numpy()


# ------------------------------------------------------------------ C1 ------
def _c1_oracle(a):
    oracle = _bench()._oracle()
    X, y = datagen.paper_shaped(189, "K20", "time")
    folds = oracle.make_folds(y, 10, a["reps"], seed=7104, custom=True)
    t0 = time.perf_counter()
    oracle.cv_grid(X, y, 10, a["reps"], [100], [12], fold_ids=folds, target=1, seed=7104, task_begin=a["lo"],
                   task_end=a["hi"])
    return (a["hi"] - a["lo"]) * 100, time.perf_counter() - t0


def c1(rfg, torch, flush, cpu=True, e2e=True):
    X, y = datagen.paper_shaped(189, "K20", "time")
    Xd, yd = torch.as_tensor(X, device="cuda"), torch.as_tensor(y, device="cuda")
    f = rfg.make_folds(yd, 10, 1, seed=7104, custom=True)
    fm = torch.empty((1, 1, 1, 10), dtype=torch.float64, device="cuda")
    run = lambda: rfg.cross_validate_grid(Xd, yd, 10, 1, [100], [12], fold_ids=f, target=1, seed=7104, out=fm)
    run()
    torch.cuda.synchronize()
    # 2,000 steps (~1 s): long enough for the clock sampler to see the timed region.  The library's
    # per-launch profiling (two cudaEventCreate + records per scope) is off while timing -- at
    # 0.3 ms per step it cost ~40 % -- and on for a separate pass that gives the kernel times
    steps = 2000
    c0 = rfg.counters()[1]
    ms, clocks = _timed(torch, run, steps, 3, flush)
    cands = (rfg.counters()[1] - c0) / (steps + 3)
    psteps = 200
    rfg.set_profiling(True)
    _timed(torch, run, psteps, 0, flush)
    prof = rfg.last_profile()
    rfg.set_profiling(False)
    B = _bench()
    kms = prof.get("small_tree", (0.0, 1))[0] / psteps
    ach = cands * B.FLOPS_PER_CANDIDATE / (kms / 1e3) / 1e12 if kms else None
    out = {"workload": "C1 paper-shaped CV (configs[0]): 189 x 12 K20 time, LOG, custom 10-fold split, 1 repeat, "
                       "100 trees, mtry 12 (1,000 trees per step)",
           "metric": "trees trained/sec", "value": 1000 / (ms / 1e3), "unit": "trees/s", "ms_per_step": ms,
           "steps": steps, "warmup": 3, "l2": "flushed between timed steps", "clocks": clocks,
           "roofline": {"bound": "alu", "kernel": "small_tree_kernel", "achieved": ach, "peak": B.FP64_PEAK_TFLOPS,
                        "unit": "TFLOP/s (fp64)", "frac": ach / B.FP64_PEAK_TFLOPS if ach else None,
                        "traffic": None, "flops_per_candidate": B.FLOPS_PER_CANDIDATE,
                        "candidates_per_step": cands, "kernel_ms_per_step": kms,
                        "kernel_share_of_step": kms / ms, "peak_source": B.FP64_PEAK_SOURCE,
                        "note": "a 10-task launch fills 10 x 100 warps: launch- and latency-bound; HBM ~0"}}
    if e2e:
        Xh, yh = _pinned(torch, X), _pinned(torch, y)

        def host_step():
            fo = rfg.make_folds(yh, 10, 1, seed=7104, custom=True)
            return rfg.cross_validate_grid(Xh, yh, 10, 1, [100], [12], fold_ids=fo, target=1, seed=7104), fo
        host_step()
        t0 = time.perf_counter()
        for _ in range(200):
            r, fo = host_step()
        dt = (time.perf_counter() - t0) / 200
        out["e2e"] = {"value": 1000 / dt, "unit": "trees/s", "ms_per_step": dt * 1e3,
                      "h2d_bytes_per_step": int(yh.nbytes * 2 + Xh.nbytes + fo.nbytes),
                      "d2h_bytes_per_step": int(fo.nbytes + r.nbytes),
                      "api": "rf_make_folds + rf_cross_validate_grid (host pointers, pinned inputs)"}
    if cpu:
        trees, sec = _c1_oracle(dict(reps=1, lo=0, hi=10))
        n = B.ncores()
        tot, wall, used = _cores(_c1_oracle, [dict(reps=n, lo=10 * i, hi=10 * i + 10) for i in range(n)])
        out["cpu_baseline"] = {"value": trees / sec, "unit": "trees/s", "cores": 1, "kind": "oracle",
                               "sample": f"the whole C1 step ({trees} trees) on 1 core ({sec:.2f} s)",
                               "n_cores": {"value": tot / wall, "unit": "trees/s", "cores": used,
                                           "sample": f"{used} pinned processes, each one repeat of C1 "
                                                     f"(different Philox folds): {tot} trees, {wall:.2f} s"},
                               **B.host_info()}
    return out


def _cores(fn, args):
    """run fn(arg) -> (units, seconds) on one pinned process per arg; wall = slowest process's
    compute time (data generation inside the processes is excluded)."""
    B = _bench()
    import multiprocessing as mp
    cores = sorted(os.sched_getaffinity(0))[:len(args)]
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    ps = [ctx.Process(target=_core_worker, args=(c, fn, a, q)) for c, a in zip(cores, args)]
    for p in ps:
        p.start()
    res = [q.get() for _ in ps]
    for p in ps:
        p.join()
    del B
    return sum(r[0] for r in res), max(r[1] for r in res), len(ps)


def _core_worker(core, fn, a, q):
    try:
        os.sched_setaffinity(0, {core})
    except OSError:
        pass
    q.put(fn(a))


# ------------------------------------------------------------------ C3 ------
def _c3_oracle(a):
    oracle = _bench()._oracle()
    X, y = datagen.scaled(100_000, 64)
    t0 = time.perf_counter()
    oracle.fit(X, y, ntree=500, tree_begin=a["t"], tree_end=a["t"] + 1, mtry=21, target=1, seed=7)
    return 1, time.perf_counter() - t0


def c3(rfg, torch, flush, cpu=True, e2e=True):
    B = _bench()
    X, y = datagen.scaled(100_000, 64)
    Q = datagen.queries(100_000, 64)
    Xd, yd, Qd = (torch.as_tensor(a, device="cuda") for a in (X, y, Q))
    holder = {}

    def run():
        holder["f"] = rfg.fit(Xd, yd, ntree=500, mtry=21, target=1, seed=7)
    run()
    torch.cuda.synchronize()
    rfg.set_profiling(True)
    rfg.row_levels(reset=True)
    ms, clocks = _timed(torch, run, 3, 1, flush)
    rl = rfg.row_levels(reset=True) / 4  # per fit (warm-up included in the count: 1 + 3 calls)
    prof = rfg.last_profile()
    rfg.set_profiling(False)
    kms = {k: v[0] / 4 for k, v in prof.items()}  # per fit (warm-up + 3 timed calls recorded)
    info = holder["f"].info()
    pred = torch.empty(100_000, dtype=torch.float64, device="cuda")
    pms, _ = _timed(torch, lambda: rfg.predict(holder["f"], Qd, out=pred), 5, 2, flush)
    p, m = 64, 21
    peak, psrc = B.hbm_peak()
    s_ms, p_ms = kms.get("large_search", 0.0), kms.get("large_partition", 0.0)
    dom = "large_search" if s_ms >= p_ms else "large_partition"
    bytes_dom = rl * (4 * m if dom == "large_search" else 8 * p)
    ach = bytes_dom / (max(s_ms, p_ms) / 1e3) / 1e9 if max(s_ms, p_ms) else None
    comb = rl * (8 * p + 4 * m) / ((s_ms + p_ms) / 1e3) / 1e9 if s_ms + p_ms else None
    out = {"workload": "C3 (configs[2]): rf_fit scaled(100,000 x 64), exact presorted splits, mtry 21, 500 trees, "
                       "bootstrap, unbounded depth, LOG target",
           "metric": "trees trained/sec", "value": 500 / (ms / 1e3), "unit": "trees/s", "ms_per_step": ms,
           "steps": 3, "warmup": 1, "l2": "flushed between timed steps", "clocks": clocks,
           "nodes_per_tree": info["total_nodes"] / 500, "row_levels_per_tree": rl / 500,
           "kernels_ms_per_fit": kms,
           "predict_100k_rows": {"ms": pms, "predictions_per_s": 1e5 / (pms / 1e3)},
           "roofline": {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak, "unit": "GB/s",
                        "frac": ach / peak if ach else None, "traffic": None,
                        "bytes_per_row_level": 4 * m if dom == "large_search" else 8 * p,
                        "algorithmic_bytes": "SURVEY 8(d) C3: search reads the m drawn lists' u32 entries "
                                             "(4m = 84 B per row-level); partition reads + writes all p lists "
                                             "(8p = 512 B); row-levels counted by the library",
                        "search_plus_partition_achieved": comb,
                        "search_plus_partition_frac": comb / peak if comb else None,
                        "peak_source": psrc}}
    if e2e:
        Xh, yh, Qh = _pinned(torch, X), _pinned(torch, y), _pinned(torch, Q)

        def host_step():
            f = rfg.fit(Xh, yh, ntree=500, mtry=21, target=1, seed=7)
            return rfg.predict(f, Qh)
        host_step()
        t0 = time.perf_counter()
        r = host_step()
        dt = time.perf_counter() - t0
        out["e2e"] = {"value": 500 / dt, "unit": "trees/s", "ms_per_step": dt * 1e3,
                      "h2d_bytes_per_step": int(Xh.nbytes + yh.nbytes + Qh.nbytes), "d2h_bytes_per_step": int(r.nbytes),
                      "api": "rf_fit + rf_predict of 100k held-out rows (host pointers, pinned inputs)"}
    if cpu:
        _, sec = _c3_oracle(dict(t=0))
        n = B.ncores()
        tot, wall, used = _cores(_c3_oracle, [dict(t=i) for i in range(n)])
        out["cpu_baseline"] = {"value": 1 / sec, "unit": "trees/s", "cores": 1, "kind": "oracle",
                               "sample": f"tree 0 of the C3 forest on 1 core ({sec:.1f} s)",
                               "n_cores": {"value": tot / wall, "unit": "trees/s", "cores": used,
                                           "sample": f"{used} pinned processes, trees 0..{used - 1} (one each), "
                                                     f"{wall:.1f} s"},
                               **B.host_info()}
    return out


# ------------------------------------------------------------------ C4 ------
C4_SAMPLE_ROWS = 1_000_000


def _c4_oracle(a):
    oracle = _bench()._oracle()
    X, y = datagen.scaled(C4_SAMPLE_ROWS, 64)
    t0 = time.perf_counter()
    oracle.fit(X, y, ntree=C4_TREES, tree_begin=a["t"], tree_end=a["t"] + 1, mtry=21, max_depth=12, split_mode=1,
               target=1, seed=7104)
    return 1, time.perf_counter() - t0


def c4(rfg, torch, flush, cpu=True, e2e=True):
    """Returns (object, forest) -- C5 reuses the forest."""
    B = _bench()
    X, y = datagen.scaled_device(C4_ROWS, 64)
    holder = {}

    def run():
        holder["f"] = None  # free the previous forest before the next fit
        holder["f"] = rfg.fit(X, y, ntree=C4_TREES, mtry=21, max_depth=12, split_mode=1, target=1, seed=7104)
    rfg.set_profiling(True)
    rfg.row_levels(reset=True)
    # two timed fits (one alone was exposed to a 13 % outlier in rd2_59 that the A/B of rd2_60 did
    # not reproduce); the profile and row-levels counters cover the warm-up fit too (3 fits)
    ms, clocks = _timed(torch, run, 2, 1)
    rl = rfg.row_levels(reset=True) / 3
    prof = rfg.last_profile()
    rfg.set_profiling(False)
    kms = {k: v[0] / 3 for k, v in prof.items()}
    info = holder["f"].info()
    m = 21
    peak, psrc = B.hbm_peak()
    # searched nodes ~ internal nodes (+ open nodes without a valid cut): (nodes - trees) / 2
    searched = (info["total_nodes"] - C4_TREES) / 2
    hist_bytes = searched * m * 256 * 12 * 2  # histograms written once and read once per searched node
    s_ms = kms.get("hist_search", 0.0)
    ach = (rl * 77 + hist_bytes) / (s_ms / 1e3) / 1e9 if s_ms else None
    fit_bytes = rl * 81 + hist_bytes
    out = {"workload": "C4 (configs[3]): rf_fit scaled(10,000,000 x 64) generated on the device, 256-bin "
                       "quantile histograms, mtry 21, max_depth 12, 1000 trees, bootstrap, LOG target, 1 GPU",
           "metric": "trees trained/sec", "value": C4_TREES / (ms / 1e3), "unit": "trees/s", "ms_per_step": ms,
           "steps": 2, "warmup": 1, "l2": "inputs (5.1 GB X, 640 MB bins) larger than L2", "clocks": clocks,
           "nodes_per_tree": info["total_nodes"] / C4_TREES, "row_levels_per_tree": rl / C4_TREES,
           "kernels_ms_per_fit": kms,
           "whole_fit_hbm": {"algorithmic_bytes": fit_bytes, "achieved": fit_bytes / (ms / 1e3) / 1e9,
                             "frac": fit_bytes / (ms / 1e3) / 1e9 / peak,
                             "roofline_s": fit_bytes / (peak * 1e9)},
           "roofline": {"bound": "hbm", "kernel": "hist_search (k_hist_build + k_hist_best)", "achieved": ach,
                        "peak": peak, "unit": "GB/s", "frac": ach / peak if ach else None, "traffic": None,
                        "bytes_per_row_level": 77,
                        "algorithmic_bytes": "SURVEY 8(d) C4: per row-level row id 4 + binned row 64 (two 32-B "
                                             "sectors) + t_q 8 + w 1 = 77 B (the partition's 4-B write is the "
                                             "partition kernel's), plus per searched node m x 256 x 12 B of "
                                             "histograms written and read",
                        "kernel_share_of_step": s_ms / ms if ms else None, "peak_source": psrc}}
    if e2e:
        Xh = torch.empty(X.shape, dtype=torch.float64, pin_memory=True)
        yh = torch.empty(y.shape, dtype=torch.float64, pin_memory=True)
        Xh.copy_(X)
        yh.copy_(y)
        Xn, yn = Xh.numpy(), yh.numpy()
        holder["f"] = None
        t0 = time.perf_counter()
        f = rfg.fit(Xn, yn, ntree=C4_TREES, mtry=21, max_depth=12, split_mode=1, target=1, seed=7104)
        e = f.export()
        dt = time.perf_counter() - t0
        d2h = sum(v.nbytes for v in e.values() if isinstance(v, np.ndarray))
        out["e2e"] = {"value": C4_TREES / dt, "unit": "trees/s", "ms_per_step": dt * 1e3,
                      "h2d_bytes_per_step": int(Xn.nbytes + yn.nbytes), "d2h_bytes_per_step": int(d2h),
                      "api": "rf_fit (host pointers, pinned 5.1 GB X) + rf_forest_export of the whole forest"}
        holder["f"] = f
        del Xh, yh
    if cpu:
        _, sec = _c4_oracle(dict(t=0))
        n = min(B.ncores(), 8)
        tot, wall, used = _cores(_c4_oracle, [dict(t=i) for i in range(n)])
        scale = C4_ROWS / C4_SAMPLE_ROWS
        out["cpu_baseline"] = {"value": 1 / (sec * scale), "unit": "trees/s", "cores": 1, "kind": "oracle",
                               "sample": f"tree 0 on the 1M-row sample scaled(1,000,000 x 64) (same recipe), "
                                         f"{sec:.1f} s incl. its cuts/binning setup; time x {scale:.0f} "
                                         "for 10M rows (growth and setup linear or n log n in rows: labelled "
                                         "extrapolation)",
                               "n_cores": {"value": tot / (wall * scale), "unit": "trees/s", "cores": used,
                                           "sample": f"{used} pinned processes, one 1M-row tree each, {wall:.1f} s, "
                                                     f"x {scale:.0f} for 10M rows (host RAM bounds the count)"},
                               **B.host_info()}
    del X, y
    return out, holder["f"]


# ------------------------------------------------------------------ C5 ------
def _c5_oracle(a):
    oracle = _bench()._oracle()
    f = a["forest"]
    Q = datagen.queries(a["rows"], 64, seed=datagen.SEED + 17 * a["i"])
    t0 = time.perf_counter()
    oracle.predict(f, Q)
    return a["rows"], time.perf_counter() - t0


def c5(rfg, torch, forest, cpu=True, e2e=True):
    B = _bench()
    Q = datagen.queries_device(C5_ROWS, 64)
    out_t = torch.empty(C5_ROWS, dtype=torch.float64, device="cuda")
    rfg.set_profiling(True)
    ms, clocks = _timed(torch, lambda: rfg.predict(forest, Q, out=out_t), 1, 1)
    rfg.set_profiling(False)
    info = forest.info()
    peak, psrc = B.hbm_peak()
    bts = C5_ROWS * (8 * 64 + 8)
    ach = bts / (ms / 1e3) / 1e9
    res = {"workload": "C5 (configs[4]): the C4 forest (1000 trees, depth <= 12) over 100,000,000 query rows "
                       "scaled(., 64, seed + 1) generated on the device, plus single-query latency",
           "metric": "predictions/sec", "value": C5_ROWS / (ms / 1e3), "unit": "predictions/s", "ms_per_step": ms,
           "steps": 1, "warmup": 1, "l2": "inputs (51.2 GB) larger than L2", "clocks": clocks,
           "tree_visits_per_s": C5_ROWS * info["ntree"] / (ms / 1e3),
           "roofline": {"bound": "hbm", "kernel": "k_predict_batch", "achieved": ach, "peak": peak, "unit": "GB/s",
                        "frac": ach / peak, "traffic": None, "bytes_per_row": 8 * 64 + 8,
                        "algorithmic_bytes": "SURVEY 8(d) C5: per query row its 64 fp64 features + the fp64 "
                                             "prediction (520 B)",
                        "peak_source": psrc,
                        "note": "the node walks bound the kernel, not HBM (SURVEY 8(d) C5): up to 13 dependent 8-B "
                                "node reads per tree, the top 7 levels from shared memory, the rest as two "
                                "64-B three-level blocks from L1/L2 (DESIGN.md sec. 5)"}}
    del Q
    # single-query latency (host API, warm): the C4 forest and a 512-tree paper-shaped forest
    q1 = datagen.queries(1, 64)
    lat = []
    for i in range(2005):
        t0 = time.perf_counter()
        rfg.predict(forest, q1)
        lat.append(time.perf_counter() - t0)
    lat = np.array(lat[5:]) * 1e3
    X2, y2 = datagen.paper_shaped(189, "K20", "time")
    f2 = rfg.fit(X2, y2, ntree=512, mtry=12, target=1, seed=3)
    lat2 = []
    for i in range(2005):
        t0 = time.perf_counter()
        rfg.predict(f2, X2[:1])
        lat2.append(time.perf_counter() - t0)
    lat2 = np.array(lat2[5:]) * 1e3
    res["single_query_ms"] = {"c4_forest_p50": float(np.percentile(lat, 50)),
                              "c4_forest_p99": float(np.percentile(lat, 99)),
                              "paper_512_tree_forest_p50": float(np.percentile(lat2, 50)),
                              "paper_512_tree_forest_p99": float(np.percentile(lat2, 99)),
                              "calls": 2000, "api": "rf_predict, host pointers, one row, copies included",
                              "paper_context_ms": "15-108 (Xeon E5-2667 v3, scikit-learn; P:46, T4/T5)"}
    if e2e:
        chunk = C5_ROWS // 10
        Qh = torch.empty((chunk, 64), dtype=torch.float64, pin_memory=True)
        Qh.copy_(datagen.queries_device(chunk, 64))
        Qn = Qh.numpy()
        rfg.predict(forest, Qn[:1000])
        t0 = time.perf_counter()
        for _ in range(10):
            r = rfg.predict(forest, Qn)
        dt = time.perf_counter() - t0
        res["e2e"] = {"value": C5_ROWS / dt, "unit": "predictions/s", "ms_per_step": dt * 1e3,
                      "h2d_bytes_per_step": int(Qn.nbytes * 10), "d2h_bytes_per_step": int(r.nbytes * 10),
                      "api": "rf_predict (host pointers): 100M rows as 10 calls of 10M rows from one pinned "
                             "5.1 GB host buffer (the first 10M query rows), predictions copied back"}
        del Qh
    if cpu:
        oracle = B._oracle()
        X3, y3 = datagen.scaled(10_000, 64)
        of = oracle.fit(X3, y3, ntree=100, mtry=21, max_depth=12, split_mode=1, target=1, seed=7105)
        rows, sec = _c5_oracle(dict(forest=of, rows=20_000, i=0))
        n = B.ncores()
        tot, wall, used = _cores(_c5_oracle, [dict(forest=of, rows=20_000, i=i) for i in range(n)])
        sc = 1000 / 100
        res["cpu_baseline"] = {"value": rows / sec / sc, "unit": "predictions/s", "cores": 1, "kind": "oracle",
                               "sample": f"{rows} query rows through the oracle's own 100-tree depth-12 forest "
                                         f"(grown on scaled(10k, 64)) in {sec:.2f} s; / {sc:.0f} for 1000 trees "
                                         "(visits linear in trees: labelled extrapolation)",
                               "n_cores": {"value": tot / wall / sc, "unit": "predictions/s", "cores": used,
                                           "sample": f"{used} pinned processes x {rows} rows, {wall:.2f} s, / {sc:.0f}"},
                               **B.host_info()}
    return res


def run_configs(rfg, torch, args, dev, flush):
    sel = [c.strip() for c in args.configs.split(",") if c.strip()]
    cpu, e2e = not args.no_cpu_baseline, not args.no_e2e
    out = {}
    forest = None
    for c in sel:
        try:
            if c == "c1":
                out["C1"] = c1(rfg, torch, flush, cpu, e2e)
            elif c == "c3":
                out["C3"] = c3(rfg, torch, flush, cpu, e2e)
            elif c == "c4":
                out["C4"], forest = c4(rfg, torch, flush, cpu, e2e)
            elif c == "c5":
                if forest is None:
                    _, forest = c4(rfg, torch, flush, False, False)
                out["C5"] = c5(rfg, torch, forest, cpu, e2e)
        except Exception as ex:  # keep the headline line even if one config fails
            out[c.upper()] = {"error": f"{type(ex).__name__}: {ex}"}
        torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c3,c4,c5")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    a = ap.parse_args()
    import torch
    import paper_2001_07104_b200 as rfg
    torch.cuda.set_device(0)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    print(json.dumps(run_configs(rfg, torch, a, torch.device("cuda", 0), flush)), flush=True)


if __name__ == "__main__":
    main()
