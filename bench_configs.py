"""Measurements of the non-headline configs of BASELINE.json.

bench.py is the driver's contract (the full CV study, configs[1]); this script
times the other configurations through the same C ABI and prints one JSON line
per config.  It is not part of the driver contract.

  C1  paper-shaped CV: 189 x 12, K20 time, 100 trees, 10-fold (trees/s)
  C3  100k x 64, exact presorted, mtry 21, unbounded depth: rf_fit (trees/s)
      [--c3-trees to bound the run]
  C5  inference: forest over query rows (predictions/s), plus single-query latency

  python bench_configs.py [--configs c1,c3,c5] [--c3-trees 16] [--c5-rows 1000000]
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


def timed(fn, reps=3, warm=1):
    import torch
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps / 1e3


def c1(rfg, torch):
    X, y = datagen.paper_shaped(189, "K20", "time")
    Xd, yd = torch.as_tensor(X, device="cuda"), torch.as_tensor(y, device="cuda")
    f = rfg.make_folds(yd, 10, 1, seed=7104, custom=True)
    sec = timed(lambda: rfg.cross_validate_grid(Xd, yd, 10, 1, [100], [12], fold_ids=f, target=1, seed=7104), 10, 3)
    return {"config": "C1 paper-shaped CV (189x12, 100 trees, mtry 12, 10-fold)", "trees": 1000,
            "seconds": sec, "trees_per_s": 1000 / sec}


def c3(rfg, torch, ntrees):
    X, y = datagen.scaled(100_000, 64)
    Xd, yd = torch.as_tensor(X, device="cuda"), torch.as_tensor(y, device="cuda")
    rfg.fit(Xd, yd, ntree=ntrees, mtry=21, target=1, seed=7)  # warm-up (allocator pool, modules)
    torch.cuda.synchronize()
    rfg.set_profiling(True)
    rfg.row_levels(reset=True)
    t0 = time.perf_counter()
    f = rfg.fit(Xd, yd, ntree=ntrees, mtry=21, target=1, seed=7)
    torch.cuda.synchronize()
    sec = time.perf_counter() - t0
    rl = rfg.row_levels(reset=True)
    prof = rfg.last_profile()
    rfg.set_profiling(False)
    info = f.info()
    kms = {k: v[0] for k, v in prof.items()}
    # HBM roofline: algorithmic bytes per row-level =
    # partition 8p (read + write a u32 entry in each of the p lists) + search 4m (the m drawn
    # lists' entries); row-levels counted by the library (rf_debug_row_levels)
    p, m = 64, 21
    grow_ms = kms.get("large_search", 0.0) + kms.get("large_partition", 0.0)
    peak, src = hbm_peak()
    achieved = rl * (8 * p + 4 * m) / (grow_ms / 1e3) / 1e9 if grow_ms else None
    part_gbs = rl * 8 * p / (kms["large_partition"] / 1e3) / 1e9 if kms.get("large_partition") else None
    return {"config": f"C3 rf_fit 100k x 64 exact, mtry 21, unbounded depth ({ntrees} of 500 trees)",
            "trees": ntrees, "seconds": sec, "trees_per_s": ntrees / sec,
            "nodes_per_tree": info["total_nodes"] / ntrees, "row_levels_per_tree": rl / ntrees,
            "kernels_ms": kms,
            "roofline": {"bound": "hbm", "unit": "GB/s", "bytes_per_row_level": 8 * p + 4 * m,
                         "achieved": achieved, "peak": peak, "frac": achieved / peak if achieved else None,
                         "partition_achieved": part_gbs,
                         "partition_frac": part_gbs / peak if part_gbs else None,
                         "kernels": "large_search + large_partition (CUDA events, rfg.last_profile)",
                         "peak_source": src}}


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, KeyError, ValueError):
        return 6650.0, "B200_PROFILING.md fallback (MEASURED_PEAKS.json absent)"


def c4(rfg, torch, ntrees, nrows):
    X, y = datagen.scaled(nrows, 64)
    Xd, yd = torch.as_tensor(X, device="cuda"), torch.as_tensor(y, device="cuda")
    del X
    # warm-up at the timed size (allocator pool and batch buffers sized as in the timed call)
    rfg.fit(Xd, yd, ntree=ntrees, mtry=21, target=1, seed=7, max_depth=12, split_mode=1)
    torch.cuda.synchronize()
    rfg.set_profiling(True)
    t0 = time.perf_counter()
    f = rfg.fit(Xd, yd, ntree=ntrees, mtry=21, target=1, seed=7, max_depth=12, split_mode=1)
    torch.cuda.synchronize()
    sec = time.perf_counter() - t0
    prof = rfg.last_profile()
    rfg.set_profiling(False)
    info = f.info()
    return {"config": f"C4 rf_fit {nrows} x 64 histogram-256, mtry 21, max_depth 12 ({ntrees} of 1000 trees, 1 GPU)",
            "trees": ntrees, "seconds": sec, "trees_per_s": ntrees / sec,
            "nodes_per_tree": info["total_nodes"] / ntrees, "kernels_ms": {k: v[0] for k, v in prof.items()}}


def c5(rfg, torch, nrows):
    X, y = datagen.scaled(20_000, 64)
    f = rfg.fit(X, y, ntree=1000, mtry=21, target=1, seed=9, max_depth=12)
    Q = torch.as_tensor(datagen.queries(nrows, 64), device="cuda")
    out = torch.empty(nrows, dtype=torch.float64, device="cuda")
    sec = timed(lambda: rfg.predict(f, Q, out=out), 3, 1)
    # single query latency (host API, warm)
    q1 = datagen.queries(1, 64)
    lat = []
    for i in range(1005):
        t0 = time.perf_counter()
        rfg.predict(f, q1)
        lat.append(time.perf_counter() - t0)
    lat = np.array(lat[5:]) * 1e3
    X2, y2 = datagen.paper_shaped(189, "K20", "time")
    f2 = rfg.fit(X2, y2, ntree=512, mtry=12, target=1, seed=3)
    q2 = X2[:1]
    lat2 = []
    for i in range(1005):
        t0 = time.perf_counter()
        rfg.predict(f2, q2)
        lat2.append(time.perf_counter() - t0)
    lat2 = np.array(lat2[5:]) * 1e3
    return {"config": f"C5 inference: 1000-tree forest (depth<=12, grown on 20k x 64) over {nrows} query rows",
            "rows": nrows, "seconds": sec, "predictions_per_s": nrows / sec,
            "tree_visits_per_s": nrows * 1000 / sec,
            "single_query_ms_p50_p99": [float(np.percentile(lat, 50)), float(np.percentile(lat, 99))],
            "single_query_512tree_paper_forest_ms_p50_p99": [float(np.percentile(lat2, 50)),
                                                              float(np.percentile(lat2, 99))],
            "paper_latency_context_ms": "15-108 ms (Xeon E5-2667 v3, sklearn, P:46 / T4-T5)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c3,c5")
    ap.add_argument("--c3-trees", type=int, default=16)
    ap.add_argument("--c5-rows", type=int, default=1_000_000)
    ap.add_argument("--c4-trees", type=int, default=32)
    ap.add_argument("--c4-rows", type=int, default=10_000_000)
    a = ap.parse_args()
    import torch
    import paper_2001_07104_b200 as rfg
    torch.cuda.set_device(0)
    for c in a.configs.split(","):
        if c == "c1":
            r = c1(rfg, torch)
        elif c == "c3":
            r = c3(rfg, torch, a.c3_trees)
        elif c == "c4":
            r = c4(rfg, torch, a.c4_trees, a.c4_rows)
        elif c == "c5":
            r = c5(rfg, torch, a.c5_rows)
        else:
            continue
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
