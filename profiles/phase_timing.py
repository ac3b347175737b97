"""Per-phase cycle split of the warp-per-tree kernel on the full-study workload.

  RF_PHASE_TIMING=1 python -m paper_2001_07104_b200.build
  RFGPU_LIB=$PWD/paper_2001_07104_b200/librfgpu_pt.so python profiles/phase_timing.py [exact|extra|mae|extra_mae]

Runs the K20/time dataset of the study (30 x 10-fold, ntree <= 1024, mtry {12,3})
once for warm-up, then once measured; prints each phase's share of the summed
warp cycles (clock64 deltas, lane 0 of every warp).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2001_07104_b200 as rfg  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "exact"
kw = {"split_mode": rfg.SPLIT_EXTRA, "bootstrap": False} if mode.startswith("extra") else {}
if mode.endswith("mae"):
    kw["criterion"] = 1
for ds in datagen.study(datagen.SEED)[:2]:
    X = torch.as_tensor(ds["X"], device="cuda")
    y = torch.as_tensor(ds["y"], device="cuda")
    custom = ds["target"] == "time"
    f = rfg.make_folds(y, 10, 30, seed=7104, custom=custom)
    args = (X, y, 10, 30, [128, 256, 512, 1024], [12, 3, 3])
    rfg.cross_validate_grid(*args, fold_ids=f, target=1 if custom else 0, seed=7104, **kw)
    rfg.phase_cycles(reset=True)
    rfg.cross_validate_grid(*args, fold_ids=f, target=1 if custom else 0, seed=7104, **kw)
    ph = rfg.phase_cycles(reset=True)
    tot = sum(ph.values()) or 1
    print(f"== {mode} {ds['gpu']}/{ds['target']} n={ds['X'].shape[0]}: {tot:.3e} warp-cycles")
    for k, v in ph.items():
        if v:
            print(f"  {k:45s} {100 * v / tot:5.1f}%")
