"""One small-tree kernel launch of the full study (K20/time dataset, 30 x 10-fold
CV, ntree <= 1024, mtry {12, 3}) for ncu captures:

  ncu --set full --import-source on --clock-control none -k regex:small_tree_kernel -c 1 \
      -o gpurun_out/prof python profiles/prof_small_launch.py [exact|extra]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2001_07104_b200 as rfg  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "exact"
kw = {"split_mode": rfg.SPLIT_EXTRA, "bootstrap": False} if mode == "extra" else {}
ds = datagen.study(datagen.SEED)[0]
X = torch.as_tensor(ds["X"], device="cuda")
y = torch.as_tensor(ds["y"], device="cuda")
f = rfg.make_folds(y, 10, 30, seed=7104, custom=True)
rfg.cross_validate_grid(X, y, 10, 30, [128, 256, 512, 1024], [12, 3, 3], fold_ids=f, target=1, seed=7104, **kw)
torch.cuda.synchronize()
