"""Tiny end-to-end workload for compute-sanitizer (run by tests/test_gpu_tools.py):
CV on a paper-shaped slice (CTA-resident kernel, exact / ExtraTrees / MAE), a fit on
the level-synchronous path (fused and tiled partitions), the histogram mode, and
batched / single-row inference.  Exits non-zero on any library error."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import datagen  # noqa: E402
import paper_2001_07104_b200 as rfg  # noqa: E402

X, y = datagen.paper_shaped(60, "K20", "time")
f = rfg.make_folds(y, 5, 1, seed=3, custom=True)
rfg.cross_validate_grid(X, y, 5, 1, [4], [3], fold_ids=f, target=1, seed=3)
rfg.cross_validate_grid(X, y, 5, 1, [4], [12], fold_ids=f, target=1, seed=3, split_mode=rfg.SPLIT_EXTRA,
                        bootstrap=False)
rfg.cross_validate_grid(X, y, 5, 1, [4], [3], fold_ids=f, target=1, seed=3, criterion=rfg.CRITERION_MAE)
Xl, yl = datagen.tiny(300, 5, 2, distinct=40)
fl = rfg.fit(Xl, yl, ntree=2, mtry=3, seed=1, debug=True)
rfg.debug_set_option("large_tiled_partition", 1)
rfg.fit(Xl, yl, ntree=2, mtry=3, seed=1)
rfg.debug_set_option("large_tiled_partition", 0)
rfg.fit(Xl, yl, ntree=2, mtry=3, seed=1, split_mode=rfg.SPLIT_HIST256, max_depth=6)
Q = np.random.default_rng(0).normal(size=(400, 5))
rfg.predict(fl, Q)
rfg.predict(fl, Q[:3])
print("sanitize case ok")
