"""Where the C1 host-API step's time goes: rf_make_folds and rf_cross_validate_grid through host
pointers (pinned inputs) vs the device twins, each timed over 200 calls (wall, synchronised)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2001_07104_b200 as rfg  # noqa: E402

X, y = datagen.paper_shaped(189, "K20", "time")
Xh = torch.empty(X.shape, dtype=torch.float64, pin_memory=True); Xh.numpy()[...] = X
yh = torch.empty(y.shape, dtype=torch.float64, pin_memory=True); yh.numpy()[...] = y
Xn, yn = Xh.numpy(), yh.numpy()
Xd, yd = torch.as_tensor(X, device="cuda"), torch.as_tensor(y, device="cuda")


def t(fn, n=200):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


fh = rfg.make_folds(yn, 10, 1, seed=7104, custom=True)
fd = rfg.make_folds(yd, 10, 1, seed=7104, custom=True)
print("make_folds host  ms", t(lambda: rfg.make_folds(yn, 10, 1, seed=7104, custom=True)))
print("make_folds dev   ms", t(lambda: rfg.make_folds(yd, 10, 1, seed=7104, custom=True)))
print("cv_grid host     ms", t(lambda: rfg.cross_validate_grid(Xn, yn, 10, 1, [100], [12], fold_ids=fh, target=1, seed=7104)))
print("cv_grid dev      ms", t(lambda: rfg.cross_validate_grid(Xd, yd, 10, 1, [100], [12], fold_ids=fd, target=1, seed=7104)))
rfg.set_profiling(True)
rfg.cross_validate_grid(Xn, yn, 10, 1, [100], [12], fold_ids=fh, target=1, seed=7104)
torch.cuda.synchronize()
print({k: (round(v[0], 4), v[1]) for k, v in rfg.last_profile().items()})
rfg.set_profiling(False)
