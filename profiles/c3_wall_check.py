"""C3 fit wall-time stability: 500-tree fits of scaled(100k, 64) in one process, each timed on
the host and with CUDA events on the stream, profiling off / on (rd2_24 .. rd2_27)."""
import sys
import time

import torch

sys.path.insert(0, '/root/repo')
import datagen  # noqa: E402
import paper_2001_07104_b200 as rfg  # noqa: E402

X, y = datagen.scaled(100_000, 64)
Xd, yd = torch.as_tensor(X, device="cuda"), torch.as_tensor(y, device="cuda")
rfg.fit(Xd, yd, ntree=500, mtry=21, target=1, seed=7)
torch.cuda.synchronize()
for prof in (False, True, False, True):
    rfg.set_profiling(prof)
    ts, ds = [], []
    for _ in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record()
        rfg.fit(Xd, yd, ntree=500, mtry=21, target=1, seed=7)
        b.record()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
        ds.append(a.elapsed_time(b))
    p = rfg.last_profile() if prof else {}
    rfg.set_profiling(False)
    print('prof', prof, 'wall', [round(t * 1e3, 1) for t in ts], 'events', [round(d, 1) for d in ds],
          {k: round(v[0] / 4, 1) for k, v in p.items()}, flush=True)
