"""Host-pointer rf_predict of 10M pinned rows through a 1000-tree depth-12 forest with the pipelined
chunking at several chunk sizes (predict_chunk_rows; 20M = one unpipelined call)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2001_07104_b200 as rfg  # noqa: E402

Xd, yd = datagen.scaled_device(1_000_000, 64)
f = rfg.fit(Xd, yd, ntree=1000, mtry=21, max_depth=12, split_mode=1, target=1, seed=7104)
n = 10_000_000
Qd = torch.as_tensor(datagen.queries(1_000_000, 64), device="cuda").repeat(10, 1)
Qh = torch.empty(Qd.shape, dtype=torch.float64, pin_memory=True)
Qh.copy_(Qd)
Qn = Qh.numpy()
out = np.empty(n)
for chunk in (0, 20_000_000, 5_000_000, 2_500_000, 1_000_000, 0):
    rfg.debug_set_option("predict_chunk_rows", chunk)
    rfg.predict(f, Qn)
    t0 = time.perf_counter()
    for _ in range(2):
        rfg.predict(f, Qn)
    dt = (time.perf_counter() - t0) / 2
    print(chunk, round(dt * 1e3, 1), "ms", round(n / dt / 1e6, 2), "M pred/s", flush=True)
rfg.debug_set_option("predict_chunk_rows", 0)
od = torch.empty(n, dtype=torch.float64, device="cuda")
rfg.predict(f, Qd, out=od)
torch.cuda.synchronize()
t0 = time.perf_counter()
rfg.predict(f, Qd, out=od)
torch.cuda.synchronize()
print("device", round((time.perf_counter() - t0) * 1e3, 1), "ms")
