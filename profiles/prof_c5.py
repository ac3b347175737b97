"""One batched-inference launch of the C5 shape for ncu (1000-tree depth<=12 forest grown
on scaled(20k, 64), 1M query rows):

  ncu --set full --import-source on --clock-control none -k regex:k_predict -s 1 -c 1 \
      -o gpurun_out/c5 python profiles/prof_c5.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2001_07104_b200 as rfg  # noqa: E402

X, y = datagen.scaled(20_000, 64)
f = rfg.fit(X, y, ntree=1000, mtry=21, target=1, seed=9, max_depth=12)
Q = torch.as_tensor(datagen.queries(1_000_000, 64), device="cuda")
out = torch.empty(Q.shape[0], dtype=torch.float64, device="cuda")
for _ in range(2):
    rfg.predict(f, Q, out=out)
torch.cuda.synchronize()
