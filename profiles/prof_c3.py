"""C3 shape (scaled(100k, 64), exact, mtry 21, unbounded depth), a few trees, for ncu
launch lists / captures of the large-path kernels:

  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3.csv \
      python profiles/prof_c3.py 8
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2001_07104_b200 as rfg  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 8
X, y = datagen.scaled(100_000, 64)
Xd, yd = torch.as_tensor(X, device="cuda"), torch.as_tensor(y, device="cuda")
rfg.fit(Xd, yd, ntree=T, mtry=21, target=1, seed=7)
torch.cuda.synchronize()
