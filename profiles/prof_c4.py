"""C4 shape (device-generated scaled(N, 64), histogram mode, mtry 21, max_depth 12), T trees,
for ncu launch lists and per-kernel profiles:

  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4.csv \
      python profiles/prof_c4.py 10000000 89
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2001_07104_b200 as rfg  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
T = int(sys.argv[2]) if len(sys.argv) > 2 else 4
Xd, yd = datagen.scaled_device(N, 64)
torch.cuda.synchronize()
rfg.fit(Xd, yd, ntree=T, mtry=21, target=1, seed=7, max_depth=12, split_mode=rfg.SPLIT_HIST256)
torch.cuda.synchronize()
