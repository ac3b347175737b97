"""C4 shape at reduced rows (scaled(N, 64), histogram mode, mtry 21, max_depth 12), a few
trees, for ncu launch lists:

  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4.csv \
      python profiles/prof_c4.py 2000000 4
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2001_07104_b200 as rfg  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
T = int(sys.argv[2]) if len(sys.argv) > 2 else 4
X, y = datagen.scaled(N, 64)
Xd, yd = torch.as_tensor(X, device="cuda"), torch.as_tensor(y, device="cuda")
rfg.fit(Xd, yd, ntree=T, mtry=21, target=1, seed=7, max_depth=12, split_mode=rfg.SPLIT_HIST256)
torch.cuda.synchronize()
