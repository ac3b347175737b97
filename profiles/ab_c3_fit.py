"""A/B of large-path builds on the C3 shape (100k x 64, exact, mtry 21, 500 trees, one batch):
per library, a warm-up fit, then two timed fits with the library's per-phase profile.

  python profiles/ab_c3_fit.py librfgpu.so librfgpu_<tag>.so ...   (alternate them for A/B/A/B)
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import json, sys, time, torch
sys.path.insert(0, %r)
import datagen, paper_2001_07104_b200 as rfg
X, y = datagen.scaled(100_000, 64)
Xd, yd = torch.as_tensor(X, device="cuda"), torch.as_tensor(y, device="cuda")
rfg.fit(Xd, yd, ntree=500, mtry=21, target=1, seed=7)
torch.cuda.synchronize()
for rep in range(2):
    rfg.set_profiling(True)
    t0 = time.perf_counter()
    rfg.fit(Xd, yd, ntree=500, mtry=21, target=1, seed=7)
    torch.cuda.synchronize()
    sec = time.perf_counter() - t0
    prof = {k: round(v[0], 2) for k, v in rfg.last_profile().items()}
    rfg.set_profiling(False)
    print(round(500 / sec, 1), round(sec * 1e3, 1), json.dumps(prof))
''' % ROOT
for lib in sys.argv[1:]:
    env = dict(os.environ, RFGPU_LIB=os.path.join(ROOT, "paper_2001_07104_b200", lib))
    print("==", lib, flush=True)
    r = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True, timeout=600)
    print(r.stdout.strip() or r.stderr[-2000:], flush=True)
