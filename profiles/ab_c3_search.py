"""A/B of the large-path split search on C3 (100k x 64, exact, mtry 21): the warp-striped kernel
per library build (round 2: RF_SEARCH_UNROLL variants of a warp-striped kernel against the
thread-serial one via a test switch -- removed after this A/B; then RF_SEARCH_PF 0/1; then the
node-parallel search threshold KS=k1,k2,... via the "node_search_min" switch).

  python profiles/ab_c3_search.py librfgpu.so librfgpu_su1.so ...
"""
import json
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
out = {}
for k in KS:
    if k:
        rfg.debug_set_option("node_search_min", k)
    rfg.fit(Xd, yd, ntree=128, mtry=21, target=1, seed=7)
    torch.cuda.synchronize()
    rfg.set_profiling(True)
    t0 = time.perf_counter()
    rfg.fit(Xd, yd, ntree=500, mtry=21, target=1, seed=7)
    torch.cuda.synchronize()
    sec = time.perf_counter() - t0
    prof = rfg.last_profile()
    rfg.set_profiling(False)
    out[str(k)] = {"trees_per_s": 500 / sec, "search_ms": prof["large_search"][0],
                                              "partition_ms": prof["large_partition"][0]}
print(json.dumps(out))
''' % ROOT
KS = [int(v) for v in os.environ.get('KS', '0').split(',')]  # 0: no switch (the option existed only for rd2_22)
CODE = CODE.replace('for k in KS:', 'for k in %r:' % KS)
for lib in sys.argv[1:]:
    env = dict(os.environ, RFGPU_LIB=os.path.join(ROOT, "paper_2001_07104_b200", lib))
    r = subprocess.run([sys.executable, "-c", CODE], capture_output=True, text=True, env=env)
    print(lib, r.stdout.strip() or r.stderr[-800:], flush=True)
