import sys, time, torch
sys.path.insert(0, '/root/repo')
import datagen, paper_2001_07104_b200 as rfg
X, y = datagen.scaled(100_000, 64)
Xd, yd = torch.as_tensor(X, device="cuda"), torch.as_tensor(y, device="cuda")
rfg.fit(Xd, yd, ntree=500, mtry=21, target=1, seed=7); torch.cuda.synchronize()
for prof in (False, True, False, True):
    rfg.set_profiling(prof)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter(); rfg.fit(Xd, yd, ntree=500, mtry=21, target=1, seed=7); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    p = rfg.last_profile() if prof else {}
    rfg.set_profiling(False)
    print('prof', prof, [round(t*1e3,1) for t in ts], {k: round(v[0]/3,1) for k, v in p.items()}, flush=True)
