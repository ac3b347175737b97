"""Multi-rank driver on the GPU box: two ranks share cuda:0 (one GPU per
gpurun call) over a gloo process group, so every collective of paper_2001_07104_b200.dist runs
between real processes while the compute goes through the real library.  Each result must equal
the single-rank run of the same call: fold-MAPE tables and assembled forests bit-identical
(no floating-point reduction), tree-sharded sums within 1e-9 relative (summation order only).
"""
import os
import tempfile

import numpy as np
import pytest

import datagen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from test_dist import run_world  # noqa: E402

K, REPS, NTREES, MTRYS, SEED = 10, 3, [16, 32], [12, 3], 7104
OUT = os.environ.get("RF_DIST_TEST_DIR") or tempfile.mkdtemp(prefix="rfdist_")


def _datasets(dev):
    out = []
    for i, (gpu, target) in enumerate([("K20", "time"), ("P100", "power"), ("V100", "time")]):
        X, y = datagen.paper_shaped(189 if target == "time" else 168, gpu, target)
        out.append(dict(X=torch.as_tensor(X, device=dev), y=torch.as_tensor(y, device=dev),
                        target=1 if target == "time" else 0, seed=SEED + i, custom=target == "time"))
    return out


def _work(rank, world):
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    import paper_2001_07104_b200 as rfg
    from paper_2001_07104_b200 import dist as rd
    ds = _datasets(dev)
    # strong-scaled study: (dataset, task) units split across the ranks
    folds = [rfg.make_folds(d["y"], K, REPS, seed=d["seed"], custom=d["custom"]) for d in ds]
    outs = [torch.empty((len(MTRYS), len(NTREES), REPS, K), dtype=torch.float64, device=dev) for _ in ds]
    units = rd.cv_study_sharded(ds, K, REPS, NTREES, MTRYS, folds=folds, outs=outs)
    assert units and all(hi > lo for _, lo, hi in units)
    np.save(f"{OUT}/study_r{rank}.npy", torch.stack(outs).cpu().numpy())
    # weak-scaled study (each rank its own repeats)
    d = ds[0]
    fm = rd.cv_task_sharded(d["X"], d["y"], K, 2, NTREES, MTRYS, custom=True, seed=d["seed"], target=1)
    np.save(f"{OUT}/weak_r{rank}.npy", fm.cpu().numpy())
    # tree-sharded CV, incl. an empty shard (1 tree over 2 ranks)
    f0 = folds[0]
    for nt, tag in ((NTREES, "tree"), ([1], "tree1")):
        fm = rd.cv_tree_sharded(d["X"], d["y"], K, REPS, f0, nt, MTRYS, target=1, seed=d["seed"])
        np.save(f"{OUT}/{tag}_r{rank}.npy", fm.cpu().numpy())
    # tree-sharded fit, assembled on every rank; row-sharded prediction
    X, y = datagen.scaled(4000, 64)
    Xd, yd = torch.as_tensor(X, device=dev), torch.as_tensor(y, device=dev)
    f = rd.fit_sharded(Xd, yd, ntree=9, mtry=21, target=1, seed=3, max_depth=10)
    e = f.export()
    np.savez(f"{OUT}/fit_r{rank}.npz", **{k: v for k, v in e.items() if isinstance(v, np.ndarray)})
    Q = torch.as_tensor(datagen.queries(3001, 64), device=dev)
    np.save(f"{OUT}/pred_r{rank}.npy", rd.predict_row_sharded(f, Q).cpu().numpy())


def test_two_ranks_match_one_rank():
    import paper_2001_07104_b200 as rfg
    os.environ["RF_DIST_TEST_DIR"] = OUT
    run_world(_work, world=2)
    dev = torch.device("cuda", 0)
    ds = _datasets(dev)
    ref = []
    for d in ds:
        f = rfg.make_folds(d["y"], K, REPS, seed=d["seed"], custom=d["custom"])
        ref.append(rfg.cross_validate_grid(d["X"], d["y"], K, REPS, NTREES, MTRYS, fold_ids=f, target=d["target"],
                                           seed=d["seed"]).cpu().numpy())
    ref = np.stack(ref)
    for r in range(2):
        got = np.load(f"{OUT}/study_r{r}.npy")
        assert np.array_equal(got.view(np.int64), ref.view(np.int64)), f"rank {r} study table"
    d = ds[0]
    fw = rfg.make_folds(d["y"], K, 4, seed=d["seed"], custom=True)
    wref = rfg.cross_validate_grid(d["X"], d["y"], K, 4, NTREES, MTRYS, fold_ids=fw, target=1,
                                   seed=d["seed"]).cpu().numpy()
    for r in range(2):
        assert np.array_equal(np.load(f"{OUT}/weak_r{r}.npy").view(np.int64), wref.view(np.int64))
    f0 = rfg.make_folds(d["y"], K, REPS, seed=d["seed"], custom=True)
    for nt, tag in ((NTREES, "tree"), ([1], "tree1")):
        tref = rfg.cross_validate_grid(d["X"], d["y"], K, REPS, nt, MTRYS, fold_ids=f0, target=1,
                                       seed=d["seed"]).cpu().numpy()
        for r in range(2):
            np.testing.assert_allclose(np.load(f"{OUT}/{tag}_r{r}.npy"), tref, rtol=1e-9, atol=0)
    X, y = datagen.scaled(4000, 64)
    e = rfg.fit(X, y, ntree=9, mtry=21, target=1, seed=3, max_depth=10).export()
    Q = datagen.queries(3001, 64)
    pref = rfg.predict(rfg.fit(X, y, ntree=9, mtry=21, target=1, seed=3, max_depth=10), Q)
    for r in range(2):
        g = np.load(f"{OUT}/fit_r{r}.npz")
        for key in ("feature", "left", "thr_index", "tree_off"):
            assert np.array_equal(g[key], e[key]), (r, key)
        assert np.array_equal(g["value"].view(np.int64), e["value"].view(np.int64))
        assert np.array_equal(np.load(f"{OUT}/pred_r{r}.npy").view(np.int64), pref.view(np.int64))


def test_bench_multi_rank_path_on_one_gpu():
    """bench.py's N > 1 path (init, strong task sharding, barriers, max over ranks, the host-API e2e
    with host-side table gathers, rank-0-only JSON line) under torchrun with two ranks.  This box has
    one GPU, so both ranks run on cuda:0 over gloo (bench.py test hooks RF_BENCH_BACKEND /
    RF_BENCH_SAME_GPU): a functional check of the driver's scaling-run command, not a measurement."""
    import json
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    env = dict(os.environ, RF_BENCH_BACKEND="gloo", RF_BENCH_SAME_GPU="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(root, "bench.py"),
                        "--gpus", "2", "--steps", "1", "--warmup", "1", "--no-configs", "--no-cpu-baseline"],
                       capture_output=True, text=True, timeout=900, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["config"]["trees_per_step"] == 6144000  # the fixed study, split over the ranks
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["gpu_launches"] > 0
