"""World-size-2 gloo tests (CPU) of the multi-GPU driver's host logic:
sharding, MAPE-table gathering in task order, partial-sum reduction and
forest assembly from tree shards (compared with the oracle's full forest)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import datagen
import oracle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world)
        q.put((rank, "ok"))
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def run_world(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for r, msg in res:
        assert msg == "ok", f"rank {r}: {msg}"


def test_shard_ranges():
    from paper_2001_07104_b200.dist import shard
    for total in (1, 7, 128, 1000, 1024):
        for world in (1, 2, 3, 8):
            rngs = [shard(total, r, world) for r in range(world)]
            assert rngs[0][0] == 0 and rngs[-1][1] == total
            assert all(rngs[i][1] == rngs[i + 1][0] for i in range(world - 1))
            assert max(h - l for l, h in rngs) - min(h - l for l, h in rngs) <= 1


def _gather_tables(rank, world):
    from paper_2001_07104_b200.dist import gather_task_tables
    k, reps_per = 10, 3
    full = torch.arange(3 * 4 * reps_per * world * k, dtype=torch.float64).reshape(3, 4, reps_per * world * k)
    lo, hi = rank * reps_per * k, (rank + 1) * reps_per * k
    got = gather_task_tables(full[:, :, lo:hi].clone(), reps_per * world * k)
    assert torch.equal(got, full)


def test_gather_task_tables():
    run_world(_gather_tables)


def _reduce(rank, world):
    from paper_2001_07104_b200.dist import reduce_partials
    x = torch.full((5,), float(rank + 1), dtype=torch.float64)
    reduce_partials(x)
    assert torch.equal(x, torch.full((5,), 3.0, dtype=torch.float64))


def test_reduce_partials():
    run_world(_reduce)


def _assemble(rank, world):
    from paper_2001_07104_b200.dist import allgather_forest_arrays, shard
    X, y = datagen.paper_shaped(189, "K20", "time")
    T = 9
    full = oracle.fit(X, y, ntree=T, mtry=3, seed=5, target=1)
    lo, hi = shard(T, rank, world)
    part = oracle.fit(X, y, ntree=T, mtry=3, seed=5, target=1, tree_begin=lo, tree_end=hi)
    feat, tv, left, lv, off = part.flatten()
    value = np.where(feat >= 0, tv, lv)
    ti = np.concatenate([t.thr_index for t in part.trees])
    arrs = allgather_forest_arrays(torch.as_tensor(feat), torch.as_tensor(left.astype(np.int64)),
                                   torch.as_tensor(value), torch.as_tensor(ti.astype(np.int64)),
                                   torch.as_tensor(off.astype(np.int64)))
    ff, ftv, fleft, flv, foff = full.flatten()
    fvalue = np.where(ff >= 0, ftv, flv)
    assert np.array_equal(arrs[0].numpy(), ff)
    assert np.array_equal(arrs[1].numpy(), fleft.astype(np.int64))
    assert np.array_equal(arrs[2].numpy().view(np.int64), fvalue.view(np.int64))
    assert np.array_equal(arrs[3].numpy(), np.concatenate([t.thr_index for t in full.trees]).astype(np.int64))
    assert np.array_equal(arrs[4].numpy(), foff.astype(np.int64))


def test_allgather_forest_matches_full_forest():
    run_world(_assemble)


def _gather_rows(rank, world):
    # importance of a tree-sharded forest: per-tree raw rows of uneven shards, rank order
    from paper_2001_07104_b200.dist import gather_rows, shard
    X, y = datagen.paper_shaped(189, "V100", "time")
    T = 7
    full = oracle.fit(X, y, ntree=T, mtry=4, seed=3, target=1)
    lo, hi = shard(T, rank, world)
    part = oracle.fit(X, y, ntree=T, mtry=4, seed=3, target=1, tree_begin=lo, tree_end=hi)
    got = gather_rows(torch.as_tensor(np.stack([t.imp_raw for t in part.trees])))
    want = np.stack([t.imp_raw for t in full.trees])
    assert np.array_equal(got.numpy(), want)
    assert np.array_equal(oracle.importance(got.numpy()), full.importance())


def test_gather_rows_importance_shards():
    run_world(_gather_rows)


def _row_sharded_predict(rank, world):
    # host logic of the row-sharded inference driver (C5): the per-rank prediction is stubbed
    # with the oracle (no GPU here); rows are sharded unevenly and gathered in row order
    import paper_2001_07104_b200.dist as D
    X, y = datagen.paper_shaped(189, "K20", "time")
    f = oracle.fit(X, y, ntree=6, mtry=4, seed=2, target=1)
    D.predict = lambda forest, Xs: torch.as_tensor(oracle.predict(f, Xs.numpy()))
    Q = torch.as_tensor(X[:101])
    got = D.predict_row_sharded(None, Q)
    assert np.array_equal(got.numpy(), oracle.predict(f, X[:101]))
    lo, hi = D.shard(101, rank, world)
    mine = D.predict_row_sharded(None, Q[lo:hi], gather=False)
    assert np.array_equal(mine.numpy(), oracle.predict(f, X[lo:hi]))


def test_row_sharded_predict():
    run_world(_row_sharded_predict)
