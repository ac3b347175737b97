"""Multi-GPU driver: one process per GPU, NCCL through torch.distributed.

The library never calls NCCL.  Work shards along the
independent axes of the method -- CV tasks (repeat, fold), trees, query rows --
and the only exchange steps are:
  * all_gather of per-rank fold-MAPE tables (task-sharded CV; bit-identical for
    any number of ranks, no floating-point reduction);
  * all_reduce(SUM) of per-row partial sums of leaf values (tree-sharded CV and
    tree-sharded prediction), then a finalize kernel (divide, exp, MAPE);
  * all_gather of node counts + padded node arrays to assemble a tree-sharded
    forest on every rank (rf_forest_import).
Everything that touches the data runs in librfgpu's kernels; this module moves
tensors between ranks and calls the C ABI through the binding.  The
collective/assembly helpers take plain tensors so they are testable with the
gloo backend on CPU (tests/test_dist.py).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import (TARGET_IDENTITY, cross_validate_grid, cv_finalize, cv_partial, fit, forest_import,
               predict, predict_finalize, predict_partial)


def shard(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous range [lo, hi) of `total` units for `rank` (balanced, rank order)."""
    return (total * rank) // world, (total * (rank + 1)) // world


def _world(group=None):
    if not dist.is_available() or not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def _host_staged(t, group=None):
    """gloo process groups (CPU tests, and several ranks sharing one GPU in the GPU tests)
    exchange host tensors: True if t is a CUDA tensor and the group's backend is gloo."""
    return isinstance(t, torch.Tensor) and t.is_cuda and dist.get_backend(group) == "gloo"


# ------------------------------------------------------------ exchanges ----
def gather_task_tables(local: torch.Tensor, task_axis_len: int, group=None) -> torch.Tensor:
    """local: [..., T_local] slice of a table whose last axis is the flat task index
    (task = rep*k + fold), ranks holding consecutive task ranges of equal length.
    Returns the full table [..., world * T_local] in task order on every rank."""
    rank, world = _world(group)
    if world == 1:
        return local
    if _host_staged(local, group):
        return gather_task_tables(local.cpu(), task_axis_len, group).to(local.device)
    local = local.contiguous()
    flat = torch.empty((world * local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(flat, local, group=group)  # concatenated along dim 0 (all backends)
    out = flat.view((world,) + tuple(local.shape))
    lead = local.shape[:-1]
    perm = list(range(1, 1 + len(lead))) + [0, 1 + len(lead)]
    return out.permute(*perm).reshape(*lead, world * local.shape[-1])


def reduce_partials(partial: torch.Tensor, group=None) -> torch.Tensor:
    """In-place all_reduce(SUM) of per-row partial sums (fp64)."""
    rank, world = _world(group)
    if world > 1:
        if _host_staged(partial, group):
            h = partial.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
            partial.copy_(h)
        else:
            dist.all_reduce(partial, op=dist.ReduceOp.SUM, group=group)
    return partial


def allgather_forest_arrays(feature, left, value, thr_index, tree_off, group=None):
    """Each rank holds a contiguous tree shard (flattened arrays, host or device tensors).
    Returns the concatenated forest arrays (rank order = tree order) on every rank."""
    rank, world = _world(group)
    if world == 1:
        return feature, left, value, thr_index, tree_off
    if _host_staged(feature, group):
        arrs = allgather_forest_arrays(feature.cpu(), left.cpu(), value.cpu(), thr_index.cpu(), tree_off.cpu(),
                                       group)
        return tuple(a.to(feature.device) for a in arrs)
    dev = feature.device
    counts = torch.tensor([feature.shape[0], tree_off.shape[0] - 1], dtype=torch.int64, device=dev)
    allc = torch.empty((world * 2,), dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(allc, counts, group=group)
    allc = allc.view(world, 2)
    nmax = int(allc[:, 0].max().item())
    tmax = int(allc[:, 1].max().item())

    def gather_padded(x, length, n):
        pad = torch.zeros((length,) + tuple(x.shape[1:]), dtype=x.dtype, device=dev)
        pad[: x.shape[0]] = x
        out = torch.empty((world * length,) + tuple(x.shape[1:]), dtype=x.dtype, device=dev)
        dist.all_gather_into_tensor(out, pad, group=group)
        out = out.view((world, length) + tuple(x.shape[1:]))
        return [out[r, : int(n[r])] for r in range(world)]

    nn = allc[:, 0].tolist()
    nt = allc[:, 1].tolist()
    feats = gather_padded(feature, nmax, nn)
    lefts = gather_padded(left, nmax, nn)
    # node values travel as raw 64-bit words so the gather is bit-exact on every backend
    vals = gather_padded(value.view(torch.int64), nmax, nn)
    tis = gather_padded(thr_index, nmax, nn)
    offs = gather_padded(tree_off[1:] - tree_off[:-1], tmax, nt)  # per-tree node counts
    sizes = torch.cat(offs)
    off = torch.zeros(sizes.shape[0] + 1, dtype=torch.int64, device=dev)
    off[1:] = torch.cumsum(sizes, 0)
    return (torch.cat(feats), torch.cat(lefts), torch.cat(vals).view(torch.float64), torch.cat(tis), off)


def gather_rows(local: torch.Tensor, group=None) -> torch.Tensor:
    """Concatenate per-rank row blocks [n_r, ...] of different lengths in rank order
    (e.g. per-tree importance sums of tree shards) on every rank."""
    rank, world = _world(group)
    if world == 1:
        return local
    if _host_staged(local, group):
        return gather_rows(local.cpu(), group).to(local.device)
    dev = local.device
    n = torch.tensor([local.shape[0]], dtype=torch.int64, device=dev)
    alln = torch.empty((world,), dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(alln, n, group=group)
    sizes = alln.tolist()
    m = max(sizes)
    pad = torch.zeros((m,) + tuple(local.shape[1:]), dtype=local.dtype, device=dev)
    pad[: local.shape[0]] = local
    out = torch.empty((world * m,) + tuple(local.shape[1:]), dtype=local.dtype, device=dev)
    dist.all_gather_into_tensor(out, pad, group=group)
    out = out.view((world, m) + tuple(local.shape[1:]))
    return torch.cat([out[r, : sizes[r]] for r in range(world)])


# -------------------------------------------------------------- drivers ----
def importance_sharded(local_forest, group=None, device=None):
    """Feature importance of a tree-sharded forest: all_gather of the per-tree split
    decrease sums of every rank's shard, combined by rf_importance_dev (same vector as
    a single-GPU fit of all trees, up to the order of fp64 sums)."""
    from . import importance_dev
    _, raw = local_forest.importance(raw=True)
    dev = device or torch.device("cuda", torch.cuda.current_device())
    full = gather_rows(torch.as_tensor(raw, device=dev), group)
    return importance_dev(full.contiguous())



def fit_sharded(X, y, *, ntree, group=None, **kw):
    """Tree-sharded rf_fit: rank r grows trees shard(ntree, r, world); the forest is
    assembled on every rank (identical to a single-GPU fit of ntree trees, R15)."""
    rank, world = _world(group)
    lo, hi = shard(ntree, rank, world)
    local = fit(X, y, ntree=ntree, tree_begin=lo, tree_end=hi, **kw) if hi > lo else None
    if local is None:
        raise ValueError("fewer trees than ranks")
    e = local.export()
    dev = X.device if isinstance(X, torch.Tensor) else torch.device("cpu")
    # unsigned arrays travel as int64 (gloo has no unsigned types); converted back below
    t = lambda a: torch.as_tensor(a.astype(np.int64) if a.dtype in (np.uint64, np.uint32) else a, device=dev)
    arrs = allgather_forest_arrays(t(e["feature"]), t(e["left"]), t(e["value"]), t(e["thr_index"]),
                                   t(e["tree_off"]), group)
    feature, left, value, thr_index, off = (a.cpu().numpy() for a in arrs)
    dev_index = dev.index if dev.type == "cuda" and dev.index is not None else 0
    return forest_import(feature, left, value, thr_index, off.astype(np.uint64), e["p"], e["F"], e["target"],
                         device=dev_index)


def predict_row_sharded(forest, X, group=None, gather=True):
    """Row-sharded batched inference: the forest is replicated, rank r
    predicts rows shard(n, r, world) of X (device tensor, the full query block or already
    this rank's rows with gather=False); no data-path collective, optionally one all_gather
    of the predictions in row order."""
    rank, world = _world(group)
    lo, hi = shard(X.shape[0], rank, world) if gather else (0, X.shape[0])
    mine = predict(forest, X[lo:hi].contiguous())
    return gather_rows(mine, group) if gather else mine


def predict_tree_sharded(local_forest, X, ntree_total, target, group=None):
    """Each rank holds a tree shard; partial sums are all-reduced, then finalized."""
    part = predict_partial(local_forest, X)
    reduce_partials(part, group)
    return predict_finalize(part, ntree_total, target)


def study_units(sizes, rank, world):
    """Strong-scaling split of a fixed CV study (SURVEY 8(e) "shard whole (dataset, rep, fold)
    tasks"): sizes[d] = tasks of dataset d; the flattened (dataset, task) list is cut into
    `world` contiguous ranges.  Returns this rank's [(d, task_lo, task_hi)] (non-empty only)."""
    total = sum(sizes)
    lo, hi = shard(total, rank, world)
    out, base = [], 0
    for d, n in enumerate(sizes):
        a, b = max(lo, base), min(hi, base + n)
        if b > a:
            out.append((d, a - base, b - base))
        base += n
    return out


def cv_task_sharded(X, y, k, repeats_per_rank, ntrees, mtrys, *, custom=False, seed=0,
                    target=TARGET_IDENTITY, group=None, **kw):
    """Weak-scaling CV study: rank r runs repeats [r R, (r+1) R) of an R*world-repeat study.
    Returns the full fold-MAPE table [n_mtry, n_ntree, R*world, k] on every rank."""
    from . import make_folds
    rank, world = _world(group)
    reps = repeats_per_rank * world
    folds = make_folds(y, k, reps, seed=seed, custom=custom)
    lo, hi = rank * repeats_per_rank * k, (rank + 1) * repeats_per_rank * k
    fm = cross_validate_grid(X, y, k, reps, ntrees, mtrys, fold_ids=folds, seed=seed, target=target,
                             task_begin=lo, task_end=hi, **kw)
    flat = fm.reshape(len(mtrys), len(ntrees), reps * k)[:, :, lo:hi].contiguous()
    full = gather_task_tables(flat, reps * k, group)
    return full.reshape(len(mtrys), len(ntrees), reps, k)


def cv_tree_sharded(X, y, k, repeats, folds, ntrees, mtrys, *, target=TARGET_IDENTITY, seed=0, group=None,
                    want_pred=False, **kw):
    """Tree-sharded CV (few tasks, many trees): per-row partial sums over each rank's
    trees, all_reduce(SUM), finalize (divide, exp, MAPE) on every rank."""
    rank, world = _world(group)
    lo, hi = shard(max(ntrees), rank, world)
    if hi > lo:
        part = cv_partial(X, y, k, repeats, folds, ntrees, mtrys, tree_begin=lo, tree_end=hi, target=target,
                          seed=seed, **kw)
    else:
        # empty shard (fewer trees than ranks): contribute zeros -- (0, 0) would mean "all trees"
        # to the C ABI and double-count the forest in the all_reduce
        n = y.shape[0]
        shape = (len(mtrys), len(ntrees), repeats, n)
        part = torch.zeros(shape, dtype=torch.float64, device=X.device) if isinstance(X, torch.Tensor) \
            else np.zeros(shape, np.float64)
    host = not isinstance(part, torch.Tensor)
    if host:
        part = torch.from_numpy(part)
    reduce_partials(part, group)
    if host:
        part = part.numpy()
    return cv_finalize(y, k, repeats, folds, ntrees, len(mtrys), part, target=target, want_pred=want_pred)


def cv_study_sharded(datasets, k, repeats, ntrees, mtrys, *, folds, outs, group=None, streams=None, **kw):
    """Strong-scaling CV study (BASELINE.json configs[1], SURVEY 8(e) CV C2): the fixed study's
    (dataset, task) units are cut into contiguous rank ranges (study_units); each rank runs
    rf_cross_validate_grid with task_begin/task_end on its units only, then the owned task
    columns of every table are all-gathered in unit order (gather_rows) and written back, so
    every rank ends with the full tables -- bit-identical for any number of ranks (no
    floating-point reduction).

    datasets: [dict(X, y, target, seed)] device tensors; folds[d]: int32 [repeats, n] device
    fold ids; outs[d]: fp64 [n_mtry, n_ntree, repeats, k] device tables (filled in place).
    streams: optional CUDA streams, one per dataset (the launches of different datasets overlap).
    Returns this rank's units [(d, lo, hi)]."""
    rank, world = _world(group)
    T = repeats * k
    units = study_units([T] * len(datasets), rank, world)
    main = torch.cuda.current_stream() if streams else None
    for d, lo, hi in units:
        ds = datasets[d]
        st = streams[d % len(streams)] if streams else None
        if st is not None:
            st.wait_stream(main)
        with torch.cuda.stream(st) if st is not None else _nullctx():
            cross_validate_grid(ds["X"], ds["y"], k, repeats, ntrees, mtrys, fold_ids=folds[d], target=ds["target"],
                                seed=ds["seed"], task_begin=lo, task_end=hi, out=outs[d], **kw)
    if streams:
        for st in streams:
            main.wait_stream(st)
    if world > 1:
        G = len(mtrys) * len(ntrees)
        mine = [outs[d].reshape(G, T)[:, lo:hi].t() for d, lo, hi in units]
        local = torch.cat(mine) if mine else torch.empty((0, G), dtype=torch.float64, device=outs[0].device)
        full = gather_rows(local.contiguous(), group)  # [sum of all units, G] in unit order
        o = 0
        for d in range(len(datasets)):
            outs[d].reshape(G, T).copy_(full[o:o + T].t())
            o += T
    return units


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False
