"""CPU oracle for the random-forest CV hot path of arXiv 2001.07104.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2001_07104_b200``) never imports it and
shares no code with it; ``datagen`` (seeded synthetic inputs) is the only
module both sides use.

The arithmetic lives in ``rf_oracle.c`` (plain single-threaded C11,
``-O2 -ffp-contract=off``), which is compiled on first use.  This module is
argument marshalling over ctypes plus numpy containers.  Each function cites
the passage of PAPER.md (``P:n``) or the DESIGN.md reading (``Rn``) it follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rf_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

STATUS = {0: "OK", 1: "ARG", 2: "EMPTY", 3: "NONFINITE", 4: "NONPOSITIVE_Y",
          5: "ARITY", 6: "TOO_FEW", 9: "OVERFLOW"}


class OracleError(RuntimeError):
    def __init__(self, code):
        super().__init__(f"oracle status {code} ({STATUS.get(code, '?')})")
        self.code = code


def build(force: bool = False) -> str:
    """Compile rf_oracle.c -> liboracle.so (gcc, -O2 -ffp-contract=off)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", "-Wall", "-o", tmp, _SRC, "-lquadmath", "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        u32, u64, i32, dbl = C.c_uint32, C.c_uint64, C.c_int32, C.c_double
        P = C.c_void_p
        _lib.or_philox.argtypes = [P, P, P]
        _lib.or_draw.argtypes = [u32, u32, u32, u32, u32, u64]
        _lib.or_draw.restype = u64
        _lib.or_mulhi64.argtypes = [u64, u64]
        _lib.or_mulhi64.restype = u64
        _lib.or_tree_key.argtypes = [u64, u32, u32, P]
        _lib.or_ln.argtypes = [dbl]
        _lib.or_ln.restype = dbl
        _lib.or_quantize.argtypes = [P, u64, C.c_int, P, P, P]
        _lib.or_make_folds.argtypes = [P, u64, u32, u32, u64, u32, P]
        _lib.or_make_folds_masked.argtypes = [P, u64, u32, u32, u64, u32, P, P]
        _lib.or_fit.argtypes = [P, u64, u32, P, u32, u32, i32, u32, u32, u32, u64,
                                u32, u32, u64, P, P, P, P, P, P, P, P, P]
        _lib.or_predict.argtypes = [P, P, P, P, P, u32, u32, P, u64, u32, P]
        _lib.or_mape.argtypes = [P, P, u64]
        _lib.or_mape.restype = dbl
        _lib.or_cv_grid.argtypes = [P, u64, u32, P, u32, i32, u32, u32, u32, u64, u32, u32, P,
                                    P, u32, P, u32, u32, u32, P, P]
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------- RNG ----
def philox(ctr, key):
    """Philox4x32-10 block (R14)."""
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    lib().or_philox(_p(c), _p(k), _p(o))
    return o


def draw(k0, k1, c1, c2, c3, i):
    return int(lib().or_draw(k0, k1, c1, c2, c3, i))


def mulhi64(u, m):
    return int(lib().or_mulhi64(u, m))


def tree_key(seed, task, t):
    o = np.zeros(2, dtype=np.uint32)
    lib().or_tree_key(seed, task, t, _p(o))
    return int(o[0]), int(o[1])


def ln(y):
    """ln correctly rounded to binary64 (R20)."""
    return float(lib().or_ln(float(y)))


def quantize(y, target):
    """t = y or ln y; F rule and t_q = rint(t * 2^F) (R7)."""
    y = np.ascontiguousarray(y, dtype=np.float64)
    t = np.zeros_like(y)
    tq = np.zeros(y.shape[0], dtype=np.int64)
    F = np.zeros(1, dtype=np.int32)
    st = lib().or_quantize(_p(y), y.shape[0], int(target), _p(t), _p(tq), _p(F))
    if st:
        raise OracleError(st)
    return t, tq, int(F[0])


def make_folds(y, k, reps, seed, custom=False):
    """Fold ids [reps][n] (R16, R17)."""
    y = np.ascontiguousarray(y, dtype=np.float64)
    out = np.zeros((reps, y.shape[0]), dtype=np.int32)
    st = lib().or_make_folds(_p(y), y.shape[0], k, reps, seed, int(custom), _p(out))
    if st:
        raise OracleError(st)
    return out


# --------------------------------------------------------------- trees ---
@dataclass
class Tree:
    feature: np.ndarray     # int32, -1 = leaf
    thr_index: np.ndarray   # uint32
    thr_value: np.ndarray   # float64
    left: np.ndarray        # uint32, right = left + 1
    leaf_value: np.ndarray  # float64
    leaf_of_row: np.ndarray | None = None  # int32 [n], -1 out of bag
    imp_raw: np.ndarray | None = None      # float64 [p]: sum of the MDI decreases per feature

    @property
    def n_nodes(self):
        return int(self.feature.shape[0])

    def predict_row(self, x):
        i = 0
        while self.feature[i] >= 0:
            i = int(self.left[i]) if x[self.feature[i]] <= self.thr_value[i] else int(self.left[i]) + 1
        return float(self.leaf_value[i])

    def max_depth(self):
        depth = np.zeros(self.n_nodes, dtype=np.int64)
        for i in range(self.n_nodes):
            if self.feature[i] >= 0:
                depth[self.left[i]] = depth[i] + 1
                depth[self.left[i] + 1] = depth[i] + 1
        return int(depth.max())


@dataclass
class Forest:
    trees: list
    F: int
    target: int

    def flatten(self):
        off = np.zeros(len(self.trees) + 1, dtype=np.uint64)
        for i, t in enumerate(self.trees):
            off[i + 1] = off[i] + t.n_nodes
        cat = lambda name: np.ascontiguousarray(np.concatenate([getattr(t, name) for t in self.trees]))
        return (cat("feature"), cat("thr_value"), cat("left"), cat("leaf_value"), off)

    def importance(self):
        """Feature importance (mean decrease in impurity), see ``importance``."""
        return importance(np.stack([t.imp_raw for t in self.trees]))


def importance(raw):
    """MDI feature importance of a forest (Table 6
    P:926-948) from per-tree sums of split decreases raw [T][p], following the
    library the paper uses (scikit-learn): each tree's vector is divided by its
    sum (trees without any decrease contribute zeros), the vectors are summed
    over trees and the result is divided by its sum."""
    raw = np.asarray(raw, dtype=np.float64)
    T, p = raw.shape
    acc = np.zeros(p)
    for t in range(T):
        s = 0.0
        for f in range(p):
            s += raw[t, f]
        if s > 0.0:
            for f in range(p):
                acc[f] += raw[t, f] / s
    tot = 0.0
    for f in range(p):
        tot += acc[f]
    return acc / tot if tot > 0.0 else acc


def fit(X, y, ntree=1, mtry=None, min_samples_split=2, max_depth=-1, bootstrap=True,
        split_mode=0, target=0, seed=0, tree_begin=0, tree_end=None, leaf_rows=False, criterion=0,
        tie_break=0):
    """Grow trees [tree_begin, tree_end) of task 0 (R2-R14).  criterion 0 = MSE
    (P:215), 1 = MAE (R32).  tie_break 0 = lowest feature (north_star), 1 = first
    drawn feature (R9)."""
    split_mode = int(split_mode) | (int(criterion) << 8) | (int(tie_break) << 9)
    X = np.ascontiguousarray(X, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    n, p = X.shape
    if mtry is None:
        mtry = max(1, p // 3)
    if tree_end is None:
        tree_end = ntree
    T = tree_end - tree_begin
    cap = max(1, 2 * n - 1)
    nn = np.zeros(T, dtype=np.uint64)
    feat = np.zeros((T, cap), dtype=np.int32)
    ti = np.zeros((T, cap), dtype=np.uint32)
    tv = np.zeros((T, cap), dtype=np.float64)
    lf = np.zeros((T, cap), dtype=np.uint32)
    lv = np.zeros((T, cap), dtype=np.float64)
    lor = np.zeros((T, n), dtype=np.int32) if leaf_rows else None
    imp = np.zeros((T, p), dtype=np.float64)
    F = np.zeros(1, dtype=np.int32)
    st = lib().or_fit(_p(X), n, p, _p(y), mtry, min_samples_split, max_depth, int(bootstrap),
                      split_mode, target, seed, tree_begin, tree_end, cap,
                      _p(nn), _p(feat), _p(ti), _p(tv), _p(lf), _p(lv), _p(lor), _p(F), _p(imp))
    if st:
        raise OracleError(st)
    trees = []
    for t in range(T):
        m = int(nn[t])
        trees.append(Tree(feat[t, :m].copy(), ti[t, :m].copy(), tv[t, :m].copy(), lf[t, :m].copy(),
                          lv[t, :m].copy(), None if lor is None else lor[t].copy(), imp[t].copy()))
    return Forest(trees, int(F[0]), target)


def predict(forest: Forest, Xq):
    """Mean of trees in tree order, exp for LOG."""
    Xq = np.ascontiguousarray(Xq, dtype=np.float64)
    feat, tv, lf, lv, off = forest.flatten()
    out = np.zeros(Xq.shape[0], dtype=np.float64)
    lib().or_predict(_p(feat), _p(tv), _p(lf), _p(lv), _p(off), len(forest.trees), forest.target,
                     _p(Xq), Xq.shape[0], Xq.shape[1], _p(out))
    return out


def mape(y, yhat):
    """Eq. 1, in percent."""
    y = np.ascontiguousarray(y, dtype=np.float64)
    yhat = np.ascontiguousarray(yhat, dtype=np.float64)
    return float(lib().or_mape(_p(y), _p(yhat), y.shape[0]))


def cv_grid(X, y, k, reps, ntrees, mtrys, fold_ids=None, min_samples_split=2, max_depth=-1,
            bootstrap=True, split_mode=0, target=0, seed=0, task_begin=0, task_end=0,
            want_pred=False, criterion=0, tie_break=0):
    """Repeated k-fold CV over an ntree x mtry grid; criterion 0 MSE, 1 MAE (R32);
    tie_break 0 lowest feature (north_star), 1 first drawn feature (R9).

    Returns fold_mape [n_mtry][n_ntree][reps][k] and optionally the per-row
    predictions [n_mtry][n_ntree][reps][n]."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    n, p = X.shape
    nt = np.ascontiguousarray(ntrees, dtype=np.uint32)
    mt = np.ascontiguousarray(mtrys, dtype=np.uint32)
    fm = np.zeros((len(mt), len(nt), reps, k), dtype=np.float64)
    pr = np.zeros((len(mt), len(nt), reps, n), dtype=np.float64) if want_pred else None
    fid = None if fold_ids is None else np.ascontiguousarray(fold_ids, dtype=np.int32)
    split_mode = int(split_mode) | (int(criterion) << 8) | (int(tie_break) << 9)
    st = lib().or_cv_grid(_p(X), n, p, _p(y), min_samples_split, max_depth, int(bootstrap),
                          split_mode, target, seed, k, reps, _p(fid), _p(nt), len(nt), _p(mt),
                          len(mt), task_begin, task_end, _p(fm), _p(pr))
    if st:
        raise OracleError(st)
    return (fm, pr) if want_pred else fm


# ------------------------------------------------- nested CV / LOO (NEXT-2) ---
NESTED_SEED_TAG = 0x4E45535445440000  # "NESTED\0\0": inner folds use seed ^ tag (R31)
APE_EDGES = (10.0, 25.0, 50.0, 100.0)  # error buckets of the LOO analysis, percent


def make_folds_masked(y, k, mask, seed, custom=False):
    """Folds of a row subset per rep (mask [reps][n] != 0): the subset is split like
    make_folds splits a dataset of those rows; other rows get -2 (R31)."""
    y = np.ascontiguousarray(y, dtype=np.float64)
    mk = np.ascontiguousarray(mask, dtype=np.uint8)
    reps, n = mk.shape
    out = np.zeros((reps, n), dtype=np.int32)
    st = lib().or_make_folds_masked(_p(y), n, k, reps, seed, int(custom), _p(mk), _p(out))
    if st:
        raise OracleError(st)
    return out


def nested_cv(X, y, k_outer, k_inner, iterations, ntrees, mtrys, custom=False, seed=0, **kw):
    """Nested cross-validation (R31), followed step by step:
    1. outer folds: make_folds(y, k_outer, iterations, seed, custom);
    2. for every (iteration it, outer fold o) -- combo c = it*k_outer + o -- the inner
       folds split the outer-training rows (outer fold id != o) with make_folds_masked
       (rep c, seed ^ NESTED_SEED_TAG); the rest is excluded (-2);
    3. inner grid CV on those fold sets (one cv_grid call, reps = combos);
    4. per combo: score of grid point g = (sum of its inner fold MAPEs in fold order) / k_inner;
       best = the lowest score, ties to the first grid point (mtry-major, then ntree);
    5. outer grid CV on the outer folds; the combo's outer score = its fold MAPE at best.
    Returns (best [it][k_outer] grid index, outer_mape [it][k_outer],
             inner_score [it][k_outer][n_mtry][n_ntree])."""
    y = np.ascontiguousarray(y, dtype=np.float64)
    n = y.shape[0]
    nm, nt = len(mtrys), len(ntrees)
    outer = make_folds(y, k_outer, iterations, seed, custom)
    C = iterations * k_outer
    mask = np.zeros((C, n), dtype=np.uint8)
    for it in range(iterations):
        for o in range(k_outer):
            mask[it * k_outer + o] = outer[it] != o
    inner = make_folds_masked(y, k_inner, mask, seed ^ NESTED_SEED_TAG, custom)
    fm_in = cv_grid(X, y, k_inner, C, ntrees, mtrys, fold_ids=inner, seed=seed ^ NESTED_SEED_TAG, **kw)
    score = np.zeros((C, nm, nt))
    best = np.zeros(C, dtype=np.int32)
    for c in range(C):
        bs, bg = None, 0
        for mi in range(nm):
            for ti in range(nt):
                s = 0.0
                for f in range(k_inner):
                    s += fm_in[mi, ti, c, f]
                s = s / k_inner
                score[c, mi, ti] = s
                if bs is None or s < bs:
                    bs, bg = s, mi * nt + ti
        best[c] = bg
    fm_out = cv_grid(X, y, k_outer, iterations, ntrees, mtrys, fold_ids=outer, seed=seed, **kw)
    outer_mape = np.zeros(C)
    for c in range(C):
        it, o = divmod(c, k_outer)
        mi, ti = divmod(int(best[c]), nt)
        outer_mape[c] = fm_out[mi, ti, it, o]
    return (best.reshape(iterations, k_outer), outer_mape.reshape(iterations, k_outer),
            score.reshape(iterations, k_outer, nm, nt))


def error_buckets(y, yhat):
    """Counts of absolute percentage errors 100 |y - yhat| / y in [0,10), [10,25), [25,50),
    [50,100), [100, inf) (the LOO analysis of P:741-754); NaN predictions are skipped."""
    counts = [0, 0, 0, 0, 0]
    for a, b in zip(np.asarray(y, dtype=np.float64), np.asarray(yhat, dtype=np.float64)):
        if b != b:
            continue
        e = 100.0 * (abs(a - b) / a)  # relative error first, as in Eq. 1
        j = 0
        while j < 4 and e >= APE_EDGES[j]:
            j += 1
        counts[j] += 1
    return np.array(counts, dtype=np.int64)
