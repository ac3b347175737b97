"""B200-native random-forest cross-validation (arXiv 2001.07104 hot path).

Thin ctypes binding over ``librfgpu.so`` (C ABI in ``include/rf.h``).  This
module only marshals arguments: every step of fitting, cross-validation and
prediction runs in the library's sm_100a CUDA kernels.  There is no CPU
fallback -- if the shared library or a CUDA device is missing, calls raise.

Inputs may be numpy arrays (host path: the library copies them to the
device) or CUDA torch tensors (device path, enqueued on torch's current
stream).  PyTorch is used only for device memory and streams.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# RFGPU_LIB selects another in-tree build of the same library (the profiling build
# librfgpu_pt.so, see build.py); the default is the product build.
LIB_PATH = os.environ.get("RFGPU_LIB") or os.path.join(_HERE, "librfgpu.so")

OK, E_ARG, E_EMPTY, E_NONFINITE, E_NONPOSITIVE_Y, E_ARITY, E_TOO_FEW, E_CUDA, E_OOM, E_OVERFLOW, \
    E_UNSUPPORTED, E_INEXACT = range(12)
STATUS_NAMES = ["OK", "ARG", "EMPTY", "NONFINITE", "NONPOSITIVE_Y", "ARITY", "TOO_FEW", "CUDA", "OOM",
                "OVERFLOW", "UNSUPPORTED", "INEXACT"]
SPLIT_EXACT, SPLIT_HIST256, SPLIT_EXTRA = 0, 1, 2
TARGET_IDENTITY, TARGET_LOG = 0, 1
CRITERION_MSE, CRITERION_MAE = 0, 1
TIE_LOWEST_FEATURE, TIE_DRAW_ORDER = 0, 1  # rf_tie_break (R9): north_star's rule is the default

# every entry point declared in include/rf.h and include/rf_debug.h
ABI_SYMBOLS = [
    "rf_params_default", "rf_fit", "rf_fit_dev", "rf_fit_debug", "rf_predict", "rf_predict_dev",
    "rf_predict_partial_dev", "rf_predict_finalize_dev", "rf_make_folds", "rf_make_folds_dev",
    "rf_make_folds_masked_dev", "rf_nested_cv", "rf_nested_cv_dev", "rf_error_buckets", "rf_error_buckets_dev",
    "rf_cross_validate_grid", "rf_cross_validate_grid_dev", "rf_cross_validate", "rf_cross_validate_dev",
    "rf_cv_partial_dev",
    "rf_cv_finalize_dev", "rf_predict_partial", "rf_cv_partial", "rf_cv_finalize", "rf_forest_free", "rf_last_error", "rf_forest_info", "rf_forest_export",
    "rf_forest_export_leaf_rows", "rf_forest_import", "rf_forest_importance", "rf_importance_dev",
    "rf_last_profile", "rf_set_profiling",
    "rf_debug_ln_dev", "rf_debug_philox_dev", "rf_debug_counters", "rf_debug_row_levels", "rf_debug_phase_cycles", "rf_debug_set_option",
]


class RFError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"rf status {code} ({STATUS_NAMES[code] if code < len(STATUS_NAMES) else '?'}): {msg}")
        self.code = code


class Params(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("ntree", C.c_uint32), ("mtry", C.c_uint32),
                ("min_samples_split", C.c_uint32), ("max_depth", C.c_int32), ("bootstrap", C.c_uint32),
                ("split_mode", C.c_uint32), ("target", C.c_uint32), ("seed", C.c_uint64),
                ("device", C.c_int32), ("tree_begin", C.c_uint32), ("tree_end", C.c_uint32),
                ("task_begin", C.c_uint32), ("task_end", C.c_uint32), ("criterion", C.c_uint32),
                ("tie_break", C.c_uint32)]


_lib = None


def lib():
    """Load librfgpu.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run `python -m paper_2001_07104_b200.build` "
                               "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        P, u32, u64, i32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int32
        pp = C.POINTER(Params)
        sig = {
            "rf_params_default": ([pp], None),
            "rf_fit": ([P, u64, u32, P, pp, P], C.c_int),
            "rf_fit_debug": ([P, u64, u32, P, pp, P], C.c_int),
            "rf_fit_dev": ([P, u64, u32, P, pp, P, P], C.c_int),
            "rf_predict": ([P, P, u64, u32, P], C.c_int),
            "rf_predict_dev": ([P, P, u64, u32, P, P], C.c_int),
            "rf_predict_partial_dev": ([P, P, u64, u32, P, P], C.c_int),
            "rf_predict_finalize_dev": ([P, u64, u32, u32, P, P], C.c_int),
            "rf_predict_partial": ([P, P, u64, u32, P], C.c_int),
            "rf_cv_partial": ([P, u64, u32, P, pp, u32, u32, P, P, u32, P, u32, P], C.c_int),
            "rf_cv_finalize": ([P, u64, u32, u32, u32, P, P, u32, u32, P, P, P, i32], C.c_int),
            "rf_make_folds": ([P, u64, u32, u32, u64, u32, P], C.c_int),
            "rf_make_folds_dev": ([P, u64, u32, u32, u64, u32, P, P], C.c_int),
            "rf_make_folds_masked_dev": ([P, u64, u32, u32, u64, u32, P, P, P], C.c_int),
            "rf_nested_cv": ([P, u64, u32, P, pp, u32, u32, u32, u32, P, u32, P, u32, P, P, P], C.c_int),
            "rf_nested_cv_dev": ([P, u64, u32, P, pp, u32, u32, u32, u32, P, u32, P, u32, P, P, P, P], C.c_int),
            "rf_error_buckets": ([P, P, u64, P], C.c_int),
            "rf_error_buckets_dev": ([P, P, u64, P, P], C.c_int),
            "rf_cross_validate_grid": ([P, u64, u32, P, pp, u32, u32, P, P, u32, P, u32, P, P], C.c_int),
            "rf_cross_validate_grid_dev": ([P, u64, u32, P, pp, u32, u32, P, P, u32, P, u32, P, P, P],
                                           C.c_int),
            "rf_cross_validate": ([P, u64, u32, P, pp, u32, u32, P, P], C.c_int),
            "rf_cross_validate_dev": ([P, u64, u32, P, pp, u32, u32, P, P, P], C.c_int),
            "rf_cv_partial_dev": ([P, u64, u32, P, pp, u32, u32, P, P, u32, P, u32, P, P], C.c_int),
            "rf_cv_finalize_dev": ([P, u64, u32, u32, u32, P, P, u32, u32, P, P, P, P], C.c_int),
            "rf_forest_free": ([P], None),
            "rf_last_error": ([], C.c_char_p),
            "rf_forest_info": ([P, P, P, P, P, P], C.c_int),
            "rf_forest_export": ([P, P, P, P, P, P], C.c_int),
            "rf_forest_export_leaf_rows": ([P, P], C.c_int),
            "rf_forest_importance": ([P, P, P], C.c_int),
            "rf_importance_dev": ([P, u32, u32, P, P], C.c_int),
            "rf_forest_import": ([P, P, P, P, P, u32, u32, i32, u32, i32, P], C.c_int),
            "rf_last_profile": ([P, P, P, u32], u32),
            "rf_set_profiling": ([C.c_int], None),
            "rf_debug_ln_dev": ([P, P, u64, P], C.c_int),
            "rf_debug_philox_dev": ([P, P, u64, P], C.c_int),
            "rf_debug_counters": ([P, P], C.c_int),
            "rf_debug_row_levels": ([P, C.c_int], C.c_int),
            "rf_debug_phase_cycles": ([P, C.c_int], C.c_int),
            "rf_debug_set_option": ([C.c_char_p, C.c_int64], C.c_int),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def _check(code):
    if code != OK:
        raise RFError(code, lib().rf_last_error().decode())


def params(**kw) -> Params:
    p = Params()
    lib().rf_params_default(C.byref(p))
    for k, v in kw.items():
        if v is None:
            continue
        if not hasattr(p, k):
            raise TypeError(f"unknown parameter {k}")
        setattr(p, k, int(v))
    return p


# ----------------------------------------------------------- marshalling --
def _is_torch(a):
    return type(a).__module__.startswith("torch")


def _torch():
    import torch
    return torch


def _stream():
    return C.c_void_p(_torch().cuda.current_stream().cuda_stream)


def _dev(t, dtype, ref=None, name="argument"):
    """A CUDA tensor argument of a *_dev entry point: must be a CUDA tensor of the expected dtype
    ("float64", "int32", "uint8") on ref's device; returned contiguous -- the caller keeps the
    returned tensor alive until the call returns.  Wrong inputs raise TypeError instead of being
    read as fp64 row-major device memory."""
    if t is None:
        return None
    torch = _torch()
    if not _is_torch(t) or not t.is_cuda:
        raise TypeError(f"{name}: expected a CUDA tensor (device path), got {type(t).__name__}")
    want = getattr(torch, dtype)
    if t.dtype != want:
        raise TypeError(f"{name}: expected dtype {want}, got {t.dtype}")
    if ref is not None and t.device != ref.device:
        raise TypeError(f"{name}: on {t.device}, expected {ref.device}")
    return t.contiguous()


def _dev_out(t, dtype, ref, name="out"):
    """An output tensor of a *_dev entry point: CUDA, dtype, ref's device, and contiguous (a
    contiguous copy would not receive the results)."""
    if _dev(t, dtype, ref, name) is not t:
        raise TypeError(f"{name}: expected a contiguous CUDA {dtype} tensor")
    return t


def _host(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _ptr(a):
    if a is None:
        return None
    if _is_torch(a):
        return C.c_void_p(a.data_ptr())
    return a.ctypes.data_as(C.c_void_p)


def _u32(vals):
    return np.ascontiguousarray(np.asarray(vals, dtype=np.uint32))


# ---------------------------------------------------------------- forest --
@dataclass
class Forest:
    """Device-resident forest handle (freed on garbage collection)."""
    handle: C.c_void_p
    n_rows: int = 0
    _freed: bool = field(default=False, repr=False)

    def __del__(self):
        try:
            if not self._freed and self.handle:
                lib().rf_forest_free(self.handle)
                self._freed = True
        except Exception:
            pass

    def info(self):
        nt, tot, F, p, tg = C.c_uint32(), C.c_uint64(), C.c_int32(), C.c_uint32(), C.c_uint32()
        _check(lib().rf_forest_info(self.handle, C.byref(nt), C.byref(tot), C.byref(F), C.byref(p),
                                    C.byref(tg)))
        return dict(ntree=nt.value, total_nodes=tot.value, F=F.value, p=p.value, target=tg.value)

    def export(self):
        """Host copies: feature, left, value, thr_index [total_nodes]; tree_off [ntree+1]."""
        inf = self.info()
        m, T = inf["total_nodes"], inf["ntree"]
        feat = np.zeros(m, np.int32)
        left = np.zeros(m, np.uint32)
        val = np.zeros(m, np.float64)
        ti = np.zeros(m, np.uint32)
        off = np.zeros(T + 1, np.uint64)
        _check(lib().rf_forest_export(self.handle, _ptr(feat), _ptr(left), _ptr(val), _ptr(ti), _ptr(off)))
        return dict(feature=feat, left=left, value=val, thr_index=ti, tree_off=off, **inf)

    def importance(self, raw=False):
        """Feature importance [p] (MDI, rf_forest_importance); raw=True also returns the
        per-tree split-decrease sums [ntree][p]."""
        inf = self.info()
        imp = np.zeros(inf["p"], np.float64)
        r = np.zeros((inf["ntree"], inf["p"]), np.float64) if raw else None
        _check(lib().rf_forest_importance(self.handle, _ptr(imp), _ptr(r)))
        return (imp, r) if raw else imp

    def leaf_rows(self):
        inf = self.info()
        out = np.zeros((inf["ntree"], self.n_rows), np.int32)
        _check(lib().rf_forest_export_leaf_rows(self.handle, _ptr(out)))
        return out

    @property
    def ntree(self):
        return self.info()["ntree"]


def forest_import(feature, left, value, thr_index, tree_off, p, F, target, device=0) -> Forest:
    h = C.c_void_p()
    feature, left = _host(feature, np.int32), _host(left, np.uint32)
    value, thr_index, tree_off = _host(value, np.float64), _host(thr_index, np.uint32), _host(tree_off, np.uint64)
    _check(lib().rf_forest_import(_ptr(feature), _ptr(left), _ptr(value), _ptr(thr_index), _ptr(tree_off),
                                  len(tree_off) - 1, p, F, target, device, C.byref(h)))
    return Forest(h)


# ------------------------------------------------------------------- API --
def fit(X, y, *, ntree=100, mtry=0, min_samples_split=2, max_depth=-1, bootstrap=True,
        split_mode=SPLIT_EXACT, target=TARGET_IDENTITY, seed=0, device=0, tree_begin=0, tree_end=0,
        debug=False, criterion=CRITERION_MSE, tie_break=TIE_LOWEST_FEATURE) -> Forest:
    """Grow a forest (rf_fit).  X: [n, p] fp64, y: [n] fp64 (numpy or CUDA tensors).
    criterion: CRITERION_MSE or CRITERION_MAE (R32); tie_break:
    TIE_LOWEST_FEATURE (north_star) or TIE_DRAW_ORDER (R9)."""
    prm = params(ntree=ntree, mtry=mtry, min_samples_split=min_samples_split, max_depth=max_depth,
                 bootstrap=int(bootstrap), split_mode=split_mode, target=target, seed=seed, device=device,
                 tree_begin=tree_begin, tree_end=tree_end, criterion=criterion, tie_break=tie_break)
    h = C.c_void_p()
    if _is_torch(X):
        if debug:
            raise ValueError("debug fits take host arrays")
        X = _dev(X, "float64", None, "X")
        y = _dev(y, "float64", X, "y")
        n, p = X.shape
        _check(lib().rf_fit_dev(_ptr(X), n, p, _ptr(y), C.byref(prm), _stream(), C.byref(h)))
    else:
        X, y = _host(X, np.float64), _host(y, np.float64)
        n, p = X.shape
        fn = lib().rf_fit_debug if debug else lib().rf_fit
        _check(fn(_ptr(X), n, p, _ptr(y), C.byref(prm), C.byref(h)))
    return Forest(h, n_rows=n)


def predict(forest: Forest, X, out=None):
    """Mean of the trees' leaf values (exp for LOG forests)."""
    if _is_torch(X):
        torch = _torch()
        X = _dev(X, "float64", None, "X")
        n, p = X.shape
        out = torch.empty(n, dtype=torch.float64, device=X.device) if out is None else _dev_out(out, "float64", X)
        _check(lib().rf_predict_dev(forest.handle, _ptr(X), n, p, _ptr(out), _stream()))
        return out
    X = _host(X, np.float64)
    n, p = X.shape
    out = np.zeros(n, np.float64)
    _check(lib().rf_predict(forest.handle, _ptr(X), n, p, _ptr(out)))
    return out


def predict_partial(forest: Forest, X, out=None):
    """Sum over this forest's trees of the leaf values (tree-shard partial): CUDA tensors in and
    out (rf_predict_partial_dev), or host arrays (rf_predict_partial)."""
    if not _is_torch(X):
        X = _host(X, np.float64)
        n, p = X.shape
        out = np.zeros(n, np.float64)
        _check(lib().rf_predict_partial(forest.handle, _ptr(X), n, p, _ptr(out)))
        return out
    torch = _torch()
    X = _dev(X, "float64", None, "X")
    n, p = X.shape
    out = torch.empty(n, dtype=torch.float64, device=X.device) if out is None else _dev_out(out, "float64", X)
    _check(lib().rf_predict_partial_dev(forest.handle, _ptr(X), n, p, _ptr(out), _stream()))
    return out


def predict_finalize(partial, ntree_total, target, out=None):
    torch = _torch()
    partial = _dev(partial, "float64", None, "partial")
    out = torch.empty_like(partial) if out is None else _dev_out(out, "float64", partial)
    _check(lib().rf_predict_finalize_dev(_ptr(partial), partial.shape[0], ntree_total, target, _ptr(out),
                                         _stream()))
    return out


def make_folds(y, k, repeats=1, seed=0, custom=False, out=None):
    """Fold ids [repeats, n] (rf_make_folds)."""
    if _is_torch(y):
        torch = _torch()
        y = _dev(y, "float64", None, "y")
        n = y.shape[0]
        out = torch.empty((repeats, n), dtype=torch.int32, device=y.device) if out is None else \
            _dev_out(out, "int32", y)
        _check(lib().rf_make_folds_dev(_ptr(y), n, k, repeats, seed, int(custom), _ptr(out), _stream()))
        return out
    y = _host(y, np.float64)
    out = np.zeros((repeats, y.shape[0]), np.int32)
    _check(lib().rf_make_folds(_ptr(y), y.shape[0], k, repeats, seed, int(custom), _ptr(out)))
    return out


def make_folds_masked(y, k, mask, seed=0, custom=False, out=None):
    """Device fold ids [reps, n] of the row subsets mask [reps, n] != 0 (others -2), R31."""
    torch = _torch()
    y = _dev(y, "float64", None, "y")
    mask = _dev(mask.to(torch.uint8), "uint8", y, "mask")
    reps, n = mask.shape
    out = torch.empty((reps, n), dtype=torch.int32, device=y.device) if out is None else _dev_out(out, "int32", y)
    _check(lib().rf_make_folds_masked_dev(_ptr(y), n, k, reps, seed, int(custom), _ptr(mask),
                                          _ptr(out), _stream()))
    return out


def nested_cv(X, y, k_outer, k_inner, iterations, ntrees, mtrys, *, custom=False, min_samples_split=2,
              max_depth=-1, bootstrap=True, split_mode=SPLIT_EXACT, target=TARGET_IDENTITY, seed=0, device=0,
              criterion=CRITERION_MSE, tie_break=TIE_LOWEST_FEATURE):
    """Nested CV (rf_nested_cv, R31): (best [it, k_outer] grid index mi*n_ntree+ti,
    outer_mape [it, k_outer], inner_score [it, k_outer, n_mtry, n_ntree])."""
    prm = params(ntree=max(ntrees), mtry=0, min_samples_split=min_samples_split, max_depth=max_depth,
                 bootstrap=int(bootstrap), split_mode=split_mode, target=target, seed=seed, device=device,
                 criterion=criterion, tie_break=tie_break)
    nt, mt = _u32(ntrees), _u32(mtrys)
    if _is_torch(X):
        torch = _torch()
        X = _dev(X, "float64", None, "X")
        y = _dev(y, "float64", X, "y")
        n, p = X.shape
        best = torch.empty((iterations, k_outer), dtype=torch.int32, device=X.device)
        om = torch.empty((iterations, k_outer), dtype=torch.float64, device=X.device)
        sc = torch.empty((iterations, k_outer, len(mt), len(nt)), dtype=torch.float64, device=X.device)
        _check(lib().rf_nested_cv_dev(_ptr(X), n, p, _ptr(y), C.byref(prm), k_outer, k_inner, iterations,
                                      int(custom), _ptr(nt), len(nt), _ptr(mt), len(mt), _ptr(best), _ptr(om),
                                      _ptr(sc), _stream()))
        return best, om, sc
    X, y = _host(X, np.float64), _host(y, np.float64)
    n, p = X.shape
    best = np.zeros((iterations, k_outer), np.int32)
    om = np.zeros((iterations, k_outer), np.float64)
    sc = np.zeros((iterations, k_outer, len(mt), len(nt)), np.float64)
    _check(lib().rf_nested_cv(_ptr(X), n, p, _ptr(y), C.byref(prm), k_outer, k_inner, iterations, int(custom),
                              _ptr(nt), len(nt), _ptr(mt), len(mt), _ptr(best), _ptr(om), _ptr(sc)))
    return best, om, sc


def error_buckets(y, yhat):
    """LOO error buckets (rf_error_buckets): counts of APE in [0,10) [10,25) [25,50) [50,100) [100,inf) %."""
    if _is_torch(y):
        torch = _torch()
        y = _dev(y, "float64", None, "y")
        yhat = _dev(yhat, "float64", y, "yhat")
        out = torch.zeros(5, dtype=torch.int64, device=y.device)
        _check(lib().rf_error_buckets_dev(_ptr(y), _ptr(yhat), y.shape[0], _ptr(out), _stream()))
        return out
    y, yhat = _host(y, np.float64), _host(yhat, np.float64)
    out = np.zeros(5, np.uint64)
    _check(lib().rf_error_buckets(_ptr(y), _ptr(yhat), y.shape[0], _ptr(out)))
    return out.astype(np.int64)


def cross_validate_grid(X, y, k, repeats, ntrees, mtrys, fold_ids=None, *, want_pred=False,
                        min_samples_split=2, max_depth=-1, bootstrap=True, split_mode=SPLIT_EXACT,
                        target=TARGET_IDENTITY, seed=0, device=0, task_begin=0, task_end=0, out=None,
                        criterion=CRITERION_MSE, tie_break=TIE_LOWEST_FEATURE):
    """fold_mape [n_mtry, n_ntree, repeats, k] (+ pred [n_mtry, n_ntree, repeats, n])."""
    prm = params(ntree=max(ntrees), mtry=0, min_samples_split=min_samples_split, max_depth=max_depth,
                 bootstrap=int(bootstrap), split_mode=split_mode, target=target, seed=seed, device=device,
                 task_begin=task_begin, task_end=task_end, criterion=criterion, tie_break=tie_break)
    nt, mt = _u32(ntrees), _u32(mtrys)
    shape = (len(mt), len(nt), repeats, k)
    if _is_torch(X):
        torch = _torch()
        X = _dev(X, "float64", None, "X")
        y = _dev(y, "float64", X, "y")
        fold_ids = _dev(fold_ids, "int32", X, "fold_ids")
        n, p = X.shape
        fm = torch.empty(shape, dtype=torch.float64, device=X.device) if out is None else _dev_out(out, "float64", X)
        pr = torch.empty((len(mt), len(nt), repeats, n), dtype=torch.float64, device=X.device) \
            if want_pred else None
        _check(lib().rf_cross_validate_grid_dev(_ptr(X), n, p, _ptr(y), C.byref(prm), k, repeats,
                                                _ptr(fold_ids), _ptr(nt), len(nt), _ptr(mt), len(mt),
                                                _ptr(fm), _ptr(pr), _stream()))
    else:
        X, y = _host(X, np.float64), _host(y, np.float64)
        n, p = X.shape
        fm = np.zeros(shape, np.float64)
        pr = np.zeros((len(mt), len(nt), repeats, n), np.float64) if want_pred else None
        fid = None if fold_ids is None else _host(fold_ids, np.int32)
        _check(lib().rf_cross_validate_grid(_ptr(X), n, p, _ptr(y), C.byref(prm), k, repeats, _ptr(fid),
                                            _ptr(nt), len(nt), _ptr(mt), len(mt), _ptr(fm), _ptr(pr)))
    return (fm, pr) if want_pred else fm


def cross_validate(X, y, k, repeats=1, fold_ids=None, *, ntree=100, mtry=0, min_samples_split=2, max_depth=-1,
                   bootstrap=True, split_mode=SPLIT_EXACT, target=TARGET_IDENTITY, seed=0, device=0, tree_begin=0,
                   tree_end=0, task_begin=0, task_end=0, criterion=CRITERION_MSE, tie_break=TIE_LOWEST_FEATURE,
                   out=None):
    """One model under repeated k-fold CV (rf_cross_validate / rf_cross_validate_dev):
    fold_mape [repeats, k] in percent.  mtry 0 = the library default (R5)."""
    prm = params(ntree=ntree, mtry=mtry, min_samples_split=min_samples_split, max_depth=max_depth,
                 bootstrap=int(bootstrap), split_mode=split_mode, target=target, seed=seed, device=device,
                 tree_begin=tree_begin, tree_end=tree_end, task_begin=task_begin, task_end=task_end,
                 criterion=criterion, tie_break=tie_break)
    if _is_torch(X):
        torch = _torch()
        X = _dev(X, "float64", None, "X")
        y = _dev(y, "float64", X, "y")
        fold_ids = _dev(fold_ids, "int32", X, "fold_ids")
        n, p = X.shape
        fm = torch.empty((repeats, k), dtype=torch.float64, device=X.device) if out is None else \
            _dev_out(out, "float64", X)
        _check(lib().rf_cross_validate_dev(_ptr(X), n, p, _ptr(y), C.byref(prm), k, repeats, _ptr(fold_ids),
                                           _ptr(fm), _stream()))
        return fm
    X, y = _host(X, np.float64), _host(y, np.float64)
    n, p = X.shape
    fm = np.zeros((repeats, k), np.float64)
    fid = None if fold_ids is None else _host(fold_ids, np.int32)
    _check(lib().rf_cross_validate(_ptr(X), n, p, _ptr(y), C.byref(prm), k, repeats, _ptr(fid), _ptr(fm)))
    return fm


def cv_partial(X, y, k, repeats, fold_ids, ntrees, mtrys, *, tree_begin, tree_end, min_samples_split=2,
               max_depth=-1, bootstrap=True, target=TARGET_IDENTITY, seed=0, out=None, split_mode=SPLIT_EXACT,
               criterion=CRITERION_MSE, tie_break=TIE_LOWEST_FEATURE):
    """Tree-sharded CV partial sums [n_mtry, n_ntree, repeats, n] (device tensors, or host arrays
    through rf_cv_partial)."""
    prm = params(ntree=max(ntrees), min_samples_split=min_samples_split, max_depth=max_depth,
                 bootstrap=int(bootstrap), target=target, seed=seed, tree_begin=tree_begin, tree_end=tree_end,
                 split_mode=split_mode, criterion=criterion, tie_break=tie_break)
    nt, mt = _u32(ntrees), _u32(mtrys)
    n, p = X.shape
    if not _is_torch(X):
        X, y, fid = _host(X, np.float64), _host(y, np.float64), _host(fold_ids, np.int32)
        out = np.zeros((len(mt), len(nt), repeats, n), np.float64)
        _check(lib().rf_cv_partial(_ptr(X), n, p, _ptr(y), C.byref(prm), k, repeats, _ptr(fid), _ptr(nt), len(nt),
                                   _ptr(mt), len(mt), _ptr(out)))
        return out
    torch = _torch()
    X = _dev(X, "float64", None, "X")
    y = _dev(y, "float64", X, "y")
    fold_ids = _dev(fold_ids, "int32", X, "fold_ids")
    out = torch.empty((len(mt), len(nt), repeats, n), dtype=torch.float64, device=X.device) if out is None else \
        _dev_out(out, "float64", X)
    _check(lib().rf_cv_partial_dev(_ptr(X), n, p, _ptr(y), C.byref(prm), k, repeats, _ptr(fold_ids), _ptr(nt),
                                   len(nt), _ptr(mt), len(mt), _ptr(out), _stream()))
    return out


def cv_finalize(y, k, repeats, fold_ids, ntrees, n_mtry, reduced, *, target=TARGET_IDENTITY, want_pred=False,
                device=0):
    """Fold MAPEs (and predictions) from all-reduced partial sums (rf_cv_finalize[_dev])."""
    n = y.shape[0]
    nt = _u32(ntrees)
    if not _is_torch(y):
        y, fid, red = _host(y, np.float64), _host(fold_ids, np.int32), _host(reduced, np.float64)
        fm = np.zeros((n_mtry, len(nt), repeats, k), np.float64)
        pr = np.zeros((n_mtry, len(nt), repeats, n), np.float64) if want_pred else None
        _check(lib().rf_cv_finalize(_ptr(y), n, target, k, repeats, _ptr(fid), _ptr(nt), len(nt), n_mtry, _ptr(red),
                                    _ptr(fm), _ptr(pr), device))
        return (fm, pr) if want_pred else fm
    torch = _torch()
    y = _dev(y, "float64", None, "y")
    fold_ids = _dev(fold_ids, "int32", y, "fold_ids")
    reduced = _dev(reduced, "float64", y, "reduced")
    fm = torch.empty((n_mtry, len(nt), repeats, k), dtype=torch.float64, device=y.device)
    pr = torch.empty((n_mtry, len(nt), repeats, n), dtype=torch.float64, device=y.device) if want_pred else None
    _check(lib().rf_cv_finalize_dev(_ptr(y), n, target, k, repeats, _ptr(fold_ids), _ptr(nt), len(nt), n_mtry,
                                    _ptr(reduced), _ptr(fm), _ptr(pr), _stream()))
    return (fm, pr) if want_pred else fm


def set_profiling(on: bool):
    lib().rf_set_profiling(int(on))


def last_profile():
    """{kernel name: (total ms, launches)} of event-bracketed launches since set_profiling(True)."""
    cap = 64
    names = (C.c_char_p * cap)()
    ms = np.zeros(cap, np.float64)
    cnt = np.zeros(cap, np.uint32)
    m = lib().rf_last_profile(C.cast(names, C.c_void_p), _ptr(ms), _ptr(cnt), cap)
    return {names[i].decode(): (float(ms[i]), int(cnt[i])) for i in range(m)}


def counters():
    """(kernel launches issued by the library, candidate splits evaluated on this device)."""
    a, c = C.c_uint64(), C.c_uint64()
    _check(lib().rf_debug_counters(C.byref(a), C.byref(c)))
    return a.value, c.value


def row_levels(reset=False):
    """Row-levels (sum over levels and trees of live in-bag rows) grown by the large-n path."""
    v = C.c_uint64()
    _check(lib().rf_debug_row_levels(C.byref(v), 1 if reset else 0))
    return v.value


def launch_count():
    return counters()[0]


PHASE_NAMES = ["tree setup (bootstrap, root, in-bag lists)", "(a) node prefixes", "(a) feature draws",
               "(a) ExtraTrees bounds", "(b) search pass 1 + scan", "(b) search pass 2 + node bests",
               "(c) decide", "(d) mark", "(e) children / emission", "(f) test-row routing",
               "(g) partition list 0", "(g) partition lists 1..p-1", "level advance", "tree end",
               "CTA prologue", "unused"]


def phase_cycles(reset=True):
    """Per-phase SM cycles of the tree kernel summed over warps (profiling build only:
    RF_PHASE_TIMING=1 python -m paper_2001_07104_b200.build, then RFGPU_LIB=.../librfgpu_pt.so)."""
    out = np.zeros(16, np.uint64)
    _check(lib().rf_debug_phase_cycles(_ptr(out), 1 if reset else 0))
    return dict(zip(PHASE_NAMES, out.tolist()))


def debug_set_option(name: str, value: int):
    """Test switch of alternative kernel paths (rf_debug_set_option)."""
    _check(lib().rf_debug_set_option(name.encode(), int(value)))


def candidate_count():
    return counters()[1]


def debug_ln(y):
    torch = _torch()
    out = torch.empty_like(y)
    _check(lib().rf_debug_ln_dev(_ptr(y), _ptr(out), y.shape[0], _stream()))
    return out


def debug_philox(ctr_key):
    """ctr_key: int tensor [m, 6] (c0..c3, k0, k1) on CUDA -> [m, 4] uint32 (as int64 tensor)."""
    torch = _torch()
    m = ctr_key.shape[0]
    inp = ctr_key.to(torch.int64).to(torch.int32).contiguous()
    out = torch.empty((m, 4), dtype=torch.int32, device=ctr_key.device)
    _check(lib().rf_debug_philox_dev(_ptr(inp), _ptr(out), m, _stream()))
    return out.to(torch.int64) & 0xFFFFFFFF


def importance_dev(raw, out=None):
    """Device: importance [p] from per-tree split-decrease sums raw [ntree][p]
    (torch float64 CUDA tensor; e.g. all-gathered tree shards), rf_importance_dev."""
    import torch
    raw = _dev(raw, "float64", None, "raw")
    T, p = raw.shape
    if out is None:
        out = torch.empty(p, dtype=torch.float64, device=raw.device)
    _check(lib().rf_importance_dev(_ptr(raw), T, p, _ptr(out), _stream()))
    return out
