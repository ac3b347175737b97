/*
 * rf.h -- C ABI of librfgpu.so, the B200 (sm_100a) implementation of the
 * random-forest cross-validation hot path of arXiv 2001.07104 (Braun et al.,
 * "A Simple Model for Portable and Fast Prediction of Execution Time and
 * Power Consumption of GPU Kernels").
 *
 * Citations: P:n = PAPER.md line n; Rn = reading n of DESIGN.md section 2
 * (where the paper is silent, ambiguous or garbled).
 *
 * The operations (sec. 3): samples x_i with labels y_i;
 * find g: X -> Y minimising the prediction error, scored by MAPE (Eq. 1,
 * P:400-403).  g is a random forest (sec. 2.2): n_estimators
 * trees, each node compares one feature with a threshold, a leaf outputs a
 * value; max_features features are considered per node split.
 * The model is trained per (GPU, target) and chosen by repeated k-fold
 * cross-validation over ntree x max_features.
 *
 * Conventions (all entry points):
 *  - Every call returns rf_status; RF_OK = 0.  No C++ exception crosses the
 *    ABI.  On error, rf_last_error() (thread-local) describes it, outputs are
 *    unspecified and any rf_forest** out is set to NULL.
 *  - Layouts: X is n x p row-major fp64; y, yhat are fp64[n]; fold ids int32.
 *  - Host-pointer functions (no suffix) borrow their inputs (not retained),
 *    copy them to the device of params->device, and return after the results
 *    are in the caller's host buffers.
 *  - *_dev functions take DEVICE pointers (same layouts) on the current CUDA
 *    device and a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  Work is enqueued on that stream; a call may synchronise the
 *    stream internally when it needs a size on the host (documented per call).
 *    Results are complete when the stream is synchronised.
 *  - Threads: every entry point may be called from several host threads at
 *    once; host-pointer calls run on a per-thread, per-device CUDA stream, so
 *    concurrent calls overlap on the GPU.  A forest handle may be read
 *    (predict, export) concurrently; rf_forest_free must not race its users.
 *  - The library never calls NCCL: multi-GPU sharding is by tree range
 *    (tree_begin/end) and CV task range (task_begin/end); the Python driver
 *    performs the collectives.
 *  - No CPU fallback: without a usable CUDA device every call returns
 *    RF_E_CUDA.
 */
#ifndef RF_H
#define RF_H

#include <stdint.h>

#if defined(__GNUC__)
#define RF_API __attribute__((visibility("default")))
#else
#define RF_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RF_OK = 0,
  RF_E_ARG = 1,            /* invalid argument / parameter combination            */
  RF_E_EMPTY = 2,          /* n == 0                                              */
  RF_E_NONFINITE = 3,      /* NaN/Inf in X or y                                   */
  RF_E_NONPOSITIVE_Y = 4,  /* y <= 0 with LOG target or in any CV call (Eq. 1)    */
  RF_E_ARITY = 5,          /* predict with p different from the forest's          */
  RF_E_TOO_FEW = 6,        /* k < 2, k > n, an empty test fold, too few rows      */
  RF_E_CUDA = 7,           /* CUDA runtime error (incl. no device)                */
  RF_E_OOM = 8,            /* device allocation failed                            */
  RF_E_OVERFLOW = 9,       /* size limits of a kernel variant exceeded           */
  RF_E_UNSUPPORTED = 10,   /* valid request outside what this build implements    */
  RF_E_INEXACT = 11        /* LOG target: ln(y) of some y could not be certified  */
                           /* correctly rounded (within ~2^-94 relative of a      */
                           /* rounding boundary; R20) -- no result is   */
                           /* produced rather than a possibly misrounded t_q      */
} rf_status;

/* Split rule.  EXACT: every boundary between consecutive distinct in-node
   values (R8).  HIST256: 256 quantile bins per (task, feature) (R23).
   EXTRA: Extremely Randomized Trees, the paper's learner: per
   drawn feature one threshold uniform in [min, max) of its in-node values
   (R29).  All three share the criterion, tie-break, stopping and leaves. */
typedef enum { RF_SPLIT_EXACT = 0, RF_SPLIT_HIST256 = 1, RF_SPLIT_EXTRA = 2 } rf_split_mode;
typedef enum { RF_TARGET_IDENTITY = 0, RF_TARGET_LOG = 1 } rf_target;
/* Split criterion.  MSE: variance reduction, leaves hold the
   weighted in-bag mean (R6, R13).  MAE (the paper's best models
   in Tables 4/5): a split minimises the summed weighted absolute
   deviations of the children from their weighted medians, leaves hold the
   weighted median (R32).  MAE is implemented for the exact and ExtraTrees
   split modes on both paths: the CTA-resident kernel (training sets of <= 255
   rows, p <= 64; the paper's datasets have 189 / 168 rows) and the
   level-synchronous one up to 12,288 training rows (the paper's n = 4,096
   sensitivity variant); histogram mode and larger training sets return
   RF_E_UNSUPPORTED.  Under MAE the targets are quantised with 2 guard bits
   (F = 62 - ceil(log2 n) - e - 2) so doubled medians and doubled absolute-
   deviation sums are exact integers below 2^63. */
typedef enum { RF_CRITERION_MSE = 0, RF_CRITERION_MAE = 1 } rf_criterion;
/* Tie-break among candidate splits with bitwise-equal scores (R9; the paper is
   silent).  LOWEST_FEATURE (default): the lowest feature index, then the
   lowest threshold -- BASELINE.json north_star's "deterministic tie-break of
   lowest feature then lowest threshold".  DRAW_ORDER: the feature drawn first
   at the node (the lowest slot of R4's partial Fisher-Yates), then the lowest
   threshold -- scikit-learn's splitter (the paper's library) visits
   the features in draw order and keeps the first best.  Both are total orders
   over a node's candidates, so the GPU's reduction order cannot change them. */
typedef enum { RF_TIE_LOWEST_FEATURE = 0, RF_TIE_DRAW_ORDER = 1 } rf_tie_break;

/* Hyper-parameters and sharding. */
typedef struct {
  uint32_t struct_size;       /* = sizeof(rf_params) (ABI versioning)                    */
  uint32_t ntree;             /* n_estimators >= 1                               */
  uint32_t mtry;              /* max_features 1..p; 0 => max(1, floor(p/3)) (R5) */
  uint32_t min_samples_split; /* >= 2: nodes with fewer distinct in-bag rows are leaves   */
  int32_t max_depth;          /* -1 = unbounded (default, R11)                    */
  uint32_t bootstrap;         /* 1: n_tr draws with replacement (R2); 0: all weights 1   */
  uint32_t split_mode;        /* rf_split_mode: exact (R8), 256-bin (R23), extra (R29)   */
  uint32_t target;            /* rf_target: LOG fits ln y, predicts exp      */
  uint64_t seed;              /* Philox key of every random draw (R14-R16)               */
  int32_t device;             /* CUDA ordinal for host-pointer calls                     */
  uint32_t tree_begin;        /* this rank's trees [tree_begin, tree_end); 0,0 = all     */
  uint32_t tree_end;
  uint32_t task_begin;        /* CV tasks (task = rep*k + fold) [task_begin, task_end);  */
  uint32_t task_end;          /*   0,0 = all; outputs of other tasks are NaN             */
  uint32_t criterion;         /* rf_criterion: MSE (default) or MAE (R32)                */
  uint32_t tie_break;         /* rf_tie_break: lowest feature (default) or draw order    */
} rf_params;

/* Fills the defaults: ntree 100, mtry 0, min_samples_split 2, max_depth -1,
   bootstrap 1, exact, IDENTITY, seed 0, device 0, no sharding, MSE,
   lowest-feature tie-break. */
RF_API void rf_params_default(rf_params* prm);

/* Opaque device-resident forest: flattened BFS nodes (16 B each:
   {int32 feature (-1 = leaf), uint32 left child (right = left+1),
    fp64 threshold or leaf value}), tree offsets, F, p, target.
   Owned by the caller; release with rf_forest_free. */
typedef struct rf_forest rf_forest;

/* rf_fit: grow trees [tree_begin, tree_end) (all if 0,0) of one forest on all
   n rows (task 0).  Tree t uses Philox key k_t = f(seed, task 0, t) (R15), so
   a forest of T trees is the prefix of any larger one and a tree shard is
   identical to the same trees of the full forest.
   Errors: RF_E_EMPTY, RF_E_NONFINITE, RF_E_NONPOSITIVE_Y (LOG), RF_E_INEXACT
   (LOG), RF_E_ARG. */
RF_API rf_status rf_fit(const double* X, uint64_t n, uint32_t p, const double* y, const rf_params* prm,
                 rf_forest** out);
/* Device twin.  Synchronises `stream` once (forest size). */
RF_API rf_status rf_fit_dev(const double* dX, uint64_t n, uint32_t p, const double* dy,
                     const rf_params* prm, void* stream, rf_forest** out);

/* rf_predict: yhat[i] = mean over the forest's trees of the leaf reached by
   row i (x[f] <= thr goes left), exp() for LOG.  Host X
   [n][p] and yhat [n]; batches above ~1 GB of X are streamed in ~512 MB
   chunks over two CUDA streams (copies overlap the walks when X is pinned;
   device memory stays at two chunks).  Synchronous.
   Errors: RF_E_ARITY (p differs), RF_E_NONFINITE. */
RF_API rf_status rf_predict(const rf_forest* f, const double* X, uint64_t n, uint32_t p, double* yhat);
RF_API rf_status rf_predict_dev(const rf_forest* f, const double* dX, uint64_t n, uint32_t p,
                         double* dyhat, void* stream);
/* Sum over this forest's trees of the leaf values (not divided, not exp'd):
   the per-rank partial of a tree-sharded forest, to be all-reduced. */
RF_API rf_status rf_predict_partial_dev(const rf_forest* f, const double* dX, uint64_t n, uint32_t p,
                                 double* dpartial, void* stream);
/* Finish a reduced partial: yhat = partial / ntree_total, exp if LOG. */
RF_API rf_status rf_predict_finalize_dev(const double* dpartial, uint64_t n, uint32_t ntree_total,
                                  uint32_t target, double* dyhat, void* stream);
/* Host twin of rf_predict_partial_dev (host X in, host partial[n] out; synchronous). */
RF_API rf_status rf_predict_partial(const rf_forest* f, const double* X, uint64_t n, uint32_t p,
                                    double* partial);

/* rf_make_folds: fold ids [repeats][n] in {-1 (always train), 0..k-1}.
   Plain (custom = 0): rows ordered by Philox keys (seed, rep), contiguous
   blocks of floor(n/k) (+1 for the first n mod k folds) (R16).
   Custom (custom = 1, time targets): the 5 largest y always train;
   the rest stratified short (<1e3 us) / medium (<1e5) / long (R17), each
   stratum in Philox order, dealt round-robin over folds.
   Errors: RF_E_TOO_FEW (k < 2, k > n, custom with n - 5 < k). */
RF_API rf_status rf_make_folds(const double* y, uint64_t n, uint32_t k, uint32_t repeats, uint64_t seed,
                        uint32_t custom, int32_t* fold_ids);
RF_API rf_status rf_make_folds_dev(const double* dy, uint64_t n, uint32_t k, uint32_t repeats,
                            uint64_t seed, uint32_t custom, int32_t* dfold_ids, void* stream);

/* Folds of a row subset per repeat (nested CV, R31): rows with
   dmask[rep*n + i] != 0 are split exactly as rf_make_folds splits a dataset
   of those rows (Philox keys indexed by the original row); the others get
   -2 (excluded: neither train nor test in the CV calls).  n <= 4096
   (RF_E_UNSUPPORTED beyond).  Stream-ordered, no synchronisation. */
RF_API rf_status rf_make_folds_masked_dev(const double* dy, uint64_t n, uint32_t k, uint32_t repeats,
                                          uint64_t seed, uint32_t custom, const uint8_t* dmask,
                                          int32_t* dfold_ids, void* stream);

/* rf_cross_validate_grid: repeated k-fold CV of every (mtry,
   ntree) grid point.  For each task (rep, fold) and each mtry,
   max(ntrees) trees are grown on the training rows (fold id != fold) and
   every ntree value is scored as a prefix (R19).  fold_ids: [repeats][n]
   (NULL => plain folds from prm->seed).  Output fold_mape
   [n_mtry][n_ntree][repeats][k] in percent (Eq. 1, on raw y).  Optional
   pred [n_mtry][n_ntree][repeats][n]: each row's prediction by the forest of
   its test fold (NaN for rows with fold -1); pass NULL to skip.
   Errors: RF_E_NONPOSITIVE_Y (any y <= 0), RF_E_INEXACT (LOG), RF_E_TOO_FEW, RF_E_ARG
   (tree_begin/end set: use rf_cv_partial), RF_E_UNSUPPORTED (n_tr > 255 in
   this build's exact small-tree kernel without the large path).
   The _dev twin synchronises `stream` once (per-task sizes). */
RF_API rf_status rf_cross_validate_grid(const double* X, uint64_t n, uint32_t p, const double* y,
                                 const rf_params* prm, uint32_t k, uint32_t repeats,
                                 const int32_t* fold_ids, const uint32_t* ntrees, uint32_t n_ntree,
                                 const uint32_t* mtrys, uint32_t n_mtry, double* fold_mape,
                                 double* pred);
RF_API rf_status rf_cross_validate_grid_dev(const double* dX, uint64_t n, uint32_t p, const double* dy,
                                     const rf_params* prm, uint32_t k, uint32_t repeats,
                                     const int32_t* dfold_ids, const uint32_t* ntrees,
                                     uint32_t n_ntree, const uint32_t* mtrys, uint32_t n_mtry,
                                     double* dfold_mape, double* dpred, void* stream);
/* rf_cross_validate: the problem statement's call:
   repeated k-fold CV of ONE model -- prm->ntree trees, prm->mtry features per
   split (0 => max(1, floor(p/3)), R5) -- returning per-fold MAPE
   fold_mape [repeats][k] in percent (Eq. 1, raw y).  fold_ids as in
   rf_cross_validate_grid ([repeats][n] in {-1, 0..k-1}; NULL => plain Philox
   folds from prm->seed, R16).  Same as rf_cross_validate_grid with the grid
   {prm->ntree} x {mtry}.  Errors: RF_E_NONPOSITIVE_Y (any y <= 0), RF_E_TOO_FEW
   (k < 2, k > n, an empty test fold), RF_E_ARG (tree_begin/end set: a rank
   cannot score a partial forest -- use rf_cv_partial), plus those of rf_fit.
   The _dev twin takes device pointers and a stream (synchronised once). */
RF_API rf_status rf_cross_validate(const double* X, uint64_t n, uint32_t p, const double* y,
                            const rf_params* prm, uint32_t k, uint32_t repeats,
                            const int32_t* fold_ids, double* fold_mape);
RF_API rf_status rf_cross_validate_dev(const double* dX, uint64_t n, uint32_t p, const double* dy,
                                       const rf_params* prm, uint32_t k, uint32_t repeats,
                                       const int32_t* dfold_ids, double* dfold_mape, void* stream);

/* Nested cross-validation ("First the scores of each hyperparameter
   combination are computed on all splits, then the best parameter combination
   is used to compute scores on all splits again"; R31), as two
   batched grid-CV launches:
     outer folds  = rf_make_folds(y, k_outer, iterations, prm->seed, custom);
     combo c = it*k_outer + o: inner folds split the rows outside outer fold o
       (rf_make_folds_masked, rep c, seed prm->seed ^ 0x4E45535445440000);
     inner grid CV over all combos (one call, tree keys from the inner seed);
     best[c] = first grid point g = mi*n_ntree + ti with the lowest
       (sum of its inner fold MAPEs in fold order) / k_inner;
     outer grid CV on the outer folds; outer_mape[c] = its fold MAPE at best[c].
   Outputs (host or device per twin): best int32 [iterations][k_outer],
   outer_mape fp64 [iterations][k_outer], inner_score fp64
   [iterations][k_outer][n_mtry][n_ntree] (or NULL).  prm->ntree/mtry are
   ignored (the grid decides); tree/task ranges must be 0.  n <= 4096.
   Errors: as rf_cross_validate_grid; RF_E_TOO_FEW if an outer-training set
   cannot hold k_inner folds. */
RF_API rf_status rf_nested_cv(const double* X, uint64_t n, uint32_t p, const double* y, const rf_params* prm,
                              uint32_t k_outer, uint32_t k_inner, uint32_t iterations, uint32_t custom,
                              const uint32_t* ntrees, uint32_t n_ntree, const uint32_t* mtrys, uint32_t n_mtry,
                              int32_t* best, double* outer_mape, double* inner_score);
RF_API rf_status rf_nested_cv_dev(const double* dX, uint64_t n, uint32_t p, const double* dy,
                                  const rf_params* prm, uint32_t k_outer, uint32_t k_inner,
                                  uint32_t iterations, uint32_t custom, const uint32_t* ntrees,
                                  uint32_t n_ntree, const uint32_t* mtrys, uint32_t n_mtry, int32_t* dbest,
                                  double* douter_mape, double* dinner_score, void* stream);

/* LOO error buckets: counts[5] of the absolute percentage error
   100 * (|y - yhat| / y) in [0,10), [10,25), [25,50), [50,100), [100,inf);
   NaN predictions (rows without a prediction) are skipped.  Leave-one-out
   itself is rf_cross_validate_grid with k = n. */
RF_API rf_status rf_error_buckets(const double* y, const double* yhat, uint64_t n, uint64_t* counts);
RF_API rf_status rf_error_buckets_dev(const double* dy, const double* dyhat, uint64_t n, uint64_t* dcounts,
                                      void* stream);

/* Tree-sharded CV (multi-GPU): per-row partial sums of
   leaf values over this rank's trees [tree_begin, tree_end) for each grid
   point: dpartial [n_mtry][n_ntree][repeats][n] (sum over the rank's trees
   that lie below each ntree prefix; not divided, not exp'd).  The caller
   all-reduces (SUM) across ranks and calls rf_cv_finalize_dev. */
RF_API rf_status rf_cv_partial_dev(const double* dX, uint64_t n, uint32_t p, const double* dy,
                            const rf_params* prm, uint32_t k, uint32_t repeats,
                            const int32_t* dfold_ids, const uint32_t* ntrees, uint32_t n_ntree,
                            const uint32_t* mtrys, uint32_t n_mtry, double* dpartial,
                            void* stream);
RF_API rf_status rf_cv_finalize_dev(const double* dy, uint64_t n, uint32_t target, uint32_t k,
                             uint32_t repeats, const int32_t* dfold_ids, const uint32_t* ntrees,
                             uint32_t n_ntree, uint32_t n_mtry, const double* dreduced,
                             double* dfold_mape, double* dpred, void* stream);
/* Host twins of the tree-sharded CV pair (host buffers in and out, synchronous; fold_ids
   are required, [repeats][n]; partial / reduced [n_mtry][n_ntree][repeats][n]; fold_mape
   [n_mtry][n_ntree][repeats][k]; pred may be NULL).  Device: prm->device. */
RF_API rf_status rf_cv_partial(const double* X, uint64_t n, uint32_t p, const double* y,
                               const rf_params* prm, uint32_t k, uint32_t repeats,
                               const int32_t* fold_ids, const uint32_t* ntrees, uint32_t n_ntree,
                               const uint32_t* mtrys, uint32_t n_mtry, double* partial);
RF_API rf_status rf_cv_finalize(const double* y, uint64_t n, uint32_t target, uint32_t k,
                                uint32_t repeats, const int32_t* fold_ids, const uint32_t* ntrees,
                                uint32_t n_ntree, uint32_t n_mtry, const double* reduced,
                                double* fold_mape, double* pred, int32_t device);

RF_API void rf_forest_free(rf_forest* f);
RF_API const char* rf_last_error(void);

/* Introspection / parity export (host copies). */
RF_API rf_status rf_forest_info(const rf_forest* f, uint32_t* ntree, uint64_t* total_nodes, int32_t* F,
                         uint32_t* p, uint32_t* target);
/* Flattened copy: feature/left/value/thr_index [total_nodes], tree_off [ntree+1].
   value = threshold of an internal node, leaf value of a leaf. */
RF_API rf_status rf_forest_export(const rf_forest* f, int32_t* feature, uint32_t* left, double* value,
                           uint32_t* thr_index, uint64_t* tree_off);
/* Leaf of every input row per tree [ntree][n] (-1 = out of bag); only if the
   forest was grown with rf_fit_debug. */
RF_API rf_status rf_forest_export_leaf_rows(const rf_forest* f, int32_t* leaf_of_row);
/* rf_fit that also records leaf_of_row (parity tests). */
RF_API rf_status rf_fit_debug(const double* X, uint64_t n, uint32_t p, const double* y,
                       const rf_params* prm, rf_forest** out);
/* Feature importance (mean decrease in impurity; SURVEY 8(f) NEXT-3, P:218-219,
   Table 6).  Each split adds W imp(node) - WL imp(L) - WR imp(R)
   (imp = in-bag weighted MSE of the quantised target, R30) to its
   feature; importance[p] (host) = the per-tree sums divided by their tree's
   total, summed over trees, divided by the grand total (scikit-learn's rule;
   all zeros if no tree has a positive decrease).  raw (host [ntree][p] or
   NULL) receives the per-tree sums in target units.  Only forests grown by
   rf_fit / rf_fit_dev carry them: RF_E_UNSUPPORTED for imported forests
   (combine shards' raw arrays with rf_importance_dev). */
RF_API rf_status rf_forest_importance(const rf_forest* f, double* importance, double* raw);
/* Device: importance[p] from per-tree sums draw [ntree][p] (e.g. all-gathered
   from tree shards), same rule.  Synchronises nothing; stream-ordered. */
RF_API rf_status rf_importance_dev(const double* draw, uint32_t ntree, uint32_t p, double* dimportance,
                                   void* stream);

/* Build a forest from flattened arrays on the host (multi-GPU assembly). */
RF_API rf_status rf_forest_import(const int32_t* feature, const uint32_t* left, const double* value,
                           const uint32_t* thr_index, const uint64_t* tree_off, uint32_t ntree,
                           uint32_t p, int32_t F, uint32_t target, int32_t device,
                           rf_forest** out);

/* Per-kernel timing of the last call on this thread (bench roofline):
   names[i] / ms[i] / launches[i] for up to cap kernels; returns the count. */
RF_API uint32_t rf_last_profile(const char** names, double* ms, uint32_t* launches, uint32_t cap);
/* 1 to record per-kernel CUDA events (adds event records, no syncs). */
RF_API void rf_set_profiling(int on);

#ifdef __cplusplus
}
#endif
#endif /* RF_H */
