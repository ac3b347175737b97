// cv.cuh -- cross-validation plumbing on the device: folds, per-task row
// sets and orders, prefix-forest scoring (Eq. 1).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace rf {

// fold ids [reps][n]; custom = paper's time split (R17); dmask (nullable,
// [reps][n], n <= 4096): split only the rows with mask != 0, the others get -2 (R31)
cudaError_t make_folds(const double* dy, int n, int k, int reps, uint64_t seed, int custom,
                       int32_t* dfold, void* ws, size_t ws_bytes, cudaStream_t s,
                       const uint8_t* dmask = nullptr);
size_t make_folds_ws_bytes(int n, int reps, int custom);

struct TaskData {
  int ntask = 0, task0 = 0, n = 0, p = 0, ntr_stride = 0;
  uint32_t* tr_rows = nullptr;  // [ntask][n]
  uint32_t* te_rows = nullptr;  // [ntask][n]
  int32_t* loc = nullptr;       // [ntask][n] local training index, -1 = test
  int32_t* ntr = nullptr;       // [ntask]
  int32_t* nte = nullptr;       // [ntask]
  uint8_t* ord = nullptr;       // [ntask][p][ntr_stride]
  uint8_t* lrank = nullptr;     // [ntask][p][ntr_stride]
};

// dfold == nullptr: a single task with every row training (rf_fit)
cudaError_t build_tasks(const int32_t* dfold, int k, const uint32_t* order, const uint32_t* grank,
                        TaskData& t, cudaStream_t s);
// small-kernel orders (n_tr <= 255): ord/lrank as u8
cudaError_t build_task_orders_u8(const uint32_t* order, const uint32_t* grank, TaskData& t,
                                 cudaStream_t s);

// per (mtry, ntree prefix, rep, fold): prediction of each test row and MAPE.
struct ScoreArgs {
  const double* partial;  // [n_mtry][ntask][nsub][nte_max]
  int n_mtry, ntask, nsub, nte_max, Cw, tree_lo;
  const uint32_t* te_rows;  // [ntask][n]
  const int32_t* nte;
  int n, k, reps, task0;
  int n_ntree;
  int ntrees[16];
  int target;
  const double* y;
  double* fold_mape;  // [n_mtry][n_ntree][reps][k]
  double* pred;       // [n_mtry][n_ntree][reps][n] or null
  double* partial_rows;  // tree-sharded mode: [n_mtry][n_ntree][reps][n] un-divided sums or null
};
cudaError_t score_cv(const ScoreArgs& a, cudaStream_t s);

// finalize reduced partial sums: pred = sum / ntree (exp for LOG), MAPE per fold
cudaError_t finalize_cv(const double* reduced, const double* y, const int32_t* fold, int n, int k,
                        int reps, int n_mtry, int n_ntree, const int* ntrees, int target,
                        double* fold_mape, double* pred, cudaStream_t s);

// nested CV (R31): mask[c][i] = outer[it][i] != o (c = it*k_outer + o); per combo the
// first grid point with the lowest mean inner MAPE; the outer MAPE at that point
cudaError_t nested_mask(const int32_t* outer, int n, int k_outer, int C, uint8_t* mask, cudaStream_t s);
cudaError_t nested_select(const double* fm_in, int nm, int nt, int C, int k_in, int32_t* best, double* score,
                          cudaStream_t s);
cudaError_t nested_pick(const double* fm_out, const int32_t* best, int nt, int C, int k_out, int iters,
                        double* outer_mape, cudaStream_t s);
// LOO error buckets: counts[5] of APE in [0,10) [10,25) [25,50) [50,100) [100,inf) %
cudaError_t ape_buckets(const double* y, const double* yhat, int64_t n, unsigned long long* counts, cudaStream_t s);

}  // namespace rf
