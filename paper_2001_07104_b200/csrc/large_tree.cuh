// large_tree.cuh -- level-synchronous growth for training sets beyond the
// CTA-resident small-tree kernel (n_tr > 255, exact or 256-bin histogram).
#pragma once
#include <string>
#include "../../include/rf.h"
#include "common.cuh"
#include "cv.cuh"
#include "host_util.cuh"
#include "prep.cuh"

namespace rf {

// Grows trees [tree_lo, tree_hi) of task 0 over all rows.  Outputs (scratch
// owned by `sc`): per-tree node blocks of capacity *cap, node counts.
rf_status fit_large(const DevData& d, const rf_params* prm, int mtry, int tree_lo, int tree_hi,
                    cudaStream_t s, Scratch& sc, Node16** nodes, uint32_t** thr_index,
                    uint32_t** nnodes, uint64_t* cap, int32_t* leaf_of_row, std::string& err);

// CV for tasks whose training sets exceed the small-tree kernel.
rf_status cv_large(const double* dX, const DevData& d, const TaskData& td, const int32_t* dfold,
                   const rf_params* prm, uint32_t k, uint32_t reps, const uint32_t* ntrees,
                   uint32_t n_ntree, const uint32_t* mtrys, uint32_t n_mtry, int tree_lo, int tree_hi,
                   int ntr_max, int nte_max, double* dfold_mape, double* dpred, double* dpartial_rows,
                   cudaStream_t s, Scratch& sc, std::string& err);

}  // namespace rf
