// large_tree.cuh -- level-synchronous growth for training sets beyond the
// CTA-resident small-tree kernel (n_tr > 255), exact split mode.
#pragma once
#include <string>
#include <vector>
#include "../../include/rf.h"
#include "common.cuh"
#include "cv.cuh"
#include "host_util.cuh"
#include "prep.cuh"

namespace rf {

// test switch (rf_debug_set_option "large_tiled_partition"): force the tiled partition
extern int g_opt_tiled_partition;
extern long long g_opt_hist_node_cap;  // test switch: histogram node-chunk cap (0 = by memory)

// Grows trees [tree_lo, tree_hi) of task 0 over all rows.  Outputs (scratch
// owned by `sc`): per-tree BFS node blocks of capacity *cap, node counts.
rf_status fit_large(const DevData& d, const rf_params* prm, int mtry, int tree_lo, int tree_hi,
                    cudaStream_t s, Scratch& sc, Node16** nodes, uint32_t** thr_index,
                    uint32_t** nnodes, uint64_t* cap, int32_t* leaf_of_row, double* imp,
                    std::string& err);

// CV tasks whose training sets exceed the small-tree kernel: for every task and
// every distinct mtry, grow trees [tree_lo, tree_hi) and write the per-chunk
// (Cw trees) sums of the test rows' leaf values into
// partial [n_mtry][ntask][nsub][nte_max] -- the layout the small-tree kernel
// produces, scored by score_cv.
rf_status cv_large_partial(const DevData& d, const TaskData& td, const rf_params* prm,
                           const std::vector<int>& mtrys, int tree_lo, int tree_hi, int Cw, int nsub,
                           int nte_max, double* partial, cudaStream_t s, Scratch& sc, std::string& err);

}  // namespace rf
