// small_tree.cuh -- interface of the warp-per-tree kernel (CTA-resident data).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "common.cuh"

namespace rf {

constexpr int kSmallMaxRows = 255;  // n_tr <= 255: u8 local indices, u8 bootstrap counts
constexpr int kSmallMaxP = 64;
constexpr int kSmallKMax = 8;       // ceil(255 / 32)
constexpr int kMaxMtry = 16;        // grid points per launch
#ifndef RF_SMALL_MAXWPB
#define RF_SMALL_MAXWPB 14
#endif
// warps per CTA (launch bound 32 x kSmallMaxWpb threads); the host picks the count with the most
// resident warps (A/B on the full study, round 1: up to 16 warps in one CTA per SM beat 2 CTAs x 7
// warps by 5 %; round 2, after the search's segment-end prefetch: the 14-warp bound -- on the C2
// shapes the host then runs two CTAs of 8 warps per SM -- beat one CTA of 16 by 3 %; 12 (158
// registers) lost 16 %, 20 (96 registers) 14 %: profiles/rd2_32_ab_occ.txt, rd2_36/38_ab_c2.txt)
constexpr int kSmallMaxWpb = RF_SMALL_MAXWPB;

struct SmallArgs {
  // dataset (device)
  const double* X;          // [n][p] canonical
  int n, p;
  const int64_t* tq;        // [n] quantised targets
  const int32_t* dF;        // quantisation exponent F (device scalar)
  const uint32_t* grank;    // [p][n] global dense ranks (fit mode: threshold index)
  // tasks (device)
  int ntask;                // tasks in this launch
  int task0;                // global id of local task 0 (Philox key)
  int row_stride;           // stride of tr_rows/te_rows rows (>= n)
  int ntr_stride;           // stride of ord/lrank per feature (>= max ntr)
  const int32_t* ntr;       // [ntask]
  const int32_t* nte;       // [ntask]
  const uint32_t* tr_rows;  // [ntask][row_stride] global training rows, ascending
  const uint32_t* te_rows;  // [ntask][row_stride] global test rows, ascending
  const uint8_t* ord;       // [ntask][p][ntr_stride] local idx sorted by x_f (stable)
  const uint8_t* lrank;     // [ntask][p][ntr_stride] dense rank of x_f among training rows
  int ntr_max, nte_max;     // over the launch's tasks
  // forest parameters
  uint64_t seed;
  int bootstrap, min_split, max_depth;
  int extra;                // ExtraTrees split mode (R29): one random threshold per drawn feature
  int mae;                  // MAE criterion (R32): absolute deviations from weighted medians
  int tie_draw;             // tie-break (R9): 0 lowest feature index (north_star), 1 first drawn
  int n_mtry;
  int mtrys[kMaxMtry];
  int tree_lo, tree_hi;     // trees [tree_lo, tree_hi)
  int Cw;                   // trees per warp job
  int nsub;                 // warp jobs per (mtry, task) = ceil((hi - lo) / Cw)
  int wpb;                  // warps per block
  // CV output: sum of leaf values per warp job and test row
  double* partial;          // [n_mtry][ntask][nsub][nte_max]
  // fit output (fit_mode = 1; ntask == 1, all rows train)
  int fit_mode;
  Node16* nodes;            // [tree_hi - tree_lo][cap]
  uint32_t* thr_index;      // [tree_hi - tree_lo][cap]
  uint32_t* tree_nnodes;    // [tree_hi - tree_lo]
  uint32_t cap;             // node capacity per tree (2 ntr - 1)
  int32_t* leaf_of_row;     // [tree_hi - tree_lo][n] or nullptr
  double* imp;              // [tree_hi - tree_lo][p] MDI decreases per tree and feature, or nullptr
  int* err;                 // device error flag
  unsigned long long* cand; // evaluated candidate splits (counter) or null
};

// shared-memory bytes per block for the launch configuration
size_t small_tree_smem_bytes(const SmallArgs& a, int mmax);
// resident CTAs per SM for a.wpb warps per CTA (0 if it does not fit)
int small_tree_ctas_per_sm(const SmallArgs& a);
cudaError_t launch_small_tree(const SmallArgs& a, cudaStream_t s);

// profiling build (RF_PHASE_TIMING): per-phase clock64 sums of the kernel's warps
constexpr int kPhases = 16;
bool small_tree_phase_timing_enabled();
cudaError_t small_tree_phase_cycles(uint64_t* out, bool reset);

}  // namespace rf
