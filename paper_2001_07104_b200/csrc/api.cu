// api.cu -- the C ABI of librfgpu.so (include/rf.h): argument validation,
// device memory, orchestration of the kernels, host<->device copies.
// Every compute step runs in this library's CUDA kernels; there is no CPU
// fallback (without a device every call returns RF_E_CUDA).
#include <algorithm>
#include <mutex>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/rf.h"
#include "../../include/rf_debug.h"
#include "common.cuh"
#include "cv.cuh"
#include "large_tree.cuh"
#include "predict.cuh"
#include "prep.cuh"
#include "small_tree.cuh"
#include "host_util.cuh"
#include "importance.cuh"

struct rf_forest {
  int device = 0;
  uint32_t ntree = 0, p = 0, target = 0;
  int32_t F = 0;
  uint64_t total_nodes = 0;
  rf::Node16* nodes = nullptr;   // device
  uint32_t* thr_index = nullptr; // device
  uint64_t* tree_off = nullptr;  // device [ntree + 1]
  std::vector<uint64_t> h_tree_off;
  int32_t* leaf_of_row = nullptr;  // device [ntree][n_rows] (debug fits)
  double* imp = nullptr;           // device [ntree][p] MDI decreases (rf_fit), null if imported
  uint64_t n_rows = 0;
  bool pooled = false;  // nodes / thr_index / tree_off from the device's stream-ordered pool
  rf::Node8* n8 = nullptr;  // compact copy for batch inference (null if a tree has >= 2^23 nodes)
  double* val = nullptr;    // fp64 threshold / leaf value beside n8 (same slots)
  uint64_t* n8_off = nullptr;  // device [ntree + 1] slot offsets of the blocked layout (null: tree_off)
};

namespace {
std::atomic<bool> g_opt_predict_node16{false};  // test switch (rf_debug_set_option "predict_node16")
std::atomic<long long> g_opt_predict_chunk{0};     // test switch "predict_chunk_rows" (0: by size)

// compact 8-byte node copy of a forest (predict.cuh Node8) on the forest's stream: the blocked
// layout (three-level 64-byte blocks below a BFS prefix, predict.cu) for shallow forests whose
// trees are all BFS-ordered (fitted forests; imported ones if they are), else the BFS-slot copy
cudaError_t attach_node8(rf_forest* f, cudaStream_t s) {
#ifdef RF_NO_NODE8
  return cudaSuccess;
#endif
  if (f->p >= 255 || f->total_nodes == 0) return cudaSuccess;
  for (uint32_t t = 0; t < f->ntree; ++t)
    if (f->h_tree_off[t + 1] - f->h_tree_off[t] >= (1ull << 23)) return cudaSuccess;
  auto dalloc = [&](auto** p, size_t bytes) {
    return f->pooled ? cudaMallocAsync((void**)p, bytes, s) : cudaMalloc((void**)p, bytes);
  };
  auto dfree = [&](void* p) { if (p) { if (f->pooled) cudaFreeAsync(p, s); else cudaFree(p); } };
  const int T = (int)f->ntree;
#ifndef RF_PRED_NOBLOCKS
  if (T <= 65536 && f->total_nodes <= (uint64_t)T * rf::kShallowNodesPerTree) {
    uint64_t* slots = nullptr;
    uint32_t* lev = nullptr;
    int* nlev = nullptr;
    int* bad = nullptr;
    cudaError_t e = dalloc(&slots, (size_t)T * 8);
    if (e == cudaSuccess) e = dalloc(&lev, (size_t)T * rf::kBlkLevStride * 4);
    if (e == cudaSuccess) e = dalloc(&nlev, (size_t)T * 4);
    if (e == cudaSuccess) e = dalloc(&bad, 4);
    if (e == cudaSuccess) e = cudaMemsetAsync(bad, 0, 4, s);
    if (e == cudaSuccess) e = rf::node8_blocked_count(f->nodes, f->tree_off, T, slots, lev, nlev, bad, s);
    std::vector<uint64_t> hs((size_t)T + 1, 0);
    int hbad = 1;
    if (e == cudaSuccess) e = cudaMemcpyAsync(hs.data() + 1, slots, (size_t)T * 8, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e == cudaSuccess && !hbad) {
      for (int t = 0; t < T; ++t) hs[t + 1] += hs[t];  // exclusive offsets
      const uint64_t total = hs[T];
      e = dalloc(&f->n8_off, ((size_t)T + 1) * 8);
      if (e == cudaSuccess) e = dalloc(&f->n8, total * sizeof(rf::Node8));
      if (e == cudaSuccess) e = dalloc(&f->val, total * sizeof(double));
      if (e == cudaSuccess) e = cudaMemcpyAsync(f->n8_off, hs.data(), ((size_t)T + 1) * 8, cudaMemcpyHostToDevice, s);
      if (e == cudaSuccess) e = cudaMemsetAsync(f->n8, 0xFF, total * sizeof(rf::Node8), s);  // padding: leaves
      if (e == cudaSuccess) e = cudaMemsetAsync(f->val, 0, total * sizeof(double), s);
      if (e == cudaSuccess) e = rf::node8_blocked_build(f->nodes, f->tree_off, T, f->n8_off, lev, nlev, f->n8, f->val, s);
      if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // (hs is freed on return)
    }
    dfree(slots); dfree(lev); dfree(nlev); dfree(bad);
    if (e != cudaSuccess || !hbad) return e;
  }
#endif
  cudaError_t e = dalloc(&f->n8, f->total_nodes * sizeof(rf::Node8));
  if (e == cudaSuccess) e = dalloc(&f->val, f->total_nodes * sizeof(double));
  if (e == cudaSuccess) e = rf::build_node8(f->nodes, f->total_nodes, f->n8, f->val, s);
  return e;
}
}  // namespace

namespace {

thread_local std::string g_err;

struct ProfRec {
  const char* name;
  cudaEvent_t a, b;
  int dev;  // the device the events belong to (current when the scope ran)
};
thread_local std::vector<ProfRec> g_prof;
thread_local bool g_prof_on = false;
using rf::ProfScope;
using rf::Scratch;

rf_status fail(rf_status st, const std::string& msg) {
  g_err = msg;
  return st;
}

rf_status cuda_fail(cudaError_t e, const char* where) {
  if (e == cudaErrorMemoryAllocation) return fail(RF_E_OOM, std::string(where) + ": out of device memory");
  return fail(RF_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(expr, where)                              \
  do {                                               \
    cudaError_t _e = (expr);                         \
    if (_e != cudaSuccess) return cuda_fail(_e, where); \
  } while (0)

// the calling thread's stream `which` (0, 1) on `device` (host-pointer entry points; 1 = the second
// stream of the pipelined rf_predict)
cudaStream_t host_stream(int device, int which = 0) {
  static thread_local std::vector<cudaStream_t> streams;
  const int i = 2 * device + which;
  if ((int)streams.size() <= i) streams.resize(i + 1, nullptr);
  if (!streams[i]) cudaStreamCreateWithFlags(&streams[i], cudaStreamNonBlocking);
  return streams[i];
}

rf_status check_device() {
  int cnt = 0;
  cudaError_t e = cudaGetDeviceCount(&cnt);
  if (e != cudaSuccess || cnt == 0) return fail(RF_E_CUDA, "no CUDA device available (no CPU fallback)");
  return RF_OK;
}

rf_status check_params(const rf_params* prm, uint32_t p, uint32_t* mtry_out) {
  if (!prm) return fail(RF_E_ARG, "params is NULL");
  if (prm->struct_size != sizeof(rf_params)) return fail(RF_E_ARG, "rf_params.struct_size mismatch");
  if (p == 0) return fail(RF_E_ARG, "p must be >= 1");
  if (p > (uint32_t)rf::kSmallMaxP && p > 4096) return fail(RF_E_ARG, "p too large");
  if (prm->min_samples_split < 2) return fail(RF_E_ARG, "min_samples_split must be >= 2");
  if (prm->max_depth < -1) return fail(RF_E_ARG, "max_depth must be >= -1");
  if (prm->split_mode > RF_SPLIT_EXTRA || prm->target > 1) return fail(RF_E_ARG, "bad split_mode/target");
  if (prm->criterion > RF_CRITERION_MAE) return fail(RF_E_ARG, "bad criterion");
  if (prm->tie_break > RF_TIE_DRAW_ORDER) return fail(RF_E_ARG, "bad tie_break");
  if (prm->criterion == RF_CRITERION_MAE && prm->split_mode == RF_SPLIT_HIST256)
    return fail(RF_E_UNSUPPORTED, "MAE criterion: exact and ExtraTrees split modes only (R32)");
  uint32_t m = prm->mtry ? prm->mtry : std::max<uint32_t>(1, p / 3);
  if (m > p) return fail(RF_E_ARG, "mtry must be <= p");
  if (mtry_out) *mtry_out = m;
  return RF_OK;
}

rf_status read_err(const int* derr, cudaStream_t s) {
  int h = 0;
  CK(cudaMemcpyAsync(&h, derr, sizeof(int), cudaMemcpyDeviceToHost, s), "err flag");
  CK(cudaStreamSynchronize(s), "sync");
  if (h & rf::kErrNonFinite) return fail(RF_E_NONFINITE, "non-finite value in X or y");
  if (h & rf::kErrNonPositive) return fail(RF_E_NONPOSITIVE_Y, "y <= 0 (LOG target or CV / MAPE)");
  if (h & rf::kErrOverflow) return fail(RF_E_OVERFLOW, "kernel size limit exceeded");
  if (h & rf::kErrInexact) return fail(RF_E_INEXACT, "ln(y) not certified correctly rounded (LOG target)");
  return RF_OK;
}

// dataset on device: canonical X, t_q, F, presort
rf_status prepare(const double* dX, const double* dy, uint64_t n, uint32_t p, int target,
                  int require_pos, bool need_sort, rf::DevData& d, Scratch& sc, cudaStream_t s, int guard = 0,
                  bool need_rank = true) {
  d.n = (int)n;
  d.p = (int)p;
  CK(sc.alloc(&d.X, n * p), "alloc X");
  CK(sc.alloc(&d.tq, n), "alloc tq");
  CK(sc.alloc(&d.F, 1), "alloc F");
  CK(sc.alloc(&d.err, 1), "alloc err");
  CK(cudaMemsetAsync(d.err, 0, sizeof(int), s), "memset");
  double* t;
  CK(sc.alloc(&t, n + 2), "alloc t");
  {
    ProfScope ps("prep", s);
    CK(rf::prep_targets(dX, dy, (int)n, (int)p, target, require_pos, guard, d, t, s), "prep");
  }
  if (need_sort) {
    CK(sc.alloc(&d.order, n * p), "alloc order");
    CK(sc.alloc(&d.grank, n * p), "alloc grank");
    size_t wsb = rf::presort_ws_bytes((int)n, (int)p);
    void* ws = nullptr;
    if (wsb) CK(sc.alloc(reinterpret_cast<char**>(&ws), wsb), "alloc presort ws");
    ProfScope ps("presort", s);
    CK(rf::presort(d, ws, wsb, s, need_rank), "presort");
  }
  return RF_OK;
}

// quantisation headroom (R32): 2 guard bits under MAE
int mae_guard(const rf_params* prm) { return prm->criterion == RF_CRITERION_MAE ? 2 : 0; }

int gcd_i(int a, int b) { return b == 0 ? a : gcd_i(b, a % b); }

int resident_warps(size_t smem_block, int wpb) {
  int per_sm = (int)std::min<size_t>(32, (227 * 1024) / std::max<size_t>(smem_block, 1));
  per_sm = std::min(per_sm, 64 / std::max(wpb, 1));
  return 148 * per_sm * wpb;
}

struct GridPlan {
  std::vector<int> mtry_distinct;
  std::vector<int> mtry_map;  // requested index -> distinct index
};

GridPlan plan_mtry(const uint32_t* mtrys, uint32_t n_mtry) {
  GridPlan g;
  for (uint32_t i = 0; i < n_mtry; ++i) {
    int m = (int)mtrys[i];
    auto it = std::find(g.mtry_distinct.begin(), g.mtry_distinct.end(), m);
    if (it == g.mtry_distinct.end()) {
      g.mtry_map.push_back((int)g.mtry_distinct.size());
      g.mtry_distinct.push_back(m);
    } else {
      g.mtry_map.push_back((int)(it - g.mtry_distinct.begin()));
    }
  }
  return g;
}

// Core of CV: fills fold_mape/pred (partial_rows == null) or per-row partial sums.
rf_status cv_core(const double* dX, uint64_t n, uint32_t p, const double* dy, const rf_params* prm,
                  uint32_t k, uint32_t reps, const int32_t* dfold_in, const uint32_t* ntrees,
                  uint32_t n_ntree, const uint32_t* mtrys, uint32_t n_mtry, double* dfold_mape,
                  double* dpred, double* dpartial_rows, cudaStream_t s) {
  if (n == 0) return fail(RF_E_EMPTY, "n == 0");
  if (k < 2 || k > n) return fail(RF_E_TOO_FEW, "need 2 <= k <= n");
  if (reps == 0) return fail(RF_E_ARG, "repeats must be >= 1");
  if (n_ntree == 0 || n_ntree > 16 || n_mtry == 0 || n_mtry > (uint32_t)rf::kMaxMtry)
    return fail(RF_E_ARG, "grid sizes: 1..16 ntree values, 1..16 mtry values");
  if (n > 0x7FFFFFFF) return fail(RF_E_ARG, "n too large");
  rf_status st = check_params(prm, p, nullptr);
  if (st) return st;
  int Tmax = 0;
  for (uint32_t i = 0; i < n_ntree; ++i) {
    if (ntrees[i] == 0) return fail(RF_E_ARG, "ntree values must be >= 1");
    Tmax = std::max(Tmax, (int)ntrees[i]);
  }
  for (uint32_t i = 0; i < n_mtry; ++i)
    if (mtrys[i] == 0 || mtrys[i] > p) return fail(RF_E_ARG, "mtry values must be in 1..p");
  int tree_lo = 0, tree_hi = Tmax;
  if (prm->tree_begin || prm->tree_end) {
    if (!dpartial_rows) return fail(RF_E_ARG, "tree sharding needs rf_cv_partial_dev");
    tree_lo = (int)prm->tree_begin;
    tree_hi = (int)std::min<uint32_t>(prm->tree_end, (uint32_t)Tmax);
    if (tree_lo > tree_hi) return fail(RF_E_ARG, "tree_begin > tree_end");
  }
  const int ntask_all = (int)(reps * k);
  int task_lo = 0, task_hi = ntask_all;
  if (prm->task_begin || prm->task_end) {
    task_lo = (int)prm->task_begin;
    task_hi = (int)std::min<uint32_t>(prm->task_end, (uint32_t)ntask_all);
    if (task_lo > task_hi) return fail(RF_E_ARG, "task_begin > task_end");
  }
  Scratch sc(s);
  rf::DevData d;
  st = prepare(dX, dy, n, p, prm->target, 1, true, d, sc, s, mae_guard(prm));
  if (st) return st;

  const int32_t* dfold = dfold_in;
  if (!dfold) {
    int32_t* f;
    CK(sc.alloc(&f, (size_t)n * reps), "alloc folds");
    size_t wsb = rf::make_folds_ws_bytes((int)n, (int)reps, 0);
    char* ws = nullptr;
    if (wsb) CK(sc.alloc(&ws, wsb), "alloc folds ws");
    CK(rf::make_folds(dy, (int)n, (int)k, (int)reps, prm->seed, 0, f, ws, wsb, s), "folds");
    dfold = f;
  }

  const size_t n_out = (size_t)n_mtry * n_ntree * reps * k;
  if (dfold_mape) CK(cudaMemsetAsync(dfold_mape, 0xFF, n_out * sizeof(double), s), "memset mape");
  if (dpred) CK(cudaMemsetAsync(dpred, 0xFF, (size_t)n_mtry * n_ntree * reps * n * sizeof(double), s), "memset pred");
  if (dpartial_rows)
    CK(cudaMemsetAsync(dpartial_rows, 0, (size_t)n_mtry * n_ntree * reps * n * sizeof(double), s), "memset partial");
  const int ntask = task_hi - task_lo;
  if (ntask == 0 || tree_hi == tree_lo) return read_err(d.err, s);

  rf::TaskData td;
  td.ntask = ntask; td.task0 = task_lo; td.n = (int)n; td.p = (int)p;
  CK(sc.alloc(&td.tr_rows, (size_t)ntask * n), "alloc tasks");
  CK(sc.alloc(&td.te_rows, (size_t)ntask * n), "alloc tasks");
  CK(sc.alloc(&td.loc, (size_t)ntask * n), "alloc tasks");
  CK(sc.alloc(&td.ntr, ntask), "alloc tasks");
  CK(sc.alloc(&td.nte, ntask), "alloc tasks");
  {
    ProfScope ps("tasks", s);
    CK(rf::build_tasks(dfold, (int)k, d.order, d.grank, td, s), "tasks");
  }
  std::vector<int32_t> hntr(ntask), hnte(ntask);
  CK(cudaMemcpyAsync(hntr.data(), td.ntr, ntask * 4, cudaMemcpyDeviceToHost, s), "d2h");
  CK(cudaMemcpyAsync(hnte.data(), td.nte, ntask * 4, cudaMemcpyDeviceToHost, s), "d2h");
  st = read_err(d.err, s);  // synchronises
  if (st) return st;
  int ntr_max = 0, nte_max = 0;
  for (int i = 0; i < ntask; ++i) {
    if (hnte[i] == 0) return fail(RF_E_TOO_FEW, "empty test fold");
    if (hntr[i] == 0) return fail(RF_E_TOO_FEW, "empty training set");
    ntr_max = std::max(ntr_max, hntr[i]);
    nte_max = std::max(nte_max, hnte[i]);
  }
  GridPlan gp = plan_mtry(mtrys, n_mtry);
  const int nmd = (int)gp.mtry_distinct.size();
  // trees per warp job / chunk: divides every prefix boundary so prefix sums align with jobs
  int g = 0;
  for (uint32_t i = 0; i < n_ntree; ++i) g = gcd_i(g, (int)ntrees[i]);
  if (tree_lo) g = gcd_i(g, tree_lo);
  if (tree_hi != Tmax) g = gcd_i(g, tree_hi);
  const int T = tree_hi - tree_lo;
  bool large = ntr_max > rf::kSmallMaxRows || (int)p > rf::kSmallMaxP || prm->split_mode == RF_SPLIT_HIST256;
  int Cw = 1, nsub = T;
  double* partial = nullptr;
  rf::SmallArgs a;
  memset(&a, 0, sizeof a);
  a.X = d.X; a.n = (int)n; a.p = (int)p; a.tq = d.tq; a.dF = d.F; a.grank = d.grank;
  a.ntask = ntask; a.task0 = task_lo; a.row_stride = (int)n; a.ntr_stride = ntr_max;
  a.ntr = td.ntr; a.nte = td.nte; a.tr_rows = td.tr_rows; a.te_rows = td.te_rows;
  a.ntr_max = ntr_max; a.nte_max = nte_max;
  a.seed = prm->seed; a.bootstrap = (int)prm->bootstrap; a.min_split = (int)prm->min_samples_split;
  a.extra = prm->split_mode == RF_SPLIT_EXTRA;
  a.mae = prm->criterion == RF_CRITERION_MAE;
  a.tie_draw = prm->tie_break == RF_TIE_DRAW_ORDER;
  a.max_depth = prm->max_depth; a.n_mtry = nmd;
  for (int i = 0; i < nmd; ++i) a.mtrys[i] = gp.mtry_distinct[i];
  a.tree_lo = tree_lo; a.tree_hi = tree_hi;
  a.err = d.err;
  a.cand = rf::candidate_counter();
  // warps per CTA: the most resident warps per SM (registers and shared memory both bound it);
  // a task shape whose CTA-resident data does not fit shared memory takes the large path
  int best_wpb = 0, best_warps = 0;
  if (!large) {
    for (int w = 1; w <= rf::kSmallMaxWpb; ++w) {
      a.wpb = w;
      const int warps = w * rf::small_tree_ctas_per_sm(a);
      if (warps > best_warps) { best_warps = warps; best_wpb = w; }
    }
    if (best_wpb == 0) large = true;
  }
  if (large) {
    for (int c = 32; c >= 1; --c)
      if (g % c == 0) { Cw = c; break; }
    nsub = (T + Cw - 1) / Cw;
    CK(sc.alloc(&partial, (size_t)nmd * ntask * nsub * nte_max), "alloc partial");
    ProfScope ps("large_cv", s);
    rf_status ls = rf::cv_large_partial(d, td, prm, gp.mtry_distinct, tree_lo, tree_hi, Cw, nsub, nte_max,
                                        partial, s, sc, g_err);
    if (ls) return ls;
  } else {
  td.ntr_stride = ntr_max;
  CK(sc.alloc(&td.ord, (size_t)ntask * p * ntr_max), "alloc ord");
  CK(sc.alloc(&td.lrank, (size_t)ntask * p * ntr_max), "alloc lrank");
  {
    ProfScope ps("task_orders", s);
    CK(rf::build_task_orders_u8(d.order, d.grank, td, s), "task orders");
  }
  a.ord = td.ord; a.lrank = td.lrank;
  a.wpb = best_wpb;
  const int resident = 148 * best_warps;
  for (int c = 16; c >= 1; --c) {
    if (g % c) continue;
    long long jobs = (long long)nmd * ntask * ((T + c - 1) / c);
    if (jobs >= 2LL * resident || c == 1) { Cw = c; break; }
  }
  a.Cw = Cw;
  a.nsub = nsub = (T + Cw - 1) / Cw;
  {
    // a launch with fewer warp jobs than resident warp slots (e.g. C1: 1,000 single-tree
    // jobs) spreads its jobs over all SMs with smaller CTAs instead of filling a few SMs
    const long long jobs = (long long)nmd * ntask * nsub;
    if (jobs < resident) {
      int w = best_wpb;
      while (w > 1 && (long long)nmd * ntask * ((nsub + w - 1) / w) < 148) --w;
      a.wpb = w;
    }
  }
  CK(sc.alloc(&partial, (size_t)nmd * ntask * a.nsub * nte_max), "alloc partial");
  a.partial = partial;
  {
    ProfScope ps("small_tree", s);
    CK(rf::launch_small_tree(a, s), "small_tree kernel");
  }
  }  // small path
  // score every distinct mtry, then copy blocks for duplicates
  double* mape_d = nullptr;
  double* pred_d = nullptr;
  double* rows_d = nullptr;
  const size_t blk_mape = (size_t)n_ntree * reps * k, blk_rows = (size_t)n_ntree * reps * n;
  if (dfold_mape) CK(sc.alloc(&mape_d, nmd * blk_mape), "alloc");
  if (dpred) CK(sc.alloc(&pred_d, nmd * blk_rows), "alloc");
  if (dpartial_rows) CK(sc.alloc(&rows_d, nmd * blk_rows), "alloc");
  if (pred_d) CK(cudaMemsetAsync(pred_d, 0xFF, nmd * blk_rows * 8, s), "memset");
  if (mape_d) CK(cudaMemsetAsync(mape_d, 0xFF, nmd * blk_mape * 8, s), "memset");
  if (rows_d) CK(cudaMemsetAsync(rows_d, 0, nmd * blk_rows * 8, s), "memset");
  rf::ScoreArgs sa;
  memset(&sa, 0, sizeof sa);
  sa.partial = partial; sa.n_mtry = nmd; sa.ntask = ntask; sa.nsub = nsub; sa.nte_max = nte_max;
  sa.Cw = Cw; sa.tree_lo = tree_lo; sa.te_rows = td.te_rows; sa.nte = td.nte; sa.n = (int)n;
  sa.k = (int)k; sa.reps = (int)reps; sa.task0 = task_lo; sa.n_ntree = (int)n_ntree;
  for (uint32_t i = 0; i < n_ntree; ++i) sa.ntrees[i] = (int)ntrees[i];
  sa.target = (int)prm->target; sa.y = dy;
  sa.fold_mape = mape_d ? mape_d : nullptr;
  sa.pred = pred_d;
  sa.partial_rows = rows_d;
  if (!mape_d && !rows_d) return read_err(d.err, s);
  if (!sa.fold_mape) {
    CK(sc.alloc(&mape_d, nmd * blk_mape), "alloc");
    sa.fold_mape = mape_d;
  }
  {
    ProfScope ps("score", s);
    CK(rf::score_cv(sa, s), "score");
  }
  for (uint32_t i = 0; i < n_mtry; ++i) {
    const int di = gp.mtry_map[i];
    if (dfold_mape)
      CK(cudaMemcpyAsync(dfold_mape + i * blk_mape, mape_d + di * blk_mape, blk_mape * 8,
                         cudaMemcpyDeviceToDevice, s), "copy");
    if (dpred)
      CK(cudaMemcpyAsync(dpred + i * blk_rows, pred_d + di * blk_rows, blk_rows * 8,
                         cudaMemcpyDeviceToDevice, s), "copy");
    if (dpartial_rows)
      CK(cudaMemcpyAsync(dpartial_rows + i * blk_rows, rows_d + di * blk_rows, blk_rows * 8,
                         cudaMemcpyDeviceToDevice, s), "copy");
  }
  // task-range outputs outside the shard stay NaN (memset 0xFF above)
  return RF_OK;
}

// gather per-tree node blocks (stride cap) into the flat forest
__global__ void k_compact_nodes(const rf::Node16* __restrict__ in, const uint32_t* __restrict__ tin,
                                const uint64_t* __restrict__ off, int T, uint64_t cap,
                                rf::Node16* out, uint32_t* tout) {
  const int t = blockIdx.y;
  if (t >= T) return;
  const uint64_t cnt = off[t + 1] - off[t];
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cnt;
       i += (uint64_t)gridDim.x * blockDim.x) {
    out[off[t] + i] = in[t * cap + i];
    tout[off[t] + i] = tin[t * cap + i];
  }
}

rf_status fit_core(const double* dX, uint64_t n, uint32_t p, const double* dy, const rf_params* prm,
                   bool debug, cudaStream_t s, rf_forest** out) {
  *out = nullptr;
  if (n == 0) return fail(RF_E_EMPTY, "n == 0");
  if (n > 0x7FFFFFFF) return fail(RF_E_ARG, "n too large");
  uint32_t mtry = 0;
  rf_status st = check_params(prm, p, &mtry);
  if (st) return st;
  if (prm->ntree == 0) return fail(RF_E_ARG, "ntree must be >= 1");
  int tree_lo = 0, tree_hi = (int)prm->ntree;
  if (prm->tree_begin || prm->tree_end) {
    tree_lo = (int)prm->tree_begin;
    tree_hi = (int)std::min(prm->tree_end, prm->ntree);
    if (tree_lo >= tree_hi) return fail(RF_E_ARG, "empty tree range");
  }
  const int T = tree_hi - tree_lo;
  Scratch sc(s);
  rf::DevData d;
  // histogram fits beyond the CTA-resident sizes need the orders (cuts) but no dense ranks
  const bool hist_large = prm->split_mode == RF_SPLIT_HIST256 && n > 4096;
  st = prepare(dX, dy, n, p, prm->target, prm->target == RF_TARGET_LOG, true, d, sc, s, mae_guard(prm), !hist_large);
  if (st) return st;
  int dev = 0;
  cudaGetDevice(&dev);

  bool small = n <= (uint64_t)rf::kSmallMaxRows && p <= (uint32_t)rf::kSmallMaxP &&
               prm->split_mode != RF_SPLIT_HIST256;
  rf::Node16* nodes_w = nullptr;
  uint32_t* tidx_w = nullptr;
  uint32_t* nn_d = nullptr;
  // leaf rows (debug) and per-tree MDI decreases [T][p] (feature importance, NEXT-3) end up owned
  // by the forest; until then this guard frees them on every early return (CK included)
  struct OwnedBufs {
    int32_t* lor = nullptr;
    double* imp = nullptr;
    ~OwnedBufs() { cudaFree(lor); cudaFree(imp); }
  } own;
  int32_t*& lor = own.lor;
  double*& imp = own.imp;
  uint64_t cap = 0;
  if (debug) CK(cudaMalloc(&lor, (size_t)T * n * sizeof(int32_t)), "alloc leaf_of_row");
  CK(cudaMalloc(&imp, (size_t)T * p * sizeof(double)), "alloc importance");
  CK(cudaMemsetAsync(imp, 0, (size_t)T * p * sizeof(double), s), "alloc importance");
  if (small) {
    rf::TaskData td;
    td.ntask = 1; td.task0 = 0; td.n = (int)n; td.p = (int)p; td.ntr_stride = (int)n;
    CK(sc.alloc(&td.tr_rows, n), "alloc");
    CK(sc.alloc(&td.te_rows, n), "alloc");
    CK(sc.alloc(&td.loc, n), "alloc");
    CK(sc.alloc(&td.ntr, 1), "alloc");
    CK(sc.alloc(&td.nte, 1), "alloc");
    CK(sc.alloc(&td.ord, (size_t)p * n), "alloc");
    CK(sc.alloc(&td.lrank, (size_t)p * n), "alloc");
    CK(rf::build_tasks(nullptr, 1, d.order, d.grank, td, s), "tasks");
    CK(rf::build_task_orders_u8(d.order, d.grank, td, s), "task orders");
    cap = 2 * n - 1;
    CK(sc.alloc(&nodes_w, (size_t)T * cap), "alloc nodes");
    CK(sc.alloc(&tidx_w, (size_t)T * cap), "alloc nodes");
    CK(sc.alloc(&nn_d, (size_t)T), "alloc nodes");
    rf::SmallArgs a;
    memset(&a, 0, sizeof a);
    a.X = d.X; a.n = (int)n; a.p = (int)p; a.tq = d.tq; a.dF = d.F; a.grank = d.grank;
    a.ntask = 1; a.task0 = 0; a.row_stride = (int)n; a.ntr_stride = (int)n;
    a.ntr = td.ntr; a.nte = td.nte; a.tr_rows = td.tr_rows; a.te_rows = td.te_rows;
    a.ord = td.ord; a.lrank = td.lrank; a.ntr_max = (int)n; a.nte_max = 0;
    a.seed = prm->seed; a.bootstrap = (int)prm->bootstrap; a.min_split = (int)prm->min_samples_split;
    a.extra = prm->split_mode == RF_SPLIT_EXTRA;
    a.mae = prm->criterion == RF_CRITERION_MAE;
    a.tie_draw = prm->tie_break == RF_TIE_DRAW_ORDER;
    a.max_depth = prm->max_depth; a.n_mtry = 1; a.mtrys[0] = (int)mtry;
    a.tree_lo = tree_lo; a.tree_hi = tree_hi; a.Cw = 1; a.nsub = T; a.wpb = 4;
    a.fit_mode = 1; a.nodes = nodes_w; a.thr_index = tidx_w; a.tree_nnodes = nn_d;
    a.cap = (uint32_t)cap; a.leaf_of_row = lor; a.imp = imp; a.err = d.err;
    a.cand = rf::candidate_counter();
    size_t smem = 0;
    for (; a.wpb >= 1; a.wpb >>= 1) {
      smem = rf::small_tree_smem_bytes(a, 0);
      if (smem <= 227 * 1024) break;
    }
    if (a.wpb == 0) {
      small = false;  // CTA-resident data does not fit shared memory: large path
    } else {
      ProfScope ps("small_tree_fit", s);
      cudaError_t e = rf::launch_small_tree(a, s);
      if (e != cudaSuccess) return cuda_fail(e, "small_tree fit");
    }
  }
  if (!small) {
    rf_status ls = rf::fit_large(d, prm, (int)mtry, tree_lo, tree_hi, s, sc, &nodes_w, &tidx_w, &nn_d,
                                 &cap, lor, imp, g_err);
    if (ls) return ls;
  }
  std::vector<uint32_t> hnn(T);
  CK(cudaMemcpyAsync(hnn.data(), nn_d, T * 4, cudaMemcpyDeviceToHost, s), "d2h");
  int32_t hF = 0;
  CK(cudaMemcpyAsync(&hF, d.F, 4, cudaMemcpyDeviceToHost, s), "d2h");
  st = read_err(d.err, s);
  if (st) return st;
  rf_forest* f = new rf_forest();
  f->imp = imp;
  own.imp = nullptr;  // owned by the forest from here on (rf_forest_free)
  f->device = dev; f->ntree = (uint32_t)T; f->p = p; f->target = prm->target; f->F = hF;
  f->h_tree_off.resize(T + 1);
  f->h_tree_off[0] = 0;
  for (int t = 0; t < T; ++t) f->h_tree_off[t + 1] = f->h_tree_off[t] + hnn[t];
  f->total_nodes = f->h_tree_off[T];
  f->leaf_of_row = own.lor;
  own.lor = nullptr;
  f->n_rows = n;
  // the forest's arrays come from the stream-ordered pool (retained): a fresh cudaMalloc of the
  // ~1 GB C3 forest per fit stalled the fit for 0.1-1 s (profiles/rd2_27_c3wall.txt)
  f->pooled = true;
  cudaError_t e = cudaMallocAsync(&f->nodes, std::max<uint64_t>(1, f->total_nodes) * sizeof(rf::Node16), s);
  if (e == cudaSuccess) e = cudaMallocAsync(&f->thr_index, std::max<uint64_t>(1, f->total_nodes) * sizeof(uint32_t), s);
  if (e == cudaSuccess) e = cudaMallocAsync(&f->tree_off, (T + 1) * sizeof(uint64_t), s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(f->tree_off, f->h_tree_off.data(), (T + 1) * 8, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) {
    dim3 grid((unsigned)std::min<uint64_t>((cap + 255) / 256, 64), (unsigned)T);
    k_compact_nodes<<<grid, 256, 0, s>>>(nodes_w, tidx_w, f->tree_off, T, cap, f->nodes, f->thr_index);
    rf::note_launch();
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = attach_node8(f, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    rf_forest_free(f);
    return cuda_fail(e, "forest assembly");
  }
  *out = f;
  return RF_OK;
}

}  // namespace

namespace rf {
static std::atomic<unsigned long long> g_launches{0};
void note_launch(int n) { g_launches.fetch_add((unsigned long long)n, std::memory_order_relaxed); }
static std::atomic<unsigned long long> g_row_levels{0};
void note_row_levels(long long n) { g_row_levels.fetch_add((unsigned long long)n, std::memory_order_relaxed); }
// per-device counter, created once under a mutex (entry points may run on several host threads)
unsigned long long* candidate_counter() {
  static unsigned long long* ptrs[64] = {nullptr};
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  if (!ptrs[dev]) {
    if (cudaMalloc(&ptrs[dev], sizeof(unsigned long long)) != cudaSuccess) return nullptr;
    cudaMemset(ptrs[dev], 0, sizeof(unsigned long long));
  }
  return ptrs[dev];
}
bool prof_enabled() { return g_prof_on; }
void prof_push(const char* name, cudaEvent_t a, cudaEvent_t b) {
  int dev = 0;
  cudaGetDevice(&dev);
  g_prof.push_back(ProfRec{name, a, b, dev});
}
thread_local std::vector<std::pair<int, cudaEvent_t>> g_evpool;  // (device, event)
cudaEvent_t prof_event() {
  int dev = 0;
  cudaGetDevice(&dev);
  for (size_t i = g_evpool.size(); i-- > 0;)
    if (g_evpool[i].first == dev) {
      cudaEvent_t e = g_evpool[i].second;
      g_evpool.erase(g_evpool.begin() + (long)i);
      return e;
    }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
void prof_recycle(cudaEvent_t e, int dev) { g_evpool.emplace_back(dev, e); }
}  // namespace rf

// ======================================================================= ABI
extern "C" {

void rf_params_default(rf_params* prm) {
  if (!prm) return;
  memset(prm, 0, sizeof *prm);
  prm->struct_size = sizeof(rf_params);
  prm->ntree = 100;
  prm->mtry = 0;
  prm->min_samples_split = 2;
  prm->max_depth = -1;
  prm->bootstrap = 1;
  prm->split_mode = RF_SPLIT_EXACT;
  prm->target = RF_TARGET_IDENTITY;
  prm->seed = 0;
  prm->device = 0;
}

const char* rf_last_error(void) { return g_err.c_str(); }

void rf_forest_free(rf_forest* f) {
  if (!f) return;
  if (f->pooled) {  // back to the pool (kept mapped): the next fit reuses it without a cudaMalloc
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(f->device);
    cudaStream_t s = host_stream(f->device);
    cudaFreeAsync(f->nodes, s);
    cudaFreeAsync(f->thr_index, s);
    cudaFreeAsync(f->tree_off, s);
    if (f->n8) cudaFreeAsync(f->n8, s);
    if (f->val) cudaFreeAsync(f->val, s);
    if (f->n8_off) cudaFreeAsync(f->n8_off, s);
    cudaSetDevice(cur);
  } else {
    cudaFree(f->nodes);
    cudaFree(f->thr_index);
    cudaFree(f->tree_off);
    cudaFree(f->n8);
    cudaFree(f->val);
    cudaFree(f->n8_off);
  }
  cudaFree(f->leaf_of_row);
  cudaFree(f->imp);
  delete f;
}

rf_status rf_fit_dev(const double* dX, uint64_t n, uint32_t p, const double* dy, const rf_params* prm,
                     void* stream, rf_forest** out) {
  if (!out) return fail(RF_E_ARG, "out is NULL");
  *out = nullptr;
  if (rf_status st = check_device()) return st;
  try {
    return fit_core(dX, n, p, dy, prm, false, static_cast<cudaStream_t>(stream), out);
  } catch (...) {
    return fail(RF_E_CUDA, "internal exception");
  }
}

static rf_status fit_host(const double* X, uint64_t n, uint32_t p, const double* y, const rf_params* prm,
                          bool debug, rf_forest** out) {
  if (!out) return fail(RF_E_ARG, "out is NULL");
  *out = nullptr;
  if (rf_status st = check_device()) return st;
  if (!prm) return fail(RF_E_ARG, "params is NULL");
  if (n == 0) return fail(RF_E_EMPTY, "n == 0");
  if (!X || !y) return fail(RF_E_ARG, "NULL input");
  CK(cudaSetDevice(prm->device), "set device");
  cudaStream_t s = host_stream(prm->device);
  try {
    Scratch sc(s);
    double *dX, *dy;
    CK(sc.alloc(&dX, n * p), "alloc");
    CK(sc.alloc(&dy, n), "alloc");
    CK(cudaMemcpyAsync(dX, X, n * p * 8, cudaMemcpyHostToDevice, s), "h2d");
    CK(cudaMemcpyAsync(dy, y, n * 8, cudaMemcpyHostToDevice, s), "h2d");
    return fit_core(dX, n, p, dy, prm, debug, s, out);
  } catch (...) {
    return fail(RF_E_CUDA, "internal exception");
  }
}

rf_status rf_fit(const double* X, uint64_t n, uint32_t p, const double* y, const rf_params* prm,
                 rf_forest** out) {
  return fit_host(X, n, p, y, prm, false, out);
}

rf_status rf_fit_debug(const double* X, uint64_t n, uint32_t p, const double* y, const rf_params* prm,
                       rf_forest** out) {
  return fit_host(X, n, p, y, prm, true, out);
}

static rf_status predict_core(const rf_forest* f, const double* dX, uint64_t n, uint32_t p, double* dout,
                              int mode, cudaStream_t s, double* host_out = nullptr) {
  if (!f) return fail(RF_E_ARG, "forest is NULL");
  if (p != f->p) return fail(RF_E_ARITY, "p differs from the forest's");
  if (n == 0) return RF_OK;
  Scratch sc(s);
  int* err;
  CK(sc.alloc(&err, 1), "alloc");
  CK(cudaMemsetAsync(err, 0, 4, s), "memset");
  const bool few = (long long)n <= rf::kFewRows;
  if (!few) CK(rf::check_finite(dX, n * p, err, s), "check");
  {
    ProfScope ps("predict", s);
    CK(rf::predict_forest(f->nodes, f->tree_off, (int)f->ntree, dX, (long long)n, (int)p, mode, dout, s,
                          few ? err : nullptr, f->total_nodes, g_opt_predict_node16 ? nullptr : f->n8,
                          g_opt_predict_node16 ? nullptr : f->val, f->n8_off),
       "predict");
  }
  if (host_out) {  // one synchronisation for result and error flag
    int h = 0;
    CK(cudaMemcpyAsync(host_out, dout, n * 8, cudaMemcpyDeviceToHost, s), "d2h");
    CK(cudaMemcpyAsync(&h, err, 4, cudaMemcpyDeviceToHost, s), "d2h");
    CK(cudaStreamSynchronize(s), "sync");
    if (h) return fail(RF_E_NONFINITE, "non-finite value in X");
    return RF_OK;
  }
  return read_err(err, s);
}

rf_status rf_predict_dev(const rf_forest* f, const double* dX, uint64_t n, uint32_t p, double* dyhat,
                         void* stream) {
  if (rf_status st = check_device()) return st;
  if (!f) return fail(RF_E_ARG, "forest is NULL");
  return predict_core(f, dX, n, p, dyhat, f->target == RF_TARGET_LOG ? 2 : 1,
                      static_cast<cudaStream_t>(stream));
}

rf_status rf_predict_partial_dev(const rf_forest* f, const double* dX, uint64_t n, uint32_t p,
                                 double* dpartial, void* stream) {
  if (rf_status st = check_device()) return st;
  return predict_core(f, dX, n, p, dpartial, 0, static_cast<cudaStream_t>(stream));
}

rf_status rf_predict_finalize_dev(const double* dpartial, uint64_t n, uint32_t ntree_total, uint32_t target,
                                  double* dyhat, void* stream) {
  if (rf_status st = check_device()) return st;
  if (ntree_total == 0) return fail(RF_E_ARG, "ntree_total must be >= 1");
  CK(rf::predict_finalize(dpartial, (long long)n, (int)ntree_total, (int)target, dyhat,
                          static_cast<cudaStream_t>(stream)), "finalize");
  return RF_OK;
}

rf_status rf_predict(const rf_forest* f, const double* X, uint64_t n, uint32_t p, double* yhat) {
  if (rf_status st = check_device()) return st;
  if (!f) return fail(RF_E_ARG, "forest is NULL");
  if (p != f->p) return fail(RF_E_ARITY, "p differs from the forest's");
  if (n == 0) return RF_OK;
  CK(cudaSetDevice(f->device), "set device");
  cudaStream_t s = host_stream(f->device);
  const int mode = f->target == RF_TARGET_LOG ? 2 : 1;
  // rows per pipeline chunk: ~512 MB of X (test switch "predict_chunk_rows")
  const uint64_t chunk = g_opt_predict_chunk > 0 ? (uint64_t)g_opt_predict_chunk
                                                 : std::max<uint64_t>(4096, (512ull << 20) / ((uint64_t)p * 8));
  if (n <= 2 * chunk) {
    Scratch sc(s);
    double *dX, *dy;
    CK(sc.alloc(&dX, n * p), "alloc");
    CK(sc.alloc(&dy, n), "alloc");
    CK(cudaMemcpyAsync(dX, X, n * p * 8, cudaMemcpyHostToDevice, s), "h2d");
    return predict_core(f, dX, n, p, dy, mode, s, yhat);
  }
  // Large batches: chunks alternate between two streams, each doing H2D -> finiteness check ->
  // walk of its chunk in order, so the copy of one chunk overlaps the walk of the other (with
  // pinned X the H2D hides behind the kernels).  The predictions of all chunks stay on the device
  // and come back in one copy at the end (a D2H into pageable memory per chunk would block the
  // host and serialise the pipeline).
  cudaStream_t st[2] = {s, host_stream(f->device, 1)};
  Scratch sc0(st[0]), sc1(st[1]);
  Scratch* sc[2] = {&sc0, &sc1};
  double *dX[2], *dy;
  int* err[2];
  CK(sc0.alloc(&dy, n), "alloc");
  for (int b = 0; b < 2; ++b) {
    CK(sc[b]->alloc(&dX[b], chunk * p), "alloc");
    CK(sc[b]->alloc(&err[b], 1), "alloc");
    CK(cudaMemsetAsync(err[b], 0, 4, st[b]), "memset");
  }
  int c = 0;
  for (uint64_t r0 = 0; r0 < n; r0 += chunk, ++c) {
    const int b = c & 1;
    const uint64_t cn = std::min(chunk, n - r0);
    CK(cudaMemcpyAsync(dX[b], X + r0 * p, cn * p * 8, cudaMemcpyHostToDevice, st[b]), "h2d");
    CK(rf::check_finite(dX[b], cn * p, err[b], st[b]), "check");
    ProfScope ps("predict", st[b]);
    CK(rf::predict_forest(f->nodes, f->tree_off, (int)f->ntree, dX[b], (long long)cn, (int)p, mode, dy + r0, st[b],
                          nullptr, f->total_nodes, g_opt_predict_node16 ? nullptr : f->n8,
                          g_opt_predict_node16 ? nullptr : f->val, f->n8_off),
       "predict");
  }
  int h[2] = {0, 0};
  CK(cudaStreamSynchronize(st[1]), "sync");  // stream 1's walks done before stream 0 copies dy
  CK(cudaMemcpyAsync(yhat, dy, n * 8, cudaMemcpyDeviceToHost, st[0]), "d2h");
  for (int b = 0; b < 2; ++b) CK(cudaMemcpyAsync(&h[b], err[b], 4, cudaMemcpyDeviceToHost, st[0]), "d2h");
  CK(cudaStreamSynchronize(st[0]), "sync");
  if (h[0] | h[1]) return fail(RF_E_NONFINITE, "non-finite value in X");
  return RF_OK;
}

rf_status rf_make_folds_dev(const double* dy, uint64_t n, uint32_t k, uint32_t repeats, uint64_t seed,
                            uint32_t custom, int32_t* dfold_ids, void* stream) {
  if (rf_status st = check_device()) return st;
  if (n == 0) return fail(RF_E_EMPTY, "n == 0");
  if (k < 2 || (!custom && k > n) || (custom && (n < 5 || n - 5 < k)))
    return fail(RF_E_TOO_FEW, "too few rows for k folds");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Scratch sc(s);
  size_t wsb = rf::make_folds_ws_bytes((int)n, (int)repeats, (int)custom);
  char* ws = nullptr;
  if (wsb) CK(sc.alloc(&ws, wsb), "alloc");
  cudaError_t e = rf::make_folds(dy, (int)n, (int)k, (int)repeats, seed, (int)custom, dfold_ids, ws, wsb, s);
  if (e == cudaErrorNotSupported) return fail(RF_E_UNSUPPORTED, "custom split limited to n <= 4096");
  CK(e, "folds");
  return RF_OK;
}

rf_status rf_make_folds_masked_dev(const double* dy, uint64_t n, uint32_t k, uint32_t repeats, uint64_t seed,
                                   uint32_t custom, const uint8_t* dmask, int32_t* dfold_ids, void* stream) {
  if (rf_status st = check_device()) return st;
  if (n == 0) return fail(RF_E_EMPTY, "n == 0");
  if (!dmask || !dfold_ids) return fail(RF_E_ARG, "NULL mask or output");
  if (k < 2) return fail(RF_E_TOO_FEW, "k < 2");
  if (n > 4096) return fail(RF_E_UNSUPPORTED, "masked folds limited to n <= 4096");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CK(rf::make_folds(dy, (int)n, (int)k, (int)repeats, seed, (int)custom, dfold_ids, nullptr, 0, s, dmask),
     "masked folds");
  return RF_OK;
}

namespace {
rf_status nested_core(const double* dX, uint64_t n, uint32_t p, const double* dy, const rf_params* prm,
                      uint32_t k_outer, uint32_t k_inner, uint32_t iterations, uint32_t custom,
                      const uint32_t* ntrees, uint32_t n_ntree, const uint32_t* mtrys, uint32_t n_mtry,
                      int32_t* dbest, double* douter, double* dscore, cudaStream_t s) {
  if (n == 0) return fail(RF_E_EMPTY, "n == 0");
  if (!prm) return fail(RF_E_ARG, "params is NULL");
  if (iterations == 0) return fail(RF_E_ARG, "iterations must be >= 1");
  if (n > 4096) return fail(RF_E_UNSUPPORTED, "nested CV limited to n <= 4096 (masked folds)");
  if (prm->tree_begin || prm->tree_end || prm->task_begin || prm->task_end)
    return fail(RF_E_ARG, "nested CV runs whole forests and all tasks");
  const uint64_t pin = custom ? 5 : 0;
  if (k_outer < 2 || k_inner < 2 || n < pin + k_outer) return fail(RF_E_TOO_FEW, "too few rows for the folds");
  // the smallest outer-training set: n - (largest outer fold)
  const uint64_t big = (n - pin + k_outer - 1) / k_outer;
  if (n - big < pin + k_inner) return fail(RF_E_TOO_FEW, "too few outer-training rows for k_inner folds");
  const int C = (int)(iterations * k_outer);
  const uint64_t seed_in = prm->seed ^ 0x4E45535445440000ull;  // R31
  Scratch sc(s);
  int32_t *outer, *inner;
  uint8_t* mask;
  double *fm_in, *fm_out;
  CK(sc.alloc(&outer, (size_t)iterations * n), "alloc");
  CK(sc.alloc(&mask, (size_t)C * n), "alloc");
  CK(sc.alloc(&inner, (size_t)C * n), "alloc");
  CK(sc.alloc(&fm_in, (size_t)n_mtry * n_ntree * C * k_inner), "alloc");
  CK(sc.alloc(&fm_out, (size_t)n_mtry * n_ntree * iterations * k_outer), "alloc");
  CK(rf::make_folds(dy, (int)n, (int)k_outer, (int)iterations, prm->seed, (int)custom, outer, nullptr, 0, s),
     "outer folds");
  CK(rf::nested_mask(outer, (int)n, (int)k_outer, C, mask, s), "mask");
  CK(rf::make_folds(dy, (int)n, (int)k_inner, C, seed_in, (int)custom, inner, nullptr, 0, s, mask),
     "inner folds");
  rf_params pin_prm = *prm;
  pin_prm.seed = seed_in;
  rf_status st = cv_core(dX, n, p, dy, &pin_prm, k_inner, (uint32_t)C, inner, ntrees, n_ntree, mtrys, n_mtry,
                         fm_in, nullptr, nullptr, s);
  if (st) return st;
  CK(rf::nested_select(fm_in, (int)n_mtry, (int)n_ntree, C, (int)k_inner, dbest, dscore, s), "select");
  st = cv_core(dX, n, p, dy, prm, k_outer, iterations, outer, ntrees, n_ntree, mtrys, n_mtry, fm_out, nullptr,
               nullptr, s);
  if (st) return st;
  CK(rf::nested_pick(fm_out, dbest, (int)n_ntree, C, (int)k_outer, (int)iterations, douter, s), "pick");
  return RF_OK;
}
}  // namespace

rf_status rf_nested_cv_dev(const double* dX, uint64_t n, uint32_t p, const double* dy, const rf_params* prm,
                           uint32_t k_outer, uint32_t k_inner, uint32_t iterations, uint32_t custom,
                           const uint32_t* ntrees, uint32_t n_ntree, const uint32_t* mtrys, uint32_t n_mtry,
                           int32_t* dbest, double* douter_mape, double* dinner_score, void* stream) {
  if (rf_status st = check_device()) return st;
  if (!dbest || !douter_mape) return fail(RF_E_ARG, "NULL output");
  try {
    return nested_core(dX, n, p, dy, prm, k_outer, k_inner, iterations, custom, ntrees, n_ntree, mtrys, n_mtry,
                       dbest, douter_mape, dinner_score, static_cast<cudaStream_t>(stream));
  } catch (...) {
    return fail(RF_E_CUDA, "internal exception");
  }
}

rf_status rf_nested_cv(const double* X, uint64_t n, uint32_t p, const double* y, const rf_params* prm,
                       uint32_t k_outer, uint32_t k_inner, uint32_t iterations, uint32_t custom,
                       const uint32_t* ntrees, uint32_t n_ntree, const uint32_t* mtrys, uint32_t n_mtry,
                       int32_t* best, double* outer_mape, double* inner_score) {
  if (rf_status st = check_device()) return st;
  if (!prm || !X || !y || !best || !outer_mape) return fail(RF_E_ARG, "NULL argument");
  CK(cudaSetDevice(prm->device), "set device");
  cudaStream_t s = host_stream(prm->device);
  try {
    Scratch sc(s);
    double *dX, *dy, *dout, *dsc = nullptr;
    int32_t* db;
    const size_t C = (size_t)iterations * k_outer;
    CK(sc.alloc(&dX, n * p), "alloc");
    CK(sc.alloc(&dy, n), "alloc");
    CK(sc.alloc(&db, C), "alloc");
    CK(sc.alloc(&dout, C), "alloc");
    if (inner_score) CK(sc.alloc(&dsc, C * n_mtry * n_ntree), "alloc");
    CK(cudaMemcpyAsync(dX, X, n * p * 8, cudaMemcpyHostToDevice, s), "h2d");
    CK(cudaMemcpyAsync(dy, y, n * 8, cudaMemcpyHostToDevice, s), "h2d");
    rf_status st = nested_core(dX, n, p, dy, prm, k_outer, k_inner, iterations, custom, ntrees, n_ntree, mtrys,
                               n_mtry, db, dout, dsc, s);
    if (st) return st;
    CK(cudaMemcpyAsync(best, db, C * 4, cudaMemcpyDeviceToHost, s), "d2h");
    CK(cudaMemcpyAsync(outer_mape, dout, C * 8, cudaMemcpyDeviceToHost, s), "d2h");
    if (inner_score) CK(cudaMemcpyAsync(inner_score, dsc, C * n_mtry * n_ntree * 8, cudaMemcpyDeviceToHost, s), "d2h");
    CK(cudaStreamSynchronize(s), "sync");
    return RF_OK;
  } catch (...) {
    return fail(RF_E_CUDA, "internal exception");
  }
}

rf_status rf_error_buckets_dev(const double* dy, const double* dyhat, uint64_t n, uint64_t* dcounts, void* stream) {
  if (rf_status st = check_device()) return st;
  if (!dcounts || (n && (!dy || !dyhat))) return fail(RF_E_ARG, "NULL argument");
  CK(rf::ape_buckets(dy, dyhat, (int64_t)n, reinterpret_cast<unsigned long long*>(dcounts),
                     static_cast<cudaStream_t>(stream)), "buckets");
  return RF_OK;
}

rf_status rf_error_buckets(const double* y, const double* yhat, uint64_t n, uint64_t* counts) {
  if (rf_status st = check_device()) return st;
  if (!counts || (n && (!y || !yhat))) return fail(RF_E_ARG, "NULL argument");
  CK(cudaSetDevice(0), "set device");  // host twin: device 0 (documented in rf.h)
  cudaStream_t s = host_stream(0);
  Scratch sc(s);
  double *dy, *dh;
  unsigned long long* dc;
  CK(sc.alloc(&dy, std::max<uint64_t>(n, 1)), "alloc");
  CK(sc.alloc(&dh, std::max<uint64_t>(n, 1)), "alloc");
  CK(sc.alloc(&dc, 5), "alloc");
  if (n) {
    CK(cudaMemcpyAsync(dy, y, n * 8, cudaMemcpyHostToDevice, s), "h2d");
    CK(cudaMemcpyAsync(dh, yhat, n * 8, cudaMemcpyHostToDevice, s), "h2d");
  }
  CK(rf::ape_buckets(dy, dh, (int64_t)n, dc, s), "buckets");
  CK(cudaMemcpyAsync(counts, dc, 5 * 8, cudaMemcpyDeviceToHost, s), "d2h");
  CK(cudaStreamSynchronize(s), "sync");
  return RF_OK;
}

rf_status rf_make_folds(const double* y, uint64_t n, uint32_t k, uint32_t repeats, uint64_t seed,
                        uint32_t custom, int32_t* fold_ids) {
  if (rf_status st = check_device()) return st;
  CK(cudaSetDevice(0), "set device");  // host twin: device 0 (documented in rf.h)
  cudaStream_t s = host_stream(0);
  Scratch sc(s);
  double* dy;
  int32_t* df;
  CK(sc.alloc(&dy, std::max<uint64_t>(n, 1)), "alloc");
  CK(sc.alloc(&df, std::max<uint64_t>(n * repeats, 1)), "alloc");
  if (n) CK(cudaMemcpyAsync(dy, y, n * 8, cudaMemcpyHostToDevice, s), "h2d");
  rf_status st = rf_make_folds_dev(dy, n, k, repeats, seed, custom, df, s);
  if (st) return st;
  CK(cudaMemcpyAsync(fold_ids, df, n * repeats * 4, cudaMemcpyDeviceToHost, s), "d2h");
  CK(cudaStreamSynchronize(s), "sync");
  return RF_OK;
}

rf_status rf_cross_validate_grid_dev(const double* dX, uint64_t n, uint32_t p, const double* dy,
                                     const rf_params* prm, uint32_t k, uint32_t repeats,
                                     const int32_t* dfold_ids, const uint32_t* ntrees, uint32_t n_ntree,
                                     const uint32_t* mtrys, uint32_t n_mtry, double* dfold_mape,
                                     double* dpred, void* stream) {
  if (rf_status st = check_device()) return st;
  if (!dfold_mape) return fail(RF_E_ARG, "fold_mape is NULL");
  try {
    return cv_core(dX, n, p, dy, prm, k, repeats, dfold_ids, ntrees, n_ntree, mtrys, n_mtry, dfold_mape,
                   dpred, nullptr, static_cast<cudaStream_t>(stream));
  } catch (...) {
    return fail(RF_E_CUDA, "internal exception");
  }
}

rf_status rf_cross_validate_grid(const double* X, uint64_t n, uint32_t p, const double* y,
                                 const rf_params* prm, uint32_t k, uint32_t repeats,
                                 const int32_t* fold_ids, const uint32_t* ntrees, uint32_t n_ntree,
                                 const uint32_t* mtrys, uint32_t n_mtry, double* fold_mape, double* pred) {
  if (rf_status st = check_device()) return st;
  if (!prm) return fail(RF_E_ARG, "params is NULL");
  if (n == 0) return fail(RF_E_EMPTY, "n == 0");
  CK(cudaSetDevice(prm->device), "set device");
  cudaStream_t s = host_stream(prm->device);
  Scratch sc(s);
  double *dX, *dy, *dm, *dp = nullptr;
  int32_t* df = nullptr;
  const size_t nm = (size_t)n_mtry * n_ntree * repeats * k, np_ = (size_t)n_mtry * n_ntree * repeats * n;
  CK(sc.alloc(&dX, n * p), "alloc");
  CK(sc.alloc(&dy, n), "alloc");
  CK(sc.alloc(&dm, nm), "alloc");
  if (pred) CK(sc.alloc(&dp, np_), "alloc");
  CK(cudaMemcpyAsync(dX, X, n * p * 8, cudaMemcpyHostToDevice, s), "h2d");
  CK(cudaMemcpyAsync(dy, y, n * 8, cudaMemcpyHostToDevice, s), "h2d");
  if (fold_ids) {
    CK(sc.alloc(&df, n * repeats), "alloc");
    CK(cudaMemcpyAsync(df, fold_ids, n * repeats * 4, cudaMemcpyHostToDevice, s), "h2d");
  }
  rf_status st = rf_cross_validate_grid_dev(dX, n, p, dy, prm, k, repeats, df, ntrees, n_ntree, mtrys,
                                            n_mtry, dm, dp, s);
  if (st) return st;
  CK(cudaMemcpyAsync(fold_mape, dm, nm * 8, cudaMemcpyDeviceToHost, s), "d2h");
  if (pred) CK(cudaMemcpyAsync(pred, dp, np_ * 8, cudaMemcpyDeviceToHost, s), "d2h");
  CK(cudaStreamSynchronize(s), "sync");
  return RF_OK;
}

rf_status rf_cross_validate(const double* X, uint64_t n, uint32_t p, const double* y, const rf_params* prm,
                            uint32_t k, uint32_t repeats, const int32_t* fold_ids, double* fold_mape) {
  if (!prm) return fail(RF_E_ARG, "params is NULL");
  uint32_t m = 0;
  if (rf_status st = check_params(prm, p, &m)) return st;
  uint32_t nt = prm->ntree;
  return rf_cross_validate_grid(X, n, p, y, prm, k, repeats, fold_ids, &nt, 1, &m, 1, fold_mape, nullptr);
}

rf_status rf_cross_validate_dev(const double* dX, uint64_t n, uint32_t p, const double* dy, const rf_params* prm,
                                uint32_t k, uint32_t repeats, const int32_t* dfold_ids, double* dfold_mape,
                                void* stream) {
  if (!prm) return fail(RF_E_ARG, "params is NULL");
  uint32_t m = 0;
  if (rf_status st = check_params(prm, p, &m)) return st;
  uint32_t nt = prm->ntree;
  return rf_cross_validate_grid_dev(dX, n, p, dy, prm, k, repeats, dfold_ids, &nt, 1, &m, 1, dfold_mape, nullptr,
                                    stream);
}

rf_status rf_cv_partial_dev(const double* dX, uint64_t n, uint32_t p, const double* dy, const rf_params* prm,
                            uint32_t k, uint32_t repeats, const int32_t* dfold_ids, const uint32_t* ntrees,
                            uint32_t n_ntree, const uint32_t* mtrys, uint32_t n_mtry, double* dpartial,
                            void* stream) {
  if (rf_status st = check_device()) return st;
  if (!dpartial) return fail(RF_E_ARG, "partial is NULL");
  try {
    return cv_core(dX, n, p, dy, prm, k, repeats, dfold_ids, ntrees, n_ntree, mtrys, n_mtry, nullptr, nullptr,
                   dpartial, static_cast<cudaStream_t>(stream));
  } catch (...) {
    return fail(RF_E_CUDA, "internal exception");
  }
}

rf_status rf_cv_finalize_dev(const double* dy, uint64_t n, uint32_t target, uint32_t k, uint32_t repeats,
                             const int32_t* dfold_ids, const uint32_t* ntrees, uint32_t n_ntree,
                             uint32_t n_mtry, const double* dreduced, double* dfold_mape, double* dpred,
                             void* stream) {
  if (rf_status st = check_device()) return st;
  if (n_ntree == 0 || n_ntree > 16) return fail(RF_E_ARG, "1..16 ntree values");
  if (!dfold_ids) return fail(RF_E_ARG, "fold ids required");
  std::vector<int> nt(ntrees, ntrees + n_ntree);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dpred) CK(cudaMemsetAsync(dpred, 0xFF, (size_t)n_mtry * n_ntree * repeats * n * 8, s), "memset");
  CK(rf::finalize_cv(dreduced, dy, dfold_ids, (int)n, (int)k, (int)repeats, (int)n_mtry, (int)n_ntree,
                     nt.data(), (int)target, dfold_mape, dpred, s), "finalize");
  return RF_OK;
}

rf_status rf_predict_partial(const rf_forest* f, const double* X, uint64_t n, uint32_t p, double* partial) {
  if (rf_status st = check_device()) return st;
  if (!f) return fail(RF_E_ARG, "forest is NULL");
  if (n == 0) return RF_OK;
  CK(cudaSetDevice(f->device), "set device");
  cudaStream_t s = host_stream(f->device);
  Scratch sc(s);
  double *dX, *dp;
  CK(sc.alloc(&dX, n * p), "alloc");
  CK(sc.alloc(&dp, n), "alloc");
  CK(cudaMemcpyAsync(dX, X, n * p * 8, cudaMemcpyHostToDevice, s), "h2d");
  return predict_core(f, dX, n, p, dp, 0, s, partial);
}

rf_status rf_cv_partial(const double* X, uint64_t n, uint32_t p, const double* y, const rf_params* prm,
                        uint32_t k, uint32_t repeats, const int32_t* fold_ids, const uint32_t* ntrees,
                        uint32_t n_ntree, const uint32_t* mtrys, uint32_t n_mtry, double* partial) {
  if (rf_status st = check_device()) return st;
  if (!prm) return fail(RF_E_ARG, "params is NULL");
  if (n == 0) return fail(RF_E_EMPTY, "n == 0");
  if (!fold_ids || !partial) return fail(RF_E_ARG, "fold ids and partial required");
  CK(cudaSetDevice(prm->device), "set device");
  cudaStream_t s = host_stream(prm->device);
  Scratch sc(s);
  double *dX, *dy, *dp;
  int32_t* df;
  const size_t np_ = (size_t)n_mtry * n_ntree * repeats * n;
  CK(sc.alloc(&dX, n * p), "alloc");
  CK(sc.alloc(&dy, n), "alloc");
  CK(sc.alloc(&dp, np_), "alloc");
  CK(sc.alloc(&df, n * repeats), "alloc");
  CK(cudaMemcpyAsync(dX, X, n * p * 8, cudaMemcpyHostToDevice, s), "h2d");
  CK(cudaMemcpyAsync(dy, y, n * 8, cudaMemcpyHostToDevice, s), "h2d");
  CK(cudaMemcpyAsync(df, fold_ids, n * repeats * 4, cudaMemcpyHostToDevice, s), "h2d");
  rf_status st = rf_cv_partial_dev(dX, n, p, dy, prm, k, repeats, df, ntrees, n_ntree, mtrys, n_mtry, dp, s);
  if (st) return st;
  CK(cudaMemcpyAsync(partial, dp, np_ * 8, cudaMemcpyDeviceToHost, s), "d2h");
  CK(cudaStreamSynchronize(s), "sync");
  return RF_OK;
}

rf_status rf_cv_finalize(const double* y, uint64_t n, uint32_t target, uint32_t k, uint32_t repeats,
                         const int32_t* fold_ids, const uint32_t* ntrees, uint32_t n_ntree, uint32_t n_mtry,
                         const double* reduced, double* fold_mape, double* pred, int32_t device) {
  if (rf_status st = check_device()) return st;
  if (!fold_ids || !reduced || !fold_mape) return fail(RF_E_ARG, "fold ids, reduced and fold_mape required");
  if (n == 0) return fail(RF_E_EMPTY, "n == 0");
  CK(cudaSetDevice(device), "set device");
  cudaStream_t s = host_stream(device);
  Scratch sc(s);
  double *dy, *dr, *dm, *dpr = nullptr;
  int32_t* df;
  const size_t np_ = (size_t)n_mtry * n_ntree * repeats * n, nm = (size_t)n_mtry * n_ntree * repeats * k;
  CK(sc.alloc(&dy, n), "alloc");
  CK(sc.alloc(&dr, np_), "alloc");
  CK(sc.alloc(&dm, nm), "alloc");
  CK(sc.alloc(&df, n * repeats), "alloc");
  if (pred) CK(sc.alloc(&dpr, np_), "alloc");
  CK(cudaMemcpyAsync(dy, y, n * 8, cudaMemcpyHostToDevice, s), "h2d");
  CK(cudaMemcpyAsync(dr, reduced, np_ * 8, cudaMemcpyHostToDevice, s), "h2d");
  CK(cudaMemcpyAsync(df, fold_ids, n * repeats * 4, cudaMemcpyHostToDevice, s), "h2d");
  rf_status st = rf_cv_finalize_dev(dy, n, target, k, repeats, df, ntrees, n_ntree, n_mtry, dr, dm, dpr, s);
  if (st) return st;
  CK(cudaMemcpyAsync(fold_mape, dm, nm * 8, cudaMemcpyDeviceToHost, s), "d2h");
  if (pred) CK(cudaMemcpyAsync(pred, dpr, np_ * 8, cudaMemcpyDeviceToHost, s), "d2h");
  CK(cudaStreamSynchronize(s), "sync");
  return RF_OK;
}

rf_status rf_forest_info(const rf_forest* f, uint32_t* ntree, uint64_t* total_nodes, int32_t* F, uint32_t* p,
                         uint32_t* target) {
  if (!f) return fail(RF_E_ARG, "forest is NULL");
  if (ntree) *ntree = f->ntree;
  if (total_nodes) *total_nodes = f->total_nodes;
  if (F) *F = f->F;
  if (p) *p = f->p;
  if (target) *target = f->target;
  return RF_OK;
}

rf_status rf_forest_export(const rf_forest* f, int32_t* feature, uint32_t* left, double* value,
                           uint32_t* thr_index, uint64_t* tree_off) {
  if (!f) return fail(RF_E_ARG, "forest is NULL");
  CK(cudaSetDevice(f->device), "set device");
  std::vector<rf::Node16> h(f->total_nodes);
  CK(cudaMemcpy(h.data(), f->nodes, f->total_nodes * sizeof(rf::Node16), cudaMemcpyDeviceToHost), "d2h");
  for (uint64_t i = 0; i < f->total_nodes; ++i) {
    if (feature) feature[i] = h[i].feat;
    if (left) left[i] = h[i].left;
    if (value) value[i] = h[i].v;
  }
  if (thr_index)
    CK(cudaMemcpy(thr_index, f->thr_index, f->total_nodes * 4, cudaMemcpyDeviceToHost), "d2h");
  if (tree_off) memcpy(tree_off, f->h_tree_off.data(), (f->ntree + 1) * 8);
  return RF_OK;
}

rf_status rf_forest_export_leaf_rows(const rf_forest* f, int32_t* leaf_of_row) {
  if (!f) return fail(RF_E_ARG, "forest is NULL");
  if (!f->leaf_of_row) return fail(RF_E_ARG, "forest was not grown with rf_fit_debug");
  CK(cudaSetDevice(f->device), "set device");
  CK(cudaMemcpy(leaf_of_row, f->leaf_of_row, (size_t)f->ntree * f->n_rows * 4, cudaMemcpyDeviceToHost), "d2h");
  return RF_OK;
}

rf_status rf_forest_importance(const rf_forest* f, double* importance, double* raw) {
  if (!f || !importance) return fail(RF_E_ARG, "forest or output is NULL");
  if (!f->imp) return fail(RF_E_UNSUPPORTED, "forest has no split statistics (imported): use rf_importance_dev");
  CK(cudaSetDevice(f->device), "set device");
  cudaStream_t s = host_stream(f->device);
  Scratch sc(s);
  double *ws, *out;
  CK(sc.alloc(&ws, (size_t)f->ntree + f->p), "alloc");
  CK(sc.alloc(&out, (size_t)f->p), "alloc");
  CK(rf::importance_combine(f->imp, (int)f->ntree, (int)f->p, out, ws, s), "importance");
  CK(cudaMemcpyAsync(importance, out, (size_t)f->p * 8, cudaMemcpyDeviceToHost, s), "d2h");
  if (raw) CK(cudaMemcpyAsync(raw, f->imp, (size_t)f->ntree * f->p * 8, cudaMemcpyDeviceToHost, s), "d2h");
  CK(cudaStreamSynchronize(s), "sync");
  return RF_OK;
}

rf_status rf_importance_dev(const double* draw, uint32_t ntree, uint32_t p, double* dimportance, void* stream) {
  if (rf_status st = check_device()) return st;
  if (!draw || !dimportance || ntree == 0 || p == 0) return fail(RF_E_ARG, "bad arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Scratch sc(s);
  double* ws;
  CK(sc.alloc(&ws, (size_t)ntree + p), "alloc");
  CK(rf::importance_combine(draw, (int)ntree, (int)p, dimportance, ws, s), "importance");
  return RF_OK;
}

rf_status rf_forest_import(const int32_t* feature, const uint32_t* left, const double* value,
                           const uint32_t* thr_index, const uint64_t* tree_off, uint32_t ntree, uint32_t p,
                           int32_t F, uint32_t target, int32_t device, rf_forest** out) {
  if (!out) return fail(RF_E_ARG, "out is NULL");
  *out = nullptr;
  if (rf_status st = check_device()) return st;
  if (ntree == 0 || !tree_off || !feature || !left || !value) return fail(RF_E_ARG, "bad arrays");
  if (p == 0 || target > RF_TARGET_LOG) return fail(RF_E_ARG, "p must be >= 1 and target 0 or 1");
  // structure check before upload: a malformed forest (e.g. a mis-gathered shard) must not make
  // the predict kernels read out of bounds or loop on a cyclic child index.  Per tree (nodes
  // tree_off[t] .. tree_off[t+1], child ids tree-local): at least one node; an internal node i
  // has 0 <= feature < p and i < left, left + 1 < node count (children follow their parent in
  // BFS order, so every walk ends); leaves have feature -1.
  if (tree_off[0] != 0) return fail(RF_E_ARG, "tree_off[0] must be 0");
  for (uint32_t t = 0; t < ntree; ++t) {
    const uint64_t a = tree_off[t], b = tree_off[t + 1];
    if (b <= a) return fail(RF_E_ARG, "tree_off must be strictly increasing (every tree has a node)");
    for (uint64_t i = a; i < b; ++i) {
      const int32_t ft = feature[i];
      if (ft < -1 || ft >= (int32_t)p) return fail(RF_E_ARG, "node feature out of range");
      if (ft >= 0 && (left[i] <= i - a || (uint64_t)left[i] + 1 >= b - a))
        return fail(RF_E_ARG, "child index out of range or not after its parent");
    }
  }
  CK(cudaSetDevice(device), "set device");
  rf_forest* f = new rf_forest();
  f->device = device; f->ntree = ntree; f->p = p; f->F = F; f->target = target;
  f->h_tree_off.assign(tree_off, tree_off + ntree + 1);
  f->total_nodes = tree_off[ntree];
  std::vector<rf::Node16> h(f->total_nodes);
  for (uint64_t i = 0; i < f->total_nodes; ++i) { h[i].feat = feature[i]; h[i].left = left[i]; h[i].v = value[i]; }
  cudaError_t e = cudaMalloc(&f->nodes, std::max<uint64_t>(1, f->total_nodes) * sizeof(rf::Node16));
  if (e == cudaSuccess) e = cudaMalloc(&f->thr_index, std::max<uint64_t>(1, f->total_nodes) * 4);
  if (e == cudaSuccess) e = cudaMalloc(&f->tree_off, (ntree + 1) * 8);
  if (e == cudaSuccess) e = cudaMemcpy(f->nodes, h.data(), f->total_nodes * sizeof(rf::Node16), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && thr_index) e = cudaMemcpy(f->thr_index, thr_index, f->total_nodes * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(f->tree_off, tree_off, (ntree + 1) * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = attach_node8(f, 0);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { rf_forest_free(f); return cuda_fail(e, "import"); }
  *out = f;
  return RF_OK;
}

void rf_set_profiling(int on) {
  for (auto& r : g_prof) { rf::prof_recycle(r.a, r.dev); rf::prof_recycle(r.b, r.dev); }
  g_prof.clear();
  g_prof_on = on != 0;
}

uint32_t rf_last_profile(const char** names, double* ms, uint32_t* launches, uint32_t cap) {
  std::vector<std::string> order;
  std::vector<double> tot;
  std::vector<uint32_t> cnt;
  for (auto& r : g_prof) {
    cudaEventSynchronize(r.b);
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    auto it = std::find(order.begin(), order.end(), std::string(r.name));
    size_t i = it - order.begin();
    if (it == order.end()) { order.push_back(r.name); tot.push_back(0.0); cnt.push_back(0); }
    tot[i] += t;
    cnt[i] += 1;
  }
  uint32_t m = (uint32_t)std::min<size_t>(cap, order.size());
  static thread_local std::vector<std::string> keep;
  keep = order;
  for (uint32_t i = 0; i < m; ++i) {
    if (names) names[i] = keep[i].c_str();
    if (ms) ms[i] = tot[i];
    if (launches) launches[i] = cnt[i];
  }
  return m;
}

rf_status rf_debug_ln_dev(const double* dy, double* dout, uint64_t n, void* stream) {
  if (rf_status st = check_device()) return st;
  CK(rf::device_ln(dy, dout, (int)n, static_cast<cudaStream_t>(stream)), "ln");
  return RF_OK;
}

rf_status rf_debug_counters(uint64_t* launches, uint64_t* candidates) {
  if (launches) *launches = rf::g_launches.load();
  if (candidates) {
    *candidates = 0;
    unsigned long long* c = rf::candidate_counter();
    if (c) CK(cudaMemcpy(candidates, c, 8, cudaMemcpyDeviceToHost), "counter");
  }
  return RF_OK;
}

rf_status rf_debug_row_levels(uint64_t* out, int reset) {
  const unsigned long long v = reset ? rf::g_row_levels.exchange(0ull) : rf::g_row_levels.load();
  if (out) *out = v;
  return RF_OK;
}

rf_status rf_debug_phase_cycles(uint64_t* out16, int reset) {
  if (!out16) return fail(RF_E_ARG, "out is NULL");
  if (!rf::small_tree_phase_timing_enabled())
    return fail(RF_E_UNSUPPORTED, "phase timing needs a library built with RF_PHASE_TIMING=1");
  if (rf_status st = check_device()) return st;
  CK(rf::small_tree_phase_cycles(out16, reset != 0), "phase cycles");
  return RF_OK;
}

rf_status rf_debug_set_option(const char* name, int64_t value) {
  if (!name) return fail(RF_E_ARG, "name is NULL");
  if (!strcmp(name, "large_tiled_partition")) {
    rf::g_opt_tiled_partition = value != 0;
    return RF_OK;
  }
  if (!strcmp(name, "predict_node16")) {  // batches walk the 16-byte nodes (the compact copy is ignored)
    g_opt_predict_node16 = value != 0;
    return RF_OK;
  }
  if (!strcmp(name, "predict_chunk_rows")) {  // rows per chunk of the pipelined host rf_predict
    if (value < 0) return fail(RF_E_ARG, "predict_chunk_rows must be >= 0");
    g_opt_predict_chunk = value;
    return RF_OK;
  }
  if (!strcmp(name, "ln_cert_margin_log2")) {  // widened margin: reaches the RF_E_INEXACT path
    if (value != 0 && (value > -2 || value < -200)) return fail(RF_E_ARG, "ln_cert_margin_log2 must be in [-200, -2] or 0");
    rf::g_opt_ln_margin_log2 = (int)value;
    return RF_OK;
  }
  if (!strcmp(name, "hist_node_chunk_cap")) {
    if (value < 0) return fail(RF_E_ARG, "hist_node_chunk_cap must be >= 0");
    rf::g_opt_hist_node_cap = value;
    return RF_OK;
  }
  return fail(RF_E_ARG, "unknown option");
}

rf_status rf_debug_philox_dev(const uint32_t* dctr_key, uint32_t* dout, uint64_t n, void* stream) {
  if (rf_status st = check_device()) return st;
  CK(rf::device_philox(dctr_key, dout, (int)n, static_cast<cudaStream_t>(stream)), "philox");
  return RF_OK;
}

}  // extern "C"
