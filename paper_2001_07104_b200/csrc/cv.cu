// cv.cu -- folds, task row sets / orders and CV scoring on the device.
//
// Folds (R16, R17): plain k-fold orders the rows
// by Philox keys draw(i) of stream (seed; rep, 0, FOLD) (ties by index) and
// cuts contiguous blocks of floor(n/k) (+1 for the first n mod k folds).
// The paper's custom split pins the 5 largest targets to training and deals
// the short / medium / long strata round-robin in Philox order.
// Scoring: MAPE, Eq. 1, in percent, on raw targets.
#include <algorithm>
#include <cub/device/device_segmented_radix_sort.cuh>
#include "common.cuh"
#include "host_util.cuh"
#include "cv.cuh"

namespace rf {
namespace {

constexpr int kFoldSmallMax = 4096;

__device__ __forceinline__ int fold_of_pos(int pos, int n, int k) {
  const int q = n / k, r = n % k;
  const int big = (q + 1) * r;
  return pos < big ? pos / (q + 1) : r + (pos - big) / q;
}

// mask (nullable) [reps][n]: only rows with mask != 0 are split (nested CV, R31); the
// others get -2.  Keys stay indexed by the original row.
__global__ void k_folds_plain_small(int n, int k, uint64_t seed, const uint8_t* __restrict__ mask,
                                    int32_t* fold) {
  extern __shared__ unsigned long long key[];
  uint8_t* act = reinterpret_cast<uint8_t*>(key + n);
  __shared__ int nact;
  const int rep = blockIdx.x;
  const uint32_t s0 = (uint32_t)seed, s1 = (uint32_t)(seed >> 32);
  if (threadIdx.x == 0) nact = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const uint8_t a = mask ? (mask[(size_t)rep * n + i] != 0) : 1;
    act[i] = a;
    key[i] = draw64(s0, s1, (uint32_t)rep, 0u, kTagFold, (uint64_t)i);
    if (a) atomicAdd(&nact, 1);
  }
  __syncthreads();
  const int na = nact;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (!act[i]) { fold[(size_t)rep * n + i] = -2; continue; }
    const unsigned long long ki = key[i];
    int pos = 0;
    for (int j = 0; j < n; ++j) {
      const unsigned long long kj = key[j];
      pos += act[j] & ((kj < ki) | ((kj == ki) & (j < i)));
    }
    fold[(size_t)rep * n + i] = fold_of_pos(pos, na, k);
  }
}

__device__ __forceinline__ int stratum_of(double y) {
  return (y < 1000.0) ? 0 : (y < 100000.0 ? 1 : 2);
}

__global__ void k_folds_custom_small(const double* __restrict__ y, int n, int k, uint64_t seed,
                                     const uint8_t* __restrict__ mask, int32_t* fold) {
  extern __shared__ unsigned long long key[];
  double* ys = reinterpret_cast<double*>(key + n);
  uint8_t* st = reinterpret_cast<uint8_t*>(ys + n);  // stratum, 3 = pinned, 4 = excluded
  uint8_t* act = st + n;
  __shared__ int cnt[3];
  const int rep = blockIdx.x;
  const uint32_t s0 = (uint32_t)seed, s1 = (uint32_t)(seed >> 32);
  if (threadIdx.x < 3) cnt[threadIdx.x] = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    ys[i] = y[i];
    act[i] = mask ? (mask[(size_t)rep * n + i] != 0) : 1;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (!act[i]) { st[i] = 4; continue; }
    const double yi = ys[i];
    int r = 0;
    for (int j = 0; j < n; ++j) r += act[j] & ((ys[j] > yi) | ((ys[j] == yi) & (j < i)));
    int s = (r < 5) ? 3 : stratum_of(yi);
    st[i] = (uint8_t)s;
    if (s < 3) {
      key[i] = draw64(s0, s1, (uint32_t)rep, (uint32_t)s, kTagStratum, (uint64_t)i);
      atomicAdd(&cnt[s], 1);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int s = st[i];
    if (s == 4) { fold[(size_t)rep * n + i] = -2; continue; }
    if (s == 3) { fold[(size_t)rep * n + i] = -1; continue; }
    const unsigned long long ki = key[i];
    int q = 0;
    for (int j = 0; j < n; ++j)
      if (st[j] == s) q += (key[j] < ki) | ((key[j] == ki) & (j < i));
    int off = 0;
    for (int t = 0; t < s; ++t) off += cnt[t];
    fold[(size_t)rep * n + i] = (off + q) % k;
  }
}

__global__ void k_fold_keys(int n, int reps, uint64_t seed, unsigned long long* keys, uint32_t* vals) {
  const uint32_t s0 = (uint32_t)seed, s1 = (uint32_t)(seed >> 32);
  const size_t total = (size_t)n * reps;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t rep = i / n, r = i - rep * n;
    keys[i] = draw64(s0, s1, (uint32_t)rep, 0u, kTagFold, (uint64_t)r);
    vals[i] = (uint32_t)r;
  }
}

__global__ void k_fold_scatter(const uint32_t* __restrict__ sorted_idx, int n, int k, int reps,
                               int32_t* fold) {
  const size_t total = (size_t)n * reps;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t rep = i / n, pos = i - rep * n;
    fold[rep * n + sorted_idx[i]] = fold_of_pos((int)pos, n, k);
  }
}

__global__ void k_seg_off(int64_t* off, int segs, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= segs) off[i] = (int64_t)i * n;
}

// one CTA per task: training / test rows (ascending) and local indices
__global__ void k_tasks(const int32_t* __restrict__ fold, int n, int k, int task0, uint32_t* tr_rows,
                        uint32_t* te_rows, int32_t* loc, int32_t* ntr, int32_t* nte) {
  const int tl = blockIdx.x;
  const int task = task0 + tl;
  const int rep = task / k, fd = task % k;
  const int32_t* fr = fold ? fold + (size_t)rep * n : nullptr;
  __shared__ uint32_t wtr[32], wte[32];
  __shared__ uint32_t ctr, cte;
  if (threadIdx.x == 0) { ctr = 0; cte = 0; }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t* TR = tr_rows + (size_t)tl * n;
  uint32_t* TE = te_rows + (size_t)tl * n;
  int32_t* L = loc + (size_t)tl * n;
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const bool valid = i < n;
    const bool test = valid && fr && fr[i] == fd;
    const bool train = valid && !test && !(fr && fr[i] == -2);  // -2: excluded row (nested CV, R31)
    if (valid && !train && !test) L[i] = -1;
    const unsigned btr = __ballot_sync(0xffffffffu, train), bte = __ballot_sync(0xffffffffu, test);
    if (lane == 0) { wtr[warp] = __popc(btr); wte[warp] = __popc(bte); }
    __syncthreads();
    uint32_t otr = ctr, ote = cte;
    for (int w = 0; w < warp; ++w) { otr += wtr[w]; ote += wte[w]; }
    if (train) {
      uint32_t li = otr + __popc(btr & lanemask_lt());
      TR[li] = (uint32_t)i;
      L[i] = (int32_t)li;
    }
    if (test) {
      TE[ote + __popc(bte & lanemask_lt())] = (uint32_t)i;
      L[i] = -1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t a = 0, b = 0;
      for (int w = 0; w < nw; ++w) { a += wtr[w]; b += wte[w]; }
      ctr += a;
      cte += b;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) { ntr[tl] = (int32_t)ctr; nte[tl] = (int32_t)cte; }
}

// one warp per (task, feature): presorted order filtered to training rows (local ids) and the
// dense rank of x among training rows
__global__ void k_task_orders_u8(const uint32_t* __restrict__ order, const uint32_t* __restrict__ grank,
                                 const int32_t* __restrict__ loc, int n, int p, int ntask,
                                 int ntr_stride, uint8_t* ord, uint8_t* lrank) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= ntask * p) return;
  const int tl = gw / p, f = gw - tl * p;
  const uint32_t* o = order + (size_t)f * n;
  const uint32_t* g = grank + (size_t)f * n;
  const int32_t* L = loc + (size_t)tl * n;
  uint8_t* OD = ord + ((size_t)tl * p + f) * ntr_stride;
  uint8_t* LR = lrank + ((size_t)tl * p + f) * ntr_stride;
  uint32_t cnt = 0;         // training rows emitted so far
  int32_t rank = -1;        // dense rank of the last emitted row
  uint32_t lastg = 0xFFFFFFFFu;
  for (int base = 0; base < n; base += 32) {
    const int j = base + lane;
    uint32_t r = 0, gv = 0;
    int32_t li = -1;
    if (j < n) { r = o[j]; li = L[r]; gv = g[r]; }
    const bool tr = li >= 0;
    const unsigned bal = __ballot_sync(0xffffffffu, tr);
    // previous training element's global rank
    const unsigned before = bal & lanemask_lt();
    const int prev_lane = before ? 31 - __clz(before) : -1;
    uint32_t pg = __shfl_sync(0xffffffffu, gv, prev_lane < 0 ? 0 : prev_lane);
    if (prev_lane < 0) pg = lastg;
    const bool inc = tr && (gv != pg);
    const unsigned binc = __ballot_sync(0xffffffffu, inc);
    if (tr) {
      const uint32_t pos = cnt + __popc(before);
      OD[pos] = (uint8_t)li;
      LR[li] = (uint8_t)(rank + __popc(binc & (lanemask_lt() | (1u << lane))));
    }
    cnt += __popc(bal);
    rank += __popc(binc);
    if (bal) lastg = __shfl_sync(0xffffffffu, gv, 31 - __clz(bal));
  }
}

// one warp per (mtry, ntree, rep, fold) of the tasks in this launch
__global__ void k_score(ScoreArgs a) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int total = a.n_mtry * a.n_ntree * a.ntask;
  if (gw >= total) return;
  const int tl = gw % a.ntask;
  const int ni = (gw / a.ntask) % a.n_ntree;
  const int mi = gw / (a.ntask * a.n_ntree);
  const int task = a.task0 + tl;
  const int rep = task / a.k, fd = task % a.k;
  const int P = a.ntrees[ni];
  int nsub_used = (P - a.tree_lo + a.Cw - 1) / a.Cw;
  if (nsub_used > a.nsub) nsub_used = a.nsub;
  if (nsub_used < 0) nsub_used = 0;
  const int nte = a.nte[tl];
  const uint32_t* te = a.te_rows + (size_t)tl * a.n;
  const double* part = a.partial + ((size_t)mi * a.ntask + tl) * a.nsub * a.nte_max;
  double esum = 0.0;  // lane 0: sequential sum in ascending test-row order
  for (int base = 0; base < nte; base += 32) {
    const int r = base + lane;
    double e = 0.0;
    if (r < nte) {
      double s = 0.0;
      for (int c = 0; c < nsub_used; ++c) s += part[(size_t)c * a.nte_max + r];
      const size_t o = (((size_t)mi * a.n_ntree + ni) * a.reps + rep) * a.n + te[r];
      if (a.partial_rows) {
        a.partial_rows[o] = s;
      } else {
        double yh = s / (double)P;
        if (a.target == 1) yh = exp(yh);
        const double yv = a.y[te[r]];
        e = fabs(yv - yh) / yv;
        if (a.pred) a.pred[o] = yh;
      }
    }
    for (int l = 0; l < 32; ++l) {
      double v = __shfl_sync(0xffffffffu, e, l);
      if (base + l < nte) esum += v;
    }
  }
  if (lane == 0 && !a.partial_rows)
    a.fold_mape[(((size_t)mi * a.n_ntree + ni) * a.reps + rep) * a.k + fd] = 100.0 * esum / (double)nte;
}

struct FinArgs {
  const double* reduced;
  const double* y;
  const int32_t* fold;
  int n, k, reps, n_mtry, n_ntree, target;
  int ntrees[16];
  double* fold_mape;
  double* pred;
};

__global__ void k_finalize(FinArgs a) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int total = a.n_mtry * a.n_ntree * a.reps * a.k;
  if (gw >= total) return;
  const int fd = gw % a.k;
  const int rep = (gw / a.k) % a.reps;
  const int ni = (gw / (a.k * a.reps)) % a.n_ntree;
  const int mi = gw / (a.k * a.reps * a.n_ntree);
  const int P = a.ntrees[ni];
  const size_t o = (((size_t)mi * a.n_ntree + ni) * a.reps + rep) * a.n;
  const int32_t* fr = a.fold + (size_t)rep * a.n;
  double esum = 0.0;
  int cnt = 0;
  for (int base = 0; base < a.n; base += 32) {
    const int i = base + lane;
    const bool mine = i < a.n && fr[i] == fd;
    double e = 0.0;
    if (mine) {
      double yh = a.reduced[o + i] / (double)P;
      if (a.target == 1) yh = exp(yh);
      e = fabs(a.y[i] - yh) / a.y[i];
      if (a.pred) a.pred[o + i] = yh;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, mine);
    for (int l = 0; l < 32; ++l) {
      double v = __shfl_sync(0xffffffffu, e, l);
      if ((bal >> l) & 1u) esum += v;
    }
    cnt += __popc(bal);
  }
  if (lane == 0)
    a.fold_mape[(((size_t)mi * a.n_ntree + ni) * a.reps + rep) * a.k + fd] =
        cnt ? 100.0 * esum / (double)cnt : __longlong_as_double(0x7ff8000000000000ll);
}

}  // namespace

size_t make_folds_ws_bytes(int n, int reps, int custom) {
  if (n <= kFoldSmallMax || custom) return 0;
  const size_t total = (size_t)n * reps;
  size_t temp = 0;
  cub::DeviceSegmentedRadixSort::SortPairs(nullptr, temp, (const unsigned long long*)nullptr,
                                           (unsigned long long*)nullptr, (const uint32_t*)nullptr,
                                           (uint32_t*)nullptr, (int64_t)total, reps,
                                           (const int64_t*)nullptr, (const int64_t*)nullptr);
  return total * (8 + 8 + 4 + 4) + (reps + 1) * 8 + temp + 256;
}

cudaError_t make_folds(const double* dy, int n, int k, int reps, uint64_t seed, int custom,
                       int32_t* dfold, void* ws, size_t ws_bytes, cudaStream_t s, const uint8_t* dmask) {
  if (reps <= 0) return cudaSuccess;
  if (custom) {
    if (n > kFoldSmallMax) return cudaErrorNotSupported;
    size_t smem = (size_t)n * 18;
    if (smem > 48 * 1024)
      allow_max_dynamic_smem(k_folds_custom_small);
    k_folds_custom_small<<<reps, 256, smem, s>>>(dy, n, k, seed, dmask, dfold);
    note_launch();
    return cudaGetLastError();
  }
  if (n <= kFoldSmallMax) {
    size_t smem = (size_t)n * 9;
    k_folds_plain_small<<<reps, 256, smem, s>>>(n, k, seed, dmask, dfold);
    note_launch();
    return cudaGetLastError();
  }
  if (dmask) return cudaErrorNotSupported;  // masked folds: n <= 4096 (nested CV)
  const size_t total = (size_t)n * reps;
  char* w = static_cast<char*>(ws);
  unsigned long long* kin = reinterpret_cast<unsigned long long*>(w);
  unsigned long long* kout = kin + total;
  uint32_t* vin = reinterpret_cast<uint32_t*>(kout + total);
  uint32_t* vout = vin + total;
  int64_t* offs = reinterpret_cast<int64_t*>((reinterpret_cast<uintptr_t>(vout + total) + 15) & ~uintptr_t(15));
  char* temp = reinterpret_cast<char*>(offs + reps + 1);
  size_t temp_bytes = ws_bytes - (size_t)(temp - w);
  k_fold_keys<<<148 * 8, 256, 0, s>>>(n, reps, seed, kin, vin);
  note_launch();
  k_seg_off<<<(reps + 1 + 127) / 128, 128, 0, s>>>(offs, reps, n);
  note_launch();
  cudaError_t e = cub::DeviceSegmentedRadixSort::SortPairs(temp, temp_bytes, kin, kout, vin, vout,
                                                           (int64_t)total, reps, offs, offs + 1, 0, 64, s);
  if (e != cudaSuccess) return e;
  k_fold_scatter<<<148 * 8, 256, 0, s>>>(vout, n, k, reps, dfold);
  note_launch();
  return cudaGetLastError();
}

cudaError_t build_tasks(const int32_t* dfold, int k, const uint32_t*, const uint32_t*, TaskData& t,
                        cudaStream_t s) {
  k_tasks<<<t.ntask, 256, 0, s>>>(dfold, t.n, k, t.task0, t.tr_rows, t.te_rows, t.loc, t.ntr, t.nte);
  note_launch();
  return cudaGetLastError();
}

cudaError_t build_task_orders_u8(const uint32_t* order, const uint32_t* grank, TaskData& t,
                                 cudaStream_t s) {
  const int warps = t.ntask * t.p;
  k_task_orders_u8<<<(warps * 32 + 255) / 256, 256, 0, s>>>(order, grank, t.loc, t.n, t.p, t.ntask,
                                                           t.ntr_stride, t.ord, t.lrank);
  note_launch();
  return cudaGetLastError();
}

cudaError_t score_cv(const ScoreArgs& a, cudaStream_t s) {
  const int warps = a.n_mtry * a.n_ntree * a.ntask;
  k_score<<<(warps * 32 + 127) / 128, 128, 0, s>>>(a);
  note_launch();
  return cudaGetLastError();
}

cudaError_t finalize_cv(const double* reduced, const double* y, const int32_t* fold, int n, int k,
                        int reps, int n_mtry, int n_ntree, const int* ntrees, int target,
                        double* fold_mape, double* pred, cudaStream_t s) {
  FinArgs a;
  a.reduced = reduced; a.y = y; a.fold = fold; a.n = n; a.k = k; a.reps = reps;
  a.n_mtry = n_mtry; a.n_ntree = n_ntree; a.target = target;
  for (int i = 0; i < n_ntree && i < 16; ++i) a.ntrees[i] = ntrees[i];
  a.fold_mape = fold_mape; a.pred = pred;
  const int warps = n_mtry * n_ntree * reps * k;
  k_finalize<<<(warps * 32 + 127) / 128, 128, 0, s>>>(a);
  note_launch();
  return cudaGetLastError();
}



// ----------------------------------------------------- nested CV (R31) ----
namespace {

// mask[c][i] = (outer fold of row i in iteration it) != o, c = it * k_outer + o
__global__ void k_nested_mask(const int32_t* __restrict__ outer, int n, int k_outer, int C, uint8_t* mask) {
  const size_t total = (size_t)C * n;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < total; q += (size_t)gridDim.x * blockDim.x) {
    const int c = (int)(q / n), i = (int)(q - (size_t)c * n);
    const int it = c / k_outer, o = c - it * k_outer;
    mask[q] = outer[(size_t)it * n + i] != o;
  }
}

// thread per combo: score of every grid point = (sum of its inner fold MAPEs in fold
// order) / k_inner; best = first minimum in grid order (mtry-major, then ntree)
__global__ void k_nested_select(const double* __restrict__ fm_in, int nm, int nt, int C, int k_in,
                                int32_t* best, double* score) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  double bs = 0.0;
  int bg = -1;
  for (int mi = 0; mi < nm; ++mi)
    for (int ti = 0; ti < nt; ++ti) {
      const double* f = fm_in + (((size_t)mi * nt + ti) * C + c) * k_in;
      double s = 0.0;
      for (int j = 0; j < k_in; ++j) s = __dadd_rn(s, f[j]);
      s = __ddiv_rn(s, (double)k_in);
      if (score) score[((size_t)c * nm + mi) * nt + ti] = s;
      if (bg < 0 || s < bs) { bs = s; bg = mi * nt + ti; }
    }
  best[c] = bg;
}

// thread per combo: the outer fold's MAPE at the selected grid point
__global__ void k_nested_pick(const double* __restrict__ fm_out, const int32_t* __restrict__ best, int nt,
                              int C, int k_out, int iters, double* outer_mape) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const int g = best[c], mi = g / nt, ti = g - mi * nt;
  const int it = c / k_out, o = c - it * k_out;
  outer_mape[c] = fm_out[(((size_t)mi * nt + ti) * iters + it) * k_out + o];
}

// APE buckets [0,10) [10,25) [25,50) [50,100) [100,inf) percent; NaN skipped
__global__ void k_ape_buckets(const double* __restrict__ y, const double* __restrict__ yhat, int64_t n,
                              unsigned long long* counts) {
  __shared__ unsigned int c[5];
  if (threadIdx.x < 5) c[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double b = yhat[i];
    if (b != b) continue;
    const double e = __dmul_rn(100.0, __ddiv_rn(fabs(__dsub_rn(y[i], b)), y[i]));
    const int j = (e < 10.0) ? 0 : (e < 25.0) ? 1 : (e < 50.0) ? 2 : (e < 100.0) ? 3 : 4;
    atomicAdd(&c[j], 1u);
  }
  __syncthreads();
  if (threadIdx.x < 5 && c[threadIdx.x]) atomicAdd(&counts[threadIdx.x], (unsigned long long)c[threadIdx.x]);
}

}  // namespace

cudaError_t nested_mask(const int32_t* outer, int n, int k_outer, int C, uint8_t* mask, cudaStream_t s) {
  const size_t total = (size_t)C * n;
  k_nested_mask<<<(unsigned)std::min<size_t>((total + 255) / 256, 148 * 8), 256, 0, s>>>(outer, n, k_outer, C, mask);
  note_launch();
  return cudaGetLastError();
}

cudaError_t nested_select(const double* fm_in, int nm, int nt, int C, int k_in, int32_t* best, double* score,
                          cudaStream_t s) {
  k_nested_select<<<(C + 127) / 128, 128, 0, s>>>(fm_in, nm, nt, C, k_in, best, score);
  note_launch();
  return cudaGetLastError();
}

cudaError_t nested_pick(const double* fm_out, const int32_t* best, int nt, int C, int k_out, int iters,
                        double* outer_mape, cudaStream_t s) {
  k_nested_pick<<<(C + 127) / 128, 128, 0, s>>>(fm_out, best, nt, C, k_out, iters, outer_mape);
  note_launch();
  return cudaGetLastError();
}

cudaError_t ape_buckets(const double* y, const double* yhat, int64_t n, unsigned long long* counts, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(counts, 0, 5 * sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  if (n <= 0) return cudaSuccess;
  k_ape_buckets<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 4), 256, 0, s>>>(y, yhat, n, counts);
  note_launch();
  return cudaGetLastError();
}

}  // namespace rf
