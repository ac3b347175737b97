// large_tree.cu -- level-synchronous exact CART growth in global memory for
// training sets beyond the CTA-resident kernel (n_tr > 255), SURVEY.md 8(d) C3.
//
// Same method and readings as small_tree.cu (sec. 2.2 P:202-215;
// DESIGN.md R2-R14): identical bootstrap, heap-keyed feature draws, exact int64
// split sums, canonical fp64 score, tie-break, thresholds, stopping, leaf values
// and BFS node order.  A batch of B trees grows one level per round; all
// kernels of a round cover every open node of every tree in the batch:
//   node_prep   feature draws (Philox keyed by heap index), reset node bests
//   search      flattened (node, drawn feature, position) elements in node-major
//               order, tiles of 128 threads x KC elements, one pass: tile sums
//               (weights and targets cached in shared memory), decoupled look-back
//               over the preceding tiles, exact prefix sums (global prefix minus
//               segment base, modular uint64) and candidate scores; per-thread run
//               bests merged into the node best with a 128-bit compare-and-swap on
//               (G key, draw slot|position) -- a total order, so the result does not
//               depend on timing.  (Gathering a thread's 16 elements at once instead
//               of one by one measured 20 % slower: 80 registers, fewer warps; staging
//               list indices first and loading entries and (w, t_q) lane-strided --
//               coalesced list reads, 8 gathers in flight per lane -- 3.5 % slower,
//               profiles/rd2_34_ab_c3.txt.)
//   (ExtraTrees, R29: extra_bounds locates each (node, slot) segment's random
//   threshold first; the search then scores only that boundary)
//   decide      split flag, threshold, first-row targets for the constancy test
//   mark        go-left flags per row, child sums (warp-aggregated atomics),
//               child constancy flags
//   children    scans over nodes: BFS ids per tree, open children, positions;
//               next-level node tables; BFS node emission
//   partition   per-position split descriptors, go-left bits per row staged in
//               shared memory; one warp streams each list with a running carry and
//               ballot ranks (the tiled count/scan/scatter variant remains for the
//               histogram mode's single list and n > 2^20)
// Per-level sizes are read back once per round (one small D2H).
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <memory>
#include <vector>

#include "large_tree.cuh"
#include "predict.cuh"

namespace rf {
namespace {

constexpr int kThreads = 128;
// resident-CTA hint of the split search (A/B via RF_DEFS: 8 per SM beat 1, 10, 12; caching the
// list entries of pass 1 in shared memory for pass 2 (+8 KB per CTA) made the search 22 % slower
// -- the shared carve-out costs L1 capacity the gathers need -- and two gathers (t_q shared, w per
// tree) instead of the packed word 44 % slower, profiles/rd2_41_ab.txt; deciding the candidate
// flags in pass 1 (bit 0 of the staged t_q) so that pass 2 reads no list entries: neutral,
// rd2_49_ab_c3.txt; gathering the
// ranks in pass 1 with the weights instead of in pass 2 measured 39 % slower, and walking the
// cursor first to issue a thread's 16 weight/target gathers back to back 18 % slower; carrying the
// tree's bootstrap weight in 4 bits of the list entries so that pass 1 gathers only the shared
// t_q (800 KB instead of the 400 MB of per-tree packed words): search -2 %, in-bag list setup
// +4.3 ms, fit time neutral, rd2_54_ab_c3.txt)
#ifndef RF_SEARCH_MINB
#define RF_SEARCH_MINB 8
#endif
#ifndef RF_SEARCH_KC
#define RF_SEARCH_KC 16
#endif
constexpr int kKC = RF_SEARCH_KC;  // elements per thread in the search tiles
constexpr int kTile = kThreads * kKC;

struct __align__(16) Best {
  unsigned long long key;  // G bits + 1 (0 = no candidate)
  // search: tie key << 56 | draw slot << 48 | position (ascending = preferred; tie key = feature
  // index (north_star) or draw slot (R9)); after decide: feature << 32 | position
  unsigned long long aux;
};

__device__ __forceinline__ bool better(unsigned long long k1, unsigned long long a1, unsigned long long k2,
                                       unsigned long long a2) {
  return k1 > k2 || (k1 == k2 && a1 < a2);
}

__device__ __forceinline__ void cas128(Best* addr, unsigned long long key, unsigned long long aux) {
  unsigned long long clo = addr->key, chi = addr->aux;
  while (better(key, aux, clo, chi)) {
    unsigned long long olo, ohi;
    asm volatile(
        "{\n .reg .b128 d, c, v;\n mov.b128 c, {%2, %3};\n mov.b128 v, {%4, %5};\n"
        " atom.global.cas.b128 d, [%6], c, v;\n mov.b128 {%0, %1}, d;\n}\n"
        : "=l"(olo), "=l"(ohi)
        : "l"(clo), "l"(chi), "l"(key), "l"(aux), "l"(addr)
        : "memory");
    if (olo == clo && ohi == chi) return;
    clo = olo;
    chi = ohi;
  }
}

struct WS2 {  // (W, S) pair for scans; S in modular uint64
  unsigned long long w, s;
};
struct WS2Sum {
  __host__ __device__ WS2 operator()(const WS2& a, const WS2& b) const { return WS2{a.w + b.w, a.s + b.s}; }
};
struct U4S {  // children scan: split count, open-children count, open positions, left count
  unsigned int sp, op, pos, nl;
};
struct U4Sum {
  __host__ __device__ U4S operator()(const U4S& a, const U4S& b) const {
    return U4S{a.sp + b.sp, a.op + b.op, a.pos + b.pos, a.nl + b.nl};
  }
};

// node table (structure of arrays), one level
struct Nodes {
  uint32_t* tree;
  uint32_t* start;  // first position in the tree's position space
  uint32_t* len;    // distinct in-bag rows
  uint32_t* W;      // sum of multiplicities
  int64_t* S;       // sum of w * t_q
  uint64_t* heap;
  uint32_t* bfs;    // BFS id within the tree
};

struct Batch {
  int B, n, p, m, ntr, mss, max_depth;
  int F;
  int nl;                   // row lists per tree: p (exact, one per feature) or 1 (histogram)
  int hist;                 // 256-bin histogram split mode (R23)
  int extra;                // ExtraTrees split mode (R29)
  int tie_draw;             // tie-break (R9): 0 lowest feature index (north_star), 1 first drawn
  int mae;                  // MAE criterion (R32): list p holds the in-bag rows in t_q order
  int64_t* med2;            // [NMAX][2] MAE: doubled weighted medians of the children (or the node)
  uint32_t* xb;             // [NMAX][m] ExtraTrees: boundary index in the (node, slot) segment or ~0
  const uint8_t* bins;      // [n][p] bin of every row (histogram mode)
  const uint8_t* binsT;     // [p][n] the same, feature-major (the count pass's one-byte reads: a node's
                            // rows are ascending in its list, so the top levels read dense runs)
  const double* cuts;       // [p][256] cut values (histogram mode)
  const int32_t* ncuts;     // [p]
  uint32_t* accN;           // [NMAX] rows going left (histogram mode)
  long long* cmm;           // [NMAX][4] child t_q min/max: minL, maxL, minR, maxR (histogram mode)
  const double* X;
  const int64_t* tq;
  const uint32_t* grank;
  const uint32_t* tr_rows;  // training rows (ascending)
  uint32_t* keys;           // [B][2]
  uint8_t* w;               // [B][n] by global row
  long long* wt;            // [B][n] (t_q << 8) | w per training row (exact when ceil(log2 n) >= 9), or null
  // list entries: row | (low 15 bits of its rank of x_f) << 17 when n <= 2^17 (exact and
  // ExtraTrees modes), else the row; every reader masks with rowMask
  int packRank;
  uint32_t rowMask;
  const uint8_t* rfit;      // [p] 1: all dense ranks of feature f < 2^15 (packed bits decide) or null
  uint8_t* side;            // [B][n]
  uint32_t* sideBits;       // [B][nbw] go-left bit per row (fused partition path) or null
  int nbw;                  // words per tree in sideBits = ceil(n / 32)
  uint32_t* L[2];           // [B][p][ntr]
  uint32_t* posNode[2];     // [B*ntr] concatenated positions -> node
  Nodes nd[2];
  uint8_t* feat;            // [NMAX][m]
  Best* best;               // [NMAX]
  uint32_t* accW;           // [NMAX]
  unsigned long long* accS; // [NMAX]
  uint8_t* nc;              // [NMAX][2]
  double* thr;              // [NMAX]
  uint32_t* thrIdx;         // [NMAX]
  WS2* nodePref;            // [NMAX] exclusive prefix of (W, S) over nodes
  U4S* chScan;              // [NMAX] children scan (exclusive)
  U4S* chVal;               // [NMAX]
  uint8_t* chFlags;         // [NMAX] bit0 left child open, bit1 right child open
  // per tree (device)
  uint32_t* tNode0;    // first node index of the tree at this level [B+1]
  uint32_t* tPos0;     // first concatenated position [B+1]
  uint32_t* tBase;     // BFS id of the first node of this level
  uint32_t* tCount;    // nodes at this level (incl. leaves created at this depth)
  // outputs
  Node16* out;         // [B][cap]
  uint32_t* outThr;    // [B][cap]
  uint32_t* outCount;  // [B]
  uint64_t cap;
  int32_t* leaf_of_row;  // [B][n] or null
  double* imp;           // [B][p] MDI decreases per tree and feature (fit), or null
  int tree0;             // global tree index of batch slot 0
  int* err;
};

// candidate aux (search order among bitwise-equal keys, R9): tie key << 56 | draw slot << 48 |
// position; the tie key is the feature index (north_star: lowest feature, then lowest
// threshold) or the draw slot (first drawn feature); f, j < 256 (p <= 255)
__device__ __forceinline__ unsigned long long cand_aux(const Batch& b, int j, int f, unsigned pos) {
  return ((unsigned long long)(b.tie_draw ? j : f) << 56) | ((unsigned long long)j << 48) | pos;
}

// ---------------------------------------------------------------- setup ------
__global__ void k_keys_boot(Batch b, uint64_t seed, int task, int bootstrap) {
  const int t = blockIdx.y;
  uint32_t k0, k1;
  tree_key(seed, (uint32_t)task, (uint32_t)(b.tree0 + t), k0, k1);
  if (blockIdx.x == 0 && threadIdx.x == 0) { b.keys[2 * t] = k0; b.keys[2 * t + 1] = k1; }
  uint8_t* w = b.w + (size_t)t * b.n;
  if (!bootstrap) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < b.ntr; j += gridDim.x * blockDim.x) w[b.tr_rows[j]] = 1;
    return;
  }
  // byte counters updated by 32-bit reductions (no return value) on the aligned word holding
  // them; the word is located from the absolute byte offset (tree slots of n bytes need not be
  // 4-aligned).  A count passing 255 would carry into the next byte (or out of the word) and
  // lower the sum of the bytes, so k_root_finish flags overflow when sum(w) != n_tr.
  const auto count = [&](uint32_t r) {
    const size_t idx = (size_t)t * b.n + r;
    const uint32_t sh = (uint32_t)(idx & 3u) * 8u;
    atomicAdd(reinterpret_cast<unsigned int*>(b.w + (idx & ~(size_t)3)), 1u << sh);
  };
  const int nblk = (b.ntr + 1) >> 1;
  for (int blk = blockIdx.x * blockDim.x + threadIdx.x; blk < nblk; blk += gridDim.x * blockDim.x) {
    uint64_t d0, d1;
    philox_pair(k0, k1, (uint32_t)blk, 0u, 0u, kTagBoot, d0, d1);
    count(b.tr_rows[mulhi64(d0, (uint64_t)b.ntr)]);
    if (2 * blk + 1 < b.ntr) count(b.tr_rows[mulhi64(d1, (uint64_t)b.ntr)]);
  }
}

// packed (t_q << 8) | w per training row of each tree: one 8-byte gather per search
// element instead of two.  |t_q| <= 2^(62 - ceil(log2 n)) (R7), so for n > 256 the
// shifted target stays below 2^61 and the packing is exact.
__global__ void k_pack_wt(Batch b) {
  const int t = blockIdx.y;
  const uint8_t* w = b.w + (size_t)t * b.n;
  long long* wt = b.wt + (size_t)t * b.n;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < b.ntr; j += gridDim.x * blockDim.x) {
    const uint32_t r = b.tr_rows[j];
    wt[r] = (long long)((unsigned long long)b.tq[r] << 8) | (long long)w[r];
  }
}

// one CTA per (tree, list): stable compaction of the task order by w > 0
// (exact: one list per feature in x order; histogram: one list of training rows)
__global__ void k_inbag_lists(Batch b, const uint32_t* __restrict__ task_order /*[nl][ntr] global rows*/) {
  const int t = blockIdx.x / b.nl, f = blockIdx.x % b.nl;
  const uint8_t* w = b.w + (size_t)t * b.n;
  const uint32_t* src = task_order + (size_t)f * b.ntr;
  uint32_t* dst = b.L[0] + ((size_t)t * b.nl + f) * b.ntr;
  using BS = cub::BlockScan<uint32_t, kThreads>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < b.ntr; base += kThreads) {
    const int j = base + threadIdx.x;
    uint32_t r = 0, keep = 0;
    if (j < b.ntr) { r = src[j]; keep = w[r] != 0; }
    uint32_t ex, tot;
    BS(tmp).ExclusiveSum(keep, ex, tot);
    if (keep) dst[carry + ex] = (b.packRank && f < b.p) ? r | ((b.grank[(size_t)f * b.n + r] & 0x7FFFu) << 17) : r;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
}

// Warp per (tree, list): the same stable compaction streamed by one warp with ballot ranks and a
// running carry (the partition kernel's pattern: 8 x 32 entries in flight per step, no block
// scans or barriers); a CTA's 8 warps take 8 lists of one tree.
constexpr int kIbwWarps = 8, kIbwSteps = 8;
__global__ void __launch_bounds__(32 * kIbwWarps) k_inbag_lists_warp(Batch b, const uint32_t* __restrict__ task_order) {
  const int t = blockIdx.y;
  const int f = blockIdx.x * kIbwWarps + (threadIdx.x >> 5);
  if (f >= b.nl) return;
  const int lane = threadIdx.x & 31;
  const uint8_t* w = b.w + (size_t)t * b.n;
  const uint32_t* src = task_order + (size_t)f * b.ntr;
  uint32_t* dst = b.L[0] + ((size_t)t * b.nl + f) * b.ntr;
  const bool pack = b.packRank && f < b.p;
  const uint32_t* gr = b.grank + (size_t)f * b.n;
  const unsigned lt = (1u << lane) - 1u;
  uint32_t carry = 0;
  for (int base = 0; base < b.ntr; base += 32 * kIbwSteps) {
    uint32_t r[kIbwSteps];
#pragma unroll
    for (int k = 0; k < kIbwSteps; ++k) {
      const int j = base + 32 * k + lane;
      r[k] = j < b.ntr ? src[j] : 0u;
    }
    bool keep[kIbwSteps];
#pragma unroll
    for (int k = 0; k < kIbwSteps; ++k) keep[k] = base + 32 * k + lane < b.ntr && w[r[k]] != 0;
#pragma unroll
    for (int k = 0; k < kIbwSteps; ++k) {
      const unsigned bal = __ballot_sync(0xffffffffu, keep[k]);
      if (keep[k]) dst[carry + __popc(bal & lt)] = pack ? r[k] | ((gr[r[k]] & 0x7FFFu) << 17) : r[k];
      carry += __popc(bal);
    }
  }
}

// Root node of every tree (W, S, distinct count, constancy) over many CTAs per tree (large n: one CTA per tree left the GPU idle at
// C4 sizes).  acc[4 t..4 t+3] = (S, D, min t_q, max t_q), initialised by k_root_init.
__global__ void k_root_init(int B, unsigned long long* acc) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= B) return;
  acc[4 * t] = 0ull;
  acc[4 * t + 1] = 0ull;
  acc[4 * t + 2] = (unsigned long long)LLONG_MAX;
  acc[4 * t + 3] = (unsigned long long)LLONG_MIN;
}

__global__ void __launch_bounds__(256) k_root_partial(Batch b, unsigned long long* acc) {
  const int t = blockIdx.y;
  const uint8_t* w = b.w + (size_t)t * b.n;
  long long S = 0;
  long long mn = LLONG_MAX, mx = LLONG_MIN;
  unsigned long long D = 0;  // distinct rows (low 32 bits) and sum of multiplicities (high 32 bits)
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < b.ntr; j += gridDim.x * blockDim.x) {
    const uint32_t r = b.tr_rows[j];
    const uint32_t wv = w[r];
    if (wv) {
      const long long v = b.tq[r];
      S += (long long)wv * v;
      mn = min(mn, v);
      mx = max(mx, v);
      D += 1ull + ((unsigned long long)wv << 32);
    }
  }
  using BR = cub::BlockReduce<long long, 256>;
  using BRu = cub::BlockReduce<unsigned long long, 256>;
  __shared__ typename BR::TempStorage t1;
  __shared__ typename BRu::TempStorage t2;
  const long long Ssum = BR(t1).Sum(S);
  __syncthreads();
  const long long mnr = BR(t1).Reduce(mn, cub::Min());
  __syncthreads();
  const long long mxr = BR(t1).Reduce(mx, cub::Max());
  __syncthreads();
  const unsigned long long Dsum = BRu(t2).Sum(D);
  if (threadIdx.x == 0 && Dsum) {
    atomicAdd(&acc[4 * t], (unsigned long long)Ssum);  // modular: exact for the int64 sum
    atomicAdd(&acc[4 * t + 1], Dsum);
    atomicMin(reinterpret_cast<long long*>(&acc[4 * t + 2]), mnr);
    atomicMax(reinterpret_cast<long long*>(&acc[4 * t + 3]), mxr);
  }
}

__global__ void k_root_finish(Batch b, const unsigned long long* acc, uint32_t* rootInfo) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= b.B) return;
  const long long Ssum = (long long)acc[4 * t];
  const unsigned int Dsum = (unsigned int)(acc[4 * t + 1] & 0xFFFFFFFFull);
  if ((acc[4 * t + 1] >> 32) != (unsigned long long)b.ntr) atomicOr(b.err, kErrOverflow);  // a count wrapped
  const long long mnr = (long long)acc[4 * t + 2], mxr = (long long)acc[4 * t + 3];
  const bool leaf = (b.max_depth == 0) || ((int)Dsum < b.mss) || (mnr == mxr);
  rootInfo[4 * t] = Dsum;
  rootInfo[4 * t + 1] = leaf;
  Node16 nd;
  nd.feat = -1; nd.left = 0;
  nd.v = scalbn(__ddiv_rn(__ll2double_rn(Ssum), __uint2double_rn((unsigned)b.ntr)), -b.F);
  if (leaf) {
    b.out[(size_t)t * b.cap] = nd;
    b.outThr[(size_t)t * b.cap] = 0;
    b.outCount[t] = 1;
  }
  reinterpret_cast<long long*>(rootInfo)[2 * t + 1] = Ssum;  // words 2,3
}

// In-bag compaction of long lists in tiles (one CTA per list left the GPU idle at C4
// sizes): per (tree, list, tile of kIbTile rows) the kept count, a device scan over all
// tiles, then a block scan + tile prefix - the list's first tile prefix per tile.
constexpr int kIbThreads = 256, kIbItems = 16, kIbTile = kIbThreads * kIbItems;

__global__ void __launch_bounds__(kIbThreads) k_inbag_count(Batch b, const uint32_t* __restrict__ task_order,
                                                            int tiles, uint32_t* cnt) {
  const int lt = blockIdx.x, tile = lt % tiles, tl = lt / tiles;  // tl = t * nl + f
  const int t = tl / b.nl, f = tl % b.nl;
  const uint8_t* w = b.w + (size_t)t * b.n;
  const uint32_t* src = task_order + (size_t)f * b.ntr;
  uint32_t c = 0;
  const int j0 = tile * kIbTile + threadIdx.x * kIbItems;
#pragma unroll
  for (int q = 0; q < kIbItems; ++q) {
    const int j = j0 + q;
    if (j < b.ntr) c += w[src[j]] != 0;
  }
  using BR = cub::BlockReduce<uint32_t, kIbThreads>;
  __shared__ typename BR::TempStorage tmp;
  const uint32_t tot = BR(tmp).Sum(c);
  if (threadIdx.x == 0) cnt[lt] = tot;
}

__global__ void __launch_bounds__(kIbThreads) k_inbag_scatter(Batch b, const uint32_t* __restrict__ task_order,
                                                              int tiles, const uint32_t* __restrict__ pref) {
  const int lt = blockIdx.x, tile = lt % tiles, tl = lt / tiles;
  const int t = tl / b.nl, f = tl % b.nl;
  const uint8_t* w = b.w + (size_t)t * b.n;
  const uint32_t* src = task_order + (size_t)f * b.ntr;
  uint32_t* dst = b.L[0] + ((size_t)t * b.nl + f) * b.ntr;
  const int j0 = tile * kIbTile + threadIdx.x * kIbItems;
  uint32_t rr[kIbItems];
  uint32_t keep = 0, c = 0;
#pragma unroll
  for (int q = 0; q < kIbItems; ++q) {
    const int j = j0 + q;
    rr[q] = j < b.ntr ? src[j] : 0u;
    const uint32_t k = (j < b.ntr && w[rr[q]] != 0) ? 1u : 0u;
    keep |= k << q;
    c += k;
  }
  using BS = cub::BlockScan<uint32_t, kIbThreads>;
  __shared__ typename BS::TempStorage tmp;
  uint32_t ex;
  BS(tmp).ExclusiveSum(c, ex);
  uint32_t o = pref[lt] - pref[(size_t)tl * tiles] + ex;
#pragma unroll
  for (int q = 0; q < kIbItems; ++q) {
    if ((keep >> q) & 1u) {
      const uint32_t r = rr[q];
      dst[o++] = (b.packRank && f < b.p) ? r | ((b.grank[(size_t)f * b.n + r] & 0x7FFFu) << 17) : r;
    }
  }
}

// -------------------------------------------------------------- per level ----
__global__ void k_node_prep(Batch b, int cur, int NO) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= NO) return;
  const Nodes& nd = b.nd[cur];
  b.best[g] = Best{0ull, ~0ull};
  b.accW[g] = 0u;
  b.accS[g] = 0ull;
  b.nc[2 * g] = 0;
  b.nc[2 * g + 1] = 0;
  // the draw order matters even for m = p under the draw-order tie-break (R9) and for the
  // ExtraTrees thresholds (keyed by draw slot, R29)
  uint8_t* fp = b.feat + (size_t)g * b.m;
  if (b.m == b.p && !b.tie_draw && !b.extra) {  // all features, order irrelevant (as small_tree.cu)
    for (int f = 0; f < b.p; ++f) fp[f] = (uint8_t)f;
    return;
  }
  uint8_t perm[256];
  for (int f = 0; f < b.p; ++f) perm[f] = (uint8_t)f;
  const uint32_t t = nd.tree[g];
  const uint32_t k0 = b.keys[2 * t], k1 = b.keys[2 * t + 1];
  const uint64_t h = nd.heap[g];
  for (int j = 0; j < b.m; j += 2) {
    uint64_t d0, d1;
    philox_pair(k0, k1, (uint32_t)(j >> 1), (uint32_t)h, (uint32_t)(h >> 32), kTagFeat, d0, d1);
    int r = j + (int)mulhi64(d0, (uint64_t)(b.p - j));
    uint8_t tmp = perm[j]; perm[j] = perm[r]; perm[r] = tmp;
    if (j + 1 < b.m) {
      r = j + 1 + (int)mulhi64(d1, (uint64_t)(b.p - j - 1));
      tmp = perm[j + 1]; perm[j + 1] = perm[r]; perm[r] = tmp;
    }
  }
  for (int j = 0; j < b.m; ++j) fp[j] = perm[j];
}

// ExtraTrees (R29): thread per (node, slot): the slot's random threshold in [lo, hi) of the
// segment (sorted by x_f) and its boundary = last segment index with x <= thr (~0 if lo = hi)
__global__ void k_extra_bounds(Batch b, int cur, long long NQ) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= NQ) return;
  const int g = (int)(q / b.m), j = (int)(q - (long long)g * b.m);
  const Nodes& nd = b.nd[cur];
  const int t = (int)nd.tree[g], f = b.feat[q];
  const uint32_t len = nd.len[g];
  const uint32_t* L = b.L[cur & 1] + ((size_t)t * b.nl + f) * b.ntr + nd.start[g];
  const double* Xf = b.X + f;
  const double lo = Xf[(size_t)(L[0] & b.rowMask) * b.p], hi = Xf[(size_t)(L[len - 1] & b.rowMask) * b.p];
  uint32_t bnd = ~0u;
  if (lo < hi) {
    const double thr = extra_thr(b.keys[2 * t], b.keys[2 * t + 1], nd.heap[g], j, lo, hi);
    uint32_t l = 0, u = len - 1;  // x[l] <= thr < x[u]
    while (u - l > 1) {
      const uint32_t mid = (l + u) >> 1;
      if (Xf[(size_t)(L[mid] & b.rowMask) * b.p] <= thr) l = mid; else u = mid;
    }
    bnd = l;
  }
  b.xb[q] = bnd;
}

__global__ void k_node_ws(Batch b, int cur, int NO, WS2* out) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= NO) return;
  out[g] = WS2{(unsigned long long)b.nd[cur].W[g], (unsigned long long)b.nd[cur].S[g]};
}

// cursor over the flattened (node g, slot j, index i) space; positions are concatenated
// over trees (node g's positions [gpos0, gpos0 + len))
struct Cursor {
  int g, j, i, len, t, start, f;
  uint32_t xb;  // ExtraTrees boundary of the segment
  uint32_t W;
  int64_t S;
  long long listBase;  // offset of list (t, f) + start
};

__device__ __forceinline__ void cursor_load(const Batch& b, const Nodes& nd, Cursor& c) {
  c.len = (int)nd.len[c.g];
  c.t = (int)nd.tree[c.g];
  c.start = (int)nd.start[c.g];
  c.W = nd.W[c.g];
  c.S = nd.S[c.g];
}
__device__ __forceinline__ void cursor_feat(const Batch& b, Cursor& c) {
  c.f = b.feat[(size_t)c.g * b.m + c.j];
  c.listBase = ((long long)c.t * b.nl + c.f) * b.ntr + c.start;
  if (b.extra) c.xb = b.xb[(size_t)c.g * b.m + c.j];
}
// element e = m * gpos0(g) + j * len + i, gpos0 = concatenated first position of g
__device__ __forceinline__ void cursor_locate(const Batch& b, const Nodes& nd, const uint32_t* posNode,
                                              const uint32_t* tPos0, long long e, Cursor& c) {
  const long long q = e / b.m;
  c.g = (int)posNode[q];
  cursor_load(b, nd, c);
  const long long gpos0 = (long long)tPos0[c.t] + c.start;
  const long long off = e - (long long)b.m * gpos0;
  c.j = (int)(off / c.len);
  c.i = (int)(off - (long long)c.j * c.len);
  cursor_feat(b, c);
}
__device__ __forceinline__ void cursor_next_segment(const Batch& b, const Nodes& nd, Cursor& c) {
  c.i = 0;
  if (++c.j == b.m) {
    c.j = 0;
    ++c.g;
    cursor_load(b, nd, c);
  }
  cursor_feat(b, c);
}

// Single-pass search (decoupled look-back): a CTA takes the next tile id from a counter,
// sums its elements (pass 1, caching each element's weight and target in shared memory),
// publishes the tile aggregate, then walks back over the predecessors' published
// aggregates / inclusive prefixes for its exclusive prefix -- no separate totals kernel
// and no device-wide scan, and pass 2 reads the cached weights/targets instead of
// gathering them again.  Tile ids follow CTA start order, and every CTA publishes its
// aggregate before it waits, so the look-back cannot deadlock.  Flags carry a per-level
// epoch ((epoch << 2) | state; state 1 = aggregate, 2 = inclusive), so the status
// array is never reset.
// Shared staging of a thread's kKC = 16 elements: slot k of thread tid at tid * 16 + (k ^ (tid & 15)).
// Thread-serial walks (all threads at the same k) then spread over the banks instead of all 32
// threads hitting one bank (stride 16 x 8 B = 128 B); lane-strided walks (16 lanes over one
// thread's slots) stay conflict-free.
#ifdef RF_SEARCH_NOSWZ
#define SWZ(tid, k) ((tid) * kKC + (k))
#else
#define SWZ(tid, k) ((tid) * kKC + ((k) ^ ((tid) & (kKC - 1))))
#endif

struct TileStat {
  unsigned long long aw, as, iw, is;  // aggregate (W, S), inclusive prefix (W, S)
};

__global__ void __launch_bounds__(kThreads, RF_SEARCH_MINB) k_search_fused(Batch b, int cur, long long E, unsigned long long* ncand,
                                                           uint32_t* tileCtr, TileStat* stat, uint32_t* flags,
                                                           uint32_t epoch) {
  __shared__ uint32_t s_tile;
  __shared__ WS2 s_pref;
  __shared__ int s_local;  // 1: the tile contains a segment start, its prefix is known locally
  __shared__ long long s_t[kTile];
  __shared__ uint8_t s_w[kTile];
  if (threadIdx.x == 0) {
    s_tile = atomicAdd(tileCtr, 1u);
    s_local = 0;
  }
  __syncthreads();
  const long long tile = s_tile;
  const Nodes& nd = b.nd[cur];
  const uint32_t* posNode = b.posNode[cur];
  const uint32_t* L = b.L[cur & 1];
  const long long e0 = tile * kTile + (long long)threadIdx.x * kKC;
  const long long e1 = min(e0 + kKC, E);
  // pass 1: thread totals (weights and targets cached).  The absolute prefix at every
  // segment start is known from the node prefixes (m bW[g] + j W[g]), so a tile that
  // contains a segment start derives its own prefix and skips the look-back.
  unsigned long long lw = 0, ls = 0;
  bool has_start = false;
  unsigned long long sbW = 0, sbS = 0;  // segment base minus the thread's sum before that start
  Cursor c0;
  if (e0 < e1) {
    cursor_locate(b, nd, posNode, b.tPos0, e0, c0);
    Cursor c = c0;
    for (long long e = e0; e < e1; ++e) {
      if (!has_start && c.i == 0) {
        has_start = true;
        sbW = (unsigned long long)b.m * b.nodePref[c.g].w + (unsigned long long)c.j * c.W - lw;
        sbS = (unsigned long long)b.m * b.nodePref[c.g].s + (unsigned long long)c.j * (unsigned long long)c.S - ls;
      }
      const uint32_t r = L[c.listBase + c.i] & b.rowMask;
      uint32_t wv;
      long long tv;
      if (b.wt) {  // (the chunk may span trees)
        const long long v = b.wt[(size_t)c.t * b.n + r];
        wv = (uint32_t)(v & 0xFF);
        tv = v >> 8;
      } else {
        wv = b.w[(size_t)c.t * b.n + r];
        tv = b.tq[r];
      }
      s_w[SWZ(threadIdx.x, (int)(e - e0))] = (uint8_t)wv;
      s_t[SWZ(threadIdx.x, (int)(e - e0))] = tv;
      lw += wv;
      ls += (unsigned long long)((long long)wv * tv);
      if (++c.i == c.len && e + 1 < e1) cursor_next_segment(b, nd, c);
    }
  }
  using BS = cub::BlockScan<WS2, kThreads>;
  __shared__ typename BS::TempStorage tmp;
  WS2 ex, agg;
  BS(tmp).ExclusiveScan(WS2{lw, ls}, ex, WS2{0ull, 0ull}, WS2Sum(), agg);
  if (has_start) {  // every such thread derives the same value (benign identical writes)
    s_pref = WS2{sbW - ex.w, sbS - ex.s};
    s_local = 1;
  }
  __syncthreads();
  if (s_local) {
    if (threadIdx.x == 0) {
      volatile TileStat* vs = stat;
      vs[tile].iw = s_pref.w + agg.w; vs[tile].is = s_pref.s + agg.s;
      __threadfence();
      reinterpret_cast<volatile uint32_t*>(flags)[tile] = (epoch << 2) | 2u;
    }
  } else if (threadIdx.x < 32) {
    // warp-wide look-back: 32 predecessors per step; aggregates are summed until the
    // nearest published inclusive prefix (tile 0 always publishes one)
    volatile TileStat* vs = stat;
    volatile uint32_t* vf = flags;
    const int lane = threadIdx.x;
    unsigned long long pw = 0, ps = 0;
    if (tile == 0) {
      if (lane == 0) {
        vs[0].iw = agg.w; vs[0].is = agg.s;
        __threadfence();
        vf[0] = (epoch << 2) | 2u;
      }
    } else {
      if (lane == 0) {
        vs[tile].aw = agg.w; vs[tile].as = agg.s;
        __threadfence();
        vf[tile] = (epoch << 2) | 1u;
      }
      for (long long k = tile - 1;; k -= 32) {
        const long long kk = k - lane;
        uint32_t fl = 0;
        if (kk >= 0) {
          do { fl = vf[kk]; } while ((fl >> 2) != epoch || (fl & 3u) == 0u);
        }
        __syncwarp();
        __threadfence();
        const unsigned incl = __ballot_sync(0xffffffffu, kk >= 0 && (fl & 2u));
        const int stop = incl ? __ffs(incl) - 1 : 31;
        unsigned long long vw = 0, vsum = 0;
        if (kk >= 0 && lane <= stop) {
          if ((fl & 2u) && lane == stop) { vw = vs[kk].iw; vsum = vs[kk].is; }
          else { vw = vs[kk].aw; vsum = vs[kk].as; }
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
          vw += __shfl_xor_sync(0xffffffffu, vw, d);
          vsum += __shfl_xor_sync(0xffffffffu, vsum, d);
        }
        pw += vw;
        ps += vsum;
        if (incl) break;
      }
      if (lane == 0) {
        vs[tile].iw = pw + agg.w; vs[tile].is = ps + agg.s;
        __threadfence();
        vf[tile] = (epoch << 2) | 2u;
      }
    }
    if (lane == 0) s_pref = WS2{pw, ps};
  }
  __syncthreads();
  unsigned long long cW = s_pref.w + ex.w, cS = s_pref.s + ex.s;
  unsigned int nc = 0;
  if (e0 < e1) {  // pass 2 (no early return: the candidate count below is a full-warp shuffle)
  Cursor c = c0;
  unsigned long long segW = (unsigned long long)b.m * b.nodePref[c.g].w + (unsigned long long)c.j * c.W;
  unsigned long long segS = (unsigned long long)b.m * b.nodePref[c.g].s + (unsigned long long)c.j * (unsigned long long)c.S;
  unsigned long long rkey = 0ull, raux = ~0ull;
  int rg = c.g;
  const uint32_t* grank = b.grank;
  bool fits = b.rfit && b.rfit[c.f];  // packed rank bits decide alone (all ranks of f < 2^15)
  // r: list entry of the current element; rk: its rank (packed: the entry's rank bits, the
  // full rank gathered only when two neighbours' low rank bits agree)
  uint32_t r = L[c.listBase + c.i];
  uint32_t rk = b.packRank ? (r >> 17) : grank[(size_t)c.f * b.n + r];
  for (long long e = e0; e < e1; ++e) {
    const uint32_t wv = s_w[SWZ(threadIdx.x, (int)(e - e0))];
    cW += wv;
    cS += (unsigned long long)((long long)wv * s_t[SWZ(threadIdx.x, (int)(e - e0))]);
    const bool hasNext = c.i + 1 < c.len;
    uint32_t rn = r, rkn = rk;
    if (hasNext) {
      rn = L[c.listBase + c.i + 1];
      bool cand;
      if (b.extra) {
        cand = (uint32_t)c.i == c.xb;  // the segment's one candidate (R29)
      } else if (b.packRank) {
        rkn = rn >> 17;
        cand = rkn != rk ||
               (!fits && grank[(size_t)c.f * b.n + (rn & 0x1FFFFu)] != grank[(size_t)c.f * b.n + (r & 0x1FFFFu)]);
      } else {
        rkn = grank[(size_t)c.f * b.n + rn];
        cand = rkn != rk;
      }
      if (cand) {
        const unsigned long long WL = cW - segW;
        const long long SL = (long long)(cS - segS);
        const unsigned long long WR = (unsigned long long)c.W - WL;
        const long long SR = c.S - SL;
        const double G = split_gain((long long)WL, SL, (long long)WR, SR);
        const unsigned long long key = (unsigned long long)__double_as_longlong(G) + 1ull;
        const unsigned long long aux = cand_aux(b, c.j, c.f, (unsigned)c.i);  // R9
        ++nc;
        if (better(key, aux, rkey, raux)) { rkey = key; raux = aux; }
      }
    }
    if (e + 1 < e1) {
      if (!hasNext) {
        const int pg = c.g;
        cursor_next_segment(b, nd, c);
        if (c.g != pg) {
          if (rkey) cas128(&b.best[pg], rkey, raux);
          rkey = 0ull; raux = ~0ull;
          rg = c.g;
        }
        fits = b.rfit && b.rfit[c.f];
        segW = (unsigned long long)b.m * b.nodePref[c.g].w + (unsigned long long)c.j * c.W;
        segS = (unsigned long long)b.m * b.nodePref[c.g].s + (unsigned long long)c.j * (unsigned long long)c.S;
        rn = L[c.listBase];
        rkn = b.packRank ? (rn >> 17) : grank[(size_t)c.f * b.n + rn];
      } else {
        ++c.i;
      }
    }
    r = rn;
    rk = rkn;
  }
  if (rkey) cas128(&b.best[rg], rkey, raux);
  }

  if (ncand) {
    unsigned long long v = nc;
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(ncand, v);
  }
}

// per feature: 1 if every dense rank fits the 15 packed rank bits of a list entry (rfit)
__global__ void k_rank_fit(const uint32_t* __restrict__ grank, int n, int p, uint32_t* maxr, uint8_t* rfit,
                           int finish) {
  const int f = blockIdx.y;
  if (finish) {
    if (blockIdx.x == 0 && threadIdx.x == 0) rfit[f] = maxr[f] < 0x8000u ? 1 : 0;
    return;
  }
  uint32_t mx = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    mx = max(mx, grank[(size_t)f * n + i]);
  for (int d = 16; d > 0; d >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, d));
  if ((threadIdx.x & 31) == 0) atomicMax(&maxr[f], mx);
}

// ------------------------------------------------------- MAE criterion (R32) ----
// Level-synchronous MAE (SURVEY 8(f) NEXT-4 on training sets beyond the CTA-resident kernel:
// the paper's n = 4,096 sensitivity variant).  Same candidates, tie-break, thresholds and
// stopping as the MSE path (R8, R9, R29, R11); a candidate's cost is D = 2 (SAD_L + SAD_R), the
// doubled weighted absolute deviations of the children from their weighted medians (exact in
// uint64 under the 2 guard bits of quantisation), key = ~D so "larger key = better" and the
// 128-bit node-best CAS apply unchanged.  Each tree carries one more row list (list p): its
// in-bag rows in (t_q, row) order, partitioned with the feature lists.  A candidate's D is one
// walk of the node's t-ordered rows that routes every row to the left or right tracker by
// rank_f(row) <= rank_f(boundary row) and stops at both weighted medians (the small kernel's
// MedTrack, scikit-learn's median rule).  One CTA per (node, draw slot): the node's t-ordered
// (rank_f, w, t_q) are staged in shared memory once (nodes up to kMaeMaxLen distinct rows), the
// candidates' (W_L, S_L) come from a chunked prefix of the feature-ordered segment, and each warp
// walks the staged list for 32 candidates in lock step (broadcast shared loads).
constexpr int kMaeMaxLen = 12288;
constexpr int kMaeThreads = 256;

struct LMed {  // weighted-median tracker (as small_tree.cu MedTrack)
  uint32_t W, cum, Wk;
  int64_t sum, Sk, m2;
  int state;  // 0 searching, 1 waiting for t_k+1, 2 done
};
__device__ __forceinline__ void lmed_init(LMed& m, uint32_t W) {
  m.W = W; m.cum = 0; m.Wk = 0; m.sum = 0; m.Sk = 0; m.m2 = 0; m.state = W ? 0 : 2;
}
__device__ __forceinline__ void lmed_push(LMed& m, uint32_t wv, int64_t t) {
  if (m.state == 0) {
    m.cum += wv;
    m.sum += (int64_t)wv * t;
    if (2u * m.cum >= m.W) {
      m.Wk = m.cum; m.Sk = m.sum;
      if (2u * m.cum == m.W) { m.m2 = t; m.state = 1; }
      else { m.m2 = 2 * t; m.state = 2; }
    }
  } else if (m.state == 1) {
    m.m2 += t;
    m.state = 2;
  }
}
__device__ __forceinline__ uint64_t lmed_sad2(const LMed& m, int64_t S) {  // sum w |2t - m2|
  return (uint64_t)m.m2 * (uint64_t)(2u * m.Wk - m.W) + 2ull * (uint64_t)(S - 2 * m.Sk);
}

__device__ __forceinline__ void mae_row(const Batch& b, int t, uint32_t r, uint32_t& wv, long long& tv) {
  if (b.wt) {
    const long long v = b.wt[(size_t)t * b.n + r];
    wv = (uint32_t)(v & 0xFF);
    tv = v >> 8;
  } else {
    wv = b.w[(size_t)t * b.n + r];
    tv = b.tq[r];
  }
}

size_t mae_search_smem(int) { return (size_t)kMaeMaxLen * 13 + (size_t)(kMaeMaxLen / 32 + 1) * 16 + 64; }

__global__ void __launch_bounds__(kMaeThreads) k_mae_search(Batch b, int cur, unsigned long long* ncand) {
  extern __shared__ __align__(16) char msm[];
  long long* tt = reinterpret_cast<long long*>(msm);                          // [len] t_q, t order
  uint32_t* trk = reinterpret_cast<uint32_t*>(tt + kMaeMaxLen);               // [len] rank_f, t order
  WS2* cpref = reinterpret_cast<WS2*>(trk + kMaeMaxLen);                       // [chunks] exclusive prefix
  uint8_t* tw = reinterpret_cast<uint8_t*>(cpref + kMaeMaxLen / 32 + 1);       // [len] w, t order
  __shared__ unsigned long long sk[kMaeThreads / 32], sa[kMaeThreads / 32];
  const int g = blockIdx.x / b.m, j = blockIdx.x % b.m;
  const Nodes& nd = b.nd[cur];
  const int t = (int)nd.tree[g], len = (int)nd.len[g];
  const int f = b.feat[(size_t)g * b.m + j];
  const uint32_t W = nd.W[g];
  const long long S = nd.S[g];
  const uint32_t* Lf = b.L[cur & 1] + ((size_t)t * b.nl + f) * b.ntr + nd.start[g];
  const uint32_t* Lt = b.L[cur & 1] + ((size_t)t * b.nl + b.p) * b.ntr + nd.start[g];
  const uint32_t* rk = b.grank + (size_t)f * b.n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = kMaeThreads / 32;
  const uint32_t xb = b.extra ? b.xb[(size_t)g * b.m + j] : 0u;
  // stage the node's rows in t order; chunk totals of the feature-ordered segment
  for (int s = threadIdx.x; s < len; s += kMaeThreads) {
    const uint32_t r = Lt[s] & b.rowMask;
    uint32_t wv;
    long long tv;
    mae_row(b, t, r, wv, tv);
    tt[s] = tv;
    tw[s] = (uint8_t)wv;
    trk[s] = rk[r];
  }
  const int nch = (len + 31) >> 5;
  for (int c = warp; c < nch; c += nw) {
    const int i = c * 32 + lane;
    uint32_t wv = 0;
    long long tv = 0;
    if (i < len) mae_row(b, t, Lf[i] & b.rowMask, wv, tv);
    unsigned long long sw = wv, ss = (unsigned long long)((long long)wv * tv);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      sw += __shfl_xor_sync(0xffffffffu, sw, d);
      ss += __shfl_xor_sync(0xffffffffu, ss, d);
    }
    if (lane == 0) cpref[c] = WS2{sw, ss};
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // exclusive prefix over the chunks (<= 384)
    unsigned long long aw = 0, as = 0;
    for (int c = 0; c < nch; ++c) {
      const WS2 v = cpref[c];
      cpref[c] = WS2{aw, as};
      aw += v.w;
      as += v.s;
    }
  }
  __syncthreads();
  unsigned long long bk = 0ull, ba = ~0ull;
  unsigned int nc = 0;
  for (int c = warp; c < nch; c += nw) {
    const int i = c * 32 + lane;
    uint32_t r = 0, wv = 0, rki = 0;
    long long tv = 0;
    if (i < len) {
      r = Lf[i] & b.rowMask;
      mae_row(b, t, r, wv, tv);
      rki = rk[r];
    }
    unsigned long long iw = wv, is = (unsigned long long)((long long)wv * tv);
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned long long yw = __shfl_up_sync(0xffffffffu, iw, d);
      const unsigned long long ys = __shfl_up_sync(0xffffffffu, is, d);
      if (lane >= d) { iw += yw; is += ys; }
    }
    const WS2 cp = cpref[c];
    const uint32_t WL = (uint32_t)(cp.w + iw);
    const long long SL = (long long)(cp.s + is);
    uint32_t rkn = __shfl_down_sync(0xffffffffu, rki, 1);
    if (lane == 31 && i + 1 < len) rkn = rk[Lf[i + 1] & b.rowMask];
    const bool cand = i + 1 < len && (b.extra ? (uint32_t)i == xb : rki != rkn);
    nc += cand ? 1u : 0u;
    // lock-step walk of the staged t-ordered rows for every candidate of the chunk
    LMed mL, mR;
    lmed_init(mL, cand ? WL : 0u);
    lmed_init(mR, cand ? W - WL : 0u);
    for (int s = 0; s < len; ++s) {
      if (((s & 7) == 0) && !__any_sync(0xffffffffu, mL.state != 2 || mR.state != 2)) break;
      const uint32_t rs = trk[s];
      const uint32_t ws = tw[s];
      const long long ts = tt[s];
      if (rs <= rki) lmed_push(mL, ws, ts); else lmed_push(mR, ws, ts);
    }
    if (cand) {
      const uint64_t D = lmed_sad2(mL, SL) + lmed_sad2(mR, S - SL);
      const unsigned long long key = ~D, aux = cand_aux(b, j, f, (unsigned)i);
      if (better(key, aux, bk, ba)) { bk = key; ba = aux; }
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const unsigned long long ok = __shfl_xor_sync(0xffffffffu, bk, d);
    const unsigned long long oa = __shfl_xor_sync(0xffffffffu, ba, d);
    if (better(ok, oa, bk, ba)) { bk = ok; ba = oa; }
  }
  if (lane == 0) { sk[warp] = bk; sa[warp] = ba; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w2 = 1; w2 < nw; ++w2)
      if (better(sk[w2], sa[w2], bk, ba)) { bk = sk[w2]; ba = sa[w2]; }
    if (bk) cas128(&b.best[g], bk, ba);
  }
  if (ncand) {
    unsigned long long v = nc;
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    if (lane == 0 && v) atomicAdd(ncand, v);
  }
}

// After the mark pass: per open node, one walk of its t-ordered rows.  Split node: the weighted
// medians of both children (their leaf values if they are not opened) and, in fit mode with
// importance, SAD2(node) for the decrease (SAD2 - D) 2^(-F-1) (R30, R32); unsplit node: its own
// median (leaf value).
__global__ void k_mae_nodes(Batch b, int cur, int NO) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= NO) return;
  const Nodes& nd = b.nd[cur];
  const int t = (int)nd.tree[g], len = (int)nd.len[g];
  const uint32_t* Lt = b.L[cur & 1] + ((size_t)t * b.nl + b.p) * b.ntr + nd.start[g];
  const Best bs = b.best[g];
  const bool split = bs.key != 0ull;
  LMed mL, mR, mA;
  const uint32_t WL = split ? b.accW[g] : 0u;
  lmed_init(mL, split ? WL : 0u);
  lmed_init(mR, split ? nd.W[g] - WL : 0u);
  lmed_init(mA, (!split || b.imp) ? nd.W[g] : 0u);
  for (int s = 0; s < len; ++s) {
    if (mL.state == 2 && mR.state == 2 && mA.state == 2) break;
    const uint32_t r = Lt[s] & b.rowMask;
    uint32_t wv;
    long long tv;
    mae_row(b, t, r, wv, tv);
    if (split) {
      const bool left = b.sideBits ? ((b.sideBits[(size_t)t * b.nbw + (r >> 5)] >> (r & 31u)) & 1u)
                                   : (b.side[(size_t)t * b.n + r] != 0);
      if (left) lmed_push(mL, wv, tv); else lmed_push(mR, wv, tv);
    }
    lmed_push(mA, wv, tv);
  }
  if (split) {
    b.med2[2 * g] = mL.m2;
    b.med2[2 * g + 1] = mR.m2;
    if (b.imp) {
      const uint64_t D = ~bs.key;
      const int f = (int)(bs.aux >> 32);  // after k_decide: feature << 32 | position
      atomicAdd(&b.imp[(size_t)t * b.p + f], scalbn(__ull2double_rn(lmed_sad2(mA, nd.S[g]) - D), -b.F - 1));
    }
  } else {
    b.med2[2 * g] = mA.m2;
  }
}

// trees whose root is a leaf: the weighted median of all in-bag rows (list p of the root level)
__global__ void k_mae_root(Batch b, const uint32_t* rootInfo) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= b.B || !rootInfo[4 * t + 1]) return;
  const uint32_t* Lt = b.L[0] + ((size_t)t * b.nl + b.p) * b.ntr;
  const uint32_t D = rootInfo[4 * t];
  LMed m;
  lmed_init(m, (uint32_t)b.ntr);
  for (uint32_t s = 0; s < D && m.state != 2; ++s) {
    uint32_t wv;
    long long tv;
    mae_row(b, t, Lt[s] & b.rowMask, wv, tv);
    lmed_push(m, wv, tv);
  }
  b.out[(size_t)t * b.cap].v = scalbn(__ll2double_rn(m.m2), -b.F - 1);
}

__global__ void k_decide(Batch b, int cur, int NO) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= NO) return;
  const Nodes& nd = b.nd[cur];
  const Best bs = b.best[g];
  if (!bs.key) return;
  const int j = (int)((bs.aux >> 48) & 0xFFull), i = (int)(bs.aux & 0xFFFFFFFFull);
  const int t = (int)nd.tree[g], f = b.feat[(size_t)g * b.m + j];
  const uint32_t* L = b.L[cur & 1] + ((size_t)t * b.nl + f) * b.ntr + nd.start[g];
  const uint32_t ra = L[i] & b.rowMask, rb = L[i + 1] & b.rowMask;
  if (b.extra) {  // the drawn threshold of slot j (R29)
    const double lo = b.X[(size_t)(L[0] & b.rowMask) * b.p + f], hi = b.X[(size_t)(L[nd.len[g] - 1] & b.rowMask) * b.p + f];
    b.thr[g] = extra_thr(b.keys[2 * t], b.keys[2 * t + 1], nd.heap[g], j, lo, hi);
  } else {
    b.thr[g] = midpoint_thr(b.X[(size_t)ra * b.p + f], b.X[(size_t)rb * b.p + f]);
  }
  b.thrIdx[g] = b.grank[(size_t)f * b.n + ra];
  b.best[g].aux = ((unsigned long long)f << 32) | (unsigned long long)i;  // slot -> feature for the later kernels
}

// positions (concatenated): go-left flags, child left sums, child constancy
__global__ void k_mark(Batch b, int cur, int NP) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  const Nodes& nd = b.nd[cur];
  int g = -1;
  unsigned int wl = 0;
  unsigned long long sl = 0;
  if (q < NP) {
    g = (int)b.posNode[cur][q];
    const Best bs = b.best[g];
    if (bs.key) {
      const int t = (int)nd.tree[g], f = (int)(bs.aux >> 32), bi = (int)(bs.aux & 0xFFFFFFFFull);
      const int start = (int)nd.start[g];
      const int i = q - (int)b.tPos0[t] - start;
      const uint32_t* L = b.L[cur & 1] + ((size_t)t * b.nl + f) * b.ntr + start;
      const uint32_t r = L[i] & b.rowMask;
      const bool left = i <= bi;
      if (b.sideBits) {
        if (left) atomicOr(&b.sideBits[(size_t)t * b.nbw + (r >> 5)], 1u << (r & 31u));
      } else {
        b.side[(size_t)t * b.n + r] = left ? 1 : 0;
      }
      const long long tv = b.tq[r];
      const long long ref = b.tq[(left ? L[0] : L[bi + 1]) & b.rowMask];
      if (tv != ref) b.nc[2 * g + (left ? 0 : 1)] = 1;
      if (left) {
        wl = b.w[(size_t)t * b.n + r];
        sl = (unsigned long long)((long long)wl * tv);
      }
    } else {
      g = -1;
    }
  }
  // warp-aggregate runs of equal g (positions of a node are contiguous)
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int og = __shfl_down_sync(0xffffffffu, g, d);
    const unsigned int ow = __shfl_down_sync(0xffffffffu, wl, d);
    const unsigned long long os = __shfl_down_sync(0xffffffffu, sl, d);
    if (lane + d < 32 && og == g) { wl += ow; sl += os; }
  }
  const int pg = __shfl_up_sync(0xffffffffu, g, 1);
  if (g >= 0 && (lane == 0 || pg != g)) {
    // wl/sl now hold the run total only for run heads whose run lies in [lane, lane+31]:
    // the doubling above sums lanes l..l+2^k-1 with equal g, which covers the whole run
    if (wl) atomicAdd(&b.accW[g], wl);
    if (sl) atomicAdd(&b.accS[g], sl);
  }
}

// ------------------------------------------------------- histogram mode ----
// 256-bin quantile histograms (R23): cuts per
// (task, feature) from the training rows; bin(x) = #{cuts < x}; per node and
// drawn feature the (W, S) sums per bin are exact integers (order-free atomics);
// the candidate after cut c is valid iff WL > 0 and WR > 0; threshold = cut
// value, threshold index = c; ties -> first drawn feature (R9), then lowest c.
constexpr int kHistThreads = 512;
// rows per histogram work item: nodes longer than one chunk add their chunk histograms with
// global atomics (m x 256 x 2 per chunk), so chunks are long (8192 rows measured 35 % slower per
// row at the top levels of C4, rd2_06)
#ifndef RF_HIST_CHUNK
#define RF_HIST_CHUNK 32768
#endif
constexpr int kHistChunk = RF_HIST_CHUNK;

// Cuts from the task's training rows sorted by x_f (R23), in three kernels over (chunk of
// kCutChunk sorted positions, feature) so the value gathers X[order[j]] use the whole GPU (one
// CTA per feature gathered 640M values with 64 CTAs on C4: 107 ms, rd2_06):
//   k_cut_count    distinct-run starts per chunk
//   k_cut_finish   one CTA per feature: D = number of distinct values; D > 256: the distinct
//                  values among s_{ceil(j ntr / 256) - 1}, j = 1..255, minus the maximum
//   k_cut_collect  D <= 256: all distinct values but the largest, in order, at their offsets
constexpr int kCutChunk = 4096;

__device__ __forceinline__ double sorted_x(const double* __restrict__ X, int p, const uint32_t* __restrict__ o,
                                           int f, long long j) {
  return X[(size_t)o[j] * p + f];
}

__global__ void __launch_bounds__(256) k_cut_count(const double* __restrict__ X, int p,
                                                   const uint32_t* __restrict__ order, int ntr, uint32_t* cnt) {
  const int f = blockIdx.y, ch = blockIdx.x, nch = gridDim.x;
  const uint32_t* o = order + (size_t)f * ntr;
  uint32_t c = 0;
  for (long long j = (long long)ch * kCutChunk + threadIdx.x; j < min((long long)ntr, (long long)(ch + 1) * kCutChunk);
       j += blockDim.x)
    c += (j == 0 || sorted_x(X, p, o, f, j) != sorted_x(X, p, o, f, j - 1)) ? 1u : 0u;
  using BR = cub::BlockReduce<uint32_t, 256>;
  __shared__ typename BR::TempStorage tmp;
  const uint32_t tot = BR(tmp).Sum(c);
  if (threadIdx.x == 0) cnt[(size_t)f * nch + ch] = tot;
}

__global__ void __launch_bounds__(256) k_cut_finish(const double* __restrict__ X, int p,
                                                    const uint32_t* __restrict__ order, int ntr, uint32_t* cnt,
                                                    int nch, double* cuts, int32_t* ncuts) {
  const int f = blockIdx.x;
  const uint32_t* o = order + (size_t)f * ntr;
  uint32_t* cf = cnt + (size_t)f * nch;
  using BS = cub::BlockScan<uint32_t, 256>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ uint32_t carry;
  __shared__ double q[256];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nch; base += 256) {  // exclusive offsets of the chunks' distinct starts
    const int i = base + threadIdx.x;
    const uint32_t v = i < nch ? cf[i] : 0u;
    uint32_t ex, tot;
    BS(tmp).ExclusiveSum(v, ex, tot);
    if (i < nch) cf[i] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  const uint32_t D = carry;
  if (threadIdx.x == 0) cnt[(size_t)p * nch + f] = D;  // read by k_cut_collect
  if (D <= 256) {  // k_cut_collect writes the values
    if (threadIdx.x == 0) ncuts[f] = (int)D - 1;
    return;
  }
  const double vmax = sorted_x(X, p, o, f, ntr - 1);
  const int jq = threadIdx.x + 1;  // 1..255
  if (jq <= 255) q[jq] = sorted_x(X, p, o, f, ((long long)jq * ntr + 255) / 256 - 1);  // ceil(jq ntr / 256) - 1
  __syncthreads();
  if (threadIdx.x == 0) {
    int c = 0;
    double last = 0.0;
    for (int j = 1; j <= 255; ++j) {
      const double v = q[j];
      if (v == vmax || (c > 0 && v == last)) continue;
      cuts[(size_t)f * 256 + c++] = v;
      last = v;
    }
    ncuts[f] = c;
  }
}

__global__ void __launch_bounds__(256) k_cut_collect(const double* __restrict__ X, int p,
                                                     const uint32_t* __restrict__ order, int ntr,
                                                     const uint32_t* __restrict__ off, const int32_t* __restrict__ ncuts,
                                                     double* cuts) {
  const int f = blockIdx.y, ch = blockIdx.x, nch = gridDim.x;
  if (off[(size_t)gridDim.y * nch + f] > 256u) return;  // D > 256: quantile cuts (k_cut_finish)
  const int nc = ncuts[f];
  const uint32_t* o = order + (size_t)f * ntr;
  const long long j0 = (long long)ch * kCutChunk, j1 = min((long long)ntr, j0 + kCutChunk);
  using BS = cub::BlockScan<uint32_t, 256>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = off[(size_t)f * nch + ch];
  __syncthreads();
  for (long long base = j0; base < j1; base += 256) {
    const long long j = base + threadIdx.x;
    uint32_t keep = 0;
    double v = 0.0;
    if (j < j1) {
      v = sorted_x(X, p, o, f, j);
      keep = (j == 0 || v != sorted_x(X, p, o, f, j - 1)) ? 1u : 0u;
    }
    uint32_t ex, tot;
    BS(tmp).ExclusiveSum(keep, ex, tot);
    if (keep && carry + ex < (uint32_t)nc) cuts[(size_t)f * 256 + carry + ex] = v;  // all but the largest
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
}

// bin(x) = #{cuts < x} for every row and feature (row-major [n][p] u8).  The cut tables of a
// group of features are staged in shared memory (8 dependent loads per element from L1/L2 made
// the binary search latency-bound: 120 ms for C4's 640M elements, rd2_07); grid-stride over
// rows, the group's columns per thread.
constexpr int kBinFeat = 16;  // features per shared-memory cut group (16 x 256 x 8 B = 32 KB)

__global__ void __launch_bounds__(256) k_bins(const double* __restrict__ X, int n, int p,
                                              const double* __restrict__ cuts, const int32_t* __restrict__ ncuts,
                                              uint8_t* bins) {
  __shared__ double sc[kBinFeat][256];
  __shared__ int snc[kBinFeat];
  const int f0 = blockIdx.y * kBinFeat, nf = min(kBinFeat, p - f0);
  for (int i = threadIdx.x; i < nf * 256; i += blockDim.x) sc[i >> 8][i & 255] = cuts[(size_t)(f0 + (i >> 8)) * 256 + (i & 255)];
  if (threadIdx.x < nf) snc[threadIdx.x] = ncuts[f0 + threadIdx.x];
  __syncthreads();
  const size_t total = (size_t)n * nf;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const size_t r = e / nf;
    const int fl = (int)(e - r * nf);
    const double x = X[r * p + f0 + fl];
    int lo = 0, hi = snc[fl];  // first index with c[idx] >= x
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (sc[fl][mid] < x) lo = mid + 1; else hi = mid;
    }
    bins[r * p + f0 + fl] = (uint8_t)lo;
  }
}

// bins [n][p] -> binsT [p][n] through 64 x 64 shared tiles (both sides coalesced)
__global__ void __launch_bounds__(256) k_bins_T(const uint8_t* __restrict__ bins, int n, int p, uint8_t* __restrict__ binsT) {
  __shared__ uint8_t tile[64][65];
  const long long r0 = (long long)blockIdx.x * 64;
  const int f0 = blockIdx.y * 64;
  for (int q = threadIdx.x; q < 64 * 64; q += blockDim.x) {
    const int rr = q >> 6, ff = q & 63;
    if (r0 + rr < n && f0 + ff < p) tile[rr][ff] = bins[(size_t)(r0 + rr) * p + f0 + ff];
  }
  __syncthreads();
  for (int q = threadIdx.x; q < 64 * 64; q += blockDim.x) {
    const int ff = q >> 6, rr = q & 63;
    if (r0 + rr < n && f0 + ff < p) binsT[(size_t)(f0 + ff) * n + r0 + rr] = tile[rr][ff];
  }
}

// Work items of the histogram build in row-range-major order: a node's list is in row-id order
// (the training rows, partitioned stably), so chunk c of a node with nch chunks covers about the
// row range [c/nch, (c+1)/nch) of the table.  Items are ordered by bucket k = floor(c kHistK / nch),
// then node, then chunk: the CTAs running at one time read the bin rows of about 1/kHistK of the
// table (40 MB at C4), which stay in L2 for the other trees' nodes instead of coming from DRAM once
// per (tree, node).  Nodes of one chunk (the deep levels) all fall in bucket 0, as before.
// Measured on C4 (rd2_63_ab_c4.txt): histogram search 4,078 ms (K = 1, node-major) -> 4,035 (16)
// -> 4,029 (64): the build is bound by its shared atomics and issue, not by the bin-row reads.
#ifndef RF_HIST_K
#define RF_HIST_K 16
#endif
constexpr int kHistK = RF_HIST_K;

__device__ __forceinline__ uint32_t hist_nch(uint32_t len) { return (len + kHistChunk - 1) / kHistChunk; }

// nch[k * cnt + (g - g0)] = chunks of node g in bucket k (chunks ceil(k nch / K) .. ceil((k+1) nch / K) - 1)
__global__ void k_hist_nchunks(Batch b, int cur, int g0, int g1, uint32_t* nch) {
  const int cnt = g1 - g0;
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= (long long)kHistK * cnt) return;
  const int k = (int)(q / cnt), g = g0 + (int)(q - (long long)k * cnt);
  const uint32_t n = hist_nch(b.nd[cur].len[g]);
  nch[q] = (uint32_t)(((unsigned long long)(k + 1) * n + kHistK - 1) / kHistK -
                      ((unsigned long long)k * n + kHistK - 1) / kHistK);
}

// multi-chunk nodes accumulate with atomics: zero their histograms first
__global__ void k_hist_zero(Batch b, int cur, int g0, int g1, uint32_t* hW, unsigned long long* hS) {
  const int g = g0 + blockIdx.x;
  if (g >= g1 || b.nd[cur].len[g] <= (uint32_t)kHistChunk) return;
  const size_t base = (size_t)(g - g0) * b.m * 256;
  for (int i = threadIdx.x; i < b.m * 256; i += blockDim.x) { hW[base + i] = 0u; hS[base + i] = 0ull; }
}

// work item = (node, chunk of <= kHistChunk rows): shared-memory histograms of the drawn
// features.  A warp takes 32 rows of the chunk at a time: the lanes load the rows' ids,
// weights and targets (coalesced ids, gathered w and t_q) and stage (byte offset of the bin
// row, w, S low word, S high word) in a per-warp shared buffer; then the warp walks the 32 rows
// one by one with the lanes over the drawn features: each step reads the row's record with one
// broadcast 16-byte shared load, lane j reads byte sF[j] of the row's 64-byte bin row (one
// coalesced access per row) and updates feature j's histogram -- the lanes of a warp never hit
// the same counter (no same-address serialisation on low-cardinality features, where a
// row-per-lane layout made whole warps collide).  The sums are kept in 32-bit shared counters
// only: W, and S = w t_q as a (lo, hi) pair whose carry is taken from the returned old lo
// (exact modular 64-bit arithmetic, order free).  A bin's three counters are adjacent, so one
// address serves all three atomics (immediate offsets); 257 bins per feature spread equal low
// bins of different features over different banks.  Measured (profiles/micro, rd2_02): one
// 64-bit shared atomicAdd compiles to a compare-and-swap loop (1.3 pair-updates/clk/SM),
// three 32-bit atomics run 3.0/clk/SM.  (Earlier variants: row per lane with u32 + u64 CAS
// atomics, 18 ms per C4 tree; a warp bitonic sort + segmented sums, 1.8x slower still; the
// per-row shuffles of the record instead of the staged broadcast, 41 instructions per row.)
constexpr int kHistBins = 257;       // bins per feature histogram in shared memory (256 + pad)
#ifndef RF_HIST_AHEAD
#define RF_HIST_AHEAD 16
#endif
constexpr int kHistRowsAhead = RF_HIST_AHEAD;  // bin-row gathers issued before their atomics

__global__ void __launch_bounds__(kHistThreads, 2) k_hist_build(Batch b, int cur, int g0, int g1,
                                                                const uint32_t* itemPref, uint32_t* hW,
                                                                unsigned long long* hS) {
  extern __shared__ __align__(16) uint4 hst[];
  const int m = b.m;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  uint4* stage = hst + warp * 32;                                               // [nwarp][32] row records
  uint32_t* hist = reinterpret_cast<uint32_t*>(hst + nwarp * 32);                // [m][kHistBins][3]
  int* sF = reinterpret_cast<int*>(hist + (size_t)m * kHistBins * 3);           // [m] drawn features
  const int item = blockIdx.x;
  const int cnt = g1 - g0;
  int lo = 0, hi = kHistK * cnt;  // (bucket, node): last index with itemPref[idx] <= item
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if ((int)itemPref[mid] <= item) lo = mid; else hi = mid;
  }
  const int kb = lo / cnt;
  const int g = g0 + (lo - kb * cnt);
  const Nodes& nd = b.nd[cur];
  const int t = (int)nd.tree[g];
  const uint32_t start = nd.start[g], len = nd.len[g];
  const uint32_t c = (uint32_t)(((unsigned long long)kb * hist_nch(len) + kHistK - 1) / kHistK) +
                     (uint32_t)(item - (int)itemPref[lo]);
  const uint32_t i0 = c * kHistChunk, i1 = min(len, i0 + (uint32_t)kHistChunk);
  __shared__ long long sTmin, sTmax;  // t_q range of the chunk's rows (node constancy, R11)
  for (int i = threadIdx.x; i < 3 * m * kHistBins; i += blockDim.x) hist[i] = 0u;
  for (int j = threadIdx.x; j < m; j += blockDim.x) sF[j] = b.feat[(size_t)g * m + j];
  if (threadIdx.x == 0) { sTmin = LLONG_MAX; sTmax = LLONG_MIN; }
  __syncthreads();
  long long tmin = LLONG_MAX, tmax = LLONG_MIN;
  const uint32_t* L = b.L[cur & 1] + (size_t)t * b.ntr + start;
  const uint8_t* w = b.w + (size_t)t * b.n;
  const long long* wt = b.wt ? b.wt + (size_t)t * b.n : nullptr;
  const uint32_t p = (uint32_t)b.p;  // host guarantees n * p < 2^32 (32-bit bin-row offsets)
  const int ngrp = (m + 31) >> 5;    // feature groups of 32 lanes (m <= 73 by the smem limit)
  for (uint32_t base = i0 + 32u * warp; base < i1; base += 32u * nwarp) {
    const uint32_t i = base + lane;
    if (i < i1) {
      const uint32_t r = L[i];
      uint32_t wv;
      long long tv;
      if (wt) {  // one 8-byte gather: (t_q << 8) | w
        const long long pk = wt[r];
        wv = (uint32_t)(pk & 0xFF);
        tv = pk >> 8;
      } else {
        wv = w[r];
        tv = b.tq[r];
      }
      const unsigned long long v = (unsigned long long)((long long)wv * tv);
      stage[lane] = make_uint4(r * p, wv, (uint32_t)v, (uint32_t)(v >> 32));
      tmin = min(tmin, tv);
      tmax = max(tmax, tv);
    }
    __syncwarp();
    const int nk = (int)min(32u, i1 - base);
    for (int gq = 0; gq < ngrp; ++gq) {
      const int j = gq * 32 + lane;
      const bool act = j < m;
      const uint8_t* bcol = b.bins + (act ? sF[j] : 0);
      uint32_t* hj = hist + (size_t)(act ? j : 0) * kHistBins * 3;
      for (int k0 = 0; k0 < nk; k0 += kHistRowsAhead) {
        uint32_t bn[kHistRowsAhead / 4];  // the gathered bins, four per register
#pragma unroll
        for (int q = 0; q < kHistRowsAhead / 4; ++q) bn[q] = 0u;
#pragma unroll
        for (int q = 0; q < kHistRowsAhead; ++q)
          if (act && k0 + q < nk) bn[q >> 2] |= (uint32_t)bcol[stage[k0 + q].x] << (8 * (q & 3));
#pragma unroll
        for (int q = 0; q < kHistRowsAhead; ++q) {
          if (act && k0 + q < nk) {
            const uint4 e = stage[k0 + q];
            uint32_t* cb = hj + 3 * ((bn[q >> 2] >> (8 * (q & 3))) & 0xFFu);
            atomicAdd(cb, e.y);
            const uint32_t old = atomicAdd(cb + 1, e.z);
            const uint32_t add = e.w + (old > ~e.z ? 1u : 0u);  // carry out of the low word
            if (add) atomicAdd(cb + 2, add);
          }
        }
      }
    }
    __syncwarp();  // the records are read before the next batch overwrites them
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    tmin = min(tmin, __shfl_xor_sync(0xffffffffu, tmin, d));
    tmax = max(tmax, __shfl_xor_sync(0xffffffffu, tmax, d));
  }
  if (lane == 0 && tmin != LLONG_MAX) {
    atomicMin(&sTmin, tmin);
    atomicMax(&sTmax, tmax);
  }
  __syncthreads();
  if (threadIdx.x == 0 && sTmin != LLONG_MAX) {
    atomicMin(&b.cmm[4 * g], sTmin);
    atomicMax(&b.cmm[4 * g + 1], sTmax);
  }
  const size_t obase = (size_t)(g - g0) * m * 256;
  const bool single = len <= (uint32_t)kHistChunk;
  for (int idx = threadIdx.x; idx < m * 256; idx += blockDim.x) {
    const int j = idx >> 8, bin = idx & 255;
    const uint32_t* cb = hist + ((size_t)j * kHistBins + bin) * 3;
    const uint32_t Wv = cb[0];
    const unsigned long long Sv = ((unsigned long long)cb[2] << 32) | cb[1];
    if (single) {
      hW[obase + idx] = Wv;
      hS[obase + idx] = Sv;
    } else if (Wv) {
      atomicAdd(&hW[obase + idx], Wv);
      atomicAdd(&hS[obase + idx], Sv);
    }
  }
}

size_t hist_build_smem(int m) {
  return (size_t)(kHistThreads / 32) * 32 * 16 + (size_t)3 * m * kHistBins * 4 + (size_t)m * 4 + 16;
}

// one CTA per node: best cut over the drawn features (warp per feature, 8 bins per lane)
__global__ void __launch_bounds__(256) k_hist_best(Batch b, int cur, int g0, int g1, const uint32_t* hW,
                                                   const unsigned long long* hS, unsigned long long* ncand) {
  const int g = g0 + blockIdx.x;
  if (g >= g1) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Nodes& nd = b.nd[cur];
  const unsigned long long Wt = nd.W[g];
  const long long St = nd.S[g];
  unsigned long long bk = 0ull, ba = ~0ull, bw = 0ull, bs = 0ull;  // best key, aux, left W, left S
  unsigned int nc = 0;
  // constant target (R11; t_q range from k_hist_build): a leaf, no candidate is searched.  The
  // children of a split are opened without a constancy pass (that needed a t_q gather per row);
  // a constant child is recognised here, one level later, with the same leaf value and BFS slot
  const bool constant = b.cmm[4 * g] == b.cmm[4 * g + 1];
  for (int j = constant ? b.m : warp; j < b.m; j += 8) {
    const int f = b.feat[(size_t)g * b.m + j];
    const int ncut = b.ncuts[f];
    const size_t base = ((size_t)(g - g0) * b.m + j) * 256 + 8 * lane;
    uint32_t w8[8];
    unsigned long long s8[8];
    uint32_t lw = 0;
    unsigned long long ls = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      w8[k] = hW[base + k];
      s8[k] = hS[base + k];
      lw += w8[k];
      ls += s8[k];
    }
    uint32_t xw = lw;
    unsigned long long xs = ls;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t yw = __shfl_up_sync(0xffffffffu, xw, d);
      const unsigned long long ys = __shfl_up_sync(0xffffffffu, xs, d);
      if (lane >= d) { xw += yw; xs += ys; }
    }
    unsigned long long cw = xw - lw, cs = xs - ls;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      cw += w8[k];
      cs += s8[k];
      const int cidx = 8 * lane + k;
      if (cidx < ncut && cw > 0 && cw < Wt) {
        const long long SL = (long long)cs;
        const double G = split_gain((long long)cw, SL, (long long)(Wt - cw), St - SL);
        const unsigned long long key = (unsigned long long)__double_as_longlong(G) + 1ull;
        const unsigned long long aux = cand_aux(b, j, f, (unsigned)cidx);  // R9
        ++nc;
        if (better(key, aux, bk, ba)) { bk = key; ba = aux; bw = cw; bs = cs; }
      }
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const unsigned long long ok = __shfl_xor_sync(0xffffffffu, bk, d);
    const unsigned long long oa = __shfl_xor_sync(0xffffffffu, ba, d);
    const unsigned long long ow = __shfl_xor_sync(0xffffffffu, bw, d);
    const unsigned long long os = __shfl_xor_sync(0xffffffffu, bs, d);
    if (better(ok, oa, bk, ba)) { bk = ok; ba = oa; bw = ow; bs = os; }
  }
  __shared__ unsigned long long sk[8], sa[8], sw[8], ss[8];
  if (lane == 0) { sk[warp] = bk; sa[warp] = ba; sw[warp] = bw; ss[warp] = bs; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w2 = 1; w2 < 8; ++w2)
      if (better(sk[w2], sa[w2], bk, ba)) { bk = sk[w2]; ba = sa[w2]; bw = sw[w2]; bs = ss[w2]; }
    b.best[g] = Best{bk, bk ? ba : ~0ull};
    if (bk) {  // the winner's left child sums straight from its histogram prefix (no row pass)
      b.accW[g] = (uint32_t)bw;
      b.accS[g] = bs;
    }
  }
  if (ncand) {
    unsigned long long v = nc;
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    if (lane == 0 && v) atomicAdd(ncand, v);
  }
}

__global__ void k_decide_hist(Batch b, int NO) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= NO) return;
  const Best bs = b.best[g];
  if (!bs.key) return;
  const int j = (int)((bs.aux >> 48) & 0xFFull), c = (int)(bs.aux & 0xFFFFFFFFull);
  const int f = b.feat[(size_t)g * b.m + j];
  b.thr[g] = b.cuts[(size_t)f * 256 + c];
  b.thrIdx[g] = (uint32_t)c;
  b.best[g].aux = ((unsigned long long)f << 32) | (unsigned long long)c;  // slot -> feature
}

__global__ void k_hist_reset(Batch b, int NO) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= NO) return;
  b.accN[g] = 0u;
  b.cmm[4 * g] = LLONG_MAX;
  b.cmm[4 * g + 1] = LLONG_MIN;
  b.cmm[4 * g + 2] = LLONG_MAX;
  b.cmm[4 * g + 3] = LLONG_MIN;
}

__global__ void k_children_count(Batch b, int cur, int NO, int depth) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= NO) return;
  const Nodes& nd = b.nd[cur];
  const Best bs = b.best[g];
  U4S v{0u, 0u, 0u, 0u};
  if (bs.key) {
    // left distinct rows: exact mode = position of the boundary + 1; histogram mode = counted
    const uint32_t nl = b.hist ? b.accN[g] : (uint32_t)(bs.aux & 0xFFFFFFFFull) + 1u;
    const uint32_t lenL = nl, lenR = nd.len[g] - nl;
    const bool capd = (b.max_depth >= 0) && (depth + 1 >= b.max_depth);
    // histogram mode: constancy of a child is found at the next level (k_hist_best)
    const bool ncL = b.hist ? true : (b.nc[2 * g] != 0);
    const bool ncR = b.hist ? true : (b.nc[2 * g + 1] != 0);
    const bool oL = !capd && (int)lenL >= b.mss && ncL;
    const bool oR = !capd && (int)lenR >= b.mss && ncR;
    v.sp = 1u;
    v.op = (oL ? 1u : 0u) + (oR ? 1u : 0u);
    v.pos = (oL ? lenL : 0u) + (oR ? lenR : 0u);
    v.nl = nl;
    b.chFlags[g] = (uint8_t)((oL ? 1u : 0u) | (oR ? 2u : 0u));
  } else {
    b.chFlags[g] = 0;
  }
  b.chVal[g] = v;
}

// per tree: next-level first node / position, BFS base, level count (from scans at tree borders)
__global__ void k_tree_update(Batch b, int NO, uint32_t* nextNode0, uint32_t* nextPos0, uint32_t* nlBase) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > b.B) return;
  const uint32_t g0 = b.tNode0[t];
  const U4S s0 = g0 < (uint32_t)NO ? b.chScan[g0] : U4S{0, 0, 0, 0};
  U4S send;
  if (NO > 0) {
    const U4S last = b.chScan[NO - 1], lv = b.chVal[NO - 1];
    send = U4S{last.sp + lv.sp, last.op + lv.op, last.pos + lv.pos, last.nl + lv.nl};
  } else {
    send = U4S{0, 0, 0, 0};
  }
  const U4S a = g0 < (uint32_t)NO ? s0 : send;
  nextNode0[t] = a.op;
  nextPos0[t] = a.pos;
  nlBase[t] = a.nl;
  if (t < b.B) {
    const uint32_t g1 = b.tNode0[t + 1];
    const U4S e = g1 < (uint32_t)NO ? b.chScan[g1] : send;
    // BFS bookkeeping: next level starts after this level's nodes; it has 2 * splits nodes
    const uint32_t splits = e.sp - a.sp;
    b.tBase[t] += b.tCount[t];
    b.tCount[t] = 2u * splits;
  }
}

__global__ void k_children_write(Batch b, int cur, int NO, const uint32_t* nextNode0, const uint32_t* nextPos0,
                                 const uint32_t* nlBase, int depth) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= NO) return;
  const Nodes& nd = b.nd[cur];
  Nodes& nx = b.nd[cur ^ 1];
  const int t = (int)nd.tree[g];
  Node16* out = b.out + (size_t)t * b.cap;
  uint32_t* outThr = b.outThr + (size_t)t * b.cap;
  const Best bs = b.best[g];
  const uint32_t me = nd.bfs[g];
  if (!bs.key) {  // open node without any candidate split: leaf (R11)
    Node16 l;
    l.feat = -1; l.left = 0;
    l.v = b.mae ? scalbn(__ll2double_rn(b.med2[2 * g]), -b.F - 1)  // weighted median (R32)
                : scalbn(__ddiv_rn(__ll2double_rn(nd.S[g]), __uint2double_rn(nd.W[g])), -b.F);
    out[me] = l;
    outThr[me] = 0;
    return;
  }
  const U4S sc = b.chScan[g], v = b.chVal[g];
  const uint32_t g0 = b.tNode0[t];
  const uint32_t splitRank = sc.sp - b.chScan[g0].sp;
  // tBase/tCount were advanced by k_tree_update: tBase = first BFS id of the next level
  const uint32_t childBase = b.tBase[t] + 2u * splitRank;
  const uint32_t WLv = b.accW[g];
  const int64_t SLv = (int64_t)b.accS[g];
  const uint32_t WRv = nd.W[g] - WLv;
  const int64_t SRv = nd.S[g] - SLv;
  const uint32_t nl = v.nl, lenR = nd.len[g] - nl;
  const bool oL = b.chFlags[g] & 1u, oR = b.chFlags[g] & 2u;
  Node16 me_n;
  me_n.feat = (int32_t)(bs.aux >> 32);
  me_n.left = childBase;
  me_n.v = b.thr[g];
  out[me] = me_n;
  outThr[me] = b.thrIdx[g];
  if (b.imp && !b.mae)  // feature importance (MDI, NEXT-3; MAE: k_mae_nodes)
    atomicAdd(&b.imp[(size_t)t * b.p + me_n.feat], mdi_decrease(WLv, SLv, WRv, SRv, b.F));
  uint32_t oi = sc.op;                             // global open index of the first child
  uint32_t ps = sc.pos - nextPos0[t];              // tree-local position of the first child
  if (oL) {
    nx.tree[oi] = (uint32_t)t; nx.start[oi] = ps; nx.len[oi] = nl; nx.W[oi] = WLv; nx.S[oi] = SLv;
    nx.heap[oi] = 2ull * nd.heap[g]; nx.bfs[oi] = childBase;
    ++oi; ps += nl;
  } else {
    Node16 l; l.feat = -1; l.left = 0;
    l.v = b.mae ? scalbn(__ll2double_rn(b.med2[2 * g]), -b.F - 1)
                : scalbn(__ddiv_rn(__ll2double_rn(SLv), __uint2double_rn(WLv)), -b.F);
    out[childBase] = l; outThr[childBase] = 0;
  }
  if (oR) {
    nx.tree[oi] = (uint32_t)t; nx.start[oi] = ps; nx.len[oi] = lenR; nx.W[oi] = WRv; nx.S[oi] = SRv;
    nx.heap[oi] = 2ull * nd.heap[g] + 1ull; nx.bfs[oi] = childBase + 1;
  } else {
    Node16 l; l.feat = -1; l.left = 0;
    l.v = b.mae ? scalbn(__ll2double_rn(b.med2[2 * g + 1]), -b.F - 1)
                : scalbn(__ddiv_rn(__ll2double_rn(SRv), __uint2double_rn(WRv)), -b.F);
    out[childBase + 1] = l; outThr[childBase + 1] = 0;
  }
  (void)nlBase;
  (void)depth;
}

// Stable partition of every (tree, list) in tiles of kPartTile positions: tile
// counts of go-left rows -> device-wide exclusive scan -> scatter (block scan +
// tile prefix - list's first tile prefix = left rows of this list before the
// element).  tileTab[2t] = first tile of tree t, tileTab[2t+1] = tiles per list.
constexpr int kPartThreads = 256, kPartItems = 8, kPartTile = kPartThreads * kPartItems;

__device__ __forceinline__ void part_locate(const Batch& b, const uint32_t* tileTab, int tile, int& t, int& f,
                                            int& k) {
  int lo = 0, hi = b.B;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if ((int)tileTab[2 * mid] <= tile) lo = mid; else hi = mid;
  }
  t = lo;
  const int rel = tile - (int)tileTab[2 * t], per = (int)tileTab[2 * t + 1];
  f = rel / per;
  k = rel - f * per;
}

__global__ void __launch_bounds__(kPartThreads) k_part_count(Batch b, int cur, const uint32_t* tileTab,
                                                             uint32_t* tileCnt) {
  int t, f, k;
  part_locate(b, tileTab, blockIdx.x, t, f, k);
  const uint32_t pos0 = b.tPos0[t], N = b.tPos0[t + 1] - pos0;
  const uint32_t* L = b.L[cur & 1] + ((size_t)t * b.nl + f) * b.ntr;
  const uint32_t* posNode = b.posNode[cur];
  const uint8_t* side = b.side + (size_t)t * b.n;
  const uint32_t i0 = (uint32_t)k * kPartTile + threadIdx.x * kPartItems;
  uint32_t c = 0;
#pragma unroll
  for (int it = 0; it < kPartItems; ++it) {
    const uint32_t i = i0 + it;
    if (i < N && b.best[posNode[pos0 + i]].key) c += side[L[i] & b.rowMask];
  }
  using BR = cub::BlockReduce<uint32_t, kPartThreads>;
  __shared__ typename BR::TempStorage tmp;
  const uint32_t tot = BR(tmp).Sum(c);
  if (threadIdx.x == 0) tileCnt[blockIdx.x] = tot;
}

// histogram mode, fused into the partition's count pass (a separate go-left pass with per-warp
// global atomics and t_q gathers for the children's constancy was 41 % of a C4 fit, rd2_06:
// every warp of a top-level node hit the same few counters): per tile of kPartTile positions
// of the single row list, the go-left decision bin(x_f) <= cut from the row's bins, the
// decisions as one byte per thread for the scatter, the tile's left count for the scatter's
// scan, and per split node its distinct left rows (per-thread runs, a warp segmented sum, a CTA
// table of the tile's first 32 nodes, one global atomic per node and CTA).  The children's
// (W, S) come from k_hist_best's histogram prefix; their constancy from the next level's build.
// (Launching the count tiles sorted by their node's split feature -- a key kernel + CUB radix sort per
// level -- so that concurrent CTAs gather from few L2-resident bin columns: count 458 -> 428 ms per C4
// fit but the whole fit 5.42 -> 5.70 s, rd2_68_ab_c4.txt; not kept.)
__global__ void __launch_bounds__(kPartThreads) k_part_count_hist(Batch b, int cur, const uint32_t* tileTab,
                                                                  uint32_t* tileCnt, uint8_t* leftBits) {
  int t, f, k;
  part_locate(b, tileTab, blockIdx.x, t, f, k);
  const uint32_t pos0 = b.tPos0[t], N = b.tPos0[t + 1] - pos0;
  const uint32_t* L = b.L[cur & 1] + (size_t)t * b.ntr;
  const uint32_t* posNode = b.posNode[cur];
  __shared__ unsigned int sN[32];
  __shared__ int sG0;
  if (threadIdx.x < 32) sN[threadIdx.x] = 0u;
  const uint32_t tile0 = (uint32_t)k * kPartTile;
  if (threadIdx.x == 0) sG0 = tile0 < N ? (int)posNode[pos0 + tile0] : 0;
  __syncthreads();
  const int g0 = sG0;
  int rg = -1;  // this thread's current run (node) and its left rows
  unsigned int rc = 0;
  auto flush = [&](int g) {  // into the CTA table, or global for nodes beyond it
    if (g < 0 || !rc) return;
    const int sl = g - g0;
    if (sl >= 0 && sl < 32) atomicAdd(&sN[sl], rc);
    else atomicAdd(&b.accN[g], rc);
  };
  uint32_t c = 0, bits = 0;
  const uint32_t i0 = tile0 + threadIdx.x * kPartItems;
  // the thread's loads in three independent rounds (node ids and rows, split rules, bins) so
  // kPartItems gathers of each round are in flight at once
  int gg[kPartItems];
  uint32_t rr[kPartItems], fc[kPartItems];
#pragma unroll
  for (int it = 0; it < kPartItems; ++it) {
    const uint32_t i = i0 + it;
    gg[it] = i < N ? (int)posNode[pos0 + i] : -1;
    rr[it] = i < N ? L[i] : 0u;
  }
#pragma unroll
  for (int it = 0; it < kPartItems; ++it) {
    fc[it] = 0xFFFFFFFFu;  // feature << 16 | cut, or none (unsplit node / past the end)
    if (gg[it] >= 0) {
      const Best bs = b.best[gg[it]];
      if (bs.key) fc[it] = (uint32_t)((bs.aux >> 32) << 16) | (uint32_t)(bs.aux & 0xFFFFull);
    }
  }
#pragma unroll
  for (int it = 0; it < kPartItems; ++it)
    if (fc[it] != 0xFFFFFFFFu)
      bits |= ((uint32_t)(b.binsT ? b.binsT[(size_t)(fc[it] >> 16) * b.n + rr[it]] : b.bins[(size_t)rr[it] * b.p + (fc[it] >> 16)]) <=
                       (fc[it] & 0xFFFFu) ? 1u : 0u) << it;
#pragma unroll
  for (int it = 0; it < kPartItems; ++it) {
    if (fc[it] == 0xFFFFFFFFu) continue;
    const int g = gg[it];
    const bool left = (bits >> it) & 1u;
    if (g != rg) {
      flush(rg);
      rg = g;
      rc = 0;
    }
    rc += left ? 1u : 0u;
    c += left ? 1u : 0u;
  }
  // the threads' last runs: warp segmented sum over equal nodes (positions of a node are
  // contiguous, so equal-node lanes are adjacent), run heads flush
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int og = __shfl_down_sync(0xffffffffu, rg, d);
    const unsigned int oc = __shfl_down_sync(0xffffffffu, rc, d);
    if (lane + d < 32 && og == rg) rc += oc;
  }
  const int pg = __shfl_up_sync(0xffffffffu, rg, 1);
  if (rg >= 0 && (lane == 0 || pg != rg)) flush(rg);
  leftBits[(size_t)blockIdx.x * kPartThreads + threadIdx.x] = (uint8_t)bits;  // read by the scatter
  using BR = cub::BlockReduce<uint32_t, kPartThreads>;
  __shared__ typename BR::TempStorage tmp;
  const uint32_t tot = BR(tmp).Sum(c);
  if (threadIdx.x == 0) tileCnt[blockIdx.x] = tot;
  __syncthreads();
  if (threadIdx.x < 32 && sN[threadIdx.x]) atomicAdd(&b.accN[g0 + (int)threadIdx.x], sN[threadIdx.x]);
}

__global__ void __launch_bounds__(kPartThreads) k_part_scatter(Batch b, int cur, const uint32_t* tileTab,
                                                               const uint32_t* tilePref, const uint32_t* nextPos0,
                                                               const uint32_t* nlBase, int debug_rows,
                                                               const uint8_t* leftBits) {
  int t, f, k;
  part_locate(b, tileTab, blockIdx.x, t, f, k);
  const Nodes& nd = b.nd[cur];
  const uint32_t pos0 = b.tPos0[t], N = b.tPos0[t + 1] - pos0;
  const uint32_t* L = b.L[cur & 1] + ((size_t)t * b.nl + f) * b.ntr;
  uint32_t* L2 = b.L[(cur & 1) ^ 1] + ((size_t)t * b.nl + f) * b.ntr;
  const uint32_t* posNode = b.posNode[cur];
  uint32_t* posNode2 = b.posNode[cur ^ 1];
  const uint8_t* side = b.side + (size_t)t * b.n;
  const uint32_t nlb = nlBase[t];
  const uint32_t npos0 = nextPos0[t];
  const int firstTile = (int)tileTab[2 * t] + f * (int)tileTab[2 * t + 1];
  const uint32_t i0 = (uint32_t)k * kPartTile + threadIdx.x * kPartItems;
  uint32_t rr[kPartItems], gg[kPartItems];
  uint32_t flags = 0, c = 0;  // bit 2it: split node, bit 2it+1: left
  // histogram mode: the go-left bits of this thread's positions from the count pass
  const uint32_t lb8 = leftBits ? leftBits[(size_t)blockIdx.x * kPartThreads + threadIdx.x] : 0u;
#pragma unroll
  for (int it = 0; it < kPartItems; ++it) {
    const uint32_t i = i0 + it;
    rr[it] = 0;
    gg[it] = 0;
    if (i < N) {
      const uint32_t g = posNode[pos0 + i];
      const uint32_t r = L[i];
      gg[it] = g;
      rr[it] = r;
      const Best bs = b.best[g];
      if (bs.key) {
        const uint32_t lf = leftBits ? ((lb8 >> it) & 1u) : side[r & b.rowMask];
        flags |= (1u | (lf << 1)) << (2 * it);
        c += lf;
      }
    }
  }
  using BS = cub::BlockScan<uint32_t, kPartThreads>;
  __shared__ typename BS::TempStorage tmp;
  uint32_t ex;
  BS(tmp).ExclusiveSum(c, ex);
  uint32_t leftBefore = (tilePref[blockIdx.x] - tilePref[firstTile]) + ex;  // left rows of this list before i0
#pragma unroll
  for (int it = 0; it < kPartItems; ++it) {
    const uint32_t i = i0 + it;
    if (i >= N) break;
    const uint32_t g = gg[it], r = rr[it];
    const bool sp = (flags >> (2 * it)) & 1u, left = (flags >> (2 * it + 1)) & 1u;
    if (sp) {
      const U4S sc = b.chScan[g];
      const uint32_t nodeLeftBase = sc.nl - nlb;  // left rows of earlier split nodes of the tree
      const uint32_t within = left ? (leftBefore - nodeLeftBase) : ((i - nd.start[g]) - (leftBefore - nodeLeftBase));
      const uint32_t nl = b.chVal[g].nl;  // distinct rows going left (both split modes)
      const uint32_t fl = b.chFlags[g];
      const bool openL = fl & 1u, openR = fl & 2u;
      if (left ? openL : openR) {
        const uint32_t child = sc.op + ((!left && openL) ? 1u : 0u);
        const uint32_t cstart = (sc.pos - npos0) + ((!left && openL) ? nl : 0u);
        const uint32_t dest = cstart + within;
        L2[dest] = r;
        if (f == 0) posNode2[npos0 + dest] = child;
      } else if (debug_rows && f == 0) {
        const uint32_t cb = b.out[(size_t)t * b.cap + nd.bfs[g]].left;
        b.leaf_of_row[(size_t)t * b.n + (r & b.rowMask)] = (int32_t)(cb + (left ? 0 : 1));
      }
      leftBefore += left;
    } else if (debug_rows && f == 0) {
      b.leaf_of_row[(size_t)t * b.n + (r & b.rowMask)] = (int32_t)nd.bfs[g];
    }
  }
}

// ---- fused multi-list partition (exact and ExtraTrees modes) -------------------
// The per-position split information is list independent, so it is computed once per
// level (k_part_desc) instead of once per (list, position); the go-left flags are one
// bit per row, staged in shared memory per tree (no global gathers); each list is
// streamed once by one warp with a running carry (no count pass, no device-wide scan).

// desc[q] for current position q: x = left rows of the earlier split nodes of the tree
// (leftBefore at the node start, the same in every list), y = node start (tree-local)
// | bit 31 = split, z / w = first next-level position (tree-local) of the left / right
// child or ~0 if that child is not open.
__global__ void k_part_desc(Batch b, int cur, int NP, const uint32_t* __restrict__ nextPos0,
                            const uint32_t* __restrict__ nlBase, uint4* __restrict__ desc) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= NP) return;
  const Nodes& nd = b.nd[cur];
  const uint32_t g = b.posNode[cur][q];
  if (!b.best[g].key) {
    desc[q] = make_uint4(0u, 0u, ~0u, ~0u);
    return;
  }
  const uint32_t t = nd.tree[g];
  const U4S sc = b.chScan[g];
  const uint32_t nl = b.chVal[g].nl, fl = b.chFlags[g];
  const uint32_t cL = sc.pos - nextPos0[t];
  desc[q] = make_uint4(sc.nl - nlBase[t], nd.start[g] | 0x80000000u, (fl & 1u) ? cL : ~0u,
                       (fl & 2u) ? cL + ((fl & 1u) ? nl : 0u) : ~0u);
}

// Warp per list: a CTA of kPWWarps warps shares one tree's go-left bitmap; each warp
// streams one list through the position space 32 x kPWSteps positions at a time (all
// loads of a step issued before use); a ballot gives every element its rank among the
// left rows before it -- no block scans, no barriers after the bitmap load.  (A/B against
// a CTA-per-list-group version with 64-bit block scans over four lists: -22 % time.  Steps of
// 32 positions in flight per warp: 8 beat 4 by 22 % and 16 (C3 partition 88.8 / 113.4 / 139.1 ms,
// profiles/rd2_33_ab_c3.txt, rd2_34_ab_c3.txt); tree-major CTA order measured neutral.)
#ifndef RF_PW_STEPS
#define RF_PW_STEPS 8
#endif
constexpr int kPWWarps = 8, kPWSteps = RF_PW_STEPS;

__global__ void __launch_bounds__(32 * kPWWarps) k_part_lists_warp(Batch b, int cur, const uint4* __restrict__ desc) {
  extern __shared__ uint32_t sbits[];
#ifdef RF_PART_TREE_X
  const int t = blockIdx.x;
  const int f = blockIdx.y * kPWWarps + (threadIdx.x >> 5);
#else
  // the list groups of one tree are adjacent CTAs: they read the tree's descriptors while
  // they are in L2
  const int t = blockIdx.y;
  const int f = blockIdx.x * kPWWarps + (threadIdx.x >> 5);
#endif
  const int lane = threadIdx.x & 31;
  const uint32_t pos0 = b.tPos0[t], N = b.tPos0[t + 1] - pos0;
  if (N == 0) return;
  const uint32_t* gb = b.sideBits + (size_t)t * b.nbw;
  for (int i = threadIdx.x; i < b.nbw; i += blockDim.x) sbits[i] = gb[i];
  __syncthreads();
  if (f >= b.nl) return;
  const uint32_t* Lsrc = b.L[cur & 1] + ((size_t)t * b.nl + f) * b.ntr;
  uint32_t* Ldst = b.L[(cur & 1) ^ 1] + ((size_t)t * b.nl + f) * b.ntr;
  const unsigned lt = (1u << lane) - 1u;
  uint32_t carry = 0;
  for (uint32_t base = 0; base < N; base += 32 * kPWSteps) {
    uint4 d[kPWSteps];
    uint32_t r[kPWSteps];
#pragma unroll
    for (int k = 0; k < kPWSteps; ++k) {
      const uint32_t i = base + 32 * k + lane;
      d[k] = i < N ? desc[pos0 + i] : make_uint4(0u, 0u, ~0u, ~0u);
      r[k] = i < N ? Lsrc[i] : 0u;
    }
#pragma unroll
    for (int k = 0; k < kPWSteps; ++k) {
      const uint32_t i = base + 32 * k + lane;
      const bool sp = (d[k].y >> 31) != 0u;
      const uint32_t row = r[k] & b.rowMask;
      const bool left = sp && ((sbits[row >> 5] >> (row & 31u)) & 1u);
      const unsigned bal = __ballot_sync(0xffffffffu, left);
      const uint32_t lb = carry + (uint32_t)__popc(bal & lt);  // left rows of this list before i
      if (sp) {
        const uint32_t wl = lb - d[k].x;
        const uint32_t dst = left ? d[k].z : d[k].w;
        if (dst != ~0u) Ldst[dst + (left ? wl : (i - (d[k].y & 0x7FFFFFFFu)) - wl)] = r[k];
      }
      carry += (uint32_t)__popc(bal);
    }
  }
}

// next-level position -> node map (one warp per next-level open node)
__global__ void k_fill_posnode(Batch b, int nxt, const uint32_t* __restrict__ counters) {
  const Nodes& nx = b.nd[nxt];
  const uint32_t NOn = counters[0];
  const int lane = threadIdx.x & 31;
  for (uint32_t oi = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; oi < NOn; oi += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t base = b.tPos0[nx.tree[oi]] + nx.start[oi], len = nx.len[oi];
    for (uint32_t i = lane; i < len; i += 32) b.posNode[nxt][base + i] = oi;
  }
}

// debug: leaf of every in-bag row that stops at this level (list 0 order)
__global__ void k_part_debug_rows(Batch b, int cur, int NP) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= NP) return;
  const Nodes& nd = b.nd[cur];
  const uint32_t g = b.posNode[cur][q];
  const uint32_t t = nd.tree[g];
  const uint32_t r = b.L[cur & 1][(size_t)t * b.nl * b.ntr + (q - b.tPos0[t])] & b.rowMask;
  if (!b.best[g].key) {
    b.leaf_of_row[(size_t)t * b.n + r] = (int32_t)nd.bfs[g];
    return;
  }
  const bool left = (b.sideBits[(size_t)t * b.nbw + (r >> 5)] >> (r & 31u)) & 1u;
  const uint32_t fl = b.chFlags[g];
  if (!(left ? (fl & 1u) : (fl & 2u))) {
    const uint32_t cb = b.out[(size_t)t * b.cap + nd.bfs[g]].left;
    b.leaf_of_row[(size_t)t * b.n + r] = (int32_t)(cb + (left ? 0u : 1u));
  }
}

__global__ void k_init_level0(Batch b, const uint32_t* rootInfo, uint32_t* counters /*[2]: NO, NP*/) {
  // single thread: root nodes of non-leaf trees, per-tree position spaces
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  uint32_t no = 0, np = 0;
  for (int t = 0; t < b.B; ++t) {
    b.tNode0[t] = no;
    b.tPos0[t] = np;
    b.tBase[t] = 0;
    b.tCount[t] = 1;
    const uint32_t D = rootInfo[4 * t];
    const bool leaf = rootInfo[4 * t + 1] != 0;
    if (!leaf) {
      Nodes& nd = b.nd[0];
      nd.tree[no] = (uint32_t)t; nd.start[no] = 0; nd.len[no] = D; nd.W[no] = (uint32_t)b.ntr;
      nd.S[no] = reinterpret_cast<const long long*>(rootInfo)[2 * t + 1];
      nd.heap[no] = 1ull; nd.bfs[no] = 0;
      ++no;
      np += D;
    }
  }
  b.tNode0[b.B] = no;
  b.tPos0[b.B] = np;
  counters[0] = no;
  counters[1] = np;
}

__global__ void k_pos_root(Batch b, int NP) {
  // positions of the root level: tree t's positions [tPos0[t], tPos0[t+1]) -> its root node
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= NP) return;
  int lo = 0, hi = b.B;
  while (hi - lo > 1) {
    const int mid = (lo + hi) / 2;
    if ((int)b.tPos0[mid] <= q) lo = mid; else hi = mid;
  }
  b.posNode[0][q] = b.tNode0[lo];
}

__global__ void k_finish_counts(Batch b) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < b.B) b.outCount[t] = b.tBase[t] + b.tCount[t];
}

__global__ void k_set_next_tree_tables(Batch b, const uint32_t* nextNode0, const uint32_t* nextPos0,
                                       uint32_t* counters) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > b.B) return;
  b.tNode0[t] = nextNode0[t];
  b.tPos0[t] = nextPos0[t];
  if (t == b.B) { counters[0] = nextNode0[t]; counters[1] = nextPos0[t]; }
}

}  // namespace

// ============================================================ host driver ====
namespace {

// ordered keys of the training rows' t_q (MAE t-order list): signed -> unsigned order
__global__ void k_tq_keys(const uint32_t* __restrict__ rows, const int64_t* __restrict__ tq, int ntr,
                          unsigned long long* keys) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < ntr) keys[j] = (unsigned long long)tq[rows[j]] ^ 0x8000000000000000ull;
}

__global__ void k_iota(uint32_t* a, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = (uint32_t)i;
}

__global__ void k_root_rows(Batch b, const uint32_t* rootInfo) {
  // leaf_of_row for trees whose root is a leaf: every in-bag row is in leaf 0
  const int t = blockIdx.y;
  if (!rootInfo[4 * t + 1]) return;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < b.ntr; j += gridDim.x * blockDim.x) {
    const uint32_t r = b.tr_rows[j];
    if (b.w[(size_t)t * b.n + r]) b.leaf_of_row[(size_t)t * b.n + r] = 0;
  }
}

inline unsigned nblk(long long n, int t) { return (unsigned)std::max<long long>(1, (n + t - 1) / t); }

#define LCK(expr)                                       \
  do {                                                  \
    cudaError_t _e = (expr);                            \
    if (_e != cudaSuccess) {                            \
      err = std::string("large path: ") + cudaGetErrorString(_e); \
      return _e == cudaErrorMemoryAllocation ? RF_E_OOM : RF_E_CUDA; \
    }                                                   \
  } while (0)

struct LargePlan {
  int B;
  long long nmax, npmax, tiles_max;
};

struct HistBufs {  // histogram mode: per-chunk-of-nodes histograms and work-item prefix
  long long cap = 0;        // nodes per chunk
  uint32_t* W = nullptr;    // [cap][m][256]
  unsigned long long* S = nullptr;
  uint32_t* nch = nullptr;  // [cap + 1]
  uint32_t* pref = nullptr; // [cap + 1]
};

struct PartBufs {  // per-level scratch: search look-back status, partition tiles, root / in-bag setup
  unsigned long long* rootAcc = nullptr;  // [B][4] root statistics accumulators
  uint32_t* ibCnt = nullptr;              // [B nl tiles] in-bag tile counts (long lists)
  uint32_t* ibPref = nullptr;
  uint32_t* tileCtr = nullptr;  // search: next tile id
  TileStat* stat = nullptr;     // search: [tiles_max] published aggregates / prefixes
  uint32_t* flags = nullptr;    // search: [tiles_max] (epoch << 2) | state, zeroed once
  uint32_t* epoch = nullptr;    // host: last search epoch
  uint4* desc = nullptr;     // [npmax] per-position split descriptors (fused path)
  uint32_t* tab = nullptr;   // [2 B]
  uint32_t* cnt = nullptr;   // [max tiles]
  uint8_t* leftBits = nullptr;  // histogram mode: [max tiles][kPartThreads] go-left bits of 8 positions
  uint32_t* pref = nullptr;  // [max tiles]
};

// Grows the batch's trees (slots [0, b.B)) to completion.  hcounters: pinned host
// buffer of >= 4 + 3 (B + 1) words.
rf_status grow_batch(Batch& b, const LargePlan& pl, const uint32_t* task_order, uint64_t seed, int task, int bootstrap,
                     void* cub_tmp, size_t cub_bytes, uint32_t* rootInfo, uint32_t* counters, uint32_t* hcounters,
                     uint32_t* nextNode0, uint32_t* nextPos0, uint32_t* nlBase, WS2* wsTmp, const HistBufs& hb,
                     const PartBufs& pb, unsigned long long* ncand, cudaStream_t s, std::string& err) {
  const size_t plSmem = (size_t)b.nbw * 4;
  std::unique_ptr<ProfScope> setup_scope(new ProfScope("large_tree_setup", s));  // bootstrap, in-bag lists, root statistics
  LCK(cudaMemsetAsync(b.w, 0, (size_t)b.B * b.n, s));
  if (b.side) LCK(cudaMemsetAsync(b.side, 0, (size_t)b.B * b.n, s));
  if (b.leaf_of_row) LCK(cudaMemsetAsync(b.leaf_of_row, 0xFF, (size_t)b.B * b.n * 4, s));
  {
#ifndef RF_BOOT_CTAS
#define RF_BOOT_CTAS 1184
#endif
    // CTAs per tree: blocks are scheduled x-fastest, so RF_BOOT_CTAS = the resident CTAs of the GPU
    // (148 x 8) keeps about one tree's count array (n bytes) hot in L2 at a time for its random
    // atomics: C4 setup 449 -> 208 ms per fit (64 CTAs per tree kept ~18 trees' 10 MB arrays in
    // flight), C3 unchanged (profiles/rd2_61_ab_c4.txt, rd2_61_ab_c3.txt)
    dim3 g(std::min<unsigned>(nblk((b.ntr + 1) / 2, 256), RF_BOOT_CTAS), b.B);
    k_keys_boot<<<g, 256, 0, s>>>(b, seed, task, bootstrap);
    note_launch();
    if (b.wt) {
      k_pack_wt<<<dim3(std::min<unsigned>(nblk(b.ntr, 256), 64), b.B), 256, 0, s>>>(b);
      note_launch();
    }
  }
  const int ibTiles = (b.ntr + kIbTile - 1) / kIbTile;
  if (ibTiles > 1 && pb.ibCnt && (long long)b.B * b.nl < 4 * 148) {
    // few long lists (histogram mode: one list per tree): tiled compaction over all
    // (tree, list, tile); with many lists the one-CTA-per-list kernel fills the GPU already
    // (and measured faster on the C3 shape)
    const int items = b.B * b.nl * ibTiles;
    k_inbag_count<<<items, kIbThreads, 0, s>>>(b, task_order, ibTiles, pb.ibCnt);
    size_t tb = cub_bytes;
    LCK(cub::DeviceScan::ExclusiveSum(cub_tmp, tb, pb.ibCnt, pb.ibPref, items, s));
    k_inbag_scatter<<<items, kIbThreads, 0, s>>>(b, task_order, ibTiles, pb.ibPref);
    note_launch(2);
  } else {
#ifdef RF_INBAG_CTA
    k_inbag_lists<<<b.B * b.nl, kThreads, 0, s>>>(b, task_order);
#else
    k_inbag_lists_warp<<<dim3((unsigned)((b.nl + kIbwWarps - 1) / kIbwWarps), (unsigned)b.B), 32 * kIbwWarps, 0, s>>>(
        b, task_order);
#endif
    note_launch();
  }
  {
    k_root_init<<<nblk(b.B, 128), 128, 0, s>>>(b.B, pb.rootAcc);
    const unsigned cpt = (unsigned)std::min<long long>(std::max<long long>(1, (b.ntr + 8191) / 8192), 256);
    k_root_partial<<<dim3(cpt, (unsigned)b.B), 256, 0, s>>>(b, pb.rootAcc);
    k_root_finish<<<nblk(b.B, 128), 128, 0, s>>>(b, pb.rootAcc, rootInfo);
    note_launch(3);
    if (b.mae) {  // root leaves hold the weighted median (R32)
      k_mae_root<<<nblk(b.B, 64), 64, 0, s>>>(b, rootInfo);
      note_launch();
    }
  }
  if (b.leaf_of_row) {
    k_root_rows<<<dim3(32, b.B), 256, 0, s>>>(b, rootInfo);
    note_launch();
  }
  k_init_level0<<<1, 1, 0, s>>>(b, rootInfo, counters);
  note_launch();
  setup_scope.reset();
  LCK(cudaMemcpyAsync(hcounters, counters, 8, cudaMemcpyDeviceToHost, s));
  uint32_t* htPos0 = hcounters + 4;            // [B + 1] per-tree first positions (host)
  uint32_t* htab = htPos0 + (b.B + 1);         // [2 B] partition tile table (host)
  LCK(cudaMemcpyAsync(htPos0, b.tPos0, (size_t)(b.B + 1) * 4, cudaMemcpyDeviceToHost, s));
  LCK(cudaStreamSynchronize(s));
  long long NO = hcounters[0], NP = hcounters[1];
  if (NP > 0) {
    k_pos_root<<<nblk(NP, 256), 256, 0, s>>>(b, (int)NP);
    note_launch();
  }
  int cur = 0, depth = 0;
  while (NO > 0) {
    note_row_levels(NP);
    // tile table of the tiled partition (per-tree position counts read back at the level start)
    uint32_t tiles = 0;
    if (!b.sideBits) {
      for (int t = 0; t < b.B; ++t) {
        const uint32_t Nt = htPos0[t + 1] - htPos0[t];
        const uint32_t per = (Nt + kPartTile - 1) / kPartTile;
        htab[2 * t] = tiles;
        htab[2 * t + 1] = per ? per : 1u;
        tiles += per * (uint32_t)b.nl;
      }
    }
    k_node_prep<<<nblk(NO, 128), 128, 0, s>>>(b, cur, (int)NO);
    note_launch();
    if (b.extra) {
      k_extra_bounds<<<nblk(NO * b.m, 128), 128, 0, s>>>(b, cur, NO * b.m);
      note_launch();
    }
    size_t tb = cub_bytes;
    if (!b.hist) {
      k_node_ws<<<nblk(NO, 256), 256, 0, s>>>(b, cur, (int)NO, wsTmp);
      note_launch();
      LCK(cub::DeviceScan::ExclusiveScan(cub_tmp, tb, wsTmp, b.nodePref, WS2Sum(), WS2{0ull, 0ull}, (int)NO, s));
      const long long E = (long long)b.m * NP;
      if (b.mae) {
        ProfScope ps("large_mae_search", s);
        k_mae_search<<<(unsigned)(NO * b.m), kMaeThreads, mae_search_smem(0), s>>>(b, cur, ncand);
        note_launch();
      } else {
        ProfScope ps("large_search", s);
        const uint32_t epoch = ++*pb.epoch;
        LCK(cudaMemsetAsync(pb.tileCtr, 0, 4, s));
        const long long tiles = (E + kTile - 1) / kTile;
        k_search_fused<<<(unsigned)tiles, kThreads, 0, s>>>(b, cur, E, ncand, pb.tileCtr, pb.stat, pb.flags, epoch);
        note_launch();
      }
      k_decide<<<nblk(NO, 128), 128, 0, s>>>(b, cur, (int)NO);
      if (b.sideBits) LCK(cudaMemsetAsync(b.sideBits, 0, (size_t)b.B * b.nbw * 4, s));
      k_mark<<<nblk(NP, 256), 256, 0, s>>>(b, cur, (int)NP);
      note_launch(2);
      if (b.mae) {  // children's medians / own median, MAE importance
        k_mae_nodes<<<nblk(NO, 64), 64, 0, s>>>(b, cur, (int)NO);
        note_launch();
      }
    } else {
      k_hist_reset<<<nblk(NO, 256), 256, 0, s>>>(b, (int)NO);
      note_launch();
      const size_t hsm = hist_build_smem(b.m);
      {
        ProfScope ps("hist_search", s);
        for (long long g0 = 0; g0 < NO; g0 += hb.cap) {
          const long long g1 = std::min<long long>(NO, g0 + hb.cap);
          const int cnt = (int)(g1 - g0);
          k_hist_nchunks<<<nblk((long long)kHistK * cnt, 256), 256, 0, s>>>(b, cur, (int)g0, (int)g1, hb.nch);
          note_launch();
          tb = cub_bytes;
          LCK(cub::DeviceScan::ExclusiveSum(cub_tmp, tb, hb.nch, hb.pref, kHistK * cnt + 1, s));
          uint32_t items = 0;
          LCK(cudaMemcpyAsync(&items, hb.pref + (size_t)kHistK * cnt, 4, cudaMemcpyDeviceToHost, s));
          LCK(cudaStreamSynchronize(s));
          k_hist_zero<<<cnt, 256, 0, s>>>(b, cur, (int)g0, (int)g1, hb.W, hb.S);
          k_hist_build<<<items, kHistThreads, hsm, s>>>(b, cur, (int)g0, (int)g1, hb.pref, hb.W, hb.S);
          k_hist_best<<<cnt, 256, 0, s>>>(b, cur, (int)g0, (int)g1, hb.W, hb.S, ncand);
          note_launch(3);
        }
      }
      k_decide_hist<<<nblk(NO, 128), 128, 0, s>>>(b, (int)NO);
      note_launch();
      // partition count pass, fused with the children's row counts and constancy (k_part_count_hist)
      ProfScope pm("hist_count", s);
      if (tiles > 0) {
        LCK(cudaMemcpyAsync(pb.tab, htab, (size_t)2 * b.B * 4, cudaMemcpyHostToDevice, s));
        k_part_count_hist<<<tiles, kPartThreads, 0, s>>>(b, cur, pb.tab, pb.cnt, pb.leftBits);
        note_launch();
      }
    }
    std::unique_ptr<ProfScope> ch_scope(new ProfScope("large_children", s));
    k_children_count<<<nblk(NO, 128), 128, 0, s>>>(b, cur, (int)NO, depth);
    note_launch();
    tb = cub_bytes;
    LCK(cub::DeviceScan::ExclusiveScan(cub_tmp, tb, b.chVal, b.chScan, U4Sum(), U4S{0u, 0u, 0u, 0u}, (int)NO, s));
    k_tree_update<<<nblk(b.B + 1, 64), 64, 0, s>>>(b, (int)NO, nextNode0, nextPos0, nlBase);
    k_children_write<<<nblk(NO, 128), 128, 0, s>>>(b, cur, (int)NO, nextNode0, nextPos0, nlBase, depth);
    note_launch(2);
    ch_scope.reset();
    if (b.sideBits) {
      ProfScope ps("large_partition", s);
      k_part_desc<<<nblk(NP, 256), 256, 0, s>>>(b, cur, (int)NP, nextPos0, nlBase, pb.desc);
      note_launch();
      if (b.leaf_of_row) {
        k_part_debug_rows<<<nblk(NP, 256), 256, 0, s>>>(b, cur, (int)NP);
        note_launch();
      }
#ifdef RF_PART_TREE_X
      k_part_lists_warp<<<dim3((unsigned)b.B, (unsigned)((b.nl + kPWWarps - 1) / kPWWarps)), 32 * kPWWarps, plSmem, s>>>(
          b, cur, pb.desc);
#else
      k_part_lists_warp<<<dim3((unsigned)((b.nl + kPWWarps - 1) / kPWWarps), (unsigned)b.B), 32 * kPWWarps, plSmem, s>>>(
          b, cur, pb.desc);
#endif
      note_launch();
    } else {
      ProfScope ps("large_partition", s);
      if (tiles > 0) {
        if (!b.hist) {  // (histogram mode: counted above, k_part_count_hist)
          LCK(cudaMemcpyAsync(pb.tab, htab, (size_t)2 * b.B * 4, cudaMemcpyHostToDevice, s));
          k_part_count<<<tiles, kPartThreads, 0, s>>>(b, cur, pb.tab, pb.cnt);
          note_launch();
        }
        tb = cub_bytes;
        LCK(cub::DeviceScan::ExclusiveSum(cub_tmp, tb, pb.cnt, pb.pref, (int)tiles, s));
        k_part_scatter<<<tiles, kPartThreads, 0, s>>>(b, cur, pb.tab, pb.pref, nextPos0, nlBase,
                                                       b.leaf_of_row ? 1 : 0, b.hist ? pb.leftBits : nullptr);
        note_launch();
      }
    }
    k_set_next_tree_tables<<<nblk(b.B + 1, 64), 64, 0, s>>>(b, nextNode0, nextPos0, counters);
    note_launch();
    if (b.sideBits) {  // next-level position -> node map (the fused partition does not write it)
      k_fill_posnode<<<std::min<unsigned>(nblk(2 * NO * 32, 256), 148 * 16), 256, 0, s>>>(b, cur ^ 1, counters);
      note_launch();
    }
    LCK(cudaMemcpyAsync(hcounters, counters, 8, cudaMemcpyDeviceToHost, s));
    LCK(cudaMemcpyAsync(htPos0, b.tPos0, (size_t)(b.B + 1) * 4, cudaMemcpyDeviceToHost, s));
    LCK(cudaStreamSynchronize(s));
    NO = hcounters[0];
    NP = hcounters[1];
    if (NO > pl.nmax || NP > pl.npmax) {
      err = "large path: level size exceeds the plan";
      return RF_E_OVERFLOW;
    }
    cur ^= 1;
    ++depth;
  }
  k_finish_counts<<<nblk(b.B, 64), 64, 0, s>>>(b);
  note_launch();
  return RF_OK;
}

}  // namespace

namespace {

// one CTA per feature: the dataset order filtered to a task's training rows (global ids)
__global__ void k_task_order_u32(const uint32_t* __restrict__ order, const int32_t* __restrict__ loc, int n,
                                 int ntr, uint32_t* out) {
  const int f = blockIdx.x;
  using BS = cub::BlockScan<uint32_t, 256>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < n; base += 256) {
    const int j = base + threadIdx.x;
    uint32_t r = 0, keep = 0;
    if (j < n) { r = order[(size_t)f * n + j]; keep = loc[r] >= 0; }
    uint32_t ex, tot;
    BS(tmp).ExclusiveSum(keep, ex, tot);
    if (keep) out[(size_t)f * ntr + carry + ex] = r;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
}

// per (test row, tree chunk): sum of the leaf values of the chunk's trees, trees in order
__global__ void k_chunk_predict(const Node16* __restrict__ nodes, uint64_t cap, int T, int Cw, int nsub,
                                const double* __restrict__ X, int p, const uint32_t* __restrict__ te_rows, int nte,
                                int nte_max, double* __restrict__ partial) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nte * nsub) return;
  const int r = idx % nte, c = idx / nte;
  const double* x = X + (size_t)te_rows[r] * p;
  double s = 0.0;
  for (int t = c * Cw; t < min(T, (c + 1) * Cw); ++t) {
    const Node16* tn = nodes + (size_t)t * cap;
    Node16 nd = tn[0];
    while (nd.feat >= 0) nd = tn[nd.left + ((x[nd.feat] <= nd.v) ? 0u : 1u)];
    s += nd.v;
  }
  partial[(size_t)c * nte_max + r] = s;
}

}  // namespace

int g_opt_tiled_partition = 0;
long long g_opt_hist_node_cap = 0;

static rf_status grow_forest(const DevData& d, const rf_params* prm, int mtry, int tree_lo, int tree_hi,
                             int task, const uint32_t* tr_rows_in, int ntr, const uint32_t* task_order,
                             cudaStream_t s, Scratch& sc, Node16** nodes_out, uint32_t** thr_out,
                             uint32_t** nn_out, uint64_t* cap_out, int32_t* leaf_of_row, double* imp, std::string& err);

rf_status fit_large(const DevData& d, const rf_params* prm, int mtry, int tree_lo, int tree_hi, cudaStream_t s,
                    Scratch& sc, Node16** nodes_out, uint32_t** thr_out, uint32_t** nn_out, uint64_t* cap_out,
                    int32_t* leaf_of_row, double* imp, std::string& err) {
  uint32_t* tr_rows;
  LCK(sc.alloc(&tr_rows, (size_t)d.n));
  k_iota<<<nblk(d.n, 256) > 1184 ? 1184 : nblk(d.n, 256), 256, 0, s>>>(tr_rows, d.n);
  note_launch();
  return grow_forest(d, prm, mtry, tree_lo, tree_hi, 0, tr_rows, d.n, d.order, s, sc, nodes_out, thr_out, nn_out,
                     cap_out, leaf_of_row, imp, err);
}

rf_status cv_large_partial(const DevData& d, const TaskData& td, const rf_params* prm,
                           const std::vector<int>& mtrys, int tree_lo, int tree_hi, int Cw, int nsub,
                           int nte_max, double* partial, cudaStream_t s, Scratch& sc, std::string& err) {
  const int T = tree_hi - tree_lo;
  const int ntask = td.ntask;
  std::vector<int32_t> hntr(ntask), hnte(ntask);
  LCK(cudaMemcpyAsync(hntr.data(), td.ntr, ntask * 4, cudaMemcpyDeviceToHost, s));
  LCK(cudaMemcpyAsync(hnte.data(), td.nte, ntask * 4, cudaMemcpyDeviceToHost, s));
  LCK(cudaStreamSynchronize(s));
  for (int tl = 0; tl < ntask; ++tl) {
    const int ntr = hntr[tl], nte = hnte[tl];
    Scratch ts(s);
    uint32_t* order;
    LCK(ts.alloc(&order, (size_t)d.p * ntr));
    k_task_order_u32<<<d.p, 256, 0, s>>>(d.order, td.loc + (size_t)tl * d.n, d.n, ntr, order);
    note_launch();
    for (size_t mi = 0; mi < mtrys.size(); ++mi) {
      Scratch fs(s);
      Node16* nodes;
      uint32_t *thr, *nn;
      uint64_t cap;
      rf_status st = grow_forest(d, prm, mtrys[mi], tree_lo, tree_hi, td.task0 + tl,
                                 td.tr_rows + (size_t)tl * d.n, ntr, order, s, fs, &nodes, &thr, &nn, &cap, nullptr,
                                 nullptr, err);
      if (st) return st;
      double* part = partial + ((size_t)mi * ntask + tl) * nsub * nte_max;
      const long long nth = (long long)nte * nsub;
      k_chunk_predict<<<nblk(nth, 128), 128, 0, s>>>(nodes, cap, T, Cw, nsub, d.X, d.p,
                                                     td.te_rows + (size_t)tl * d.n, nte, nte_max, part);
      note_launch();
    }
  }
  return RF_OK;
}

static rf_status grow_forest(const DevData& d, const rf_params* prm, int mtry, int tree_lo, int tree_hi,
                             int task, const uint32_t* tr_rows_in, int ntr, const uint32_t* task_order,
                             cudaStream_t s, Scratch& sc, Node16** nodes_out, uint32_t** thr_out,
                             uint32_t** nn_out, uint64_t* cap_out, int32_t* leaf_of_row, double* imp, std::string& err) {
  if (d.p > 255) {
    err = "large path: p <= 255";
    return RF_E_UNSUPPORTED;
  }
  const bool hist = prm->split_mode == RF_SPLIT_HIST256;
  const bool extra = prm->split_mode == RF_SPLIT_EXTRA;
  const bool mae = prm->criterion == RF_CRITERION_MAE;
  const int n = d.n, p = d.p, T = tree_hi - tree_lo;
  if (mae && (hist || ntr > kMaeMaxLen)) {
    err = "MAE criterion on the level-synchronous path: exact and ExtraTrees modes, training sets of <= 12288 rows (R32)";
    return RF_E_UNSUPPORTED;
  }
  const int nlists = hist ? 1 : p + (mae ? 1 : 0);  // MAE: list p = in-bag rows in t_q order
  uint64_t cap = 2ull * (uint64_t)ntr - 1ull;
  if (prm->max_depth >= 0 && prm->max_depth < 40) cap = std::min<uint64_t>(cap, (2ull << prm->max_depth) - 1ull);
  // open nodes per level per tree <= min(ntr / 2, 2^(max_depth - 1))
  long long open_max = ntr / 2 + 1;
  if (prm->max_depth >= 1 && prm->max_depth < 31) open_max = std::min<long long>(open_max, 1ll << (prm->max_depth - 1));
  // batch size: the row lists dominate (2 lists-per-tree x ntr x 4 B per tree)
  const size_t per_tree = (size_t)2 * nlists * ntr * 4 + (size_t)ntr * 8 + (size_t)n * 2 +
                          (size_t)open_max * (128 + (extra ? 4 * (size_t)mtry : 0));
  // trees per batch: per-level launch and sync costs are shared by the batch, so batches are
  // as large as the working-set budget allows (of the 180 GB HBM)
#ifndef RF_LARGE_BMAX
#define RF_LARGE_BMAX 512
#endif
#ifndef RF_LARGE_BUDGET_GB
#define RF_LARGE_BUDGET_GB 32
#endif
  int B = (int)std::max<size_t>(
      1, std::min<size_t>(RF_LARGE_BMAX, ((size_t)RF_LARGE_BUDGET_GB << 30) / std::max<size_t>(per_tree, 1)));
  B = std::min(B, (int)std::min<long long>(INT_MAX, (long long)INT_MAX / std::max(ntr, 1)));  // positions: int
  B = std::min(B, T);
  B = (T + (T + B - 1) / B - 1) / ((T + B - 1) / B);  // equal batches (the same count of batches)
  LargePlan pl;
  pl.B = B;
  pl.nmax = (long long)B * open_max;
  pl.npmax = (long long)B * ntr;
  pl.tiles_max = hist ? 1 : ((long long)mtry * pl.npmax + kTile - 1) / kTile;

  Batch b;
  memset(&b, 0, sizeof b);
  b.B = B; b.n = n; b.p = p; b.m = mtry; b.ntr = ntr; b.mss = (int)prm->min_samples_split;
  b.max_depth = prm->max_depth;
  b.X = d.X; b.tq = d.tq; b.grank = d.grank; b.err = d.err;
  b.nl = nlists;
  b.packRank = (!hist && n <= (1 << 17)) ? 1 : 0;
  b.rowMask = b.packRank ? 0x1FFFFu : 0xFFFFFFFFu;
  if (b.packRank) {
    uint32_t* maxr;
    uint8_t* rfit;
    LCK(sc.alloc(&maxr, (size_t)p));
    LCK(sc.alloc(&rfit, (size_t)p));
    LCK(cudaMemsetAsync(maxr, 0, (size_t)p * 4, s));
    k_rank_fit<<<dim3(std::min<unsigned>(nblk(n, 256), 64), (unsigned)p), 256, 0, s>>>(d.grank, n, p, maxr, rfit, 0);
    k_rank_fit<<<dim3(1, (unsigned)p), 32, 0, s>>>(d.grank, n, p, maxr, rfit, 1);
    note_launch(2);
    b.rfit = rfit;
  }
  b.hist = hist ? 1 : 0;
  b.extra = extra ? 1 : 0;
  b.tie_draw = prm->tie_break == RF_TIE_DRAW_ORDER ? 1 : 0;
  b.mae = mae ? 1 : 0;
  if (extra) LCK(sc.alloc(&b.xb, (size_t)pl.nmax * mtry));
  HistBufs hb;
  const uint32_t* list_src = task_order;
  if (mae) {
    // per-task list sources [p + 1][ntr]: the p feature orders and the training rows in
    // (t_q, row) order (a stable radix sort of the ascending rows by their ordered t_q)
    uint32_t* src;
    unsigned long long *kin, *kout;
    LCK(sc.alloc(&src, (size_t)(p + 1) * ntr));
    LCK(sc.alloc(&kin, (size_t)ntr));
    LCK(sc.alloc(&kout, (size_t)ntr));
    LCK(cudaMemcpyAsync(src, task_order, (size_t)p * ntr * 4, cudaMemcpyDeviceToDevice, s));
    k_tq_keys<<<nblk(ntr, 256), 256, 0, s>>>(tr_rows_in, d.tq, ntr, kin);
    note_launch();
    size_t tb = 0;
    LCK(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, kout, tr_rows_in, src + (size_t)p * ntr, ntr, 0, 64, s));
    char* tmp;
    LCK(sc.alloc(&tmp, tb + 16));
    LCK(cub::DeviceRadixSort::SortPairs(tmp, tb, kin, kout, tr_rows_in, src + (size_t)p * ntr, ntr, 0, 64, s));
    list_src = src;
    LCK(allow_max_dynamic_smem(k_mae_search));
  }
  if (hist) {
    // cuts of this task's training rows (R23) and the bins of every row
    double* cuts;
    int32_t* ncuts;
    uint8_t* bins;
    LCK(sc.alloc(&cuts, (size_t)p * 256));
    LCK(sc.alloc(&ncuts, (size_t)p));
    LCK(sc.alloc(&bins, (size_t)n * p));
    uint8_t* binsT = nullptr;
    {
      ProfScope ps("hist_binning", s);
      const int nch = (ntr + kCutChunk - 1) / kCutChunk;
      uint32_t* ccnt;
      LCK(sc.alloc(&ccnt, (size_t)nch * p + p));  // chunk counts -> offsets, then D per feature
      k_cut_count<<<dim3((unsigned)nch, (unsigned)p), 256, 0, s>>>(d.X, p, task_order, ntr, ccnt);
      k_cut_finish<<<p, 256, 0, s>>>(d.X, p, task_order, ntr, ccnt, nch, cuts, ncuts);
      k_cut_collect<<<dim3((unsigned)nch, (unsigned)p), 256, 0, s>>>(d.X, p, task_order, ntr, ccnt, ncuts, cuts);
      note_launch(2);
      k_bins<<<dim3(std::min<unsigned>(nblk((long long)n * kBinFeat, 256), 148 * 8), (unsigned)((p + kBinFeat - 1) / kBinFeat)),
               256, 0, s>>>(d.X, n, p, cuts, ncuts, bins);
      note_launch(2);
#ifndef RF_NO_BINST
      LCK(sc.alloc(&binsT, (size_t)n * p));
      k_bins_T<<<dim3((unsigned)((n + 63) / 64), (unsigned)((p + 63) / 64)), 256, 0, s>>>(bins, n, p, binsT);
      note_launch();
#endif
    }
    b.cuts = cuts;
    b.ncuts = ncuts;
    b.bins = bins;
    b.binsT = binsT;
    LCK(sc.alloc(&b.accN, (size_t)pl.nmax));
    LCK(sc.alloc(&b.cmm, (size_t)pl.nmax * 4));
    hb.cap = std::max<long long>(1, std::min<long long>(pl.nmax, ((long long)2 << 30) / ((long long)mtry * 256 * 12)));
    if (g_opt_hist_node_cap > 0) hb.cap = std::min<long long>(hb.cap, g_opt_hist_node_cap);  // test switch
    LCK(sc.alloc(&hb.W, (size_t)hb.cap * mtry * 256));
    LCK(sc.alloc(&hb.S, (size_t)hb.cap * mtry * 256));
    LCK(sc.alloc(&hb.nch, (size_t)kHistK * hb.cap + 1));
    LCK(sc.alloc(&hb.pref, (size_t)kHistK * hb.cap + 1));
    LCK(cudaMemsetAsync(hb.nch, 0, ((size_t)kHistK * hb.cap + 1) * 4, s));
    const size_t hsm = hist_build_smem(mtry);
    if ((uint64_t)n * (uint64_t)p >= (1ull << 32)) {
      err = "histogram mode: n * p must be < 2^32 (32-bit bin-row offsets)";
      return RF_E_UNSUPPORTED;
    }
    if (hsm > 227 * 1024) {
      err = "histogram mode: mtry too large for the shared-memory staging of the drawn bins";
      return RF_E_UNSUPPORTED;
    }
    LCK(allow_max_dynamic_smem(k_hist_build));
    list_src = tr_rows_in;  // one node-grouped list of training rows
  }
  int32_t hF = 0;
  LCK(cudaMemcpyAsync(&hF, d.F, 4, cudaMemcpyDeviceToHost, s));
  LCK(cudaStreamSynchronize(s));
  b.F = hF;
  b.tr_rows = tr_rows_in;
  LCK(sc.alloc(&b.keys, (size_t)2 * B));
  LCK(sc.alloc(&b.w, (size_t)B * n + 4));
#ifndef RF_NO_WT
  if (n > 256) LCK(sc.alloc(&b.wt, (size_t)B * n));  // packed (t_q << 8) | w gathers
#endif
  if (!hist) LCK(sc.alloc(&b.side, (size_t)B * n));  // histogram mode decides from the bins
  // fused partition path (exact / ExtraTrees): go-left bits per row, staged per tree in
  // shared memory by the partition CTAs (n <= 2^20 rows: <= 128 KB)
  b.nbw = (n + 31) / 32;
  const bool fused_part = !hist && n <= (1 << 20) && !g_opt_tiled_partition;
  if (fused_part) LCK(sc.alloc(&b.sideBits, (size_t)B * b.nbw));
  for (int i = 0; i < 2; ++i) {
    LCK(sc.alloc(&b.L[i], (size_t)B * nlists * ntr));
    LCK(sc.alloc(&b.posNode[i], (size_t)pl.npmax));
    Nodes& nd = b.nd[i];
    LCK(sc.alloc(&nd.tree, (size_t)pl.nmax));
    LCK(sc.alloc(&nd.start, (size_t)pl.nmax));
    LCK(sc.alloc(&nd.len, (size_t)pl.nmax));
    LCK(sc.alloc(&nd.W, (size_t)pl.nmax));
    LCK(sc.alloc(&nd.S, (size_t)pl.nmax));
    LCK(sc.alloc(&nd.heap, (size_t)pl.nmax));
    LCK(sc.alloc(&nd.bfs, (size_t)pl.nmax));
  }
  LCK(sc.alloc(&b.feat, (size_t)pl.nmax * mtry));
  if (mae) LCK(sc.alloc(&b.med2, (size_t)pl.nmax * 2));
  LCK(sc.alloc(&b.best, (size_t)pl.nmax));
  LCK(sc.alloc(&b.accW, (size_t)pl.nmax));
  LCK(sc.alloc(&b.accS, (size_t)pl.nmax));
  LCK(sc.alloc(&b.nc, (size_t)pl.nmax * 2));
  LCK(sc.alloc(&b.thr, (size_t)pl.nmax));
  LCK(sc.alloc(&b.thrIdx, (size_t)pl.nmax));
  LCK(sc.alloc(&b.nodePref, (size_t)pl.nmax));
  LCK(sc.alloc(&b.chScan, (size_t)pl.nmax));
  LCK(sc.alloc(&b.chVal, (size_t)pl.nmax));
  LCK(sc.alloc(&b.chFlags, (size_t)pl.nmax));
  LCK(sc.alloc(&b.tNode0, (size_t)B + 1));
  LCK(sc.alloc(&b.tPos0, (size_t)B + 1));
  LCK(sc.alloc(&b.tBase, (size_t)B));
  LCK(sc.alloc(&b.tCount, (size_t)B));
  WS2* wsTmp;
  LCK(sc.alloc(&wsTmp, (size_t)pl.nmax));
  uint32_t *rootInfo, *counters, *nextNode0, *nextPos0, *nlBase;
  LCK(sc.alloc(&rootInfo, (size_t)4 * B));
  LCK(sc.alloc(&counters, 2));
  LCK(sc.alloc(&nextNode0, (size_t)B + 1));
  LCK(sc.alloc(&nextPos0, (size_t)B + 1));
  LCK(sc.alloc(&nlBase, (size_t)B + 1));
  uint32_t* hcounters = nullptr;
  // pinned level counters: one grow-only buffer per host thread (cudaMallocHost / cudaFreeHost
  // per fit stalled the host for up to hundreds of ms, rd2_24_c3wall.txt)
  {
    static thread_local uint32_t* tl_buf = nullptr;
    static thread_local size_t tl_words = 0;
    const size_t need = (size_t)(4 + 3 * (B + 1));
    if (tl_words < need) {
      if (tl_buf) cudaFreeHost(tl_buf);
      tl_buf = nullptr;
      tl_words = 0;
      LCK(cudaMallocHost(&tl_buf, need * 4));
      tl_words = need;
    }
    hcounters = tl_buf;
  }
  PartBufs pbufs;
  const long long max_tiles = (long long)nlists * (B + pl.npmax / kPartTile + 1) + 1;
  LCK(sc.alloc(&pbufs.tab, (size_t)2 * B));
  LCK(sc.alloc(&pbufs.rootAcc, (size_t)4 * B));
  const long long ibItems = (long long)B * nlists * ((ntr + kIbTile - 1) / kIbTile);
  if ((ntr + kIbTile - 1) / kIbTile > 1 && (long long)B * nlists < 4 * 148) {
    LCK(sc.alloc(&pbufs.ibCnt, (size_t)ibItems));
    LCK(sc.alloc(&pbufs.ibPref, (size_t)ibItems));
  }
  uint32_t search_epoch = 0;
  pbufs.epoch = &search_epoch;
  LCK(sc.alloc(&pbufs.tileCtr, 1));
  LCK(sc.alloc(&pbufs.stat, (size_t)pl.tiles_max + 1));
  LCK(sc.alloc(&pbufs.flags, (size_t)pl.tiles_max + 1));
  LCK(cudaMemsetAsync(pbufs.flags, 0, ((size_t)pl.tiles_max + 1) * 4, s));
  if (fused_part) {
    LCK(sc.alloc(&pbufs.desc, (size_t)pl.npmax));
    LCK(allow_max_dynamic_smem(k_part_lists_warp));
  }
  LCK(sc.alloc(&pbufs.cnt, (size_t)max_tiles));
  if (hist) LCK(sc.alloc(&pbufs.leftBits, (size_t)max_tiles * kPartThreads));
  LCK(sc.alloc(&pbufs.pref, (size_t)max_tiles));
  // CUB temp storage for the largest scan
  size_t cb1 = 0, cb2 = 0, cb3 = 0;
  cub::DeviceScan::ExclusiveScan(nullptr, cb1, wsTmp, b.nodePref, WS2Sum(), WS2{0ull, 0ull}, (int)pl.nmax, s);
  cub::DeviceScan::ExclusiveScan(nullptr, cb3, b.chVal, b.chScan, U4Sum(), U4S{0u, 0u, 0u, 0u}, (int)pl.nmax, s);
  if (pbufs.ibCnt) cub::DeviceScan::ExclusiveSum(nullptr, cb2, pbufs.ibCnt, pbufs.ibPref, (int)ibItems, s);
  size_t cb4 = 0, cb5 = 0;
  if (hist) cub::DeviceScan::ExclusiveSum(nullptr, cb4, hb.nch, hb.pref, (int)(kHistK * hb.cap + 1), s);
  cub::DeviceScan::ExclusiveSum(nullptr, cb5, pbufs.cnt, pbufs.pref, (int)max_tiles, s);
  const size_t cub_bytes = std::max(std::max(std::max(cb1, cb4), std::max(cb2, cb3)), cb5);
  char* cub_tmp;
  LCK(sc.alloc(&cub_tmp, cub_bytes + 16));
  // outputs
  Node16* out;
  uint32_t *outThr, *outCount;
  LCK(sc.alloc(&out, (size_t)T * cap));
  LCK(sc.alloc(&outThr, (size_t)T * cap));
  LCK(sc.alloc(&outCount, (size_t)T));
  b.cap = cap;
  for (int t0 = 0; t0 < T; t0 += B) {
    const int nb = std::min(B, T - t0);
    b.B = nb;
    b.tree0 = tree_lo + t0;
    b.out = out + (size_t)t0 * cap;
    b.outThr = outThr + (size_t)t0 * cap;
    b.outCount = outCount + t0;
    b.leaf_of_row = leaf_of_row ? leaf_of_row + (size_t)t0 * n : nullptr;
    b.imp = imp ? imp + (size_t)t0 * p : nullptr;
    rf_status st = grow_batch(b, pl, list_src, prm->seed, task, (int)prm->bootstrap, cub_tmp, cub_bytes, rootInfo,
                              counters, hcounters, nextNode0, nextPos0, nlBase, wsTmp, hb, pbufs, candidate_counter(),
                              s, err);
    if (st) return st;
  }
  *nodes_out = out;
  *thr_out = outThr;
  *nn_out = outCount;
  *cap_out = cap;
  return RF_OK;
}

}  // namespace rf
