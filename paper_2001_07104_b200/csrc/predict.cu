// predict.cu -- batched forest inference (each node compares
// one feature with a threshold until a leaf's value is reached; the forest
// outputs the mean of its trees; exp() for LOG targets).
//
// One thread per query row walks every tree of the flattened BFS forest
// (16-byte nodes, one 128-bit load per visit), several trees at a time, and sums
// the leaf values in tree order (bit-identical to walking them one by one).  The
// forest (C5: 64 MB) stays L2-resident; the rows' features come from shared memory
// (p <= 192, fp32 with an exact fp64 fallback) or from a feature-major copy of the row block (wider rows).  Few rows
// (single-query latency) take a CTA per row with threads over trees.
#include <cuda_bf16.h>

#include "common.cuh"
#include "host_util.cuh"
#include "predict.cuh"

#include <cub/block/block_scan.cuh>

#include <algorithm>

namespace rf {
namespace {

// Tree walks are chains of dependent loads (node -> feature -> child), so one walk at a
// time leaves the SM waiting on L2 latency.  Each thread walks kG trees at once (kG
// independent chains in flight), then adds their leaf values in tree order, so the sum is
// bit-identical to walking the trees one by one.
// The feature values are read from a feature-major copy of the row block (XT[f][r]):
// the 32 lanes of a warp are 32 consecutive rows, and wherever they visit the same
// node (the top levels of every tree) they read the same feature, i.e. 256 contiguous
// bytes instead of 32 separate 512-byte-strided lines (ncu: L1 throughput was the
// limiter of the row-major version).
constexpr int kG = 8;

__global__ void __launch_bounds__(256) k_predict(const Node16* __restrict__ nodes,
                                                 const uint64_t* __restrict__ tree_off, int T,
                                                 const double* __restrict__ XT, long long n, int p,
                                                 int mode, double* __restrict__ out) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n;
       r += (long long)gridDim.x * blockDim.x) {
    const double* x = XT + r;  // feature f of row r at x[f * n]
    double s = 0.0;
    int t = 0;
    for (; t + kG <= T; t += kG) {
      const Node16* tn[kG];
      Node16 nd[kG];
#pragma unroll
      for (int g = 0; g < kG; ++g) {
        tn[g] = nodes + __ldg(tree_off + t + g);
        nd[g] = tn[g][0];
      }
      bool open = true;
      while (open) {
        open = false;
#pragma unroll
        for (int g = 0; g < kG; ++g) {
          if (nd[g].feat >= 0) {
            nd[g] = tn[g][nd[g].left + ((__ldg(x + (size_t)nd[g].feat * n) <= nd[g].v) ? 0u : 1u)];
            open = true;
          }
        }
      }
#pragma unroll
      for (int g = 0; g < kG; ++g) s += nd[g].v;
    }
    for (; t < T; ++t) {
      const Node16* tn = nodes + tree_off[t];
      Node16 nd = tn[0];
      while (nd.feat >= 0) nd = tn[nd.left + ((__ldg(x + (size_t)nd.feat * n) <= nd.v) ? 0u : 1u)];
      s += nd.v;
    }
    if (mode == 1) s = s / (double)T;
    if (mode == 2) s = exp(s / (double)T);
    out[r] = s;
  }
}

// Shared-memory variant (p <= kSmemMaxP): a CTA stages its kSmemRows rows feature-major in
// shared memory (row stride kSmemRows + 1 words: conflict-free when 32 lanes read one feature of 32
// rows), so the L1 serves only the node loads (ncu of the global-memory variants: L1
// throughput was the limiter, half of it the feature loads).  Same interleaving of trees
// and tree-order sums.  (A/B: fp32 staging + exact fallback beat fp64 staging by 24 %, 12
// trees per thread beat 8 and 16.)
#ifndef RF_PRED_SMEM_G
#define RF_PRED_SMEM_G 12
#endif
// rows per CTA: 256 (with the blocked node layout 256 beat 128 by 0.9 % and 64 was 2.3x slower on C5,
// rd2_80_ab_c5.txt; with the BFS-slot layout 128 had been best)
#ifndef RF_PRED_ROWS
#define RF_PRED_ROWS 256
#endif
constexpr int kSmemRows = RF_PRED_ROWS, kSmemMaxP = 192, kGs = RF_PRED_SMEM_G;

// Features staged as fp32 (half the shared memory per row -> more resident warps).  The
// comparison stays exact: rounding to nearest is monotonic, so float(x) < float(thr)
// implies x <= thr and float(x) > float(thr) implies x > thr; only float(x) ==
// float(thr) is undecided, and then the fp64 value is read from X.
constexpr int kSmemStrideF = kSmemRows + 1;

__device__ __forceinline__ bool le_exact(float xf, double thr, const double* xrow, int f) {
  const float tf = __double2float_rn(thr);
  if (xf < tf) return true;
  if (xf > tf) return false;
  return __ldg(xrow + f) <= thr;
}

// kStage > 0: the first kStage nodes (BFS order) of the group's kGs trees are staged in shared
// memory for every group -- the top levels, which every row visits (a prefix of the BFS order
// holds all nodes above the first level that has a node at index >= kStage) -- so the first
// levels' dependent node loads hit shared memory; deeper nodes come from L1/L2.  Taken for
// shallow forests (C5: depth 12, +46 %, profiles/rd2_22_ab_c5_stage.txt); deep unbounded trees
// (C3: ~49 levels) lose, because the per-group barrier waits for the longest walk of the CTA.
#ifndef RF_PRED_STAGE
#define RF_PRED_STAGE 63
#endif

template <int kStage>
__global__ void __launch_bounds__(kSmemRows) k_predict_smem(const Node16* __restrict__ nodes,
                                                           const uint64_t* __restrict__ tree_off, int T,
                                                           const double* __restrict__ X, long long n, int p,
                                                           int mode, double* __restrict__ out) {
  extern __shared__ __align__(16) float xsf[];  // [p][kSmemStrideF] rows, then [kGs][kStage] nodes
  Node16* sn = reinterpret_cast<Node16*>(xsf + ((p * kSmemStrideF + 3) & ~3));
  const long long r0 = (long long)blockIdx.x * kSmemRows;
  const int nr = (int)min((long long)kSmemRows, n - r0);
  const double* Xb = X + r0 * p;
  for (int q = threadIdx.x; q < nr * p; q += kSmemRows) {
    const int i = q / p, f = q - i * p;
    xsf[f * kSmemStrideF + i] = __double2float_rn(Xb[q]);
  }
  __syncthreads();
  const int i = threadIdx.x;
  const bool live = i < nr;  // (no early exit: every thread takes part in the node staging)
  const float* x = xsf + min(i, nr - 1);  // feature f at x[f * kSmemStrideF]
  const double* xrow = Xb + (size_t)min(i, nr - 1) * p;
  double s = 0.0;
  int t = 0;
  for (; t + kGs <= T; t += kGs) {
    if (kStage > 0) {
      __syncthreads();  // the previous group's nodes are no longer read
      for (int q = threadIdx.x; q < kGs * kStage; q += kSmemRows) {
        const int g = q / kStage, k = q - g * kStage;
        const uint64_t o0 = __ldg(tree_off + t + g), o1 = __ldg(tree_off + t + g + 1);
        if (o0 + k < o1) reinterpret_cast<uint4*>(sn)[q] = __ldg(reinterpret_cast<const uint4*>(nodes + o0 + k));
      }
      __syncthreads();
    }
    const Node16* tn[kGs];
    Node16 nd[kGs];
#pragma unroll
    for (int g = 0; g < kGs; ++g) {
      tn[g] = nodes + __ldg(tree_off + t + g);
      nd[g] = kStage > 0 ? sn[g * kStage] : tn[g][0];
    }
    bool open = live;
    while (open) {
      open = false;
#pragma unroll
      for (int g = 0; g < kGs; ++g) {
        if (nd[g].feat >= 0) {
          const int f = nd[g].feat;
          const uint32_t c = nd[g].left + (le_exact(x[f * kSmemStrideF], nd[g].v, xrow, f) ? 0u : 1u);
          nd[g] = (kStage > 0 && c < (uint32_t)kStage) ? sn[g * kStage + c] : tn[g][c];
          open = true;
        }
      }
    }
#pragma unroll
    for (int g = 0; g < kGs; ++g) s += nd[g].v;
  }
  if (!live) return;
  for (; t < T; ++t) {
    const Node16* tn = nodes + tree_off[t];
    Node16 nd = tn[0];
    while (nd.feat >= 0) {
      const int f = nd.feat;
      nd = tn[nd.left + (le_exact(x[f * kSmemStrideF], nd.v, xrow, f) ? 0u : 1u)];
    }
    s += nd.v;
  }
  if (mode == 1) s = s / (double)T;
  if (mode == 2) s = exp(s / (double)T);
  out[r0 + i] = s;
}
// Compact-node variant (Node8, forests built with a compact copy): rows staged quantised (below),
// the same tree groups, interleaving and tree-order sums; a walk carries the node index and reads
// 8-byte nodes, the exact threshold (on an fp32 tie) and the leaf value from val[].  The staged
// BFS prefix holds kStage8 nodes per tree for the same shared memory as the 16-byte layout's
// kStage (one more tree level in shared memory): 19.2 -> 21.3 M predictions/s on C5 with fp32
// staging (127 staged nodes beat 63 and 255, 12 trees per thread beat 10 and 16; rd2_43/44; with
// 2-level blocks 12 still beat 8 (2.2x slower) and 16 (-13 %), rd2_56_ab_c5.txt.  Splitting each walk
// into a fixed count of shared-memory steps (depths 0..5) and a global-only loop, to drop the
// per-step select, measured 2.3x slower, rd2_65_ab_c5.txt).
#ifndef RF_PRED_STAGE8
#define RF_PRED_STAGE8 127
#endif
#ifndef RF_PRED_G8
#define RF_PRED_G8 12
#endif
constexpr int kG8 = RF_PRED_G8;
// staged row values and node thresholds quantised by q = RN_bf16 o RN_fp32 (RF_PRED_FP32: RN_fp32):
// q is monotonic, so q(x) < q(thr) implies x <= thr and q(x) > q(thr) implies x > thr; only
// q(x) = q(thr) reads the fp64 values.  bf16 halves the staged rows (128 x 64 features: 16 KB) --
// more resident CTAs -- for a few more fp64 tie reads: 21.3 -> 26.2 M predictions/s on C5
// (profiles/rd2_44_ab_c5.txt).  Staging order-preserving 16-bit keys of the bf16 values instead (two
// integer compares, no bf16 -> fp32 conversion per step) measured neutral (+0.1 %, rd2_67_ab_c5.txt).
#ifndef RF_PRED_FP32
typedef __nv_bfloat16 XStage;
__device__ __forceinline__ float q_thr(double v) { return __bfloat162float(__float2bfloat16_rn(__double2float_rn(v))); }
__device__ __forceinline__ XStage q_stage(double v) { return __float2bfloat16_rn(__double2float_rn(v)); }
__device__ __forceinline__ float x_of(XStage v) { return __bfloat162float(v); }
#else
typedef float XStage;
__device__ __forceinline__ float q_thr(double v) { return __double2float_rn(v); }
__device__ __forceinline__ XStage q_stage(double v) { return __double2float_rn(v); }
__device__ __forceinline__ float x_of(XStage v) { return v; }
#endif
__host__ __device__ constexpr size_t xstage_bytes(int p) { return ((size_t)p * kSmemStrideF * sizeof(XStage) + 15) / 16 * 16; }

constexpr uint32_t kBlkPrefix = 128;
// levels per block (RF_PRED_BLK_LV): 3 -> 8-slot (64-byte) blocks of 7 nodes.  C5 (rd2_55..58):
// BFS slots 25.7 M predictions/s; 2-level 32-byte blocks 28.5 M; 3-level 30.5 M; 3-level with an L1
// prefetch of the block's second sector on entry 27.3 M; 4-level (128-byte) 27.4 M.
#ifndef RF_PRED_BLK_LV
#define RF_PRED_BLK_LV 3
#endif
constexpr int kBlkLv = RF_PRED_BLK_LV;
constexpr int kBlkSlots = 1 << kBlkLv;

template <int kStage>
__global__ void __launch_bounds__(kSmemRows) k_predict_smem8(const Node8* __restrict__ nodes,
                                                            const double* __restrict__ val,
                                                            const uint64_t* __restrict__ tree_off, int T,
                                                            const double* __restrict__ X, long long n, int p,
                                                            int mode, double* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char sm8[];  // [p][kSmemStrideF] rows, then [kG8][kStage] nodes
  XStage* xsf8 = reinterpret_cast<XStage*>(sm8);
  Node8* sn = reinterpret_cast<Node8*>(sm8 + xstage_bytes(p));
  const long long r0 = (long long)blockIdx.x * kSmemRows;
  const int nr = (int)min((long long)kSmemRows, n - r0);
  const double* Xb = X + r0 * p;
  for (int q = threadIdx.x; q < nr * p; q += kSmemRows) {
    const int i = q / p, f = q - i * p;
    xsf8[f * kSmemStrideF + i] = q_stage(Xb[q]);
  }
  __syncthreads();
  const int i = threadIdx.x;
  const bool live = i < nr;  // (no early exit: every thread takes part in the node staging)
  const XStage* x = xsf8 + min(i, nr - 1);
  const double* xrow = Xb + (size_t)min(i, nr - 1) * p;
  double s = 0.0;
  int t = 0;
  for (; t + kG8 <= T; t += kG8) {
    if (kStage > 0) {
      __syncthreads();  // the previous group's nodes are no longer read
      for (int q = threadIdx.x; q < kG8 * kStage; q += kSmemRows) {
        const int g = q / kStage, k = q - g * kStage;
        const uint64_t o0 = __ldg(tree_off + t + g), o1 = __ldg(tree_off + t + g + 1);
        if (o0 + k < o1) reinterpret_cast<uint2*>(sn)[q] = __ldg(reinterpret_cast<const uint2*>(nodes + o0 + k));
      }
      __syncthreads();
    }
    uint64_t base[kG8];
    Node8 nd[kG8];
    uint32_t idx[kG8];
#pragma unroll
    for (int g = 0; g < kG8; ++g) {
      base[g] = __ldg(tree_off + t + g);
      idx[g] = 0u;
      nd[g] = kStage > 0 ? sn[g * kStage] : nodes[base[g]];
    }
    bool open = live;
    while (open) {
      open = false;
#pragma unroll
      for (int g = 0; g < kG8; ++g) {
        const uint32_t f = nd[g].fl & 0xFFu;
        if (f != 0xFFu) {
          const float xf = x_of(x[f * kSmemStrideF]);
          // q decides unless q(x) = q(thr) (monotonic rounding), then the fp64 values do
          const bool le = xf < nd[g].tf || (xf == nd[g].tf && __ldg(xrow + f) <= __ldg(val + base[g] + idx[g]));
          idx[g] = ((nd[g].fl >> 8) & 0x7FFFFFu) + (le ? 0u : ((nd[g].fl >> 31) ? (uint32_t)kBlkSlots : 1u));
          nd[g] = (kStage > 0 && idx[g] < (uint32_t)kStage) ? sn[g * kStage + idx[g]] : nodes[base[g] + idx[g]];
          open = true;
        }
      }
    }
#pragma unroll
    for (int g = 0; g < kG8; ++g) s += __ldg(val + base[g] + idx[g]);
  }
  if (!live) return;
  for (; t < T; ++t) {
    const uint64_t b0 = tree_off[t];
    uint32_t id = 0;
    Node8 nd = nodes[b0];
    while ((nd.fl & 0xFFu) != 0xFFu) {
      const uint32_t f = nd.fl & 0xFFu;
      const float xf = x_of(x[f * kSmemStrideF]);
      const bool le = xf < nd.tf || (xf == nd.tf && xrow[f] <= val[b0 + id]);
      id = ((nd.fl >> 8) & 0x7FFFFFu) + (le ? 0u : ((nd.fl >> 31) ? (uint32_t)kBlkSlots : 1u));
      nd = nodes[b0 + id];
    }
    s += val[b0 + id];
  }
  if (mode == 1) s = s / (double)T;
  if (mode == 2) s = exp(s / (double)T);
  out[r0 + i] = s;
}

__global__ void k_build_node8(const Node16* __restrict__ nodes, uint64_t total, Node8* __restrict__ n8,
                              double* __restrict__ val) {
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < total; q += (uint64_t)gridDim.x * blockDim.x) {
    const Node16 nd = nodes[q];
    Node8 c;
    c.fl = nd.feat < 0 ? 0xFFu : ((uint32_t)nd.feat | (nd.left << 8));
    c.tf = nd.feat < 0 ? 0.0f : q_thr(nd.v);
    n8[q] = c;
    val[q] = nd.v;
  }
}

// ---- blocked compact layout (BFS-ordered forests: every fitted one).  Per tree: BFS levels 0..6
// (<= 127 nodes) keep their BFS slots 0..126 (slot 127 is padding); below them the tree is cut into
// blocks of kBlkLv levels -- kBlkSlots slots holding a block root P (depth 7, 7 + kBlkLv, ...) and
// its descendants in heap order (children of offset o at 2o + 1, 2o + 2), 64 bytes for 3 levels;
// the blocks of one level are numbered in BFS order, so sibling blocks are adjacent.  A walk then
// fetches one block per three levels below the prefix instead of one node per level.  Child
// addressing stays "left + (go right ? stride : 0)": stride 1 inside the prefix and inside a block,
// kBlkSlots (the adjacent block) from a depth-6 node or a block's bottom level, flagged by bit 31 of
// the node word (left slot < 2^23).
constexpr int kBlkMaxLevels = kBlkLevStride - 1;

__device__ __forceinline__ bool blk_root_depth(int d) { return d >= 7 && (d - 7) % kBlkLv == 0; }

// level d of a BFS tree: [s_d, s_{d+1}); s_{d+1} - s_d = 2 x (internal nodes of level d - 1).  One CTA
// per tree: lev[t][d] = s_d (d <= levels), nlev[t] = levels, slots[t] = 128 + 4 x (nodes at
// block-root depths); bad[0] |= 1 if a tree is not in the BFS order this assumes (children of the
// j-th internal node of a level at s_{d+1} + 2j), is deeper than kBlkMaxLevels or needs >= 2^23 slots.
__global__ void __launch_bounds__(256) k_blk_count(const Node16* __restrict__ nodes, const uint64_t* __restrict__ tree_off,
                                                   uint64_t* __restrict__ slots, uint32_t* __restrict__ lev,
                                                   int* __restrict__ nlev, int* bad) {
  using BS = cub::BlockScan<uint32_t, 256>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ uint32_t s_carry;
  const int t = blockIdx.x;
  const uint64_t o0 = tree_off[t], len = tree_off[t + 1] - o0;
  const Node16* tn = nodes + o0;
  uint32_t* lv = lev + (size_t)t * (kBlkMaxLevels + 1);
  uint64_t st = 0, en = 1, roots = 0;
  bool fail = false;
  int d = 0;
  while (st < en) {
    if (en > len || d >= kBlkMaxLevels) { fail = true; break; }  // (uniform: every thread has st, en)
    if (threadIdx.x == 0) { s_carry = 0; lv[d] = (uint32_t)st; }
    __syncthreads();
    for (uint64_t b = st; b < en; b += 256) {
      const uint64_t i = b + threadIdx.x;
      const uint32_t in = (i < en && tn[i].feat >= 0) ? 1u : 0u;
      uint32_t ex, tot;
      BS(tmp).ExclusiveSum(in, ex, tot);
      const uint32_t c0 = s_carry;
      if (in && tn[i].left != en + 2ull * (c0 + ex)) fail = true;
      __syncthreads();
      if (threadIdx.x == 0) s_carry = c0 + tot;
      __syncthreads();
    }
    if (blk_root_depth(d)) roots += en - st;
    const uint64_t cnt = s_carry;
    st = en;
    en = en + 2 * cnt;
    ++d;
    __syncthreads();
  }
  fail = __syncthreads_or(fail);
  if (en != len) fail = true;  // every node reached by the level walk
  const uint64_t sl = kBlkPrefix + (uint64_t)kBlkSlots * roots;
  if (sl >= (1ull << 23)) fail = true;
  if (threadIdx.x == 0) {
    slots[t] = sl;
    nlev[t] = d;
    if (!fail) lv[d] = (uint32_t)st;
    if (fail) atomicOr(bad, 1);
  }
}

// One CTA per tree (after k_blk_count passed): every node of the prefix levels and every block
// (written by its root's thread, with both children) in parallel, level by level.
__global__ void __launch_bounds__(256) k_blk_build(const Node16* __restrict__ nodes, const uint64_t* __restrict__ tree_off,
                                                   const uint64_t* __restrict__ n8_off, const uint32_t* __restrict__ lev,
                                                   const int* __restrict__ nlev, Node8* __restrict__ n8,
                                                   double* __restrict__ val) {
  __shared__ uint32_t s_st[kBlkMaxLevels + 1];   // level starts (tree-local BFS index)
  __shared__ uint32_t s_blk[kBlkMaxLevels + 1];  // blocks of the block-root levels before level d
  const int t = blockIdx.x;
  const Node16* tn = nodes + tree_off[t];
  Node8* out = n8 + n8_off[t];
  double* vo = val + n8_off[t];
  const int nl = nlev[t];
  const uint32_t* lv = lev + (size_t)t * (kBlkMaxLevels + 1);
  for (int d = threadIdx.x; d <= nl; d += blockDim.x) s_st[d] = lv[d];
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t blk = 0;
    for (int d = 0; d <= nl; ++d) {
      s_blk[d] = blk;
      if (d < nl && blk_root_depth(d)) blk += s_st[d + 1] - s_st[d];
    }
  }
  __syncthreads();
  // new slot of the j-th node of block-root level d
  auto root_slot = [&](int d, uint32_t j) { return kBlkPrefix + (uint32_t)kBlkSlots * (s_blk[d] + j); };
  auto put = [&](uint32_t slot, const Node16& nd, uint32_t left, uint32_t wide) {
    Node8 c;
    c.fl = nd.feat < 0 ? 0xFFu : ((uint32_t)nd.feat | (left << 8) | (wide << 31));
    c.tf = nd.feat < 0 ? 0.0f : q_thr(nd.v);
    out[slot] = c;
    vo[slot] = nd.v;
  };
  for (int d = 0; d < nl; ++d) {
    const uint32_t st = s_st[d], en = s_st[d + 1];
    if (d < 7) {
      for (uint32_t i = st + threadIdx.x; i < en; i += blockDim.x) {
        const Node16 nd = tn[i];
        if (d < 6 || nd.feat < 0) put(i, nd, nd.left, 0u);
        else put(i, nd, root_slot(7, nd.left - s_st[7]), 1u);
      }
    } else if (blk_root_depth(d)) {
      // the block of root i: heap positions o = 0 .. kBlkSlots - 2 (level l holds o = 2^l - 1 ..),
      // in-block children of o at 2o + 1, 2o + 2; the bottom level's children are the roots of
      // adjacent blocks kBlkLv levels down
      for (uint32_t i = st + threadIdx.x; i < en; i += blockDim.x) {
        const uint32_t me = root_slot(d, i - st);
        int64_t pos[kBlkSlots - 1];
        pos[0] = i;
#pragma unroll
        for (int o = 1; o < kBlkSlots - 1; ++o) pos[o] = -1;
#pragma unroll
        for (int o = 0; o < kBlkSlots - 1; ++o) {
          if (pos[o] < 0) continue;
          const Node16 nd = tn[pos[o]];
          const int lvl = 31 - __clz(o + 1);
          if (lvl < kBlkLv - 1) {
            if (nd.feat >= 0) { pos[2 * o + 1] = nd.left; pos[2 * o + 2] = nd.left + 1; }
            put(me + o, nd, me + 2 * o + 1, 0u);
          } else {
            put(me + o, nd, nd.feat >= 0 ? root_slot(d + kBlkLv, nd.left - s_st[d + kBlkLv]) : 0u, 1u);
          }
        }
      }
    }
  }
}

// rows [r0, r0 + cn) of X (row-major, n x p) -> XT (p x cn, feature-major), 32 x 32 tiles
__global__ void k_transpose(const double* __restrict__ X, long long r0, long long cn, int p, double* __restrict__ XT) {
  __shared__ double tile[32][33];
  const long long rb = blockIdx.x * 32LL;
  const int fb = blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const long long r = rb + k;
    const int f = fb + threadIdx.x;
    if (r < cn && f < p) tile[k][threadIdx.x] = X[(r0 + r) * p + f];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int f = fb + k;
    const long long r = rb + threadIdx.x;
    if (r < cn && f < p) XT[(size_t)f * cn + r] = tile[threadIdx.x][k];
  }
}

// Few rows (single-query latency, T4/T5 of the paper): one CTA per row, threads
// over trees (tree t -> thread t mod 256, each thread in tree order), a fixed-shape
// block reduction (deterministic), finiteness check of the row in the same kernel.
constexpr int kFewThreads = 256;

__global__ void __launch_bounds__(kFewThreads) k_predict_few(const Node16* __restrict__ nodes,
                                                             const uint64_t* __restrict__ tree_off, int T,
                                                             const double* __restrict__ X, int p, int mode,
                                                             double* __restrict__ out, int* err) {
  const long long r = blockIdx.x;
  const double* x = X + r * p;
  bool bad = false;
  for (int j = threadIdx.x; j < p; j += kFewThreads) bad |= !isfinite(x[j]);
  if (bad) atomicOr(err, 1);
  double s = 0.0;
  for (int t = threadIdx.x; t < T; t += kFewThreads) {
    const Node16* tn = nodes + tree_off[t];
    Node16 nd = tn[0];
    while (nd.feat >= 0) nd = tn[nd.left + ((x[nd.feat] <= nd.v) ? 0u : 1u)];
    s += nd.v;
  }
  // fixed-order block reduction: warps by shuffles, then warp sums in warp order
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) s += __shfl_down_sync(0xffffffffu, s, d);
  __shared__ double ws[kFewThreads / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < kFewThreads / 32; ++w) tot += ws[w];
    if (mode == 1) tot = tot / (double)T;
    if (mode == 2) tot = exp(tot / (double)T);
    out[r] = tot;
  }
}

__global__ void k_pred_finalize(const double* partial, long long n, int T, int target, double* out) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n;
       r += (long long)gridDim.x * blockDim.x) {
    double s = partial[r] / (double)T;
    out[r] = target == 1 ? exp(s) : s;
  }
}

__global__ void k_check_finite(const double* X, size_t total, int* err) {
  bool bad = false;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x)
    bad |= !isfinite(X[i]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(err, 1);
}

}  // namespace

cudaError_t node8_blocked_count(const Node16* nodes, const uint64_t* tree_off, int T, uint64_t* slots, uint32_t* lev,
                                int* nlev, int* bad, cudaStream_t s) {
  k_blk_count<<<(unsigned)T, 256, 0, s>>>(nodes, tree_off, slots, lev, nlev, bad);
  note_launch();
  return cudaGetLastError();
}

cudaError_t node8_blocked_build(const Node16* nodes, const uint64_t* tree_off, int T, const uint64_t* n8_off,
                                const uint32_t* lev, const int* nlev, Node8* n8, double* val, cudaStream_t s) {
  k_blk_build<<<(unsigned)T, 256, 0, s>>>(nodes, tree_off, n8_off, lev, nlev, n8, val);
  note_launch();
  return cudaGetLastError();
}

cudaError_t build_node8(const Node16* nodes, uint64_t total, Node8* n8, double* val, cudaStream_t s) {
  if (!total) return cudaSuccess;
  const uint64_t blocks = std::min<uint64_t>((total + 255) / 256, 148 * 16);
  k_build_node8<<<(unsigned)blocks, 256, 0, s>>>(nodes, total, n8, val);
  note_launch();
  return cudaGetLastError();
}

cudaError_t predict_forest(const Node16* nodes, const uint64_t* tree_off, int T, const double* X,
                           long long n, int p, int mode, double* out, cudaStream_t s, int* err_few,
                           uint64_t total_nodes, const Node8* n8, const double* val, const uint64_t* n8_off) {
  if (n <= 0) return cudaSuccess;
  if (err_few && n <= kFewRows) {  // latency path: rows checked for finiteness in-kernel
    k_predict_few<<<(unsigned)n, kFewThreads, 0, s>>>(nodes, tree_off, T, X, p, mode, out, err_few);
    note_launch();
    return cudaGetLastError();
  }
  if (n8 && val && p <= kSmemMaxP) {
    const bool stage = RF_PRED_STAGE8 > 0 && total_nodes > 0 && total_nodes <= (uint64_t)T * kShallowNodesPerTree;
    const size_t smem = xstage_bytes(p) + (stage ? (size_t)kG8 * RF_PRED_STAGE8 * sizeof(Node8) : 0);
    auto kern = stage ? k_predict_smem8<RF_PRED_STAGE8> : k_predict_smem8<0>;
    cudaError_t e = allow_max_dynamic_smem(kern);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)((n + kSmemRows - 1) / kSmemRows), kSmemRows, smem, s>>>(n8, val, n8_off ? n8_off : tree_off, T, X,
                                                                              n, p, mode, out);
    note_launch();
    return cudaGetLastError();
  }
  if (p <= kSmemMaxP) {
    const bool stage = RF_PRED_STAGE > 0 && total_nodes > 0 && total_nodes <= (uint64_t)T * kShallowNodesPerTree;
    const size_t smem = (size_t)((p * kSmemStrideF + 3) & ~3) * 4 + (stage ? (size_t)kGs * RF_PRED_STAGE * sizeof(Node16) : 0);
    auto kern = stage ? k_predict_smem<RF_PRED_STAGE> : k_predict_smem<0>;
    cudaError_t e = allow_max_dynamic_smem(kern);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)((n + kSmemRows - 1) / kSmemRows), kSmemRows, smem, s>>>(nodes, tree_off, T, X, n, p, mode, out);
    note_launch();
    return cudaGetLastError();
  }
  // wide rows: blocks of <= ~512 MB transposed at a time
  const long long chunk = std::max<long long>(4096, (512LL << 20) / (8LL * p));
  Scratch sc(s);
  double* XT;
  cudaError_t e = sc.alloc(&XT, (size_t)std::min(n, chunk) * p);
  if (e != cudaSuccess) return e;
  for (long long r0 = 0; r0 < n; r0 += chunk) {
    const long long cn = std::min(chunk, n - r0);
    k_transpose<<<dim3((unsigned)((cn + 31) / 32), (unsigned)((p + 31) / 32)), dim3(32, 8), 0, s>>>(X, r0, cn, p, XT);
    long long blocks = (cn + 255) / 256;
    if (blocks > 148LL * 64) blocks = 148LL * 64;
    k_predict<<<(unsigned)blocks, 256, 0, s>>>(nodes, tree_off, T, XT, cn, p, mode, out + r0);
    note_launch(2);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t predict_finalize(const double* partial, long long n, int T, int target, double* out,
                             cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  long long blocks = (n + 255) / 256;
  if (blocks > 148LL * 16) blocks = 148LL * 16;
  k_pred_finalize<<<(unsigned)blocks, 256, 0, s>>>(partial, n, T, target, out);
  note_launch();
  return cudaGetLastError();
}

cudaError_t check_finite(const double* X, size_t total, int* err, cudaStream_t s) {
  if (!total) return cudaSuccess;
  size_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_check_finite<<<(unsigned)blocks, 256, 0, s>>>(X, total, err);
  note_launch();
  return cudaGetLastError();
}

}  // namespace rf
