// small_tree.cu -- warp-per-tree exact CART growth for small training sets
// (n_tr <= 255), the hot kernel of the paper-shaped CV study (SURVEY.md 8(d)
// C1/C2).  One warp grows one whole tree level-synchronously with all of its
// data resident in shared memory; the CTA's warps share the task's presorted
// feature orders, local ranks, quantised targets and test rows.
//
// Method (sec. 2.2; R2-R14):
//   bootstrap n_tr draws -> integer weights w (R2); per node draw mtry
//   features by partial Fisher-Yates keyed by heap index (R4, R14); for every
//   drawn feature scan the node's rows in x order, exact int64 prefix sums
//   WL = sum w, SL = sum w t_q (R7), score G = SL^2/WL + SR^2/WR in canonical
//   fp64 (R6, R28) at every boundary between distinct values (R8); best by
//   (G desc, feature or draw slot asc, threshold rank asc) (R9); threshold midway (R8);
//   leaf if depth cap, < min_split distinct rows, constant t_q or no
//   candidate (R11); leaf value fl(S/W) 2^-F (R13).
//   ExtraTrees (split_mode 2, R29): the only candidate of a
//   (node, slot) segment is the boundary of its random threshold, given as a
//   dense-rank threshold found by a binary search in a shared-memory table of
//   the task's distinct values; everything else is shared.
//   MAE criterion (R32): the candidates are the same; a
//   candidate's cost D = 2 (SAD_L + SAD_R), the doubled weighted absolute
//   deviations of the children from their weighted medians, is exact in
//   uint64 (2 guard bits of quantisation keep it below 2^63) and is found by
//   one walk of the node's rows in t_q order (an extra row list, partitioned
//   like the feature lists): the walk stops at both children's weighted
//   medians and SAD = m2 (2 W_<=k - W) + 2 (S - 2 S_<=k) needs only the
//   cumulative sums there.  Best = lowest D (key ~D), same tie-break; leaves
//   hold the weighted median (a second walk per node after the mark pass).
//
// Per level the warp runs three lane-serial passes (each lane owns a
// contiguous chunk; lane totals are combined by one warp scan):
//   search    over (node, drawn feature, position) in node-major order, so a
//             node's candidates are contiguous: node bests need no atomics --
//             nodes inside a lane's chunk are resolved by that lane, nodes on
//             chunk borders by one segmented warp reduction;
//   mark      go-left flags, left sums, child constancy;
//   partition all p feature lists, stable, ping-pong buffers.
// fl(a / W) for the integer weights W <= 255 uses a table of y = RN(1/W) and
// one Markstein correction q + fma(a - W q) y, which returns exactly RN(a/W)
// (Markstein's theorem).
//
// CV mode routes the task's test rows level by level and accumulates their
// leaf values per warp job; fit mode writes BFS-ordered 16-byte nodes.
#include "host_util.cuh"
#include "small_tree.cuh"

namespace rf {
namespace {

// All shared-memory arrays are 32-bit offsets into one extern __shared__ symbol:
// the compiler then addresses them as shared memory directly (LDS/STS with a
// register offset) instead of converting generic pointers, and each handle costs
// one register instead of two.
extern __shared__ __align__(16) char g_smem[];

template <typename T>
struct SA {
  uint32_t off;
  template <typename I>
  __device__ __forceinline__ T& operator[](I i) const {
    return reinterpret_cast<T*>(g_smem + off)[i];
  }
  __device__ __forceinline__ SA operator+(int i) const { return SA{off + (uint32_t)i * (uint32_t)sizeof(T)}; }
  __device__ __forceinline__ T* ptr() const { return reinterpret_cast<T*>(g_smem + off); }
};

struct Carve {
  size_t off;
  __host__ __device__ explicit Carve(size_t start = 0) : off(start) {}
  template <typename T>
  __host__ __device__ SA<T> take(size_t count, size_t align = 8) {
    off = (off + align - 1) / align * align;
    SA<T> p{(uint32_t)off};
    off += count * sizeof(T);
    return p;
  }
};

struct CtaSmem {
  SA<uint8_t> ord;    // [p][ntr_max] local rows in x order
  SA<uint8_t> lrank;  // [p][ntr_max] dense rank of x among training rows, by local row
  SA<int64_t> tq;     // [ntr_max]
  SA<double2> rcp2;   // [256] (w, RN(1/w))
  SA<double> xte;     // [nte_max][p]
  SA<double> xs;      // ExtraTrees: [p][ntr_max] distinct training values of x_f by dense rank
  SA<uint8_t> tord;   // MAE: [ntr_max] local rows in (t_q, local index) order
  SA<uint32_t> trr;   // [ntr_max] global row of each local row (threshold values, decide step)
};

struct NodeSet {  // open nodes of one level
  SA<uint8_t> start;
  SA<uint8_t> len;
  SA<uint16_t> W;
  SA<int64_t> S;
  SA<uint64_t> heap;
  SA<uint16_t> bfs;
};

struct WarpSmem {
  SA<uint8_t> w;       // [ntr_max] bootstrap multiplicities
  SA<uint8_t> listA;   // [p][ntr_max]
  SA<uint8_t> listB;   // [p][ntr_max]
  SA<uint8_t> pnA;     // [ntr_max] position -> open node
  SA<uint8_t> pnB;
  SA<uint8_t> side;    // [ntr_max] by local row: 1 = goes left
  SA<uint8_t> trash;   // [32] target of the partition's discarded entries, one byte per lane
  NodeSet cur, nxt;
  SA<uint8_t> feat;    // [NM][fs] drawn features (partial Fisher-Yates), in draw order
  SA<uint8_t> xb;      // ExtraTrees: [NM][fs] rank threshold per draw slot (last rank with x <= thr) or kNone
  SA<unsigned long long> bkey;  // best key (G bits + 1; 0 = none); after decide: threshold bits
  SA<uint32_t> baux;   // best (feature << 8 | position); bit 31 = split
  SA<uint32_t> bW;     // search: prefix base of W; then the best's left W
  SA<uint64_t> bS;     // search: prefix base of S; then the best's left S; then the partition record
  SA<uint8_t> ncb;     // [NM][2] child non-constant flags (decide, mark); aliases chOpen, which (e)
                       // writes for node k after its lane has read them
  SA<uint8_t> chOpen;  // [NM][2] open index of the children or kNone
  // leaf values of a split node's leaf children (or of an unsplit node itself) for the test-row
  // routing (f) live in cur.S[k] (left / the node) and cur.heap[k] (right) as fp64 bits: (e) has
  // read both for node k (its lane only) and nothing reads them before the level advance
  SA<uint16_t> chBase; // BFS id of the left child
  SA<uint32_t> thrIdx; // fit mode: threshold rank
  SA<uint32_t> desc;   // [ntr_max] partition descriptor per position (shared by all lists);
                       // aliases bkey (free once the level's thresholds are used, (g))
  SA<int64_t> med2;    // MAE: [NM][2] doubled weighted medians of the children (or of the node)
  SA<uint64_t> bD;     // MAE fit: [NM] cost D of the chosen split (importance)
  SA<ulonglong2> mq;   // MAE + ExtraTrees: [kMaeQ] ring of queued search candidates (mae_flush)
  SA<unsigned long long> mkey;  // MAE: [NM] best queued candidate per open node (key, aux, WL, SL)
  SA<uint32_t> maux;
  SA<uint32_t> mWL;
  SA<int64_t> mSL;
};

constexpr uint8_t kNone = 0xFF;
// The search reads the list entry after a segment's last one and the tables indexed by it (row id
// < 256: lrank, w, tq) without a bounds select; the value is never used, and this much shared
// memory past the last region keeps every such read inside the allocation (tq[255] is 2040 B past
// the table's start).
constexpr size_t kReadSlack = 2048;
constexpr int kMaeQ = 64;  // MAE candidate ring: <= 31 pending + one loop step's 32 appends

__host__ __device__ inline int nmax_of(int ntr_max) { return ntr_max / 2 + 1; }
// m = p under the lowest-feature tie-break (north_star; exact mode): the drawn set is all features and
// the winner does not depend on the draw order, so no draws are made and slot j is feature j
__host__ __device__ inline bool no_draws(int m, int p, int tie_draw, bool extra) { return m == p && !tie_draw && !extra; }
// per-node stride of the drawn-feature table: the largest m that draws (p > 16: the whole in-place
// permutation), 0 when no grid point draws (saves shared memory: more resident warps)
__host__ __device__ inline int feat_stride_of(const SmallArgs& a) {
  int fs = 0;
  for (int i = 0; i < a.n_mtry; ++i)
    if (!no_draws(a.mtrys[i], a.p, a.tie_draw, a.extra != 0)) fs = max(fs, a.p > 16 ? a.p : a.mtrys[i]);
  return fs;
}
// per-feature stride of the row lists: a multiple of 4 (32-bit list words in (g))
__host__ __device__ inline int stride_of(int ntr_max) { return (ntr_max + 3) & ~3; }

__host__ __device__ inline void carve_cta(Carve& c, CtaSmem& s, int p, int ntr_max, int nte_max, bool extra,
                                          bool mae) {
  // the reciprocal table first: offset 0 is a compile-time constant, so the search loop
  // addresses it without rematerialising the carve arithmetic (ncu: ~10 instructions per
  // iteration otherwise, the kernel runs at the 128-register cap)
  s.rcp2 = c.take<double2>(256, 16);
  s.tq = c.take<int64_t>(ntr_max, 16);
  s.ord = c.take<uint8_t>((size_t)p * ntr_max, 16);
  s.lrank = c.take<uint8_t>((size_t)p * ntr_max, 16);
  s.xte = c.take<double>((size_t)nte_max * p, 16);
  s.xs = extra ? c.take<double>((size_t)p * ntr_max, 16) : SA<double>{0u};
  s.tord = mae ? c.take<uint8_t>(ntr_max, 16) : SA<uint8_t>{0u};
  s.trr = c.take<uint32_t>(ntr_max, 16);
}

// BFS ids are needed only when nodes are emitted (fit mode); CV mode routes test rows by
// open-node index and leaves them out (saves shared memory: 16 warps fit on the C2 shapes)
__host__ __device__ inline void carve_nodeset(Carve& c, NodeSet& s, int NM, bool fit) {
  s.start = c.take<uint8_t>(NM, 4);
  s.len = c.take<uint8_t>(NM, 4);
  s.W = c.take<uint16_t>(NM, 4);
  s.S = c.take<int64_t>(NM, 8);
  s.heap = c.take<uint64_t>(NM, 8);
  s.bfs = fit ? c.take<uint16_t>(NM, 4) : SA<uint16_t>{0u};
}

// row lists per tree: the p feature lists, plus the t_q-ordered list under MAE (list p)
__host__ __device__ inline int nlists_of(int p, bool mae) { return p + (mae ? 1 : 0); }

__host__ __device__ inline void carve_warp(Carve& c, WarpSmem& s, int p, int ntr_max, int fs, bool extra,
                                           bool fit, bool mae) {
  const int NM = nmax_of(ntr_max);
  const int P = nlists_of(p, mae);
  s.w = c.take<uint8_t>((ntr_max + 3) / 4 * 4, 16);
  s.listA = c.take<uint8_t>((size_t)P * ntr_max, 16);
  s.listB = c.take<uint8_t>((size_t)P * ntr_max, 16);
  s.pnA = c.take<uint8_t>(ntr_max, 4);
  s.pnB = c.take<uint8_t>(ntr_max, 4);
  s.side = c.take<uint8_t>(ntr_max, 4);
  s.trash = c.take<uint8_t>(32, 4);
  carve_nodeset(c, s.cur, NM, fit);
  carve_nodeset(c, s.nxt, NM, fit);
  s.feat = c.take<uint8_t>((size_t)NM * fs, 4);
  s.xb = extra ? c.take<uint8_t>((size_t)NM * fs, 4) : SA<uint8_t>{0u};
  s.bkey = c.take<unsigned long long>(NM, 16);  // 16-aligned: desc aliases it (uint4 loads)
  s.baux = c.take<uint32_t>(NM, 4);
  s.bW = c.take<uint32_t>(NM, 4);
  s.bS = c.take<uint64_t>(NM, 8);
  s.chOpen = c.take<uint8_t>((size_t)NM * 2, 4);
  s.ncb = s.chOpen;
  s.chBase = fit ? c.take<uint16_t>(NM, 4) : SA<uint16_t>{0u};
  s.thrIdx = fit ? c.take<uint32_t>(NM, 4) : SA<uint32_t>{0u};
  s.desc = SA<uint32_t>{s.bkey.off};  // ntr_max * 4 <= NM * 8 bytes
  s.med2 = mae ? c.take<int64_t>((size_t)NM * 2, 8) : SA<int64_t>{0u};
  s.bD = (mae && fit) ? c.take<uint64_t>(NM, 8) : SA<uint64_t>{0u};
  s.mq = (mae && extra) ? c.take<ulonglong2>(kMaeQ, 16) : SA<ulonglong2>{0u};
  s.mkey = (mae && extra) ? c.take<unsigned long long>(NM, 8) : SA<unsigned long long>{0u};
  s.mSL = (mae && extra) ? c.take<int64_t>(NM, 8) : SA<int64_t>{0u};
  s.maux = (mae && extra) ? c.take<uint32_t>(NM, 4) : SA<uint32_t>{0u};
  s.mWL = (mae && extra) ? c.take<uint32_t>(NM, 4) : SA<uint32_t>{0u};
}

// ---------------------------------------------------------------- warp ops --
// Out of line (one copy each): every inlined shuffle carries divergence-handling
// code, and the kernel's per-level code must fit the instruction caches.
struct Scan32 { uint32_t ex, tot; };
struct Scan64 { uint64_t ex, tot; };

__device__ __noinline__ Scan32 wscan32(uint32_t v) {
  const int lane = threadIdx.x & 31;
  uint32_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  return Scan32{x - v, __shfl_sync(0xffffffffu, x, 31)};
}

__device__ __noinline__ Scan64 wscan64(uint64_t v) {
  const int lane = threadIdx.x & 31;
  uint64_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  return Scan64{x - v, __shfl_sync(0xffffffffu, x, 31)};
}

__device__ __forceinline__ uint32_t wscan_u32(uint32_t v, uint32_t& total) {
  const Scan32 s = wscan32(v);
  total = s.tot;
  return s.ex;
}
__device__ __forceinline__ uint64_t wscan_u64(uint64_t v, uint64_t& total) {
  const Scan64 s = wscan64(v);
  total = s.tot;
  return s.ex;
}

__device__ __noinline__ int64_t wsum_i64(int64_t v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}
__device__ __noinline__ int64_t wmin_i64(int64_t v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) { int64_t o = __shfl_xor_sync(0xffffffffu, v, d); v = o < v ? o : v; }
  return v;
}
__device__ __noinline__ int64_t wmax_i64(int64_t v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) { int64_t o = __shfl_xor_sync(0xffffffffu, v, d); v = o > v ? o : v; }
  return v;
}

// Rarely executed helpers are out of line: the kernel's hot per-level code must fit
// the instruction caches (ncu showed no_instruction stalls with everything inlined).
// RN(a / w) for an integer 1 <= w <= 255 with y = RN(1/w): one Markstein correction
__device__ __forceinline__ double div_small(double a, double dw, double y) {
  const double q = __dmul_rn(a, y);
  const double r = __fma_rn(-dw, q, a);
  return __fma_rn(r, y, q);
}

// leaf value fl(fl(S) / W) 2^-F (R13), the division by the reciprocal table (W <= 255)
__device__ __noinline__ double leaf_value(int64_t S, double2 wy, int F) {
  return scalbn(div_small(__ll2double_rn(S), wy.x, wy.y), -F);
}

__device__ __noinline__ void philox_pair_ool(uint32_t k0, uint32_t k1, uint32_t b, uint32_t c1, uint32_t c2,
                                             uint32_t c3, uint64_t& d0, uint64_t& d1) {
  philox_pair(k0, k1, b, c1, c2, c3, d0, d1);
}

// total order of candidates: key (G bits + 1) descending, aux (tie key, draw slot, position)
// ascending; tie key = feature index (north_star, default) or draw slot (R9)
__device__ __forceinline__ bool better(unsigned long long k1, uint32_t a1, unsigned long long k2, uint32_t a2) {
  return k1 > k2 || (k1 == k2 && a1 < a2);
}

// ------------------------------------------------------- MAE criterion (R32) --
// Doubled weighted median of a row set walked in t_q order (scikit-learn's rule, the
// oracle's median2): k = the first element with 2 cum_k >= W; m2 = t_k + t_k+1 if
// 2 cum_k == W, else 2 t_k.  The tracker also keeps W_<=k and S_<=k, from which
// the doubled absolute-deviation sum is SAD2 = sum w |2t - m2|
//   = m2 (2 W_<=k - W) + 2 (S - 2 S_<=k)
// (rows up to k lie at or below m2 / 2, the rest at or above).  All exact in
// (modular) 64-bit integers: |t_q| <= 2^(60 - ceil(log2 n)) under 2 guard bits.
struct MedTrack {
  uint32_t W;          // total weight of the set
  uint32_t cum;        // running weight
  int64_t sum;         // running weighted sum
  uint32_t Wk;         // weight up to and including k
  int64_t Sk;          // weighted sum up to and including k
  int64_t m2;          // doubled median
  int state;           // 0 searching, 1 waiting for t_k+1, 2 done
};

__device__ __forceinline__ void med_init(MedTrack& m, uint32_t W) {
  m.W = W; m.cum = 0; m.sum = 0; m.Wk = 0; m.Sk = 0; m.m2 = 0; m.state = W ? 0 : 2;
}

__device__ __forceinline__ void med_push(MedTrack& m, uint32_t wv, int64_t t) {
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

// SAD2 of the tracked set with total weighted sum S
__device__ __forceinline__ uint64_t med_sad2(const MedTrack& m, int64_t S) {
  return (uint64_t)m.m2 * (uint64_t)(2u * m.Wk - m.W) + 2ull * (uint64_t)(S - 2 * m.Sk);
}

// Search key of one MAE candidate: ~D with D = SAD2(left) + SAD2(right) < 2^63, so the
// key is > 0 and "larger key = better" keeps the MSE path's reduction and tie-break (R9).
// tl: the node's rows in t order (len ln); left rows are those with lrank_f <= thr.
// m2L, m2R (if not null): the children's doubled medians (their leaf values if it wins).
__device__ __forceinline__ unsigned long long mae_walk(SA<uint8_t> tl, int ln, SA<uint8_t> lr, uint32_t thr,
                                                       SA<uint8_t> w, SA<int64_t> tq, uint32_t WL, int64_t SL,
                                                       uint32_t WR, int64_t SR, int64_t& m2L, int64_t& m2R) {
  MedTrack mL, mR;
  med_init(mL, WL);
  med_init(mR, WR);
  #pragma unroll 1
  for (int i = 0; i < ln; ++i) {
    const uint8_t r = tl[i];
    const uint32_t wv = w[r];
    const int64_t t = tq[r];
    if ((uint32_t)lr[r] <= thr) med_push(mL, wv, t); else med_push(mR, wv, t);
    if (mL.state == 2 && mR.state == 2) break;
  }
  m2L = mL.m2;
  m2R = mR.m2;
  return ~(med_sad2(mL, SL) + med_sad2(mR, SR));
}
// (Issuing the next element's loads one step ahead in this walk measured 2.9x slower for
// ExtraTrees + MAE -- profiles/r03k_mae_pf_ab.txt -- and is not used.)
__device__ __noinline__ unsigned long long mae_key(SA<uint8_t> tl, int ln, SA<uint8_t> lr, uint32_t thr,
                                                   SA<uint8_t> w, SA<int64_t> tq, uint32_t WL, int64_t SL,
                                                   uint32_t WR, int64_t SR) {
  int64_t a, b;
  return mae_walk(tl, ln, lr, thr, w, tq, WL, SL, WR, SR, a, b);
}

// Doubled weighted median (and, if sad2 != null, the doubled SAD) of the rows of a t-ordered
// segment selected by sel: 0 = all rows, 1 = side[r] != 0 (left child), 2 = side[r] == 0.
// Rows with weight 0 are absent (w = 0 adds nothing).
__device__ __noinline__ int64_t seg_median2(SA<uint8_t> tl, int ln, SA<uint8_t> w, SA<int64_t> tq,
                                            SA<uint8_t> side, int sel, uint32_t W, int64_t S, uint64_t* sad2) {
  MedTrack m;
  med_init(m, W);
  #pragma unroll 1
  for (int i = 0; i < ln && m.state != 2; ++i) {
    const uint8_t r = tl[i];
    if (sel == 1 && !side[r]) continue;
    if (sel == 2 && side[r]) continue;
    const uint32_t wv = w[r];
    if (wv) med_push(m, wv, tq[r]);
  }
  if (sad2) *sad2 = med_sad2(m, S);
  return m.m2;
}

// MAE candidate queue (R32).  The search loop appends its candidates to a per-warp ring
// (ballot-compacted; entry = node k | feature f << 8 | boundary rank << 16 | aux << 24 |
// WL << 48, and SL) and every 32 queued candidates are scored here one per lane, so each
// lane walks one candidate's t-ordered rows instead of the warp waiting on the few lanes
// that hold a candidate in a loop step (ExtraTrees: one candidate per segment).  The keys
// merge into the per-node best (mkey ...) under the search's total order (R9), which does
// not depend on the order in which candidates are merged.
__device__ __noinline__ void mae_flush(SA<ulonglong2> q, uint32_t qh, int nq, NodeSet cur, SA<uint8_t> L, int p,
                                       int ntr_max, SA<uint8_t> lrank, SA<uint8_t> w, SA<int64_t> tq,
                                       SA<unsigned long long> mkey, SA<uint32_t> maux, SA<uint32_t> mWL,
                                       SA<int64_t> mSL, SA<int64_t> med2) {
  const int lane = threadIdx.x & 31;
  __syncwarp();  // the entries written by every lane are visible
  int k = -1 - lane;
  unsigned long long key = 0ull;
  uint32_t aux = 0u, WL = 0u;
  int64_t SL = 0, m2L = 0, m2R = 0;
  if (lane < nq) {
    const ulonglong2 e = q[(qh + (uint32_t)lane) & (kMaeQ - 1)];
    k = (int)(e.x & 0xFFu);
    const int f = (int)((e.x >> 8) & 0xFFu);
    const uint32_t thr = (uint32_t)((e.x >> 16) & 0xFFu);
    aux = (uint32_t)((e.x >> 24) & 0xFFFFFFu);
    WL = (uint32_t)((e.x >> 48) & 0xFFFFu);
    SL = (int64_t)e.y;
    const uint32_t Wk = cur.W[k];
    const int64_t Sk = cur.S[k];
    key = mae_walk(L + (p * ntr_max + cur.start[k]), cur.len[k], lrank + f * ntr_max, thr, w, tq, WL, SL,
                   Wk - WL, Sk - SL, m2L, m2R);
  }
  __syncwarp();  // every entry is read before its ring slot is reused
  // the lowest lane of each node's group merges the group's candidates, then the node best
  bool lead = lane < nq;
  #pragma unroll 1
  for (int s = 0; s < nq; ++s) {
    const int ok = __shfl_sync(0xffffffffu, k, s);
    const unsigned long long okey = __shfl_sync(0xffffffffu, key, s);
    const uint32_t oaux = __shfl_sync(0xffffffffu, aux, s);
    const uint32_t oWL = __shfl_sync(0xffffffffu, WL, s);
    const int64_t oSL = __shfl_sync(0xffffffffu, SL, s);
    const int64_t om2L = __shfl_sync(0xffffffffu, m2L, s);
    const int64_t om2R = __shfl_sync(0xffffffffu, m2R, s);
    if (ok == k && s != lane) {
      if (s < lane) lead = false;
      else if (better(okey, oaux, key, aux)) { key = okey; aux = oaux; WL = oWL; SL = oSL; m2L = om2L; m2R = om2R; }
    }
  }
  if (lead && better(key, aux, mkey[k], maux[k])) {
    mkey[k] = key; maux[k] = aux; mWL[k] = WL; mSL[k] = SL;
    med2[2 * k] = m2L; med2[2 * k + 1] = m2R;  // the children's medians of the node's best so far
  }
  __syncwarp();
}

__device__ __noinline__ double median_leaf(int64_t m2, int F) { return scalbn(__ll2double_rn(m2), -F - 1); }

// ------------------------------------------------- profiling build only --
// RF_PHASE_TIMING: lane 0 of every warp adds the clock64 delta since the previous
// mark to g_phase_cyc[i] (phase names: DESIGN.md sec. 6).  Compiled out otherwise.
__device__ unsigned long long g_phase_cyc[kPhases];
#ifdef RF_PHASE_TIMING
#define PT_MARK(i)                                                              \
  do {                                                                          \
    const long long _t = clock64();                                             \
    if (lane == 0) atomicAdd(&g_phase_cyc[i], (unsigned long long)(_t - pt0)); \
    pt0 = _t;                                                                   \
  } while (0)
#else
#define PT_MARK(i) \
  do {             \
  } while (0)
#endif

// -------------------------------------------------------------- the kernel --
// TM: max test rows per lane.  kExtra: ExtraTrees split mode (R29).  kMae: MAE criterion (R32).
template <bool kFit, int TM, bool kExtra, bool kMae>
__global__ void __launch_bounds__(32 * kSmallMaxWpb, (kSmallMaxWpb <= 8 ? 2 : 1)) small_tree_kernel(SmallArgs a) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int p = a.p;
  const int ntr_max = stride_of(a.ntr_max);  // list stride: 4-byte aligned words (g)
#ifdef RF_PHASE_TIMING
  long long pt0 = clock64();
#endif

  // work item of this CTA: (mtry index, task, chunk of warp jobs)
  const int cta_per_mt = (a.nsub + a.wpb - 1) / a.wpb;
  int bid = blockIdx.x;
  const int cchunk = bid % cta_per_mt;
  bid /= cta_per_mt;
  const int tl = bid % a.ntask;
  const int mi = bid / a.ntask;
  // (through a shuffle: the compiler keeps it in a register instead of re-reading the parameter bank
  // with a dynamic index inside the search loop's divergent segment ends; A/B -2 %, rd2_38)
  const int m = __shfl_sync(0xffffffffu, a.mtrys[mi], 0);
  constexpr bool extra = kExtra;
  const int fs = feat_stride_of(a);
  const bool nodraw = no_draws(m, p, a.tie_draw, extra);

  Carve cv;
  CtaSmem cs;
  carve_cta(cv, cs, p, ntr_max, kFit ? 0 : a.nte_max, extra, kMae);
  WarpSmem ws;
  {
    const size_t cta_bytes = (cv.off + 15) / 16 * 16;
    Carve cw;
    WarpSmem dummy;
    carve_warp(cw, dummy, p, ntr_max, fs, extra, kFit, kMae);
    const size_t per_warp = (cw.off + 15) / 16 * 16;
    Carve mine(cta_bytes + per_warp * warp);
    carve_warp(mine, ws, p, ntr_max, fs, extra, kFit, kMae);
  }

  const int ntr = a.ntr[tl];
  const int nte = kFit ? 0 : a.nte[tl];
  const int F = *a.dF;
  const uint32_t* tr_rows = a.tr_rows + (size_t)tl * a.row_stride;

  // ---- CTA-shared task data
  {
    const uint8_t* go = a.ord + (size_t)tl * p * a.ntr_stride;
    const uint8_t* gr = a.lrank + (size_t)tl * p * a.ntr_stride;
    #pragma unroll 1
    for (int i = threadIdx.x; i < p * ntr; i += blockDim.x) {
      const int f = i / ntr, j = i - f * ntr;
      cs.ord[f * ntr_max + j] = go[(size_t)f * a.ntr_stride + j];
      cs.lrank[f * ntr_max + j] = gr[(size_t)f * a.ntr_stride + j];
      // ExtraTrees: value table by dense rank (rows of equal value write the same value)
      if (extra) cs.xs[f * ntr_max + gr[(size_t)f * a.ntr_stride + j]] = a.X[(size_t)tr_rows[j] * p + f];
    }
    #pragma unroll 1
    for (int i = threadIdx.x; i < ntr; i += blockDim.x) {
      const uint32_t g = tr_rows[i];
      cs.trr[i] = g;
      cs.tq[i] = a.tq[g];
    }
    if (kMae) {
      // t order of the training rows: rank of (t_q, local index) by counting (n_tr <= 255)
      __syncthreads();
      #pragma unroll 1
      for (int i = threadIdx.x; i < ntr; i += blockDim.x) {
        const int64_t ti = cs.tq[i];
        int rk = 0;
        #pragma unroll 1
        for (int j = 0; j < ntr; ++j) {
          const int64_t tj = cs.tq[j];
          rk += (tj < ti) || (tj == ti && j < i);
        }
        cs.tord[rk] = (uint8_t)i;
      }
    }
    #pragma unroll 1
    for (int i = threadIdx.x; i < 256; i += blockDim.x)
      cs.rcp2[i] = make_double2((double)i, i ? __ddiv_rn(1.0, (double)i) : 0.0);
    if (!kFit) {
      const uint32_t* te_rows = a.te_rows + (size_t)tl * a.row_stride;
      #pragma unroll 1
      for (int i = threadIdx.x; i < nte * p; i += blockDim.x) {
        const int r = i / p, f = i - r * p;
        cs.xte[i] = a.X[(size_t)te_rows[r] * p + f];
      }
    }
  }
  __syncthreads();
  PT_MARK(14);

  const int sub = cchunk * a.wpb + warp;
  if (sub >= a.nsub) return;
  const int t_begin = a.tree_lo + sub * a.Cw;
  const int t_end = min(t_begin + a.Cw, a.tree_hi);
  const int task = a.task0 + tl;

  uint32_t ncand = 0;  // candidate splits evaluated by this lane
  double acc[TM];      // test row lane + 32 s
#pragma unroll
  for (int s = 0; s < TM; ++s) acc[s] = 0.0;

  for (int t = t_begin; t < t_end; ++t) {
    uint32_t k0, k1;
    tree_key(a.seed, (uint32_t)task, (uint32_t)t, k0, k1);
    const size_t tree_slot = (size_t)(t - a.tree_lo);

    // ---- bootstrap (R2): n_tr draws with replacement -> u8 counts (n_tr <= 255)
    const SA<uint32_t> w32{ws.w.off};
    #pragma unroll 1
    for (int i = lane; i < (ntr + 3) / 4; i += 32) w32[i] = 0u;
    __syncwarp();
    if (a.bootstrap) {
      const int nblk = (ntr + 1) >> 1;
      #pragma unroll 1
      for (int b = lane; b < nblk; b += 32) {
        uint64_t d0, d1;
        philox_pair_ool(k0, k1, (uint32_t)b, 0u, 0u, kTagBoot, d0, d1);
        const uint32_t i0 = (uint32_t)mulhi64(d0, (uint64_t)ntr);
        atomicAdd(&w32[i0 >> 2], 1u << ((i0 & 3) * 8));
        if (2 * b + 1 < ntr) {
          const uint32_t i1 = (uint32_t)mulhi64(d1, (uint64_t)ntr);
          atomicAdd(&w32[i1 >> 2], 1u << ((i1 & 3) * 8));
        }
      }
    } else {
      #pragma unroll 1
      for (int i = lane; i < ntr; i += 32) ws.w[i] = 1;
    }
    __syncwarp();

    if (kFit && a.leaf_of_row)
      #pragma unroll 1
      for (int i = lane; i < ntr; i += 32)
        if (!ws.w[i]) a.leaf_of_row[tree_slot * a.n + tr_rows[i]] = -1;

    // ---- root statistics
    int64_t S = 0, mn = INT64_MAX, mx = INT64_MIN;
    uint32_t D = 0;
    #pragma unroll 1
    for (int i = lane; i < ntr; i += 32) {
      const uint32_t wv = ws.w[i];
      if (wv) {
        const int64_t v = cs.tq[i];
        S += (int64_t)wv * v;
        mn = v < mn ? v : mn;
        mx = v > mx ? v : mx;
        ++D;
      }
    }
    S = wsum_i64(S);
    mn = wmin_i64(mn);
    mx = wmax_i64(mx);
    D = (uint32_t)wsum_i64((int64_t)D);
    const uint32_t Wroot = (uint32_t)ntr;  // sum of multiplicities = n_tr draws

    uint32_t tcur = 0;  // packed: test row s -> open node (byte s), 0xFF = finished
    const bool root_leaf = (a.max_depth == 0) || ((int)D < a.min_split) || (mn == mx);
    if (root_leaf) {
      const double v = kMae ? median_leaf(seg_median2(cs.tord, ntr, ws.w, cs.tq, ws.w, 0, Wroot, S, nullptr), F)
                            : leaf_value(S, cs.rcp2[Wroot], F);
#pragma unroll
      for (int s = 0; s < TM; ++s)
        if (lane + 32 * s < nte) acc[s] += v;
      if (kFit && lane == 0) {
        Node16 nd;
        nd.feat = -1; nd.left = 0; nd.v = v;
        a.nodes[tree_slot * a.cap] = nd;
        a.thr_index[tree_slot * a.cap] = 0;
        a.tree_nnodes[tree_slot] = 1;
      }
      if (kFit && a.leaf_of_row)
        #pragma unroll 1
        for (int i = lane; i < ntr; i += 32)
          if (ws.w[i]) a.leaf_of_row[tree_slot * a.n + tr_rows[i]] = 0;
      __syncwarp();
      continue;
    }

    // ---- in-bag lists: stable compaction of the presorted orders by w > 0
    SA<uint8_t> L = ws.listA;
    SA<uint8_t> L2 = ws.listB;
    SA<uint8_t> pn = ws.pnA;
    SA<uint8_t> pn2 = ws.pnB;
    NodeSet cur = ws.cur, nxt = ws.nxt;
    #pragma unroll 1
    for (int f = 0; f < nlists_of(p, kMae); ++f) {
      // four entries per lane (one 32-bit word of the order), four ballots per step
      const SA<uint8_t> src = (kMae && f == p) ? cs.tord : cs.ord + f * ntr_max;
      const unsigned lt = lanemask_lt();
      uint32_t off = 0;
      #pragma unroll 1
      for (int c = 0; c < ntr; c += 128) {
        const int j = c + 4 * lane;
        const uint32_t rows4 = j < ntr ? *reinterpret_cast<const uint32_t*>(src.ptr() + j) : 0u;
        bool keep[4];
        unsigned bal[4];
        uint32_t before = off;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          keep[q] = j + q < ntr && ws.w[(rows4 >> (8 * q)) & 0xFFu] != 0;
          bal[q] = __ballot_sync(0xffffffffu, keep[q]);
          before += __popc(bal[q] & lt);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (keep[q]) L[f * ntr_max + before] = (uint8_t)(rows4 >> (8 * q));
          before += keep[q] ? 1u : 0u;
        }
        off += __popc(bal[0]) + __popc(bal[1]) + __popc(bal[2]) + __popc(bal[3]);
      }
    }
    #pragma unroll 1
    for (int i = lane; i < (int)D; i += 32) pn[i] = 0;
    if (lane == 0) {
      cur.start[0] = 0; cur.len[0] = (uint8_t)D; cur.W[0] = (uint16_t)Wroot; cur.S[0] = S;
      cur.heap[0] = 1ull;
      if (kFit) cur.bfs[0] = 0;
    }
    __syncwarp();

    int nOpen = 1;
    int N = (int)D;
    uint32_t curBase = 0, levelCount = 1;
    int depth = 0;
    PT_MARK(0);

    while (nOpen > 0) {
      // ---------------- (a) per node: prefix bases, reset best, feature draws
      {
        uint32_t carryW = 0;
        uint64_t carryS = 0;
        #pragma unroll 1
        for (int b0 = 0; b0 < nOpen; b0 += 32) {
          const int k = b0 + lane;
          const bool act = k < nOpen;
          const uint32_t Wk = act ? cur.W[k] : 0u;
          const uint64_t Sk = act ? (uint64_t)cur.S[k] : 0ull;
          uint32_t tW;
          uint64_t tS;
          const uint32_t eW = wscan_u32(Wk, tW);
          const uint64_t eS = wscan_u64(Sk, tS);
          if (act) {
            ws.bW[k] = carryW + eW;  // prefix of W over earlier open nodes
            ws.bS[k] = carryS + eS;
            ws.bkey[k] = 0ull;
            ws.baux[k] = 0x7FFFFFFFu;
          }
          carryW += tW;
          carryS += tS;
        }
      }
      PT_MARK(1);
      // feature draws (R4): partial Fisher-Yates; the draw order matters even for m = p
      // (ties go to the first drawn feature, R9).
      const int nblk = (m + 1) >> 1;
      // m = p under the lowest-feature tie-break (north_star; exact mode): the drawn set is all
      // features and the winner does not depend on the draw order, so the draws are skipped and
      // slot j holds feature j (same trees as the oracle's Fisher-Yates; ExtraTrees keeps its
      // draws: its thresholds are keyed by draw slot, R29)
      if (nodraw) {
        // nothing to draw: slot j is feature j (feat_of)
      } else if (p <= 16) {
        // L lanes per node share its Philox blocks; the swap indices (4 bits per slot) are
        // OR-combined across the group, then one lane applies the swaps to a nibble-packed
        // permutation in a register
        int Lg = 1;
        while (Lg * 2 * nOpen <= 32 && Lg < nblk) Lg *= 2;
        #pragma unroll 1
        for (int base = 0; base < nOpen * Lg; base += 32) {
          const int q = base + lane;
          const int k = q / Lg, sub = q & (Lg - 1);
          uint64_t sw = 0;
          if (k < nOpen) {
            const uint64_t h = cur.heap[k];
            #pragma unroll 1
            for (int b = sub; b < nblk; b += Lg) {
              uint64_t d0, d1;
              philox_pair_ool(k0, k1, (uint32_t)b, (uint32_t)h, (uint32_t)(h >> 32), kTagFeat, d0, d1);
              const int j = 2 * b;
              sw |= (uint64_t)(j + (int)mulhi64(d0, (uint64_t)(p - j))) << (4 * j);
              if (j + 1 < m) sw |= (uint64_t)(j + 1 + (int)mulhi64(d1, (uint64_t)(p - j - 1))) << (4 * j + 4);
            }
          }
          #pragma unroll 1
          for (int d = 1; d < Lg; d <<= 1) sw |= __shfl_xor_sync(0xffffffffu, sw, d);
          if (k < nOpen && sub == 0) {
            const SA<uint8_t> fp = ws.feat + k * fs;
            uint64_t perm = 0xFEDCBA9876543210ull;
            #pragma unroll 1
            for (int j = 0; j < m; ++j) {
              const int r = (int)((sw >> (4 * j)) & 0xFull);
              const uint64_t x = ((perm >> (4 * j)) ^ (perm >> (4 * r))) & 0xFull;
              perm ^= (x << (4 * j)) | (x << (4 * r));
              fp[j] = (uint8_t)((perm >> (4 * j)) & 0xFull);
            }
          }
        }
      } else {
      #pragma unroll 1
      for (int k = lane; k < nOpen; k += 32) {
        const SA<uint8_t> fp = ws.feat + k * fs;
        const uint64_t h = cur.heap[k];
        {
          #pragma unroll 1
          for (int f = 0; f < p; ++f) fp[f] = (uint8_t)f;
          #pragma unroll 1
          for (int j = 0; j < m; j += 2) {
            uint64_t d0, d1;
            philox_pair_ool(k0, k1, (uint32_t)(j >> 1), (uint32_t)h, (uint32_t)(h >> 32), kTagFeat, d0, d1);
            int r = j + (int)mulhi64(d0, (uint64_t)(p - j));
            uint8_t tmp = fp[j]; fp[j] = fp[r]; fp[r] = tmp;
            if (j + 1 < m) {
              r = j + 1 + (int)mulhi64(d1, (uint64_t)(p - j - 1));
              tmp = fp[j + 1]; fp[j + 1] = fp[r]; fp[r] = tmp;
            }
          }
        }
      }
      }
      __syncwarp();
      PT_MARK(2);
      if (extra) {
        // ExtraTrees (R29): per (node, draw slot) the random threshold in [lo, hi) of the
        // segment's values and its rank threshold = last dense rank with x <= thr
        // (kNone if lo = hi); one Philox block serves two slots
        #pragma unroll 1
        for (int q = lane; q < nOpen * nblk; q += 32) {
          const int k = q / nblk, b = q - k * nblk;
          const uint64_t h = cur.heap[k];
          uint64_t d0, d1;
          philox_pair_ool(k0, k1, (uint32_t)b, (uint32_t)h, (uint32_t)(h >> 32), kTagThr, d0, d1);
          const int st = cur.start[k], ln = cur.len[k];
          #pragma unroll 1
          for (int s = 0; s < 2 && 2 * b + s < m; ++s) {
            const int j = 2 * b + s;
            const int f = ws.feat[k * fs + j];
            const int fb = f * ntr_max;
            const int rlo = cs.lrank[fb + L[fb + st]], rhi = cs.lrank[fb + L[fb + st + ln - 1]];
            uint8_t bnd = kNone;
            if (rlo < rhi) {
              const double thr = extra_thr_draw(s ? d1 : d0, cs.xs[fb + rlo], cs.xs[fb + rhi]);
              int l = rlo, u = rhi;  // xs[l] <= thr < xs[u]
              while (u - l > 1) {
                const int mid = (l + u) >> 1;
                if (cs.xs[fb + mid] <= thr) l = mid; else u = mid;
              }
              bnd = (uint8_t)l;
            }
            ws.xb[k * fs + j] = bnd;
          }
        }
        __syncwarp();
        PT_MARK(3);
      }

      // ---------------- (b) search pass over (node, feature slot, position), node-major
      {
        const int E = m * N;
        const int Kc = (E + 31) >> 5;
        const int e0 = min(lane * Kc, E), e1 = min(e0 + Kc, E);
        const int cnt = e1 - e0;  // this lane's elements; the loops below run Kc steps in lock-step
        // cursor over (node k, feature slot j, index i in the segment)
        int k, j, i, st, ln, f, lbase;
        uint32_t Wk;
        int64_t Sk;
        {
          const int e = min(e0, E - 1);
          k = pn[min(e / m, N - 1)];
          st = cur.start[k];
          ln = cur.len[k];
          Wk = cur.W[k];
          Sk = cur.S[k];
          const int off = e - m * st;
          j = off / ln;
          i = off - j * ln;
          f = nodraw ? j : ws.feat[k * fs + j];
          lbase = f * ntr_max;
        }
        const int k_init = k, j_init = j, i_init = i, st_init = st, ln_init = ln, f_init = f;
        const uint32_t W_init = Wk;
        const int64_t S_init = Sk;
        // pass 1, direct form: a lane's start prefix is the segment base (m bW[k] + j W_k)
        // plus the sum over the segment's elements before i0 -- or, when shorter, W_k minus
        // the sum from i0 to the segment end.  Cost min(i0, ln - i0) per lane instead of Kc
        // plus a warp scan; taken when the warp's largest such cost is below Kc (deeper levels;
        // A/B on the full study: -6.5 % step time).
        const bool fwd = i <= ln - i;
        const int cdir = cnt > 0 ? (fwd ? i : ln - i) : 0;
        const int cmax = __reduce_max_sync(0xffffffffu, (unsigned)cdir);
        uint32_t cW;
        uint64_t cS;
        if (cmax < Kc) {
          const int q0 = fwd ? 0 : i;
          uint32_t pw = 0;
          uint64_t ps = 0;
          #pragma unroll 1
          for (int c = 0; c < cmax; ++c) {
            if (c < cdir) {
              const uint8_t r = L[lbase + st + q0 + c];
              const uint32_t wv = ws.w[r];
              pw += wv;
              ps += (uint64_t)((int64_t)wv * cs.tq[r]);
            }
          }
          cW = (uint32_t)m * ws.bW[k] + (uint32_t)j * Wk + (fwd ? pw : Wk - pw);
          cS = (uint64_t)m * ws.bS[k] + (uint64_t)j * (uint64_t)Sk + (fwd ? ps : (uint64_t)Sk - ps);
        } else {
        // pass 1: lane totals
          uint32_t lw = 0;
          uint64_t ls = 0;
          // the next element's row id is loaded while this element's weight and target load.
          // (Adding a whole segment's sums (W_k, S_k) instead of walking it measured 2.5 %
          // slower: the divergent variable-stride loop costs more than the skipped loads.)
          uint8_t r1 = L[lbase + st + i];
          #pragma unroll 1
          for (int c = 0; c < Kc; ++c) {
            const bool act = c < cnt;
            const uint8_t r = r1;
            const uint32_t wv = act ? (uint32_t)ws.w[r] : 0u;
            const int64_t tv = cs.tq[r];
            if (++i == ln && c + 1 < cnt) {
              i = 0;
              if (++j == m) {
                j = 0;
                ++k;
                st = cur.start[k];
                ln = cur.len[k];
              }
              f = nodraw ? j : ws.feat[k * fs + j];
              lbase = f * ntr_max;
            }
            r1 = L[lbase + st + min(i, ln - 1)];
            lw += wv;
            ls += (uint64_t)((int64_t)wv * tv);
          }
          uint32_t tW;
          uint64_t tS;
          cW = wscan_u32(lw, tW);
          cS = wscan_u64(ls, tS);
        }

        PT_MARK(4);
        // pass 2: prefix sums, candidates at distinct-value boundaries, best per node run
        k = k_init; j = j_init; i = i_init; st = st_init; ln = ln_init; f = f_init; lbase = f * ntr_max;
        Wk = W_init; Sk = S_init;
        const int hk = cnt > 0 ? k : -1;  // head node
        int rk = hk;                      // current run node
        unsigned long long hkey = 0ull, rkey = 0ull;
        uint32_t haux = 0x7FFFFFFFu, raux = 0x7FFFFFFFu;
        uint32_t hWL = 0, rWL = 0;   // left sums of the best candidate (children sums)
        int64_t hSL = 0, rSL = 0;
        // left sums of the current segment up to the element (relative to the segment start: they
        // restart at 0 at every segment start, the previous segment's sums having reached (W_k, S_k))
        uint32_t WLr = cW - ((uint32_t)m * ws.bW[k] + (uint32_t)j * Wk);
        int64_t SLr = (int64_t)(cS - ((uint64_t)m * ws.bS[k] + (uint64_t)j * (uint64_t)Sk));
        // MSE: the run best's key minus one, signed (-1 = none): G >= 0, so its bits compare as
        // signed integers and no "+ 1" is formed per candidate (exported as key = rkm1 + 1)
        long long rkm1 = -1;
        uint8_t r = L[lbase + st + i];
        uint32_t rkr = cs.lrank[lbase + r];
        // the element's weight and target are loaded one iteration ahead (off the
        // critical path of the prefix sums -> reciprocal table -> fp64 score chain)
        uint32_t wr = ws.w[r];
        int64_t tr = cs.tq[r];
        int xbj = extra ? (int)ws.xb[k * fs + j] : (int)kNone;  // ExtraTrees boundary of the segment
        // candidate aux minus the index: tie key << 16 | draw slot << 8 | node start, tie key =
        // the feature (north_star) or the draw slot (R9); ascending aux = preferred among equal keys
        const bool tie_draw = a.tie_draw != 0;
        uint32_t auxb = ((uint32_t)(tie_draw ? j : f) << 16) | ((uint32_t)j << 8) | (uint32_t)st;
        // the following segment (next draw slot of node k, or slot 0 of node k + 1): its feature
        // and start, fetched one segment ahead so that the element loop reads the next segment's
        // first entry on its main path (a select of the address) and a segment end only moves
        // registers -- segment ends are divergent (lanes reach them at different steps) and, with
        // ~10-element segments, fall in most lock-step iterations of the warp.  (Reads for a node
        // past the last open one return stale bytes that are never used; the feature is clamped
        // to < p so that the addresses formed from it stay inside shared memory.)
        int nf, nst;
        if (j + 1 < m) { nf = nodraw ? j + 1 : ws.feat[k * fs + j + 1]; nst = st; }
        else { nf = nodraw ? 0 : min((int)ws.feat[(k + 1) * fs], p - 1); nst = cur.start[k + 1]; }
        uint32_t qh = 0u, qt = 0u;  // MAE candidate ring: head, tail
        if (kMae && kExtra) {
          #pragma unroll 1
          for (int kk = lane; kk < nOpen; kk += 32) { ws.mkey[kk] = 0ull; ws.maux[kk] = 0x7FFFFFFFu; }
          __syncwarp();
        }
        // reciprocal-table entries of the next element, loaded one iteration ahead
        double2 ylN = cs.rcp2[(WLr + wr) & 0xFFu], yrN = cs.rcp2[(Wk - (WLr + wr)) & 0xFFu];
        #pragma unroll 1
        for (int c = 0; c < Kc; ++c) {
          const bool act = c < cnt;
          const uint32_t wv = act ? wr : 0u;
          WLr += wv;
          SLr += (int64_t)wv * tr;
          const bool hasNext = i + 1 < ln;
          // next element: this segment's next entry or the following segment's first (after the
          // lane's last element a stale row id < 256 is read and not used: every load below stays
          // inside the CTA's shared memory)
          const int nfb = nf * ntr_max;
          uint8_t rn = L[hasNext ? lbase + st + i + 1 : nfb + nst];
          uint32_t rkn = cs.lrank[(hasNext ? lbase : nfb) + rn];
          wr = ws.w[rn];
          tr = cs.tq[rn];
          const uint32_t WL = WLr;
          const int64_t SL = SLr;
          const uint32_t WR = Wk - WL;
          const int64_t SR = Sk - SL;
          const double dSL = __ll2double_rn(SL), dSR = __ll2double_rn(SR);
          const double2 yl = ylN, yr = yrN;  // = rcp2[WL], rcp2[WR] for active lanes
          const double gl = div_small(__dmul_rn(dSL, dSL), yl.x, yl.y);
          const double gr = div_small(__dmul_rn(dSR, dSR), yr.x, yr.y);
          const bool cand = act && hasNext && (extra ? (rkr <= (uint32_t)xbj && rkn > (uint32_t)xbj) : rkr != rkn);
          unsigned long long key;
          const uint32_t aux = auxb + (uint32_t)i;  // tie key << 16 | draw slot << 8 | position (R9)
          if (kMae && kExtra) {  // R32: queued, scored one per lane by mae_flush (left = rank <= rkr)
            key = 0ull;
            const uint32_t bal = __ballot_sync(0xffffffffu, cand);
            if (cand) {
              const uint32_t slot = (qt + (uint32_t)__popc(bal & ((1u << lane) - 1u))) & (kMaeQ - 1);
              ws.mq[slot] = make_ulonglong2((unsigned long long)k | ((unsigned long long)f << 8) |
                                                ((unsigned long long)rkr << 16) |
                                                ((unsigned long long)(aux & 0xFFFFFFu) << 24) |
                                                ((unsigned long long)WL << 48),
                                            (unsigned long long)SL);
            }
            qt += (uint32_t)__popc(bal);
            if (qt - qh >= 32u) {  // warp-uniform
              mae_flush(ws.mq, qh, 32, cur, L, p, ntr_max, cs.lrank, ws.w, cs.tq, ws.mkey, ws.maux, ws.mWL, ws.mSL, ws.med2);
              qh += 32u;
            }
          } else if (kMae) {  // exact CART: nearly every element is a candidate, scored in place
            key = cand ? mae_key(L + (p * ntr_max + st), ln, cs.lrank + lbase, rkr, ws.w, cs.tq, WL, SL, WR, SR)
                       : 0ull;
          } else {
            key = 0ull;
            const long long kb = __double_as_longlong(__dadd_rn(gl, gr));
            // a lane's running best improves O(log n) times over a segment: the update is a rare
            // branch rather than selects on every candidate
            if (__builtin_expect(cand && kb >= rkm1, 0)) {
              if (kb > rkm1 || aux < raux) { rkm1 = kb; raux = aux; rWL = WL; rSL = SL; }
            }
          }
          ncand += cand;
          if (kMae && better(key, aux, rkey, raux)) { rkey = key; raux = aux; rWL = WL; rSL = SL; }
          if (!hasNext && c + 1 < cnt) {
            // end of segment: next feature slot or next node.  Segments are contiguous in the
            // flattened order and each holds all rows of its node: the next segment's left sums
            // start at 0
            i = 0;
            WLr = 0u;
            SLr = 0;
            if (++j == m) {
              j = 0;
              if (!kMae) rkey = (unsigned long long)(rkm1 + 1);
              // node k complete inside this lane (no other lane reads its bW/bS any more)
              if (k == hk) { hkey = rkey; haux = raux; hWL = rWL; hSL = rSL; }
              else { ws.bkey[k] = rkey; ws.baux[k] = raux; ws.bW[k] = rWL; ws.bS[k] = (uint64_t)rSL; }
              rkey = 0ull; raux = 0x7FFFFFFFu;
              rkm1 = -1;
              ++k;
              rk = k;
              ln = cur.len[k];
              Wk = cur.W[k];
              Sk = cur.S[k];
            }
            f = nf;
            st = nst;
            lbase = nfb;
            if (extra) xbj = ws.xb[k * fs + j];
            auxb = ((uint32_t)(tie_draw ? j : f) << 16) | ((uint32_t)j << 8) | (uint32_t)st;
            if (j + 1 < m) { nf = nodraw ? j + 1 : ws.feat[k * fs + j + 1]; }
            else { nf = nodraw ? 0 : min((int)ws.feat[(k + 1) * fs], p - 1); nst = cur.start[k + 1]; }
          } else if (act) {
            ++i;
          }
          {
            const uint32_t WLn = WLr + wr;
            ylN = cs.rcp2[WLn & 0xFFu];
            yrN = cs.rcp2[(Wk - WLn) & 0xFFu];
          }
          r = rn;
          rkr = rkn;
        }
        if (!kMae) rkey = (unsigned long long)(rkm1 + 1);
        if (cnt > 0 && rk == hk) { hkey = rkey; haux = raux; hWL = rWL; hSL = rSL; }
        if (kMae && kExtra) {
          #pragma unroll 1
          while (qt != qh) {
            const int nq = (int)min(qt - qh, 32u);
            mae_flush(ws.mq, qh, nq, cur, L, p, ntr_max, cs.lrank, ws.w, cs.tq, ws.mkey, ws.maux, ws.mWL, ws.mSL, ws.med2);
            qh += (uint32_t)nq;
          }
        }
        // every lane has read its start node's prefix bases (bW/bS) before any lane
        // overwrites a border node's entries with its best below (racecheck)
        __syncwarp();
        // nodes on chunk borders: segmented suffix reduction of the head partials
        unsigned long long vkey = hkey;
        uint32_t vaux = haux, vWL = hWL;
        int64_t vSL = hSL;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int ok = __shfl_down_sync(0xffffffffu, hk, d);
          const unsigned long long okey = __shfl_down_sync(0xffffffffu, vkey, d);
          const uint32_t oaux = __shfl_down_sync(0xffffffffu, vaux, d);
          const uint32_t oWL = __shfl_down_sync(0xffffffffu, vWL, d);
          const int64_t oSL = __shfl_down_sync(0xffffffffu, vSL, d);
          if (lane + d < 32 && hk >= 0 && ok == hk && better(okey, oaux, vkey, vaux)) {
            vkey = okey; vaux = oaux; vWL = oWL; vSL = oSL;
          }
        }
        const int prev_tail = __shfl_up_sync(0xffffffffu, rk, 1);
        const unsigned long long prev_tkey = __shfl_up_sync(0xffffffffu, rkey, 1);
        const uint32_t prev_taux = __shfl_up_sync(0xffffffffu, raux, 1);
        const uint32_t prev_tWL = __shfl_up_sync(0xffffffffu, rWL, 1);
        const int64_t prev_tSL = __shfl_up_sync(0xffffffffu, rSL, 1);
        const int prev_head = __shfl_up_sync(0xffffffffu, hk, 1);
        const int next_head = __shfl_down_sync(0xffffffffu, hk, 1);
        if (hk >= 0) {
          // the first lane whose head is hk writes it, merging the previous lane's tail run
          if (lane == 0 || prev_head != hk) {
            if (lane > 0 && prev_tail == hk && better(prev_tkey, prev_taux, vkey, vaux)) {
              vkey = prev_tkey; vaux = prev_taux; vWL = prev_tWL; vSL = prev_tSL;
            }
            ws.bkey[hk] = vkey; ws.baux[hk] = vaux; ws.bW[hk] = vWL; ws.bS[hk] = (uint64_t)vSL;
          }
          // a tail run that does not continue into the next lane is a complete node
          if (rk != hk && !(lane < 31 && next_head == rk)) {
            ws.bkey[rk] = rkey; ws.baux[rk] = raux; ws.bW[rk] = rWL; ws.bS[rk] = (uint64_t)rSL;
          }
        }
      }
      __syncwarp();
      if (kMae && kExtra) {  // the queued candidates' per-node bests replace the (empty) in-loop ones
        #pragma unroll 1
        for (int kk = lane; kk < nOpen; kk += 32) {
          ws.bkey[kk] = ws.mkey[kk]; ws.baux[kk] = ws.maux[kk]; ws.bW[kk] = ws.mWL[kk];
          ws.bS[kk] = (uint64_t)ws.mSL[kk];
        }
        __syncwarp();
      }
      PT_MARK(5);

      // ---------------- (c) decisions and thresholds; first-row targets of the children
      #pragma unroll 1
      for (int k = lane; k < nOpen; k += 32) {
        const unsigned long long key = ws.bkey[k];
        ws.ncb[2 * k] = 0;
        ws.ncb[2 * k + 1] = 0;
        if (key) {
          const uint32_t aux = ws.baux[k];
          const int j = (int)((aux >> 8) & 0xFFu), bp = (int)(aux & 0xFFu);
          const int f = nodraw ? j : ws.feat[k * fs + j];
          const uint8_t ra = L[f * ntr_max + bp], rb = L[f * ntr_max + bp + 1];
          const uint32_t ga = cs.trr[ra], gb = cs.trr[rb];
          double thr;
          if (extra) {  // the drawn threshold of slot j (R29), recomputed from the segment's range
            const int st = cur.start[k], fb = f * ntr_max;
            const double lo = cs.xs[fb + cs.lrank[fb + L[fb + st]]];
            const double hi = cs.xs[fb + cs.lrank[fb + L[fb + st + cur.len[k] - 1]]];
            thr = extra_thr(k0, k1, cur.heap[k], j, lo, hi);
          } else {
            // (read-only-path loads (__ldg) here measured equal, profiles/r03n_x_ldg_ab.txt;
            // deferring these loads past the mark pass 0.5 % slower, rd2_19_ab_defer_thr.txt)
            thr = midpoint_thr(a.X[(size_t)ga * p + f], a.X[(size_t)gb * p + f]);
          }
          if (kMae && kFit) ws.bD[k] = ~key;  // cost D of the chosen split (importance)
          ws.bkey[k] = (unsigned long long)__double_as_longlong(thr);
          ws.baux[k] = ((uint32_t)f << 8) | (uint32_t)bp | 0x80000000u;  // feature, boundary, split flag
          if (kFit) ws.thrIdx[k] = a.grank[(size_t)f * a.n + ga];
          // child first-row targets for the constancy test in (d): in the next level's node table,
          // which (e) fills only after (d)
          nxt.S[k] = cs.tq[L[f * ntr_max + cur.start[k]]];
          nxt.heap[k] = (uint64_t)cs.tq[rb];
        }
      }
      __syncwarp();
      PT_MARK(6);

      // ---------------- (d) mark pass: go-left flags, child constancy (lock-step, no atomics)
      #pragma unroll 1
      for (int base = 0; base < N; base += 32) {
        const int pos = base + lane;
        if (pos < N) {
          const int k = pn[pos];
          const uint32_t aux = ws.baux[k];
          if (aux & 0x80000000u) {
            const int f = (int)((aux >> 8) & 0xFFu);
            const uint8_t r = L[f * ntr_max + pos];
            const int sd = pos <= (int)(aux & 0xFFu) ? 0 : 1;
            ws.side[r] = (uint8_t)(1 - sd);
            if (cs.tq[r] != (sd ? (int64_t)nxt.heap[k] : nxt.S[k])) ws.ncb[2 * k + sd] = 1;
          }
        }
      }
      __syncwarp();
      PT_MARK(7);

      // ---------------- (d') MAE (R32): weighted medians of the children of split nodes (leaf
      // values) and of unsplit open nodes, by one walk of the node's t-ordered rows each
      if (kMae) {
        #pragma unroll 1
        for (int k = lane; k < nOpen; k += 32) {
          const SA<uint8_t> tl = L + (p * ntr_max + cur.start[k]);
          const int ln = cur.len[k];
          const uint32_t aux = ws.baux[k];
          if (aux & 0x80000000u) {
            const uint32_t WLv = ws.bW[k];
            const int64_t SLv = (int64_t)ws.bS[k];
            if (!kExtra) {  // ExtraTrees: mae_flush stored the winning candidate's child medians
              ws.med2[2 * k] = seg_median2(tl, ln, ws.w, cs.tq, ws.side, 1, WLv, SLv, nullptr);
              ws.med2[2 * k + 1] = seg_median2(tl, ln, ws.w, cs.tq, ws.side, 2, cur.W[k] - WLv, cur.S[k] - SLv, nullptr);
            }
            if (kFit && a.imp) {  // importance: (SAD2(node) - D) 2^(-F-1) (R30, R32)
              uint64_t sad = 0;
              seg_median2(tl, ln, ws.w, cs.tq, ws.side, 0, cur.W[k], cur.S[k], &sad);
              ws.bD[k] = sad - ws.bD[k];
            }
          } else {
            ws.med2[2 * k] = seg_median2(tl, ln, ws.w, cs.tq, ws.side, 0, cur.W[k], cur.S[k], nullptr);
          }
        }
        __syncwarp();
      }

      // ---------------- (e) children, node emission, next-level tables
      int nSplitTotal = 0, nOpenNext = 0, Nnext = 0, NL = 0;
      {
        uint32_t carrySplit = 0, carryOpen = 0, carryPos = 0, carryL = 0;
        #pragma unroll 1
        for (int b0 = 0; b0 < nOpen; b0 += 32) {
          const int k = b0 + lane;
          const bool act = k < nOpen;
          const uint32_t aux = act ? ws.baux[k] : 0u;
          const bool sp = act && (aux & 0x80000000u);
          uint32_t WLv = 0, WRv = 0, lenL = 0, lenR = 0, nl = 0;
          int64_t SLv = 0, SRv = 0;
          bool openL = false, openR = false;
          if (sp) {
            WLv = ws.bW[k];
            SLv = (int64_t)ws.bS[k];
            WRv = cur.W[k] - WLv;
            SRv = cur.S[k] - SLv;
            nl = (aux & 0xFFu) - cur.start[k] + 1;
            lenL = nl;
            lenR = cur.len[k] - nl;
            const bool capd = (a.max_depth >= 0) && (depth + 1 >= a.max_depth);
            openL = !capd && (int)lenL >= a.min_split && ws.ncb[2 * k];
            openR = !capd && (int)lenR >= a.min_split && ws.ncb[2 * k + 1];
          }
          // the four counters share one warp scan, one byte each: every total is <= 255
          // (splits and open children <= N/2 < 128, positions and left rows <= N <= 255)
          uint32_t tPacked;
          const uint32_t ePacked = wscan_u32((sp ? 1u : 0u) | (((openL ? 1u : 0u) + (openR ? 1u : 0u)) << 8) |
                                                 (((openL ? lenL : 0u) + (openR ? lenR : 0u)) << 16) |
                                                 ((sp ? nl : 0u) << 24),
                                             tPacked);
          const uint32_t eSp = ePacked & 0xFFu, eOpen = (ePacked >> 8) & 0xFFu, ePos = (ePacked >> 16) & 0xFFu,
                         eL = ePacked >> 24;
          const uint32_t tSp = tPacked & 0xFFu, tOpen = (tPacked >> 8) & 0xFFu, tPos = (tPacked >> 16) & 0xFFu,
                         tL = tPacked >> 24;
          if (sp) {
            const uint32_t childBase = curBase + levelCount + 2 * (carrySplit + eSp);
            if (kFit) ws.chBase[k] = (uint16_t)childBase;
            uint32_t oi = carryOpen + eOpen;
            uint32_t ps = carryPos + ePos;
            double vL = 0.0, vR = 0.0;
            if (openL) {
              nxt.start[oi] = (uint8_t)ps; nxt.len[oi] = (uint8_t)lenL;
              nxt.W[oi] = (uint16_t)WLv; nxt.S[oi] = SLv;
              nxt.heap[oi] = 2ull * cur.heap[k];
              if (kFit) nxt.bfs[oi] = (uint16_t)childBase;
              ws.chOpen[2 * k] = (uint8_t)oi;
              ++oi; ps += lenL;
            } else {
              vL = kMae ? median_leaf(ws.med2[2 * k], F) : leaf_value(SLv, cs.rcp2[WLv], F);
              ws.chOpen[2 * k] = kNone;
            }
            if (openR) {
              nxt.start[oi] = (uint8_t)ps; nxt.len[oi] = (uint8_t)lenR;
              nxt.W[oi] = (uint16_t)WRv; nxt.S[oi] = SRv;
              nxt.heap[oi] = 2ull * cur.heap[k] + 1ull;
              if (kFit) nxt.bfs[oi] = (uint16_t)(childBase + 1);
              ws.chOpen[2 * k + 1] = (uint8_t)oi;
            } else {
              vR = kMae ? median_leaf(ws.med2[2 * k + 1], F) : leaf_value(SRv, cs.rcp2[WRv], F);
              ws.chOpen[2 * k + 1] = kNone;
            }
            cur.S[k] = __double_as_longlong(vL);  // routing leaf values (cur.S / cur.heap are read above)
            cur.heap[k] = (uint64_t)__double_as_longlong(vR);
            {
              // packed partition record: start | baseL | dstL | dstR | openL | openR | split
              const uint64_t dL = openL ? nxt.start[ws.chOpen[2 * k]] : kNone;
              const uint64_t dR = openR ? nxt.start[ws.chOpen[2 * k + 1]] : kNone;
              ws.bS[k] = (uint64_t)cur.start[k] | ((uint64_t)((carryL + eL) & 0xFFu) << 8) | (dL << 16) |
                         (dR << 24) | ((uint64_t)ws.chOpen[2 * k] << 32) |
                         ((uint64_t)ws.chOpen[2 * k + 1] << 40) | (1ull << 48);
            }
            if (kFit) {
              Node16* tn = a.nodes + tree_slot * a.cap;
              uint32_t* ti = a.thr_index + tree_slot * a.cap;
              const uint32_t me = cur.bfs[k];
              Node16 nd;
              nd.feat = (int32_t)((aux >> 8) & 0xFFu);
              nd.left = childBase;
              nd.v = __longlong_as_double((long long)ws.bkey[k]);
              tn[me] = nd;
              ti[me] = ws.thrIdx[k];
              if (!openL) { Node16 l; l.feat = -1; l.left = 0; l.v = vL; tn[childBase] = l; ti[childBase] = 0; }
              if (!openR) { Node16 r; r.feat = -1; r.left = 0; r.v = vR; tn[childBase + 1] = r; ti[childBase + 1] = 0; }
              if (a.imp)  // feature importance (MDI, NEXT-3; MAE: R32)
                atomicAdd(&a.imp[tree_slot * p + nd.feat],
                          kMae ? scalbn(__ull2double_rn(ws.bD[k]), -F - 1) : mdi_decrease(WLv, SLv, WRv, SRv, F));
            }
          } else if (act) {
            // open node without any candidate split: leaf (R11)
            const double v = kMae ? median_leaf(ws.med2[2 * k], F) : leaf_value(cur.S[k], cs.rcp2[cur.W[k]], F);
            cur.S[k] = __double_as_longlong(v);
            ws.bS[k] = 0ull;  // partition record: not split
            if (kFit) {
              Node16 nd;
              nd.feat = -1; nd.left = 0; nd.v = v;
              a.nodes[tree_slot * a.cap + cur.bfs[k]] = nd;
              a.thr_index[tree_slot * a.cap + cur.bfs[k]] = 0;
            }
          }
          carrySplit += tSp;
          carryOpen += tOpen;
          carryPos += tPos;
          carryL += tL;
        }
        nSplitTotal = (int)carrySplit;
        nOpenNext = (int)carryOpen;
        Nnext = (int)carryPos;
        NL = (int)carryL;
      }
      __syncwarp();
      PT_MARK(8);

      // ---------------- (f) route the task's test rows one level down
      if (!kFit) {
#pragma unroll
        for (int s = 0; s < TM; ++s) {
          const int r = lane + 32 * s;
          const uint32_t c = (tcur >> (8 * s)) & 0xFFu;
          if (r < nte && c != kNone) {
            const int k = (int)c;
            const uint32_t aux = ws.baux[k];
            uint32_t nc_;
            if (!(aux & 0x80000000u)) {
              acc[s] += __longlong_as_double(cur.S[k]);
              nc_ = kNone;
            } else {
              const int f = (int)((aux >> 8) & 0xFFu);
              const double thr = __longlong_as_double((long long)ws.bkey[k]);
              const int sd = (cs.xte[(size_t)r * p + f] <= thr) ? 0 : 1;
              nc_ = ws.chOpen[2 * k + sd];
              if (nc_ == kNone) acc[s] += __longlong_as_double(sd ? (long long)cur.heap[k] : cur.S[k]);
            }
            tcur = (tcur & ~(0xFFu << (8 * s))) | (nc_ << (8 * s));
          }
        }
      }
      PT_MARK(9);
      __syncwarp();  // the routing above reads the thresholds in bkey, which desc aliases

      // ---------------- (g) stable partition of all p lists (feature-major), ping-pong.
      // One pass in 32-element chunks: a ballot of go-left flags gives every
      // element its rank among the left rows before it; the node record gives
      // the child segments (bS[k] holds the packed record, see (e)).
      const bool rows_debug = kFit && a.leaf_of_row != nullptr;
      if (nOpenNext > 0 || rows_debug) {
        const unsigned lt = lanemask_lt();
        // list 0: also writes the next level's position -> node map (and debug leaf rows).
        // (Folding list 0 into the four-wide pass below, with the descriptors and child
        // indices built in a pass of their own, measured 2 % slower.)
        // builds the per-position descriptor shared by the other lists:
        //   dL | dR << 8 | leftBase << 16 | start << 24, or ~0 for positions of unsplit nodes
        uint32_t carry = 0;
        #pragma unroll 1
        for (int base = 0; base < N; base += 32) {
          const int pos = base + lane;
          const bool valid = pos < N;
          uint64_t info = 0;
          uint8_t r = 0;
          int k = 0;
          bool left = false;
          if (valid) {
            k = pn[pos];
            info = ws.bS[k];
            r = L[pos];
            left = ((info >> 48) & 1u) && ws.side[r];
            ws.desc[pos] = ((info >> 48) & 1u) ? (uint32_t)((info >> 16) & 0xFFFFu) |
                                                     ((uint32_t)((info >> 8) & 0xFFu) << 16) |
                                                     ((uint32_t)(info & 0xFFu) << 24)
                                               : 0xFFFFFFFFu;
          }
          const unsigned bal = __ballot_sync(0xffffffffu, left);
          if (valid) {
            if ((info >> 48) & 1u) {
              const uint32_t st = (uint32_t)(info & 0xFFu);
              const uint32_t leftBefore = carry + __popc(bal & lt) - (uint32_t)((info >> 8) & 0xFFu);
              const uint32_t sh = left ? 0u : 8u;
              const uint32_t d = (uint32_t)(info >> (16 + sh)) & 0xFFu;  // child segment start
              if (d != kNone) {
                const uint32_t dest = d + (left ? leftBefore : ((uint32_t)pos - st) - leftBefore);
                L2[dest] = r;
                pn2[dest] = (uint8_t)(info >> (32 + sh));
              } else if (rows_debug) {
                a.leaf_of_row[tree_slot * a.n + tr_rows[r]] = (int32_t)(ws.chBase[k] + (left ? 0 : 1));
              }
            } else if (rows_debug) {
              a.leaf_of_row[tree_slot * a.n + tr_rows[r]] = (int32_t)cur.bfs[k];
            }
          }
          carry += __popc(bal);
        }
        // descriptors of the padding positions N .. 4 ceil(N / 4) - 1 (read by the four-wide pass)
        if (lane < ((4 - (N & 3)) & 3)) ws.desc[N + lane] = 0xFFFFFFFFu;
        __syncwarp();
        PT_MARK(10);
        // lists 1..p-1, flattened feature-major in chunks of 4 positions (one 32-bit word of
        // a list, one 16-byte load of descriptors): chunk c -> list 1 + c / nc4, positions
        // 4 (c % nc4) .. +3 (c / nc4 exactly via a float reciprocal: c < 2^16).  Four
        // ballots give each element its rank among the left rows before it.  (Issuing the next
        // step's loads one step ahead measured 0.9 % slower, profiles/rd2_20_ab_part_pf.txt.)
        const int nc4 = (N + 3) >> 2;
        const int C = (nlists_of(p, kMae) - 1) * nc4;
        // the lane's chunk (list fi + 1, word q) advances by 32 chunks per step
        const int dfi = 32 / nc4, dq = 32 - dfi * nc4;
        int fi = lane / nc4, q = lane - fi * nc4;
        carry = 0;
        #pragma unroll 1
        for (int base = 0; base < C; base += 32) {
          const bool valid = base + lane < C;
          const int q4 = q * 4;
          const int f = fi + 1;
          uint32_t rows4 = 0;
          uint4 d4 = make_uint4(~0u, ~0u, ~0u, ~0u);
          if (valid) {
            rows4 = *reinterpret_cast<const uint32_t*>(L.ptr() + f * ntr_max + q4);
            d4 = *reinterpret_cast<const uint4*>(ws.desc.ptr() + q4);
          }
          uint32_t dsc[4] = {d4.x, d4.y, d4.z, d4.w};
          bool left[4];
          unsigned bal[4];
          uint32_t before = carry;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            // (padding positions N .. 4 nc4 - 1 hold ~0 descriptors, written by the list-0 pass)
            left[i] = dsc[i] != 0xFFFFFFFFu && ws.side[(rows4 >> (8 * i)) & 0xFFu];
            bal[i] = __ballot_sync(0xffffffffu, left[i]);
            before += __popc(bal[i] & lt);
          }
          before -= (uint32_t)fi * (uint32_t)NL;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const uint32_t d = left[i] ? (dsc[i] & 0xFFu) : ((dsc[i] >> 8) & 0xFFu);
            const uint32_t leftBefore = before - ((dsc[i] >> 16) & 0xFFu);
            const uint32_t dest = d + (left[i] ? leftBefore : ((uint32_t)(q4 + i) - (dsc[i] >> 24)) - leftBefore);
            // entries of leaf children, unsplit nodes and padding (d = kNone) go to a trash byte:
            // an unconditional store instead of a branch per entry
            const uint32_t at = d != kNone ? L2.off + (uint32_t)(f * ntr_max) + dest : ws.trash.off + (uint32_t)lane;
            SA<uint8_t>{at}[0] = (uint8_t)(rows4 >> (8 * i));
            before += left[i] ? 1u : 0u;
          }
          carry += __popc(bal[0]) + __popc(bal[1]) + __popc(bal[2]) + __popc(bal[3]);
          q += dq;
          fi += dfi;
          if (q >= nc4) { q -= nc4; ++fi; }
        }
      }
      PT_MARK(11);
      // advance to the next level
      {
        const NodeSet tmp = cur; cur = nxt; nxt = tmp;
        const SA<uint8_t> t8 = L; L = L2; L2 = t8;
        const SA<uint8_t> tp = pn; pn = pn2; pn2 = tp;
      }
      curBase += levelCount;
      levelCount = 2u * (uint32_t)nSplitTotal;
      nOpen = nOpenNext;
      N = Nnext;
      ++depth;
      __syncwarp();
      PT_MARK(12);
    }
    if (kFit && lane == 0) a.tree_nnodes[tree_slot] = curBase + levelCount;
    __syncwarp();
    PT_MARK(13);
  }

  if (a.cand) {
    unsigned long long c = ncand;
    for (int d = 16; d > 0; d >>= 1) c += __shfl_xor_sync(0xffffffffu, c, d);
    if (lane == 0) atomicAdd(a.cand, c);
  }
  if (!kFit) {
    double* out = a.partial + (((size_t)mi * a.ntask + tl) * a.nsub + sub) * a.nte_max;
#pragma unroll
    for (int s = 0; s < TM; ++s) {
      const int r = lane + 32 * s;
      if (r < nte) out[r] = acc[s];
    }
  }
}

}  // namespace

size_t small_tree_smem_bytes(const SmallArgs& a, int /*mmax*/) {
  Carve c;
  CtaSmem cs;
  carve_cta(c, cs, a.p, stride_of(a.ntr_max), a.fit_mode ? 0 : a.nte_max, a.extra != 0, a.mae != 0);
  const size_t cta = (c.off + 15) / 16 * 16;
  Carve w;
  WarpSmem ws;
  carve_warp(w, ws, a.p, stride_of(a.ntr_max), feat_stride_of(a), a.extra != 0, a.fit_mode != 0, a.mae != 0);
  const size_t per_warp = (w.off + 15) / 16 * 16;
  return cta + per_warp * a.wpb + kReadSlack;
}

// calls fn(kernel) with the variant for (fit mode, test rows per lane, split mode, criterion)
template <bool kFit, int TM, bool kExtra, typename Fn>
static auto with_crit(const SmallArgs& a, Fn&& fn) {
  return a.mae ? fn(small_tree_kernel<kFit, TM, kExtra, true>) : fn(small_tree_kernel<kFit, TM, kExtra, false>);
}
template <bool kFit, int TM, typename Fn>
static auto with_split(const SmallArgs& a, Fn&& fn) {
  return a.extra ? with_crit<kFit, TM, true>(a, fn) : with_crit<kFit, TM, false>(a, fn);
}
template <typename Fn>
static auto with_variant(const SmallArgs& a, Fn&& fn) {
  if (a.fit_mode) return with_split<true, 1>(a, fn);
  const int TMn = (a.nte_max + 31) / 32;
  if (TMn <= 1) return with_split<false, 1>(a, fn);
  if (TMn <= 2) return with_split<false, 2>(a, fn);
  return with_split<false, 8>(a, fn);
}

int small_tree_ctas_per_sm(const SmallArgs& a) {
  const size_t smem = small_tree_smem_bytes(a, 0);
  if (smem > 227 * 1024) return 0;
  return with_variant(a, [&](void (*kern)(SmallArgs)) {
    if (allow_max_dynamic_smem(kern) != cudaSuccess) return 0;
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, 32 * a.wpb, smem) != cudaSuccess) return 0;
    return nb;
  });
}

bool small_tree_phase_timing_enabled() {
#ifdef RF_PHASE_TIMING
  return true;
#else
  return false;
#endif
}

cudaError_t small_tree_phase_cycles(uint64_t* out, bool reset) {
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpyFromSymbol(out, g_phase_cyc, sizeof(unsigned long long) * kPhases);
  if (e == cudaSuccess && reset) {
    static const unsigned long long zeros[kPhases] = {};
    e = cudaMemcpyToSymbol(g_phase_cyc, zeros, sizeof zeros);
  }
  return e;
}

cudaError_t launch_small_tree(const SmallArgs& a, cudaStream_t s) {
  const size_t smem = small_tree_smem_bytes(a, 0);
  const int cta_per_mt = (a.nsub + a.wpb - 1) / a.wpb;
  const long long grid = (long long)a.n_mtry * a.ntask * cta_per_mt;
  if (grid <= 0) return cudaSuccess;
  return with_variant(a, [&](void (*kern)(SmallArgs)) {
    cudaError_t e = allow_max_dynamic_smem(kern);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)grid, 32 * a.wpb, smem, s>>>(a);
    note_launch();
    return cudaGetLastError();
  });
}

}  // namespace rf
