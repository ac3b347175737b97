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
//   (G desc, feature asc, threshold rank asc) (R9); threshold midway (R8);
//   leaf if depth cap, < min_split distinct rows, constant t_q or no
//   candidate (R11); leaf value fl(S/W) 2^-F (R13).
//
// Layout per warp (shared memory): in-bag row lists of every feature, each
// node-grouped and x-sorted (u8 local row ids), a position -> open-node map,
// node tables of the current and the next level.  Per level: m search passes
// (lane-serial runs of K = ceil(N/32) positions + one warp scan; node sums
// recovered as global prefix minus the node's base), one mark pass (go-left
// flags, child sums, child constancy), p stable in-place partition passes
// (ballot-free: lane-serial counts + warp scan).
//
// CV mode routes the task's test rows level by level and accumulates their
// leaf values per warp job; fit mode writes BFS-ordered 16-byte nodes.
#include "small_tree.cuh"

namespace rf {
namespace {

struct Carve {
  char* base;
  size_t off;
  __host__ __device__ Carve(char* b) : base(b), off(0) {}
  template <typename T>
  __host__ __device__ T* take(size_t count, size_t align = 8) {
    off = (off + align - 1) / align * align;
    T* p = reinterpret_cast<T*>(base + off);
    off += count * sizeof(T);
    return p;
  }
};

struct CtaSmem {
  uint8_t* ord;     // [p][ntr_max]
  uint8_t* lrank;   // [p][ntr_max]
  int64_t* tq;      // [ntr_max]
  double* xte;      // [nte_max][p]
};

struct NodeSet {  // one level of open nodes
  uint8_t* start;
  uint8_t* len;
  uint32_t* W;
  int64_t* S;
  uint64_t* heap;
  uint32_t* bfs;
};

struct WarpSmem {
  uint8_t* w;       // [ntr_max] bootstrap multiplicities
  uint8_t* list;    // [p][ntr_max]
  uint8_t* pnode;   // [ntr_max]
  uint8_t* pnode2;  // [ntr_max]
  uint8_t* side;    // [ntr_max] by local row: 1 = goes left
  NodeSet cur, nxt;
  uint32_t* baseW;
  int64_t* baseS;
  uint8_t* feat;    // [NMAX][p]
  unsigned long long* bestKey;
  uint32_t* bestF;
  uint32_t* bestPos;
  unsigned long long* passKey;
  uint32_t* passPos;
  uint8_t* split;
  double* thr;
  uint32_t* thrIdx;
  uint32_t* WL;
  int64_t* SL;
  int64_t* tqfL;
  int64_t* tqfR;
  uint8_t* nc;      // bit0: left child non-constant, bit1: right
  uint8_t* chOpen;  // [NMAX][2]
  double* chVal;    // [NMAX][2]
  uint32_t* baseL;
};

__host__ __device__ inline int nmax_of(int ntr_max) { return ntr_max / 2 + 1; }

__host__ __device__ inline void carve_cta(Carve& c, CtaSmem& s, int p, int ntr_max, int nte_max) {
  s.ord = c.take<uint8_t>((size_t)p * ntr_max, 16);
  s.lrank = c.take<uint8_t>((size_t)p * ntr_max, 16);
  s.tq = c.take<int64_t>(ntr_max, 16);
  s.xte = c.take<double>((size_t)nte_max * p, 16);
}

__host__ __device__ inline void carve_nodeset(Carve& c, NodeSet& s, int NM) {
  s.start = c.take<uint8_t>(NM, 4);
  s.len = c.take<uint8_t>(NM, 4);
  s.W = c.take<uint32_t>(NM, 4);
  s.S = c.take<int64_t>(NM, 8);
  s.heap = c.take<uint64_t>(NM, 8);
  s.bfs = c.take<uint32_t>(NM, 4);
}

__host__ __device__ inline void carve_warp(Carve& c, WarpSmem& s, int p, int ntr_max, bool need_feat) {
  const int NM = nmax_of(ntr_max);
  s.w = c.take<uint8_t>((ntr_max + 3) / 4 * 4, 16);
  s.list = c.take<uint8_t>((size_t)p * ntr_max, 16);
  s.pnode = c.take<uint8_t>(ntr_max, 4);
  s.pnode2 = c.take<uint8_t>(ntr_max, 4);
  s.side = c.take<uint8_t>(ntr_max, 4);
  carve_nodeset(c, s.cur, NM);
  carve_nodeset(c, s.nxt, NM);
  s.baseW = c.take<uint32_t>(NM, 4);
  s.baseS = c.take<int64_t>(NM, 8);
  s.feat = need_feat ? c.take<uint8_t>((size_t)NM * p, 4) : nullptr;
  s.bestKey = c.take<unsigned long long>(NM, 8);
  s.bestF = c.take<uint32_t>(NM, 4);
  s.bestPos = c.take<uint32_t>(NM, 4);
  s.passKey = c.take<unsigned long long>(NM, 8);
  s.passPos = c.take<uint32_t>(NM, 4);
  s.split = c.take<uint8_t>(NM, 4);
  s.thr = c.take<double>(NM, 8);
  s.thrIdx = c.take<uint32_t>(NM, 4);
  s.WL = c.take<uint32_t>(NM, 4);
  s.SL = c.take<int64_t>(NM, 8);
  s.tqfL = c.take<int64_t>(NM, 8);
  s.tqfR = c.take<int64_t>(NM, 8);
  s.nc = c.take<uint8_t>((NM + 3) / 4 * 4, 4);
  s.chOpen = c.take<uint8_t>((size_t)NM * 2, 4);
  s.chVal = c.take<double>((size_t)NM * 2, 8);
  s.baseL = c.take<uint32_t>(NM, 4);
}

// ---------------------------------------------------------------- warp ops --
__device__ __forceinline__ uint32_t wscan_u32(uint32_t v, uint32_t& total) {
  const int lane = threadIdx.x & 31;
  uint32_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  total = __shfl_sync(0xffffffffu, x, 31);
  return x - v;
}

__device__ __forceinline__ int64_t wscan_i64(int64_t v, int64_t& total) {
  const int lane = threadIdx.x & 31;
  int64_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  total = __shfl_sync(0xffffffffu, x, 31);
  return x - v;
}

__device__ __forceinline__ int64_t wsum_i64(int64_t v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}
__device__ __forceinline__ int64_t wmin_i64(int64_t v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) { int64_t o = __shfl_xor_sync(0xffffffffu, v, d); v = o < v ? o : v; }
  return v;
}
__device__ __forceinline__ int64_t wmax_i64(int64_t v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) { int64_t o = __shfl_xor_sync(0xffffffffu, v, d); v = o > v ? o : v; }
  return v;
}

__device__ __forceinline__ double leaf_value(int64_t S, uint32_t W, int F) {
  return scalbn(__ddiv_rn(__ll2double_rn(S), __ll2double_rn((long long)W)), -F);
}

constexpr uint8_t kNone = 0xFF;

// -------------------------------------------------------------- the kernel --
// KM: max positions per lane (ceil(n_tr/32)); TM: max test rows per lane.
template <bool kFit, int KM, int TM>
__global__ void __launch_bounds__(128) small_tree_kernel(SmallArgs a) {
  extern __shared__ __align__(16) char smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int p = a.p;
  const int ntr_max = a.ntr_max;

  // work item of this CTA: (mtry index, task, chunk of warp jobs)
  const int cta_per_mt = (a.nsub + a.wpb - 1) / a.wpb;
  int bid = blockIdx.x;
  const int cchunk = bid % cta_per_mt;
  bid /= cta_per_mt;
  const int tl = bid % a.ntask;
  const int mi = bid / a.ntask;
  const int mtry = a.mtrys[mi];
  const bool need_feat = mtry < p;
  bool any_feat = false;
  for (int i = 0; i < a.n_mtry; ++i) any_feat |= (a.mtrys[i] < p);

  Carve cv(smem);
  CtaSmem cs;
  carve_cta(cv, cs, p, ntr_max, kFit ? 0 : a.nte_max);
  WarpSmem ws;
  {
    size_t cta_bytes = (cv.off + 15) / 16 * 16;
    Carve cw(nullptr);
    WarpSmem dummy;
    carve_warp(cw, dummy, p, ntr_max, any_feat);
    size_t per_warp = (cw.off + 15) / 16 * 16;
    Carve mine(smem + cta_bytes + per_warp * warp);
    carve_warp(mine, ws, p, ntr_max, any_feat);
  }

  const int ntr = a.ntr[tl];
  const int nte = kFit ? 0 : a.nte[tl];
  const int F = *a.dF;
  const uint32_t* tr_rows = a.tr_rows + (size_t)tl * a.row_stride;

  // ---- CTA-shared task data
  {
    const uint8_t* go = a.ord + (size_t)tl * p * a.ntr_stride;
    const uint8_t* gr = a.lrank + (size_t)tl * p * a.ntr_stride;
    for (int i = threadIdx.x; i < p * ntr; i += blockDim.x) {
      int f = i / ntr, j = i - f * ntr;
      cs.ord[f * ntr_max + j] = go[(size_t)f * a.ntr_stride + j];
      cs.lrank[f * ntr_max + j] = gr[(size_t)f * a.ntr_stride + j];
    }
    for (int i = threadIdx.x; i < ntr; i += blockDim.x) cs.tq[i] = a.tq[tr_rows[i]];
    if (!kFit) {
      const uint32_t* te_rows = a.te_rows + (size_t)tl * a.row_stride;
      for (int i = threadIdx.x; i < nte * p; i += blockDim.x) {
        int r = i / p, f = i - r * p;
        cs.xte[i] = a.X[(size_t)te_rows[r] * p + f];
      }
    }
  }
  __syncthreads();

  const int sub = cchunk * a.wpb + warp;
  if (sub >= a.nsub) return;
  const int t_begin = a.tree_lo + sub * a.Cw;
  const int t_end = min(t_begin + a.Cw, a.tree_hi);
  const int task = a.task0 + tl;

  double acc[TM];  // test row lane + 32 s
#pragma unroll
  for (int s = 0; s < TM; ++s) acc[s] = 0.0;

  for (int t = t_begin; t < t_end; ++t) {
    uint32_t k0, k1;
    tree_key(a.seed, (uint32_t)task, (uint32_t)t, k0, k1);
    const size_t tree_slot = (size_t)(t - a.tree_lo);

    // ---- bootstrap (R2): n_tr draws with replacement -> u8 counts (n_tr <= 255)
    for (int i = lane; i < (ntr + 3) / 4; i += 32) reinterpret_cast<uint32_t*>(ws.w)[i] = 0u;
    __syncwarp();
    if (a.bootstrap) {
      const int nblk = (ntr + 1) >> 1;
      for (int b = lane; b < nblk; b += 32) {
        uint64_t d0, d1;
        philox_pair(k0, k1, (uint32_t)b, 0u, 0u, kTagBoot, d0, d1);
        uint32_t i0 = (uint32_t)mulhi64(d0, (uint64_t)ntr);
        atomicAdd(reinterpret_cast<uint32_t*>(ws.w) + (i0 >> 2), 1u << ((i0 & 3) * 8));
        if (2 * b + 1 < ntr) {
          uint32_t i1 = (uint32_t)mulhi64(d1, (uint64_t)ntr);
          atomicAdd(reinterpret_cast<uint32_t*>(ws.w) + (i1 >> 2), 1u << ((i1 & 3) * 8));
        }
      }
    } else {
      for (int i = lane; i < ntr; i += 32) ws.w[i] = 1;
    }
    __syncwarp();

    if (kFit && a.leaf_of_row)
      for (int i = lane; i < ntr; i += 32)
        if (!ws.w[i]) a.leaf_of_row[tree_slot * a.n + tr_rows[i]] = -1;

    // ---- root statistics
    int64_t S = 0, mn = INT64_MAX, mx = INT64_MIN;
    uint32_t D = 0;
    for (int i = lane; i < ntr; i += 32) {
      uint32_t wv = ws.w[i];
      if (wv) {
        int64_t v = cs.tq[i];
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
      double v = leaf_value(S, Wroot, F);
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
        for (int i = lane; i < ntr; i += 32)
          if (ws.w[i]) a.leaf_of_row[tree_slot * a.n + tr_rows[i]] = 0;
      __syncwarp();
      continue;
    }

    // ---- in-bag lists: stable compaction of the presorted orders by w > 0
    for (int f = 0; f < p; ++f) {
      uint32_t off = 0;
      for (int c = 0; c < ntr; c += 32) {
        int j = c + lane;
        uint8_t r = 0;
        bool keep = false;
        if (j < ntr) { r = cs.ord[f * ntr_max + j]; keep = ws.w[r] != 0; }
        unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (keep) ws.list[f * ntr_max + off + __popc(bal & lanemask_lt())] = r;
        off += __popc(bal);
      }
    }
    for (int i = lane; i < (int)D; i += 32) ws.pnode[i] = 0;
    if (lane == 0) {
      ws.cur.start[0] = 0; ws.cur.len[0] = (uint8_t)D; ws.cur.W[0] = Wroot; ws.cur.S[0] = S;
      ws.cur.heap[0] = 1ull; ws.cur.bfs[0] = 0;
    }
    __syncwarp();

    int nOpen = 1;
    int N = (int)D;
    uint32_t curBase = 0, levelCount = 1;
    int depth = 0;

    while (nOpen > 0) {
      const int K = (N + 31) >> 5;
      const int pbeg = lane * K;
      const int pend = min(pbeg + K, N);  // this lane's positions [pbeg, pend)

      // (a) node bases (prefix trick), reset best, (b) feature draws
      {
        uint32_t carryW = 0;
        int64_t carryS = 0;
        for (int b0 = 0; b0 < nOpen; b0 += 32) {
          int k = b0 + lane;
          bool act = k < nOpen;
          uint32_t Wk = act ? ws.cur.W[k] : 0u;
          int64_t Sk = act ? ws.cur.S[k] : 0;
          uint32_t tW;
          int64_t tS;
          uint32_t eW = wscan_u32(Wk, tW);
          int64_t eS = wscan_i64(Sk, tS);
          if (act) {
            ws.baseW[k] = carryW + eW;
            ws.baseS[k] = carryS + eS;
            ws.bestKey[k] = 0ull;
            ws.bestF[k] = 0u;
            ws.bestPos[k] = 0u;
            if (need_feat) {
              uint8_t* fp = ws.feat + (size_t)k * p;
              for (int f = 0; f < p; ++f) fp[f] = (uint8_t)f;
              const uint64_t h = ws.cur.heap[k];
              const uint32_t hlo = (uint32_t)h, hhi = (uint32_t)(h >> 32);
              for (int j = 0; j < mtry; j += 2) {
                uint64_t d0, d1;
                philox_pair(k0, k1, (uint32_t)(j >> 1), hlo, hhi, kTagFeat, d0, d1);
                int r = j + (int)mulhi64(d0, (uint64_t)(p - j));
                uint8_t tmp = fp[j]; fp[j] = fp[r]; fp[r] = tmp;
                if (j + 1 < mtry) {
                  r = j + 1 + (int)mulhi64(d1, (uint64_t)(p - j - 1));
                  tmp = fp[j + 1]; fp[j + 1] = fp[r]; fp[r] = tmp;
                }
              }
            }
          }
          carryW += tW;
          carryS += tS;
        }
      }
      __syncwarp();

      // (d) search passes: one per drawn-feature slot j
      for (int j = 0; j < mtry; ++j) {
        for (int k = lane; k < nOpen; k += 32) { ws.passKey[k] = 0ull; ws.passPos[k] = 0xFFFFFFFFu; }
        // pass 1: lane totals; first element's (node, rank) for the left neighbour lane
        uint32_t lw = 0;
        int64_t ls = 0;
        uint32_t fn = kNone, frk = 0;
        for (int pos = pbeg; pos < pend; ++pos) {
          int k = ws.pnode[pos];
          int f = need_feat ? ws.feat[(size_t)k * p + j] : j;
          uint8_t r = ws.list[f * ntr_max + pos];
          uint32_t w_ = ws.w[r];
          lw += w_;
          ls += (int64_t)w_ * cs.tq[r];
          if (pos == pbeg) { fn = (uint32_t)k; frk = cs.lrank[f * ntr_max + r]; }
        }
        uint32_t totW;
        int64_t totS;
        uint32_t cW = wscan_u32(lw, totW);
        int64_t cS = wscan_i64(ls, totS);
        uint32_t nfn = __shfl_down_sync(0xffffffffu, fn, 1);
        uint32_t nfrk = __shfl_down_sync(0xffffffffu, frk, 1);
        if (lane == 31) nfn = kNone;
        __syncwarp();
        // pass 2: prefix sums, candidates at distinct-value boundaries, per-run best -> atomicMax
        unsigned long long gk[KM];
        unsigned long long runKey = 0ull;
        int runNode = -1;
#pragma unroll
        for (int i = 0; i < KM; ++i) {
          gk[i] = 0ull;
          const int pos = pbeg + i;
          if (pos < pend) {
            int k = ws.pnode[pos];
            int f = need_feat ? ws.feat[(size_t)k * p + j] : j;
            uint8_t r = ws.list[f * ntr_max + pos];
            uint32_t w_ = ws.w[r];
            cW += w_;
            cS += (int64_t)w_ * cs.tq[r];
            uint32_t nk, nrk;
            if (pos + 1 < pend) {
              nk = ws.pnode[pos + 1];
              nrk = (nk == (uint32_t)k) ? cs.lrank[f * ntr_max + ws.list[f * ntr_max + pos + 1]] : 0u;
            } else {
              nk = nfn;
              nrk = nfrk;
            }
            if (nk == (uint32_t)k && nrk != cs.lrank[f * ntr_max + r]) {
              uint32_t WLv = cW - ws.baseW[k];
              int64_t SLv = cS - ws.baseS[k];
              double G = split_gain((int64_t)WLv, SLv, (int64_t)(ws.cur.W[k] - WLv), ws.cur.S[k] - SLv);
              gk[i] = (unsigned long long)__double_as_longlong(G) + 1ull;
            }
            if (k != runNode) {
              if (runKey) atomicMax(&ws.passKey[runNode], runKey);
              runNode = k;
              runKey = 0ull;
            }
            runKey = gk[i] > runKey ? gk[i] : runKey;
          }
        }
        if (runKey) atomicMax(&ws.passKey[runNode], runKey);
        __syncwarp();
#pragma unroll
        for (int i = 0; i < KM; ++i)
          if (gk[i]) {
            int k = ws.pnode[pbeg + i];
            if (gk[i] == ws.passKey[k]) atomicMin(&ws.passPos[k], (uint32_t)(pbeg + i));
          }
        __syncwarp();
        for (int k = lane; k < nOpen; k += 32) {
          unsigned long long pk = ws.passKey[k];
          if (pk) {
            uint32_t f = need_feat ? ws.feat[(size_t)k * p + j] : (uint32_t)j;
            unsigned long long bk = ws.bestKey[k];
            if (pk > bk || (pk == bk && f < ws.bestF[k])) {
              ws.bestKey[k] = pk;
              ws.bestF[k] = f;
              ws.bestPos[k] = ws.passPos[k];
            }
          }
        }
        __syncwarp();
      }

      // (e) decisions; first-row targets of the children for the constancy test
      for (int k = lane; k < nOpen; k += 32) {
        bool sp = ws.bestKey[k] != 0ull;
        ws.split[k] = sp;
        if (sp) {
          int f = ws.bestF[k];
          ws.tqfL[k] = cs.tq[ws.list[f * ntr_max + ws.cur.start[k]]];
          ws.tqfR[k] = cs.tq[ws.list[f * ntr_max + ws.bestPos[k] + 1]];
        }
      }
      for (int k4 = lane; k4 < (nOpen + 3) / 4; k4 += 32) reinterpret_cast<uint32_t*>(ws.nc)[k4] = 0u;
      __syncwarp();

      // (f) mark pass: go-left flags, left sums at the chosen boundary, child constancy, threshold
      {
        uint32_t lw = 0;
        int64_t ls = 0;
        for (int pos = pbeg; pos < pend; ++pos) {
          int k = ws.pnode[pos];
          if (!ws.split[k]) continue;
          int f = ws.bestF[k];
          uint8_t r = ws.list[f * ntr_max + pos];
          uint32_t w_ = ws.w[r];
          lw += w_;
          ls += (int64_t)w_ * cs.tq[r];
          bool left = pos <= (int)ws.bestPos[k];
          ws.side[r] = left ? 1 : 0;
          int64_t ref = left ? ws.tqfL[k] : ws.tqfR[k];
          if (cs.tq[r] != ref)  // child not constant (two bits per node byte: word atomics)
            atomicOr(reinterpret_cast<unsigned int*>(ws.nc + (k & ~3)), (left ? 1u : 2u) << ((k & 3) * 8));
        }
        uint32_t tW;
        int64_t tS;
        uint32_t cW = wscan_u32(lw, tW);
        int64_t cS = wscan_i64(ls, tS);
        for (int pos = pbeg; pos < pend; ++pos) {
          int k = ws.pnode[pos];
          if (!ws.split[k]) continue;
          int f = ws.bestF[k];
          uint8_t r = ws.list[f * ntr_max + pos];
          uint32_t w_ = ws.w[r];
          cW += w_;
          cS += (int64_t)w_ * cs.tq[r];
          if (pos == (int)ws.bestPos[k]) {
            // prefix over split nodes only; made node-relative in (g)
            ws.WL[k] = cW;
            ws.SL[k] = cS;
            uint8_t rb = ws.list[f * ntr_max + pos + 1];
            uint32_t ga = tr_rows[r], gb = tr_rows[rb];
            double xa = a.X[(size_t)ga * p + f], xb = a.X[(size_t)gb * p + f];
            ws.thr[k] = midpoint_thr(xa, xb);
            if (kFit) ws.thrIdx[k] = a.grank[(size_t)f * a.n + ga];
          }
        }
      }
      __syncwarp();

      // (g) children, node emission, next-level tables
      int nSplitTotal = 0, nOpenNext = 0, Nnext = 0;
      {
        uint32_t carryW = 0, carrySplit = 0, carryOpen = 0, carryPos = 0, carryL = 0;
        int64_t carryS = 0;
        for (int b0 = 0; b0 < nOpen; b0 += 32) {
          int k = b0 + lane;
          bool act = k < nOpen;
          bool sp = act && ws.split[k];
          uint32_t tW, tSp, tOpen, tPos, tL;
          int64_t tS;
          uint32_t eW = wscan_u32(sp ? ws.cur.W[k] : 0u, tW);
          int64_t eS = wscan_i64(sp ? ws.cur.S[k] : 0, tS);
          uint32_t eSp = wscan_u32(sp ? 1u : 0u, tSp);
          uint32_t WLv = 0, WRv = 0, lenL = 0, lenR = 0, nl = 0;
          int64_t SLv = 0, SRv = 0;
          bool openL = false, openR = false;
          if (sp) {
            WLv = ws.WL[k] - (carryW + eW);
            SLv = ws.SL[k] - (carryS + eS);
            WRv = ws.cur.W[k] - WLv;
            SRv = ws.cur.S[k] - SLv;
            nl = ws.bestPos[k] - ws.cur.start[k] + 1;
            lenL = nl;
            lenR = ws.cur.len[k] - nl;
            const bool capd = (a.max_depth >= 0) && (depth + 1 >= a.max_depth);
            const uint8_t ncb = ws.nc[k];
            openL = !capd && (int)lenL >= a.min_split && (ncb & 1);
            openR = !capd && (int)lenR >= a.min_split && (ncb & 2);
          }
          uint32_t eOpen = wscan_u32((openL ? 1u : 0u) + (openR ? 1u : 0u), tOpen);
          uint32_t ePos = wscan_u32((openL ? lenL : 0u) + (openR ? lenR : 0u), tPos);
          uint32_t eL = wscan_u32(sp ? nl : 0u, tL);
          if (sp) {
            const uint32_t childBase = curBase + levelCount + 2 * (carrySplit + eSp);
            ws.baseL[k] = carryL + eL;
            ws.baseW[k] = childBase;  // baseW is dead after the search passes
            uint32_t oi = carryOpen + eOpen;
            uint32_t ps = carryPos + ePos;
            double vL = 0.0, vR = 0.0;
            if (openL) {
              ws.nxt.start[oi] = (uint8_t)ps; ws.nxt.len[oi] = (uint8_t)lenL;
              ws.nxt.W[oi] = WLv; ws.nxt.S[oi] = SLv;
              ws.nxt.heap[oi] = 2ull * ws.cur.heap[k]; ws.nxt.bfs[oi] = childBase;
              ws.chOpen[2 * k] = (uint8_t)oi;
              ++oi; ps += lenL;
            } else {
              vL = leaf_value(SLv, WLv, F);
              ws.chOpen[2 * k] = kNone;
            }
            if (openR) {
              ws.nxt.start[oi] = (uint8_t)ps; ws.nxt.len[oi] = (uint8_t)lenR;
              ws.nxt.W[oi] = WRv; ws.nxt.S[oi] = SRv;
              ws.nxt.heap[oi] = 2ull * ws.cur.heap[k] + 1ull; ws.nxt.bfs[oi] = childBase + 1;
              ws.chOpen[2 * k + 1] = (uint8_t)oi;
            } else {
              vR = leaf_value(SRv, WRv, F);
              ws.chOpen[2 * k + 1] = kNone;
            }
            ws.chVal[2 * k] = vL;
            ws.chVal[2 * k + 1] = vR;
            if (kFit) {
              Node16* tn = a.nodes + tree_slot * a.cap;
              uint32_t* ti = a.thr_index + tree_slot * a.cap;
              const uint32_t me = ws.cur.bfs[k];
              Node16 nd;
              nd.feat = (int32_t)ws.bestF[k]; nd.left = childBase; nd.v = ws.thr[k];
              tn[me] = nd;
              ti[me] = ws.thrIdx[k];
              if (!openL) { Node16 l; l.feat = -1; l.left = 0; l.v = vL; tn[childBase] = l; ti[childBase] = 0; }
              if (!openR) { Node16 r; r.feat = -1; r.left = 0; r.v = vR; tn[childBase + 1] = r; ti[childBase + 1] = 0; }
            }
          } else if (act) {
            // open node without any candidate split: leaf (R11)
            double v = leaf_value(ws.cur.S[k], ws.cur.W[k], F);
            ws.chVal[2 * k] = v;
            if (kFit) {
              Node16 nd;
              nd.feat = -1; nd.left = 0; nd.v = v;
              a.nodes[tree_slot * a.cap + ws.cur.bfs[k]] = nd;
              a.thr_index[tree_slot * a.cap + ws.cur.bfs[k]] = 0;
            }
          }
          carryW += tW;
          carryS += tS;
          carrySplit += tSp;
          carryOpen += tOpen;
          carryPos += tPos;
          carryL += tL;
        }
        nSplitTotal = (int)carrySplit;
        nOpenNext = (int)carryOpen;
        Nnext = (int)carryPos;
      }
      __syncwarp();

      // (h) route the task's test rows one level down
      if (!kFit) {
#pragma unroll
        for (int s = 0; s < TM; ++s) {
          const int r = lane + 32 * s;
          uint32_t c = (tcur >> (8 * s)) & 0xFFu;
          if (r < nte && c != kNone) {
            const int k = (int)c;
            uint32_t nc_;
            if (!ws.split[k]) {
              acc[s] += ws.chVal[2 * k];
              nc_ = kNone;
            } else {
              const int sd = (cs.xte[(size_t)r * p + ws.bestF[k]] <= ws.thr[k]) ? 0 : 1;
              nc_ = ws.chOpen[2 * k + sd];
              if (nc_ == kNone) acc[s] += ws.chVal[2 * k + sd];
            }
            tcur = (tcur & ~(0xFFu << (8 * s))) | (nc_ << (8 * s));
          }
        }
      }

      // (i) stable in-place partition of every feature list; leaf rows dropped
      for (int f = 0; f < p; ++f) {
        uint32_t rows4[(KM + 3) / 4];
        uint32_t sides = 0;  // 2 bits per element: 0 drop, 1 left, 2 right
        uint32_t lc = 0;
#pragma unroll
        for (int i = 0; i < KM; ++i) {
          const int pos = pbeg + i;
          if ((i & 3) == 0) rows4[i >> 2] = 0;
          if (pos < pend) {
            uint8_t r = ws.list[f * ntr_max + pos];
            rows4[i >> 2] |= (uint32_t)r << (8 * (i & 3));
            uint32_t s_ = ws.split[ws.pnode[pos]] ? (ws.side[r] ? 1u : 2u) : 0u;
            sides |= s_ << (2 * i);
            lc += (s_ == 1u);
          }
        }
        uint32_t tl_;
        uint32_t run = wscan_u32(lc, tl_);
        __syncwarp();
#pragma unroll
        for (int i = 0; i < KM; ++i) {
          const int pos = pbeg + i;
          if (pos < pend) {
            const int k = ws.pnode[pos];
            const uint32_t s_ = (sides >> (2 * i)) & 3u;
            const uint8_t r = (uint8_t)(rows4[i >> 2] >> (8 * (i & 3)));
            if (s_) {
              const uint32_t leftBefore = run - ws.baseL[k];
              const int sideIdx = (s_ == 1u) ? 0 : 1;
              const uint8_t c = ws.chOpen[2 * k + sideIdx];
              if (c != kNone) {
                uint32_t within = (s_ == 1u) ? leftBefore : (uint32_t)(pos - ws.cur.start[k]) - leftBefore;
                uint32_t dest = ws.nxt.start[c] + within;
                ws.list[f * ntr_max + dest] = r;
                if (f == 0) ws.pnode2[dest] = c;
              } else if (kFit && f == 0 && a.leaf_of_row) {
                a.leaf_of_row[tree_slot * a.n + tr_rows[r]] = (int32_t)(ws.baseW[k] + sideIdx);
              }
            } else if (kFit && f == 0 && a.leaf_of_row) {
              a.leaf_of_row[tree_slot * a.n + tr_rows[r]] = (int32_t)ws.cur.bfs[k];
            }
            if (s_ == 1u) ++run;
          }
        }
        __syncwarp();
      }

      // advance to the next level
      {
        NodeSet tmp = ws.cur; ws.cur = ws.nxt; ws.nxt = tmp;
        uint8_t* tp = ws.pnode; ws.pnode = ws.pnode2; ws.pnode2 = tp;
      }
      curBase += levelCount;
      levelCount = 2u * (uint32_t)nSplitTotal;
      nOpen = nOpenNext;
      N = Nnext;
      ++depth;
      __syncwarp();
    }
    if (kFit && lane == 0) a.tree_nnodes[tree_slot] = curBase + levelCount;
    __syncwarp();
  }

  if (!kFit) {
    double* out = a.partial + (((size_t)mi * a.ntask + tl) * a.nsub + sub) * a.nte_max;
#pragma unroll
    for (int s = 0; s < TM; ++s) {
      int r = lane + 32 * s;
      if (r < nte) out[r] = acc[s];
    }
  }
}

}  // namespace

size_t small_tree_smem_bytes(const SmallArgs& a, int /*mmax*/) {
  bool any_feat = false;
  for (int i = 0; i < a.n_mtry; ++i) any_feat |= (a.mtrys[i] < a.p);
  Carve c(nullptr);
  CtaSmem cs;
  carve_cta(c, cs, a.p, a.ntr_max, a.fit_mode ? 0 : a.nte_max);
  size_t cta = (c.off + 15) / 16 * 16;
  Carve w(nullptr);
  WarpSmem ws;
  carve_warp(w, ws, a.p, a.ntr_max, any_feat);
  size_t per_warp = (w.off + 15) / 16 * 16;
  return cta + per_warp * a.wpb;
}

template <bool kFit, int KM, int TM>
static cudaError_t launch_t(const SmallArgs& a, size_t smem, unsigned grid, cudaStream_t s) {
  auto kern = small_tree_kernel<kFit, KM, TM>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, 32 * a.wpb, smem, s>>>(a);
  return cudaGetLastError();
}

template <bool kFit, int TM>
static cudaError_t launch_k(const SmallArgs& a, size_t smem, unsigned grid, cudaStream_t s) {
  const int K = (a.ntr_max + 31) / 32;
  if (K <= 4) return launch_t<kFit, 4, TM>(a, smem, grid, s);
  if (K <= 6) return launch_t<kFit, 6, TM>(a, smem, grid, s);
  return launch_t<kFit, 8, TM>(a, smem, grid, s);
}

cudaError_t launch_small_tree(const SmallArgs& a, cudaStream_t s) {
  size_t smem = small_tree_smem_bytes(a, 0);
  int cta_per_mt = (a.nsub + a.wpb - 1) / a.wpb;
  long long grid = (long long)a.n_mtry * a.ntask * cta_per_mt;
  if (grid <= 0) return cudaSuccess;
  if (a.fit_mode) return launch_k<true, 1>(a, smem, (unsigned)grid, s);
  const int TMn = (a.nte_max + 31) / 32;
  if (TMn <= 1) return launch_k<false, 1>(a, smem, (unsigned)grid, s);
  if (TMn <= 2) return launch_k<false, 2>(a, smem, (unsigned)grid, s);
  return launch_k<false, 8>(a, smem, (unsigned)grid, s);
}

}  // namespace rf
