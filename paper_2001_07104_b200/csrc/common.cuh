// common.cuh -- shared device helpers of librfgpu (sm_100a).
//
// Philox4x32-10 counter-based generator (Salmon et al. SC'11; Random123
// constants), the draw(i) / mulhi64 conventions and the stream tags of
// DESIGN.md R14-R16.  This is the CUDA path's own implementation; the oracle
// has an independent one (oracle/rf_oracle.c) and both are pinned to the
// Random123 KAT vectors (tests/golden/philox_kat.txt).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace rf {

constexpr uint32_t kPhiloxM0 = 0xD2511F53u;
constexpr uint32_t kPhiloxM1 = 0xCD9E8D57u;
constexpr uint32_t kPhiloxW0 = 0x9E3779B9u;
constexpr uint32_t kPhiloxW1 = 0xBB67AE85u;

// stream tags in counter word 3 (R14-R17)
constexpr uint32_t kTagFold = 0xD0u;
constexpr uint32_t kTagStratum = 0xD1u;
constexpr uint32_t kTagKeyDeriv = 0x4Bu;
constexpr uint32_t kTagBoot = 0xB0u;
constexpr uint32_t kTagFeat = 0xF0u;
constexpr uint32_t kTagThr = 0xE7u;  // ExtraTrees thresholds (R29)

struct U4 { uint32_t x, y, z, w; };

__host__ __device__ __forceinline__ U4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2,
                                                     uint32_t c3, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
#if defined(__CUDA_ARCH__)
    uint32_t hi0 = __umulhi(kPhiloxM0, c0), lo0 = kPhiloxM0 * c0;
    uint32_t hi1 = __umulhi(kPhiloxM1, c2), lo1 = kPhiloxM1 * c2;
#else
    uint64_t p0 = (uint64_t)kPhiloxM0 * c0, p1 = (uint64_t)kPhiloxM1 * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
#endif
    uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += kPhiloxW0;
    k1 += kPhiloxW1;
  }
  return U4{c0, c1, c2, c3};
}

// the two 64-bit draws of block b: draw(2b) = (w1<<32)|w0, draw(2b+1) = (w3<<32)|w2
__host__ __device__ __forceinline__ void philox_pair(uint32_t k0, uint32_t k1, uint32_t b,
                                                     uint32_t c1, uint32_t c2, uint32_t c3,
                                                     uint64_t& even, uint64_t& odd) {
  U4 o = philox4x32_10(b, c1, c2, c3, k0, k1);
  even = ((uint64_t)o.y << 32) | o.x;
  odd = ((uint64_t)o.w << 32) | o.z;
}

__host__ __device__ __forceinline__ uint64_t draw64(uint32_t k0, uint32_t k1, uint32_t c1,
                                                    uint32_t c2, uint32_t c3, uint64_t i) {
  U4 o = philox4x32_10((uint32_t)(i >> 1), c1, c2, c3, k0, k1);
  return (i & 1) ? (((uint64_t)o.w << 32) | o.z) : (((uint64_t)o.y << 32) | o.x);
}

// floor(u * m / 2^64)
__host__ __device__ __forceinline__ uint64_t mulhi64(uint64_t u, uint64_t m) {
#if defined(__CUDA_ARCH__)
  return __umul64hi(u, m);
#else
  return (uint64_t)(((unsigned __int128)u * m) >> 64);
#endif
}

// per-tree key k_t: lanes 0,1 of Philox(key = seed, ctr = (t, task, 0, KEYDERIV))
__host__ __device__ __forceinline__ void tree_key(uint64_t seed, uint32_t task, uint32_t t,
                                                  uint32_t& k0, uint32_t& k1) {
  U4 o = philox4x32_10(t, task, 0u, kTagKeyDeriv, (uint32_t)seed, (uint32_t)(seed >> 32));
  k0 = o.x;
  k1 = o.y;
}

// 16-byte flattened node
struct __align__(16) Node16 {
  int32_t feat;   // -1 = leaf
  uint32_t left;  // BFS id of left child (right = left + 1), relative to the tree
  double v;       // threshold (internal) or leaf value
};

// canonical split score G = fl(fl(fl(SL*SL)/WL) + fl(fl(SR*SR)/WR)) (R6, R28); no contraction
__device__ __forceinline__ double split_gain(int64_t WL, int64_t SL, int64_t WR, int64_t SR) {
  double dSL = __ll2double_rn(SL), dWL = __ll2double_rn(WL);
  double dSR = __ll2double_rn(SR), dWR = __ll2double_rn(WR);
  double a = __ddiv_rn(__dmul_rn(dSL, dSL), dWL);
  double b = __ddiv_rn(__dmul_rn(dSR, dSR), dWR);
  return __dadd_rn(a, b);
}

// threshold between consecutive distinct values a < b (R8)
__device__ __forceinline__ double midpoint_thr(double a, double b) {
  double t = __dadd_rn(__dmul_rn(a, 0.5), __dmul_rn(b, 0.5));
  return (t == b) ? a : t;
}

// ExtraTrees threshold of draw slot j at heap node h (R29):
// u = (draw(j) of stream (k_t; h_lo, h_hi, 0xE7) >> 11) 2^-53 (exact),
// thr = fl(fl(fl(hi - lo) u) + lo), replaced by lo unless thr < hi.
__device__ __forceinline__ double extra_thr_draw(uint64_t d, double lo, double hi) {
  const double u = __dmul_rn(__ull2double_rn(d >> 11), 0x1p-53);
  const double t = __dadd_rn(__dmul_rn(__dsub_rn(hi, lo), u), lo);
  return t < hi ? t : lo;
}
__device__ __forceinline__ double extra_thr(uint32_t k0, uint32_t k1, uint64_t h, int j, double lo, double hi) {
  uint64_t d0, d1;
  philox_pair(k0, k1, (uint32_t)(j >> 1), (uint32_t)h, (uint32_t)(h >> 32), kTagThr, d0, d1);
  return extra_thr_draw((j & 1) ? d1 : d0, lo, hi);
}

// Mean decrease in impurity of one split (feature importance, SURVEY 8(f) NEXT-3;
// P:218-219): W imp(node) - WL imp(L) - WR imp(R) = (SL WR - SR WL)^2 / (W WL WR),
// scaled by 2^-2F to target units.  The numerator is exact in __int128 and rounded
// once (plus the split into two 64-bit halves); the rest is fp64 (relative error
// a few ulp; the sums over splits run in atomics, so importances carry a ~1e-15
// order dependence -- the parity bar is 1e-9).
__device__ __forceinline__ double mdi_decrease(int64_t WL, int64_t SL, int64_t WR, int64_t SR, int F) {
  const __int128 num = (__int128)SL * WR - (__int128)SR * WL;
  const bool neg = num < 0;
  const unsigned __int128 u = neg ? (unsigned __int128)(-num) : (unsigned __int128)num;
  const double dn = __dadd_rn(__dmul_rn(__ull2double_rn((unsigned long long)(u >> 64)), 0x1p64),
                              __ull2double_rn((unsigned long long)u));
  const double den = __dmul_rn(__dmul_rn(__ll2double_rn(WL + WR), __ll2double_rn(WL)), __ll2double_rn(WR));
  return scalbn(__ddiv_rn(__dmul_rn(dn, dn), den), -2 * F);
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

}  // namespace rf
