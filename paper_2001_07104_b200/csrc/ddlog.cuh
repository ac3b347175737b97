// ddlog.cuh -- ln(y) correctly rounded to binary64 (R20).
//
// The time targets are fitted as ln(t).  Because the
// quantised target t_q = rint(ln(y) 2^F) (R7) feeds exact integer split sums,
// ln must be the same bits on every implementation; the reading adopted is
// "ln correctly rounded".  Evaluated in double-double (~104 bits):
//   y = 2^e m, m in [sqrt(1/2), sqrt(2));  s = (m-1)/(m+1), |s| <= 0.1716
//   ln m = 2 sum_{k=0}^{21} s^(2k+1)/(2k+1)      (truncation < 2^-110 rel.)
//   ln y = e ln2 + ln m,  ln2 as a double-double constant,
// then rounded once.  Misrounding needs ln y within ~2^-100 relative of a
// rounding boundary.  __host__ __device__ so the host self-test can run it.
#pragma once
#include <cmath>

namespace rf {

#if defined(__CUDA_ARCH__)
#define RF_ADD(a, b) __dadd_rn((a), (b))
#define RF_SUB(a, b) __dsub_rn((a), (b))
#define RF_MUL(a, b) __dmul_rn((a), (b))
#define RF_DIV(a, b) __ddiv_rn((a), (b))
#define RF_FMA(a, b, c) __fma_rn((a), (b), (c))
#else
#define RF_ADD(a, b) ((a) + (b))
#define RF_SUB(a, b) ((a) - (b))
#define RF_MUL(a, b) ((a) * (b))
#define RF_DIV(a, b) ((a) / (b))
#define RF_FMA(a, b, c) std::fma((a), (b), (c))
#endif

struct DD { double hi, lo; };

__host__ __device__ inline DD dd_two_sum(double a, double b) {
  double s = RF_ADD(a, b);
  double bb = RF_SUB(s, a);
  double e = RF_ADD(RF_SUB(a, RF_SUB(s, bb)), RF_SUB(b, bb));
  return DD{s, e};
}
__host__ __device__ inline DD dd_quick(double a, double b) {
  double s = RF_ADD(a, b);
  double e = RF_SUB(b, RF_SUB(s, a));
  return DD{s, e};
}
__host__ __device__ inline DD dd_two_prod(double a, double b) {
  double p = RF_MUL(a, b);
  double e = RF_FMA(a, b, -p);
  return DD{p, e};
}
__host__ __device__ inline DD dd_add(DD a, DD b) {
  DD s = dd_two_sum(a.hi, b.hi);
  DD t = dd_two_sum(a.lo, b.lo);
  s.lo = RF_ADD(s.lo, t.hi);
  s = dd_quick(s.hi, s.lo);
  s.lo = RF_ADD(s.lo, t.lo);
  return dd_quick(s.hi, s.lo);
}
__host__ __device__ inline DD dd_neg(DD a) { return DD{-a.hi, -a.lo}; }
__host__ __device__ inline DD dd_mul(DD a, DD b) {
  DD p = dd_two_prod(a.hi, b.hi);
  p.lo = RF_ADD(p.lo, RF_ADD(RF_MUL(a.hi, b.lo), RF_MUL(a.lo, b.hi)));
  return dd_quick(p.hi, p.lo);
}
__host__ __device__ inline DD dd_mul_d(DD a, double b) {
  DD p = dd_two_prod(a.hi, b);
  p.lo = RF_ADD(p.lo, RF_MUL(a.lo, b));
  return dd_quick(p.hi, p.lo);
}
__host__ __device__ inline DD dd_div(DD a, DD b) {
  double q1 = RF_DIV(a.hi, b.hi);
  DD r = dd_add(a, dd_neg(dd_mul_d(b, q1)));
  double q2 = RF_DIV(r.hi, b.hi);
  r = dd_add(r, dd_neg(dd_mul_d(b, q2)));
  double q3 = RF_DIV(r.hi, b.hi);
  DD q = dd_quick(q1, q2);
  return dd_add(q, DD{q3, 0.0});
}

__host__ __device__ inline double ln_correctly_rounded(double y) {
  // y > 0, finite
  const DD kLn2 = {0x1.62e42fefa39efp-1, 0x1.abc9e3b39803fp-56};
  int e;
  double m = frexp(y, &e);  // y = m 2^e, m in [0.5, 1)
  if (m < 0x1.6a09e667f3bcdp-1) {
    m = RF_MUL(m, 2.0);
    e -= 1;
  }
  DD num = DD{RF_SUB(m, 1.0), 0.0};  // exact (Sterbenz)
  DD den = dd_two_sum(m, 1.0);
  DD s = dd_div(num, den);
  DD s2 = dd_mul(s, s);
  DD P = dd_div(DD{1.0, 0.0}, DD{43.0, 0.0});
  for (int k = 20; k >= 0; --k) {
    P = dd_add(dd_mul(P, s2), dd_div(DD{1.0, 0.0}, DD{(double)(2 * k + 1), 0.0}));
  }
  DD lnm = dd_mul_d(dd_mul(s, P), 2.0);
  DD el = dd_mul_d(kLn2, (double)e);
  DD r = dd_add(el, lnm);
  return RF_ADD(r.hi, r.lo);
}

}  // namespace rf
