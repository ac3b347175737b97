// ddlog.cuh -- ln(y) correctly rounded to binary64 (R20).
//
// The time targets are fitted as ln(t).  Because the
// quantised target t_q = rint(ln(y) 2^F) (R7) feeds exact integer split sums,
// ln must be the same bits on every implementation; the reading adopted is
// "ln correctly rounded".  Evaluated in double-double (~104 bits):
//   y = 2^e m, m in [sqrt(1/2), sqrt(2));  s = (m-1)/(m+1), |s| <= 0.1716
//   ln m = 2 sum_{k=0}^{21} s^(2k+1)/(2k+1)      (truncation < 2^-110 rel.)
//   ln y = e ln2 + ln m,  ln2 as a double-double constant,
// then rounded once.  Rounding test (Ziv): the double-double value r carries a
// relative error below 2^-95 (a margin of >= 2^4 over the evaluation's largest
// error, measured against 200-bit mpmath by tests/test_ddlog_host.py); the
// rounded result is certified when r -/+ 2^-94 |r| round to the same double
// (the "- / +" offsets themselves err by < 2^-105 |r|), i.e. when ln y is not
// within ~2^-94 relative of a rounding boundary.  The structured hard cases
// (y = 1 + k 2^-52, small k: ln y within ~2^-105 of a midpoint) take a separate
// branch for |y - 1| <= 2^-26 that decides the rounding with ~2^-125 error
// (ln1p_tiny_checked).  An uncertified value (none is known for binary64
// inputs; ~2^-41 of random inputs would fall there) makes the calling entry
// point fail with RF_E_INEXACT instead of risking a misrounded t_q.
// __host__ __device__ so the host test can run it.
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

// double-double ln(y), y > 0 finite (unrounded)
__host__ __device__ inline DD ln_dd(double y) {
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
  return dd_add(el, lnm);
}

// certification margin of the rounding test, as a power of two (the tests widen it through
// rf_debug_set_option "ln_cert_margin_log2" to reach the failure path)
constexpr int kLnCertLog2 = -94;

// RN(hi + lo); certified = every value within 2^margin_log2 |hi| of hi + lo rounds to it too
// (round-to-nearest is monotone, so the two ends decide)
__host__ __device__ inline double dd_round_checked(DD r, bool& certified, int margin_log2) {
  const double d = RF_ADD(r.hi, r.lo);
  const double eps = RF_MUL(fabs(r.hi), ldexp(1.0, margin_log2));
  certified = RF_ADD(r.hi, RF_SUB(r.lo, eps)) == d && RF_ADD(r.hi, RF_ADD(r.lo, eps)) == d;
  return d;
}

// ln(1 + x) for 0 < |x| <= 2^-26, x = y - 1 exact (Sterbenz).  The structured hard cases of ln
// live here: for x = k 2^-52 with small k, x - x^2/2 can sit on a rounding midpoint of binary64
// (or within ~2^-105 relative of one, e.g. y = 1 - 2^-52) and x^3/3 decides -- closer than the
// double-double evaluation above can certify.  So: v = x - x^2/2 + x^3/3 - x^4/4 + x^5/5
// (truncation < 2^-132 |x|) as s + tail with s + e = x + RN(-x^2/2) exact (two_sum), the tail
// e + lo(-x^2/2) + (x^3/3 - x^4/4 + x^5/5) in double-double (error < 2^-125 |s| all told), and
// RN(s + tail) decided by comparing the tail with the exact half-gaps to s's neighbours.  The
// true value is never a midpoint (ln(1 + x) is transcendental for x != 0), so the decision is
// certified when the tail's distance to both half-gaps exceeds the error bound.
__host__ __device__ inline double ln1p_tiny_checked(double x, bool& certified) {
  const DD x2 = dd_two_prod(x, x);                                        // x^2 exact
  const DD b = DD{RF_MUL(x2.hi, -0.5), RF_MUL(x2.lo, -0.5)};              // -x^2/2 exact
  DD c = dd_div(dd_mul_d(x2, x), DD{3.0, 0.0});                          // x^3/3
  const double x4 = RF_MUL(x2.hi, x2.hi);
  c = dd_add(c, DD{RF_ADD(RF_MUL(x4, -0.25), RF_MUL(RF_MUL(x4, x), 0.2)), 0.0});  // - x^4/4 + x^5/5
  const DD se = dd_two_sum(x, b.hi);                                     // x + b.hi = s + e
  const DD T = dd_add(DD{se.lo, 0.0}, dd_add(DD{b.lo, 0.0}, c));          // the tail
  const double sv = se.hi;
  const double up = nextafter(sv, 1.0), dn = nextafter(sv, -1.0);       // |s| < 1
  const double hu = RF_MUL(RF_SUB(up, sv), 0.5), hd = RF_MUL(RF_SUB(dn, sv), 0.5);  // exact half-gaps
  const double delta = RF_MUL(fabs(sv), 0x1p-125);
  // sign of tail - h with its uncertainty: (a1, a2) = tail.hi - h exactly, + tail.lo
  const DD au = dd_two_sum(T.hi, -hu), ad = dd_two_sum(T.hi, -hd);
  const double du = RF_ADD(au.hi, RF_ADD(au.lo, T.lo)), dd = RF_ADD(ad.hi, RF_ADD(ad.lo, T.lo));
  const double uu = RF_ADD(delta, RF_MUL(RF_ADD(RF_ADD(fabs(au.lo), fabs(T.lo)), fabs(du)), 0x1p-51));
  const double ud = RF_ADD(delta, RF_MUL(RF_ADD(RF_ADD(fabs(ad.lo), fabs(T.lo)), fabs(dd)), 0x1p-51));
  certified = fabs(du) > uu && fabs(dd) > ud;
  return du > 0.0 ? up : (dd < 0.0 ? dn : sv);
}

// ln(y) rounded to binary64; certified = the rounding test passed (see the header)
__host__ __device__ inline double ln_cr_checked(double y, bool& certified, int margin_log2 = kLnCertLog2) {
  const double x = RF_SUB(y, 1.0);
  if (x != 0.0 && fabs(x) <= 0x1p-26) return ln1p_tiny_checked(x, certified);
  return dd_round_checked(ln_dd(y), certified, margin_log2);
}

}  // namespace rf
