// Host build of the product's double-double ln (paper_2001_07104_b200/csrc/ddlog.cuh) for
// tests/test_ddlog_host.py: g++ -O2 -ffp-contract=off (IEEE binary64, no contraction, the
// same operation sequence as the device's __dadd_rn/__dmul_rn/__fma_rn intrinsics).
//   mode 0: stdin doubles y -> stdout records (hi, lo, RN result, certified) of ln_dd / ln_cr_checked
//   mode 1: stdin pairs (hi, lo) -> stdout records (RN result, certified) of dd_round_checked
#define __host__
#define __device__
#include <cstdio>
#include <cstdlib>
#include "ddlog.cuh"

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  const int margin = argc > 2 ? atoi(argv[2]) : rf::kLnCertLog2;
  if (mode == 0) {
    double y;
    while (fread(&y, 8, 1, stdin) == 1) {
      const rf::DD r = rf::ln_dd(y);
      bool ok;
      const double d = rf::ln_cr_checked(y, ok, margin);
      const double rec[4] = {r.hi, r.lo, d, ok ? 1.0 : 0.0};
      fwrite(rec, 8, 4, stdout);
    }
  } else {
    double hl[2];
    while (fread(hl, 8, 2, stdin) == 2) {
      bool ok;
      const double d = rf::dd_round_checked(rf::DD{hl[0], hl[1]}, ok, margin);
      const double rec[2] = {d, ok ? 1.0 : 0.0};
      fwrite(rec, 8, 2, stdout);
    }
  }
  return 0;
}
