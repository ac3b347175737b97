// prep.cuh -- dataset preparation on the device: validation, target
// transform, quantisation (R7, R20, R22) and per-feature presort.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace rf {

enum : int { kErrNonFinite = 1, kErrNonPositive = 2, kErrOverflow = 4, kErrInexact = 8 };
// test switch (rf_debug_set_option "ln_cert_margin_log2"): margin of ln's rounding test, 0 = default
extern int g_opt_ln_margin_log2;

// Device-resident prepared dataset.
struct DevData {
  int n = 0, p = 0;
  double* X = nullptr;        // [n][p] canonical (-0.0 -> +0.0)
  int64_t* tq = nullptr;      // [n]
  int32_t* F = nullptr;       // device scalar
  uint32_t* order = nullptr;  // [p][n] stable order by x_f
  uint32_t* grank = nullptr;  // [p][n] dense rank of x_f over all rows
  int* err = nullptr;         // device flags (kErr*)
};

// X -> canonical copy, checks finiteness; y -> t (ln if LOG) -> F, t_q.
// require_pos: y > 0 required (LOG target or CV).  guard: extra headroom bits of
// the quantisation (2 under the MAE criterion, R32: F = 62 - ceil(log2 n) - e - 2).
cudaError_t prep_targets(const double* dX, const double* dy, int n, int p, int target,
                         int require_pos, int guard, DevData& d, double* scratch_t, cudaStream_t s);
// stable per-feature order + dense ranks (needs workspace for large n)
// ranks = false: orders only (the histogram mode needs no dense ranks; large n only)
cudaError_t presort(DevData& d, void* ws, size_t ws_bytes, cudaStream_t s, bool ranks = true);
size_t presort_ws_bytes(int n, int p);

// device ln correctly rounded (exposed for tests via the API)
cudaError_t device_ln(const double* dy, double* dout, int n, cudaStream_t s);
// Philox4x32-10 blocks for (c0,c1,c2,c3,k0,k1) tuples (KAT tests)
cudaError_t device_philox(const uint32_t* ctr_key, uint32_t* out, int n, cudaStream_t s);

}  // namespace rf
