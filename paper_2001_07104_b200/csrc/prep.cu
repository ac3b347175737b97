// prep.cu -- device-side dataset preparation.
//   * X: finiteness check, -0.0 -> +0.0 (R22)
//   * y: finiteness, positivity (LOG / CV), t = y or ln y correctly rounded
//     (R20), F = 62 - ceil(log2 n) - e(max|t|), t_q = rint(t 2^F)
//     (R7: every weighted node sum fits int64 exactly)
//   * presort: per feature the stable order of rows by x and the dense rank
//     of x over all n rows (threshold index, R10).  Small n: one CTA per
//     feature ranks by counting in shared memory; large n: CUB segmented
//     radix sort of order-preserving u64 keys + a per-feature rank scan.
#include <algorithm>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_segmented_radix_sort.cuh>
#include "common.cuh"
#include "host_util.cuh"
#include "ddlog.cuh"
#include "prep.cuh"

namespace rf {
namespace {

__global__ void k_prep_X(const double* __restrict__ X, double* __restrict__ Xc, size_t total,
                         int* err) {
  bool bad = false;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    double x = X[i];
    const bool fin = isfinite(x);
    bad |= !fin;
    // canonical copy: -0.0 -> +0.0; non-finite entries are flagged (the call fails with
    // RF_E_NONFINITE) and replaced so that downstream kernels stay in bounds
    Xc[i] = (!fin || x == 0.0) ? 0.0 : x;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(err, kErrNonFinite);
}

__global__ void k_prep_y(const double* __restrict__ y, double* __restrict__ t, int n, int target,
                         int require_pos, unsigned long long* maxbits, int* err, int ln_margin_log2) {
  unsigned long long m = 0;
  int e = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double v = y[i];
    if (!isfinite(v)) { e |= kErrNonFinite; v = 1.0; }
    if ((require_pos || target == 1) && !(v > 0.0)) { e |= kErrNonPositive; v = 1.0; }
    double tv = v;
    if (target == 1) {
      bool certified;
      tv = ln_cr_checked(v, certified, ln_margin_log2);
      if (!certified) e |= kErrInexact;  // ln y too close to a rounding boundary (ddlog.cuh)
    }
    t[i] = tv;
    unsigned long long b = (unsigned long long)__double_as_longlong(fabs(tv));
    m = b > m ? b : m;
  }
  for (int d = 16; d > 0; d >>= 1) {
    unsigned long long o = __shfl_xor_sync(0xffffffffu, m, d);
    m = o > m ? o : m;
  }
  e = __reduce_or_sync(0xffffffffu, e);
  if ((threadIdx.x & 31) == 0) {
    if (m) atomicMax(maxbits, m);
    if (e) atomicOr(err, e);
  }
}

__device__ __forceinline__ int quant_F(unsigned long long maxbits, int n, int guard) {
  double M = __longlong_as_double((long long)maxbits);
  if (M == 0.0) return 0;
  int ex;
  double fr = frexp(M, &ex);
  int eM = (fr == 0.5) ? ex - 1 : ex;
  int c = 0;
  while ((1ull << c) < (unsigned long long)n) ++c;
  return 62 - c - eM - guard;  // guard = 2 under MAE (R32)
}

__global__ void k_quant(const double* __restrict__ t, int n, const unsigned long long* maxbits, int guard,
                        int64_t* __restrict__ tq, int32_t* Fout) {
  const int F = quant_F(*maxbits, n, guard);
  if (blockIdx.x == 0 && threadIdx.x == 0) *Fout = F;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    tq[i] = __double2ll_rn(scalbn(t[i], F));
}

__global__ void k_ln(const double* y, double* out, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
  {
    bool certified;
    out[i] = ln_cr_checked(y[i], certified);
  }
}

// ---- presort, small n: one CTA per feature, column in shared memory
constexpr int kSmallSortMax = 4096;

__global__ void k_presort_small(const double* __restrict__ X, int n, int p, uint32_t* order,
                                uint32_t* grank) {
  extern __shared__ double col[];
  uint8_t* first = reinterpret_cast<uint8_t*>(col + n);
  const int f = blockIdx.x;
  for (int i = threadIdx.x; i < n; i += blockDim.x) col[i] = X[(size_t)i * p + f];
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double x = col[i];
    int lt = 0, eqb = 0;
    for (int j = 0; j < n; ++j) {
      const double v = col[j];
      lt += (v < x);
      eqb += (v == x) & (j < i);
    }
    order[(size_t)f * n + lt + eqb] = (uint32_t)i;
    first[i] = (eqb == 0);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double x = col[i];
    int r = 0;
    for (int j = 0; j < n; ++j) r += first[j] & (col[j] < x);
    grank[(size_t)f * n + i] = (uint32_t)r;
  }
}

// ---- presort, large n
__device__ __forceinline__ unsigned long long ordered_key(double x) {
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void k_make_keys(const double* __restrict__ X, int n, int p, unsigned long long* keys,
                            uint32_t* vals) {
  const size_t total = (size_t)n * p;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t f = i / n, r = i - f * n;
    keys[i] = ordered_key(X[r * p + f]);
    vals[i] = (uint32_t)r;
  }
}

// one CTA per feature: dense rank by scanning the sorted keys in tiles
__global__ void k_rank_sorted(const unsigned long long* __restrict__ skeys,
                              const uint32_t* __restrict__ order, int n, uint32_t* grank) {
  const int f = blockIdx.x;
  const unsigned long long* k = skeys + (size_t)f * n;
  const uint32_t* o = order + (size_t)f * n;
  __shared__ uint32_t wsum[32];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + threadIdx.x;
    uint32_t flag = (i < n && i > 0 && k[i] != k[i - 1]) ? 1u : 0u;
    uint32_t x = flag;
    for (int d = 1; d < 32; d <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      uint32_t v = lane < nw ? wsum[lane] : 0u;
      for (int d = 1; d < 32; d <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= d) v += y;
      }
      if (lane < nw) wsum[lane] = v;
    }
    __syncthreads();
    const uint32_t incl = x + (warp ? wsum[warp - 1] : 0u) + carry;
    if (i < n) grank[(size_t)f * n + o[i]] = incl;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = incl;
    __syncthreads();
  }
}

}  // namespace

int g_opt_ln_margin_log2 = 0;

cudaError_t prep_targets(const double* dX, const double* dy, int n, int p, int target,
                         int require_pos, int guard, DevData& d, double* scratch_t, cudaStream_t s) {
  unsigned long long* maxbits = reinterpret_cast<unsigned long long*>(scratch_t + n);
  cudaMemsetAsync(maxbits, 0, sizeof(unsigned long long), s);
  const size_t total = (size_t)n * p;
  int gx = (int)std::min<size_t>((total + 255) / 256, 148 * 16);
  k_prep_X<<<gx > 0 ? gx : 1, 256, 0, s>>>(dX, d.X, total, d.err);
  note_launch();
  int gy = std::min((n + 255) / 256, 148 * 8);
  const int margin = g_opt_ln_margin_log2 ? g_opt_ln_margin_log2 : kLnCertLog2;
  k_prep_y<<<gy > 0 ? gy : 1, 256, 0, s>>>(dy, scratch_t, n, target, require_pos, maxbits, d.err, margin);
  note_launch();
  k_quant<<<gy > 0 ? gy : 1, 256, 0, s>>>(scratch_t, n, maxbits, guard, d.tq, d.F);
  note_launch();
  return cudaGetLastError();
}

size_t presort_ws_bytes(int n, int p) {
  if (n <= kSmallSortMax) return 0;
  const size_t total = (size_t)n * p;
  size_t temp = 0, temp2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, temp, (const unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, n);
  cub::DeviceSegmentedRadixSort::SortPairs(nullptr, temp2, (const unsigned long long*)nullptr,
                                           (unsigned long long*)nullptr, (const uint32_t*)nullptr,
                                           (uint32_t*)nullptr, (int64_t)total, p, (const int64_t*)nullptr,
                                           (const int64_t*)nullptr);
  temp = std::max(temp, temp2);
  return total * (8 + 8 + 4) + (size_t)(p + 1) * 8 + temp + 256;  // keys x2, values, offsets, CUB temp
}

namespace {
__global__ void k_seg_offsets(int64_t* off, int p, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= p) off[i] = (int64_t)i * n;
}
}  // namespace

cudaError_t presort(DevData& d, void* ws, size_t ws_bytes, cudaStream_t s, bool ranks) {
  const int n = d.n, p = d.p;
  if (n <= kSmallSortMax) {
    size_t smem = (size_t)n * 8 + n;
    if (smem > 48 * 1024)
      allow_max_dynamic_smem(k_presort_small);
    k_presort_small<<<p, 256, smem, s>>>(d.X, n, p, d.order, d.grank);
    note_launch();
    return cudaGetLastError();
  }
  const size_t total = (size_t)n * p;
  char* w = static_cast<char*>(ws);
  unsigned long long* kin = reinterpret_cast<unsigned long long*>(w);
  unsigned long long* kout = kin + total;
  uint32_t* vin = reinterpret_cast<uint32_t*>(kout + total);
  int64_t* offs = reinterpret_cast<int64_t*>((reinterpret_cast<uintptr_t>(vin + total) + 15) & ~uintptr_t(15));
  char* temp = reinterpret_cast<char*>(offs + p + 1);
  size_t temp_bytes = ws_bytes - (size_t)(temp - w);
  k_make_keys<<<148 * 8, 256, 0, s>>>(d.X, n, p, kin, vin);
  note_launch();
  k_seg_offsets<<<(p + 1 + 127) / 128, 128, 0, s>>>(offs, p, n);
  note_launch();
  // long columns: one device-wide radix sort per feature (CUB's segmented sort gives a segment
  // to one CTA, which left the GPU idle -- 190 ms for C4's 64 x 10M keys, rd2_06); short ones:
  // the segmented sort (64 separate sorts of 100k keys took 8 ms against its 2 ms)
  if (n < (1 << 20)) {
    cudaError_t e = cub::DeviceSegmentedRadixSort::SortPairs(temp, temp_bytes, kin, kout, vin, d.order,
                                                             (int64_t)total, p, offs, offs + 1, 0, 64, s);
    if (e != cudaSuccess) return e;
  } else {
    for (int f = 0; f < p; ++f) {
      size_t tb = temp_bytes;
      const size_t o = (size_t)f * n;
      cudaError_t e = cub::DeviceRadixSort::SortPairs(temp, tb, kin + o, kout + o, vin + o, d.order + o, n, 0, 64, s);
      if (e != cudaSuccess) return e;
    }
  }
  if (ranks) {
    k_rank_sorted<<<p, 1024, 0, s>>>(kout, d.order, n, d.grank);
    note_launch();
  }
  return cudaGetLastError();
}

namespace {
__global__ void k_philox(const uint32_t* in, uint32_t* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t* q = in + 6 * i;
  U4 o = philox4x32_10(q[0], q[1], q[2], q[3], q[4], q[5]);
  out[4 * i] = o.x; out[4 * i + 1] = o.y; out[4 * i + 2] = o.z; out[4 * i + 3] = o.w;
}
}  // namespace

cudaError_t device_philox(const uint32_t* ctr_key, uint32_t* out, int n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  k_philox<<<(n + 127) / 128, 128, 0, s>>>(ctr_key, out, n);
  note_launch();
  return cudaGetLastError();
}

cudaError_t device_ln(const double* dy, double* dout, int n, cudaStream_t s) {
  k_ln<<<std::max(1, std::min((n + 255) / 256, 148 * 8)), 256, 0, s>>>(dy, dout, n);
  note_launch();
  return cudaGetLastError();
}

}  // namespace rf
