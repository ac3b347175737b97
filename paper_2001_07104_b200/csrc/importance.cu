// importance.cu -- feature importance of a forest (
// PAPER.md P:218-219, Table 6): mean decrease in impurity.
//
// The growth kernels add each split's decrease (common.cuh mdi_decrease) to
// raw[tree][feature]; these kernels turn raw[T][p] into the importance vector
// with the rule of the library the paper uses (R30).  Three tiny
// launches, deterministic (fixed summation order).
#include <cub/block/block_reduce.cuh>

#include "host_util.cuh"
#include "importance.cuh"

namespace rf {
namespace {

constexpr int kThreads = 256;

// one CTA per tree: row sum
__global__ void k_imp_rowsum(const double* __restrict__ raw, int p, double* __restrict__ rowsum) {
  const int t = blockIdx.x;
  double v = 0.0;
  for (int f = threadIdx.x; f < p; f += blockDim.x) v += raw[(size_t)t * p + f];
  using BR = cub::BlockReduce<double, kThreads>;
  __shared__ typename BR::TempStorage tmp;
  const double s = BR(tmp).Sum(v);
  if (threadIdx.x == 0) rowsum[t] = s;
}

// thread per feature: sum over trees of the normalised rows, in tree order
__global__ void k_imp_accum(const double* __restrict__ raw, int T, int p, const double* __restrict__ rowsum,
                            double* __restrict__ acc) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= p) return;
  double a = 0.0;
  for (int t = 0; t < T; ++t) {
    const double s = rowsum[t];
    if (s > 0.0) a += raw[(size_t)t * p + f] / s;
  }
  acc[f] = a;
}

// one CTA: divide by the total
__global__ void k_imp_final(const double* __restrict__ acc, int p, double* __restrict__ out) {
  double v = 0.0;
  for (int f = threadIdx.x; f < p; f += blockDim.x) v += acc[f];
  using BR = cub::BlockReduce<double, kThreads>;
  __shared__ typename BR::TempStorage tmp;
  __shared__ double tot;
  const double s = BR(tmp).Sum(v);
  if (threadIdx.x == 0) tot = s;
  __syncthreads();
  for (int f = threadIdx.x; f < p; f += blockDim.x) out[f] = tot > 0.0 ? acc[f] / tot : acc[f];
}

}  // namespace

cudaError_t importance_combine(const double* raw, int T, int p, double* out, double* ws, cudaStream_t s) {
  if (T <= 0 || p <= 0) return cudaSuccess;
  double* rowsum = ws;
  double* acc = ws + T;
  k_imp_rowsum<<<T, kThreads, 0, s>>>(raw, p, rowsum);
  k_imp_accum<<<(p + kThreads - 1) / kThreads, kThreads, 0, s>>>(raw, T, p, rowsum, acc);
  k_imp_final<<<1, kThreads, 0, s>>>(acc, p, out);
  note_launch(3);
  return cudaGetLastError();
}

}  // namespace rf
