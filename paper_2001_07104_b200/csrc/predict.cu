// predict.cu -- batched forest inference (each node compares
// one feature with a threshold until a leaf's value is reached; the forest
// outputs the mean of its trees; exp() for LOG targets).
//
// One thread per query row walks every tree of the flattened BFS forest
// (16-byte nodes, one 128-bit load per visit) and sums the leaf values in
// tree order.  The forest (C1/C2: ~2 MB) stays L1/L2-resident; rows are read
// with 8-byte loads.  Tuned variants live beside it (predict_kernel_*).
#include "common.cuh"
#include "host_util.cuh"
#include "predict.cuh"

namespace rf {
namespace {

__global__ void __launch_bounds__(256) k_predict(const Node16* __restrict__ nodes,
                                                 const uint64_t* __restrict__ tree_off, int T,
                                                 const double* __restrict__ X, long long n, int p,
                                                 int mode, double* __restrict__ out) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n;
       r += (long long)gridDim.x * blockDim.x) {
    const double* x = X + r * p;
    double s = 0.0;
    for (int t = 0; t < T; ++t) {
      const Node16* tn = nodes + tree_off[t];
      uint32_t i = 0;
      Node16 nd = tn[0];
      while (nd.feat >= 0) {
        i = nd.left + ((x[nd.feat] <= nd.v) ? 0u : 1u);
        nd = tn[i];
      }
      s += nd.v;
    }
    if (mode == 1) s = s / (double)T;
    if (mode == 2) s = exp(s / (double)T);
    out[r] = s;
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

cudaError_t predict_forest(const Node16* nodes, const uint64_t* tree_off, int T, const double* X,
                           long long n, int p, int mode, double* out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  long long blocks = (n + 255) / 256;
  if (blocks > 148LL * 64) blocks = 148LL * 64;
  k_predict<<<(unsigned)blocks, 256, 0, s>>>(nodes, tree_off, T, X, n, p, mode, out);
  note_launch();
  return cudaGetLastError();
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
