// predict.cuh -- forest inference launchers.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "common.cuh"

namespace rf {
// rows up to this count take the latency kernel (one CTA per row, threads over trees)
constexpr long long kFewRows = 256;
// mode 0: un-divided sum (tree-shard partial); 1: mean; 2: exp(mean) (LOG).
// err_few: if non-null and n <= kFewRows, the latency kernel also checks the rows
// for non-finite values (flag bit 0); otherwise the caller checks separately.
// total_nodes (if known): forests of shallow trees (<= 16384 nodes per tree on average) have
// the top BFS nodes of each tree group staged in shared memory (see k_predict_smem).
cudaError_t predict_forest(const Node16* nodes, const uint64_t* tree_off, int T, const double* X,
                           long long n, int p, int mode, double* out, cudaStream_t s, int* err_few = nullptr,
                           uint64_t total_nodes = 0);
cudaError_t predict_finalize(const double* partial, long long n, int T, int target, double* out,
                             cudaStream_t s);
cudaError_t check_finite(const double* X, size_t total, int* err, cudaStream_t s);
}  // namespace rf
