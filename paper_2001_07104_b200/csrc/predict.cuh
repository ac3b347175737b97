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
// Compact copy of a forest for batch inference: 8-byte nodes (feature | left child << 8, the
// feature 0xFF marking a leaf; the threshold rounded to fp32) and the exact fp64 value of every
// node (threshold or leaf value) beside them.  Trees of < 2^23 nodes, p < 255.
struct __align__(8) Node8 {
  uint32_t fl;  // feature (0xFF: leaf) | tree-local left child slot << 8 (23 bits) | wide << 31
                // (right child = left + (wide ? 8 : 1): the blocked layout, predict.cu)
  float tf;     // fp32(threshold), round to nearest (exact decisions: see k_predict_smem8)
};
cudaError_t build_node8(const Node16* nodes, uint64_t total, Node8* n8, double* val, cudaStream_t s);
// Blocked compact layout of a fitted (BFS-ordered) forest (predict.cu): count -> slots[t] per tree,
// level starts lev [T][kBlkLevStride], nlev[T] (bad |= 1 if the forest does not qualify), then build
// into n8 / val at n8_off (exclusive sums of slots).
constexpr int kBlkLevStride = 2049;
// forests of shallow trees (<= this many nodes per tree on average) take the staged-prefix kernel and
// the blocked layout; deep forests the BFS-slot copy without staging (the blocked layout measured
// 28.0 -> 25.6 M predictions/s on the C3 forest, ~126k nodes per tree: its padding outweighs the
// fewer fetches there, rd2_52/59 bench lines)
constexpr uint64_t kShallowNodesPerTree = 16384;
cudaError_t node8_blocked_count(const Node16* nodes, const uint64_t* tree_off, int T, uint64_t* slots, uint32_t* lev,
                                int* nlev, int* bad, cudaStream_t s);
cudaError_t node8_blocked_build(const Node16* nodes, const uint64_t* tree_off, int T, const uint64_t* n8_off,
                                const uint32_t* lev, const int* nlev, Node8* n8, double* val, cudaStream_t s);
// n8 / val (optional): the compact copy; batches then walk 8-byte nodes (twice the nodes per
// staged byte and per cache line).
cudaError_t predict_forest(const Node16* nodes, const uint64_t* tree_off, int T, const double* X,
                           long long n, int p, int mode, double* out, cudaStream_t s, int* err_few = nullptr,
                           uint64_t total_nodes = 0, const Node8* n8 = nullptr, const double* val = nullptr,
                           const uint64_t* n8_off = nullptr);
cudaError_t predict_finalize(const double* partial, long long n, int T, int target, double* out,
                             cudaStream_t s);
cudaError_t check_finite(const double* X, size_t total, int* err, cudaStream_t s);
}  // namespace rf
