// importance.cuh -- feature importance (mean decrease in impurity) of a forest.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace rf {

// out[p] from the per-tree split-decrease sums raw[T][p] (scikit-learn's rule,
// DESIGN.md R30): each tree's row divided by its sum (rows summing to 0
// contribute nothing), summed over trees in tree order, divided by the total.
// ws: >= (T + p) doubles of device scratch.
cudaError_t importance_combine(const double* raw, int T, int p, double* out, double* ws, cudaStream_t s);

}  // namespace rf
