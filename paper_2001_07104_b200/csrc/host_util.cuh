// host_util.cuh -- host-side helpers shared by the library's translation units:
// stream-ordered scratch allocations and per-kernel CUDA-event profiling.
#pragma once
#include <cuda_runtime.h>
#include <vector>

namespace rf {

// stream-ordered scratch allocations (cudaMallocAsync pool), freed at scope exit
struct Scratch {
  cudaStream_t s;
  std::vector<void*> ptrs;
  explicit Scratch(cudaStream_t st) : s(st) {}
  ~Scratch() {
    for (void* p : ptrs) cudaFreeAsync(p, s);
  }
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  template <typename T>
  cudaError_t alloc(T** p, size_t count) {
    if (count == 0) count = 1;
    void* q = nullptr;
    cudaError_t e = cudaMallocAsync(&q, count * sizeof(T), s);
    if (e == cudaSuccess) {
      ptrs.push_back(q);
      *p = static_cast<T*>(q);
    }
    return e;
  }
};

// count of this library's kernel launches (rf_debug_counters); defined in api.cu
void note_launch(int n = 1);
// device counter of evaluated candidate splits (algorithmic work of the split search)
unsigned long long* candidate_counter();

// per-kernel event timing (enabled by rf_set_profiling); defined in api.cu
bool prof_enabled();
void prof_push(const char* name, cudaEvent_t a, cudaEvent_t b);

struct ProfScope {
  const char* name;
  cudaEvent_t a = nullptr, b = nullptr;
  cudaStream_t s;
  bool on;
  ProfScope(const char* nm, cudaStream_t st) : name(nm), s(st), on(prof_enabled()) {
    if (!on) return;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
  }
  ~ProfScope() {
    if (!on) return;
    cudaEventRecord(b, s);
    prof_push(name, a, b);
  }
};

}  // namespace rf
