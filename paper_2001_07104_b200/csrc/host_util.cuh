// host_util.cuh -- host-side helpers shared by the library's translation units:
// stream-ordered scratch allocations and per-kernel CUDA-event profiling.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <atomic>
#include <mutex>
#include <vector>

namespace rf {

// Keep freed scratch memory in the device's default pool (release threshold = max):
// with the default threshold 0 the pool returns its memory to the driver at every
// synchronisation, and the next call maps it again (a 128-tree large-path batch
// allocates ~5 GB: re-mapping it cost ~1.5 s per rf_fit call).  Once per device.
// Per-device flags behind a mutex: entry points may be called from several host threads.
inline void retain_pool() {
  static std::atomic<bool> done[64] = {};
  static std::mutex mu;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || done[dev].load(std::memory_order_acquire)) return;
  std::lock_guard<std::mutex> lk(mu);
  if (done[dev].load(std::memory_order_relaxed)) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[dev].store(true, std::memory_order_release);
}

// Opt a kernel into the device's full dynamic shared memory (minus its static shared
// memory).  Always the same value for a kernel, so host threads launching it concurrently
// with different dynamic sizes cannot invalidate each other's launches (setting the exact
// size per call raced: one thread lowered the limit under another's launch).
template <typename K>
inline cudaError_t allow_max_dynamic_smem(K kern) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  int optin = 0;
  e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return e;
  cudaFuncAttributes fa;
  e = cudaFuncGetAttributes(&fa, kern);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes);
}

// stream-ordered scratch allocations (cudaMallocAsync pool), freed at scope exit
struct Scratch {
  cudaStream_t s;
  std::vector<void*> ptrs;
  explicit Scratch(cudaStream_t st) : s(st) { retain_pool(); }
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
void note_row_levels(long long n);
// device counter of evaluated candidate splits (algorithmic work of the split search)
unsigned long long* candidate_counter();

// per-kernel event timing (enabled by rf_set_profiling); defined in api.cu
bool prof_enabled();
void prof_push(const char* name, cudaEvent_t a, cudaEvent_t b);
// a timing event of the current device from the thread's pool (created on first need; the records'
// events return to the pool when profiling is reset, so steady-state scopes create none)
cudaEvent_t prof_event();

struct ProfScope {
  const char* name;
  cudaEvent_t a = nullptr, b = nullptr;
  cudaStream_t s;
  bool on;
  ProfScope(const char* nm, cudaStream_t st) : name(nm), s(st), on(prof_enabled()) {
    if (!on) return;
    a = prof_event();
    b = prof_event();
    cudaEventRecord(a, s);
  }
  ~ProfScope() {
    if (!on) return;
    cudaEventRecord(b, s);
    prof_push(name, a, b);
  }
};

}  // namespace rf
