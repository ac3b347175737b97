// microbench.cu -- B200 unit-throughput measurements behind DESIGN.md sec. 6.
//
//   fp64   : DFMA / DMUL / DADD throughput (the fp64 peak the C1/C2 roofline uses;
//            MEASURED_PEAKS.json has none) -- independent chains, full occupancy
//   atoms  : shared-memory histogram update cost for the C4 histogram build: per update
//            one (W, S) pair into 21 x 256 bins at random addresses, in the variants
//              u32+u64cas  atomicAdd(u32) + atomicAdd(u64) (ptxas: ATOMS + CAS loop)
//              2xu32       two atomicAdd(u32), no return
//              3xu32       three atomicAdd(u32), no return
//              u32r+u32    one atomicAdd(u32) with its return value used + one without
//              1xu32       one atomicAdd(u32)
//   mma    : legacy warp mma.sync m16n8k32 s8 (int32 accumulate) throughput
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb microbench.cu && ./mb
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; } } while (0)

template <int OP>
__global__ void k_fp64(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
         x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (OP == 0) {
        x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
        x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
      } else if (OP == 1) {
        x0 = __dmul_rn(x0, a); x1 = __dmul_rn(x1, a); x2 = __dmul_rn(x2, a); x3 = __dmul_rn(x3, a);
        x4 = __dmul_rn(x4, a); x5 = __dmul_rn(x5, a); x6 = __dmul_rn(x6, a); x7 = __dmul_rn(x7, a);
      } else {
        x0 = __dadd_rn(x0, b); x1 = __dadd_rn(x1, b); x2 = __dadd_rn(x2, b); x3 = __dadd_rn(x3, b);
        x4 = __dadd_rn(x4, b); x5 = __dadd_rn(x5, b); x6 = __dadd_rn(x6, b); x7 = __dadd_rn(x7, b);
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

constexpr int kM = 21, kBins = 256;

template <int V>
__global__ void __launch_bounds__(256) k_atoms(unsigned long long* sink, int iters) {
  extern __shared__ __align__(16) char sm[];
  uint32_t* w32 = reinterpret_cast<uint32_t*>(sm);
  unsigned long long* s64 = reinterpret_cast<unsigned long long*>(sm + kM * kBins * 4);
  uint32_t* s32a = reinterpret_cast<uint32_t*>(sm + kM * kBins * 4);
  uint32_t* s32b = reinterpret_cast<uint32_t*>(sm + kM * kBins * 8);
  for (int i = threadIdx.x; i < kM * kBins * 3; i += blockDim.x) w32[i] = 0u;
  __syncthreads();
  uint32_t h = 0x9E3779B9u * (threadIdx.x + 1) + blockIdx.x * 7919u;
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 4
    for (int j = 0; j < kM; ++j) {
      h ^= h << 13; h ^= h >> 17; h ^= h << 5;
      const int idx = j * kBins + (h & 255u);
      const uint32_t wv = 1u + (h >> 30);
      const unsigned long long sv = (unsigned long long)h * 977u;
      if (V == 0) { atomicAdd(&w32[idx], wv); atomicAdd(&s64[idx], sv); }
      if (V == 1) { atomicAdd(&w32[idx], wv); atomicAdd(&s32a[idx], (uint32_t)sv); }
      if (V == 2) { atomicAdd(&w32[idx], wv); atomicAdd(&s32a[idx], (uint32_t)sv); atomicAdd(&s32b[idx], (uint32_t)(sv >> 32)); }
      if (V == 3) { const uint32_t o = atomicAdd(&s32a[idx], (uint32_t)sv); atomicAdd(&w32[idx], wv + (o > ~(uint32_t)sv ? 1u : 0u)); }
      if (V == 4) { atomicAdd(&w32[idx], wv); }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kM * kBins; i += blockDim.x) acc += w32[i];
  if (acc == 0xFFFFFFFFu) sink[0] = acc;
}

__global__ void k_mma(int* out, int iters) {
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x1234, b1 = a0 ^ 0x777;
  int c[4][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      asm volatile(
          "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
          : "+r"(c[u][0]), "+r"(c[u][1]), "+r"(c[u][2]), "+r"(c[u][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  int s = 0;
  for (int u = 0; u < 4; ++u) s += c[u][0] + c[u][1] + c[u][2] + c[u][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  cudaDeviceProp pr;
  CK(cudaGetDeviceProperties(&pr, 0));
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const int sms = pr.multiProcessorCount;
  printf("device %s, %d SMs, max SM clock %.0f MHz\n", pr.name, sms, clk_khz / 1e3);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  // ---- fp64
  {
    double* out;
    CK(cudaMalloc(&out, (size_t)sms * 8 * 256 * 8));
    const int iters = 4096;
    const char* names[3] = {"DFMA", "DMUL", "DADD"};
    for (int op = 0; op < 3; ++op) {
      auto launch = [&]() {
        if (op == 0) k_fp64<0><<<sms * 8, 256>>>(out, iters, 0.999999, 1e-9);
        if (op == 1) k_fp64<1><<<sms * 8, 256>>>(out, iters, 0.999999, 1e-9);
        if (op == 2) k_fp64<2><<<sms * 8, 256>>>(out, iters, 0.999999, 1e-9);
      };
      launch();
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) launch();
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = 5.0 * sms * 8 * 256 * (double)iters * 64;
      printf("fp64 %s: %.2f Tops/s (%s %.2f TFLOP/s)\n", names[op], ops / (ms / 1e3) / 1e12,
             op == 0 ? "2 flops/FMA:" : "1 flop/op:", ops * (op == 0 ? 2 : 1) / (ms / 1e3) / 1e12);
    }
    cudaFree(out);
  }
  // ---- shared atomics
  {
    unsigned long long* sink;
    CK(cudaMalloc(&sink, 8));
    const size_t smem = (size_t)kM * kBins * 12;
    const char* names[5] = {"u32+u64cas", "2xu32", "3xu32", "u32r+u32", "1xu32"};
    const int iters = 256;
    for (int v = 0; v < 5; ++v) {
      auto launch = [&]() {
        if (v == 0) k_atoms<0><<<sms * 3, 256, smem>>>(sink, iters);
        if (v == 1) k_atoms<1><<<sms * 3, 256, smem>>>(sink, iters);
        if (v == 2) k_atoms<2><<<sms * 3, 256, smem>>>(sink, iters);
        if (v == 3) k_atoms<3><<<sms * 3, 256, smem>>>(sink, iters);
        if (v == 4) k_atoms<4><<<sms * 3, 256, smem>>>(sink, iters);
      };
      CK(cudaFuncSetAttribute(k_atoms<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      CK(cudaFuncSetAttribute(k_atoms<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      CK(cudaFuncSetAttribute(k_atoms<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      CK(cudaFuncSetAttribute(k_atoms<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      CK(cudaFuncSetAttribute(k_atoms<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      launch();
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) launch();
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      const double upd = 5.0 * sms * 3 * 256 * (double)iters * kM;
      const double per_clk_sm = upd / (ms / 1e3) / sms / (clk_khz * 1e3);
      printf("atoms %-11s: %.1f G updates/s = %.3f updates/clk/SM (%.2f SM-cycles per update)\n", names[v],
             upd / (ms / 1e3) / 1e9, per_clk_sm, 1.0 / per_clk_sm);
    }
    cudaFree(sink);
  }
  // ---- mma.sync int8
  {
    int* out;
    CK(cudaMalloc(&out, (size_t)sms * 8 * 256 * 4));
    const int iters = 4096;
    k_mma<<<sms * 8, 256>>>(out, iters);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k_mma<<<sms * 8, 256>>>(out, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    const double mmas = 5.0 * sms * 8 * 8 * (double)iters * 4;  // warp-level mma instructions
    printf("mma.sync m16n8k32 u8: %.2f T int-ops/s (%.3f mma/clk/SM)\n", mmas * 4096 * 2 / (ms / 1e3) / 1e12,
           mmas / (ms / 1e3) / sms / (clk_khz * 1e3));
    cudaFree(out);
  }
  return 0;
}
