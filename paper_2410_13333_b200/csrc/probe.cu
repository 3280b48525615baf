// Speed probe and straggler emulation kernels.
//  * probe_copy: HBM stream copy used with a fixed GEMM by malleus_probe_speed (PAPER.md:742-745:
//    CUDA-event timing of computation to estimate straggling rates).
//  * spin_ns: one-thread spin on %globaltimer (DUTY-cycle emulation).
//  * hog: persistent kernel that occupies whole SMs (1024 threads, ~200 KB smem, FMA loop) until
//    a host-mapped flag is set: an SM-limited slowdown standing in for the paper's extra
//    compute processes.
#include "kernels.h"

namespace mls {

__global__ void probe_copy_kernel(long long n, const float4* __restrict__ src, float4* __restrict__ dst) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

cudaError_t probe_copy(long long n, const float* src, float* dst, cudaStream_t st) {
  probe_copy_kernel<<<148 * 8, 256, 0, st>>>(n / 4, (const float4*)src, (float4*)dst); count_launch();
  return cudaGetLastError();
}

__global__ void spin_kernel(long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while ((long long)(t - t0) < ns);
}

cudaError_t spin_ns(long long ns, cudaStream_t st) {
  if (ns <= 0) return cudaSuccess;
  spin_kernel<<<1, 32, 0, st>>>(ns); count_launch();
  return cudaGetLastError();
}

constexpr int HOG_SMEM = 200 * 1024;

__global__ void __launch_bounds__(1024, 1) hog_kernel(volatile int* stop, int* started, float seed) {
  extern __shared__ float hsm[];
  float a[24];
#pragma unroll
  for (int i = 0; i < 24; ++i) a[i] = seed + i;
  if (threadIdx.x == 0) { atomicAdd_system(started, 1); __threadfence_system(); }
  int it = 0;
  while (true) {
#pragma unroll 4
    for (int k = 0; k < 256; ++k)
#pragma unroll
      for (int i = 0; i < 24; ++i) a[i] = fmaf(a[i], 0.999999f, 1e-7f);
    if ((++it & 7) == 0 && *stop) break;
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 24; ++i) s += a[i];
  if (s == 12345.678f) hsm[threadIdx.x] = s;  // keep the loop alive
}

cudaError_t hog_start(int n_sms, volatile int* stop_flag, cudaStream_t st) {
  if (n_sms <= 0) return cudaSuccess;
  cudaFuncSetAttribute(hog_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, HOG_SMEM);
  static int* started = nullptr;  // host-mapped pinned counter
  static int* dstarted = nullptr;
  cudaError_t e;
  if (!started) {
    e = cudaHostAlloc((void**)&started, sizeof(int), cudaHostAllocMapped);
    if (e != cudaSuccess) return e;
    e = cudaHostGetDevicePointer((void**)&dstarted, started, 0);
    if (e != cudaSuccess) return e;
  }
  *(volatile int*)started = 0;
  hog_kernel<<<n_sms, 1024, HOG_SMEM, st>>>(stop_flag, dstarted, 1.0f); count_launch();
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  // wait (bounded, ~1 s) until every hog block is resident
  for (long i = 0; i < 100000000L && *(volatile int*)started < n_sms; ++i) {
  }
  return cudaSuccess;
}

}  // namespace mls
