// Speed probe and straggler emulation kernels.
//  * probe_copy: HBM stream copy used with a fixed GEMM by malleus_probe_speed (PAPER.md:742-745:
//    CUDA-event timing of computation to estimate straggling rates).
//  * spin_ns: one-thread spin on %globaltimer (DUTY-cycle emulation).
// (An SM-occupying "HOG" kernel was tried for S19 and removed: a resident persistent kernel
// deadlocks every device-wide synchronisation of the process; DUTY is the emulation.)
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

}  // namespace mls
