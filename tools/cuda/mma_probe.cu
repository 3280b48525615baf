// Standalone tcgen05.mma throughput probe (not part of the library): back-to-back MMAs of one shape
// from one CTA per SM, operands resident in smem / TMEM, timed with clock64 around N issues + commit
// wait.  Reports cycles per instruction for SS (A, B in smem) and TS (A in TMEM) forms.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2410_13333_b200/csrc -o mma_probe mma_probe.cu
#include <cstdio>
#include <cuda_bf16.h>
#include "ptx.cuh"
using namespace mls;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) probe(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 112 * 1024 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(&slot, 512);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t id = umma_idesc_bf16(128, N, false, false);
    const uint32_t a = smem_u32(smem), b = a + 32768;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t bd = umma_desc_sw128(b + (kk >> 2) * 32768 + (kk & 3) * 32, 16, 1024);
        if (TS) umma_f16_ts(tb, tb + 256 + kk * 8, bd, id, 1);
        else umma_f16(tb, umma_desc_sw128(a + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024), bd, id, 1);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = (t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tb, 512); }
}

template <int N, bool TS>
void run(const char* name, int blocks) {
  long long* d;
  cudaMalloc(&d, blocks * sizeof(long long));
  auto k = probe<N, TS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
  const int iters = 2000;
  k<<<blocks, 128, 120 * 1024>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
  long long h[148];
  cudaMemcpy(h, d, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < blocks; ++i) mx = h[i] > mx ? h[i] : mx;
  const double per = mx / (iters * 8.0);
  const double flop_per_clk = 2.0 * 128 * N * 16 / per;
  printf("%-28s blocks %3d: %6.1f cycles/instr  (%5.0f flop/clk/SM, ideal %d cycles)\n", name, blocks, per,
         flop_per_clk, 128 * N / 256);
  cudaFree(d);
}

int main() {
  for (int blocks : {1, 148}) {
    run<64, false>("SS M128 N64 K16", blocks);
    run<128, false>("SS M128 N128 K16", blocks);
    run<256, false>("SS M128 N256 K16", blocks);
    run<64, true>("TS M128 N64 K16", blocks);
    run<128, true>("TS M128 N128 K16", blocks);
    run<256, true>("TS M128 N256 K16", blocks);
  }
  return 0;
}
