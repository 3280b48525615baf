// Standalone check of the tcgen05 "ts" MMA form (A from TMEM) used by the attention backward:
// D[128 x 64] = A[128 x 64] * B[64 x 64]^T with A written to TMEM by tcgen05.st (packed bf16
// pairs, lane = row) and B K-major 128B-swizzled in smem.  Prints the max error vs a host GEMM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2410_13333_b200/csrc -o ts_probe ts_probe.cu
#include <cstdio>
#include <cmath>
#include <vector>
#include <cuda_bf16.h>
#include "ptx.cuh"
using namespace mls;

__global__ void __launch_bounds__(128, 1) ts_kernel(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D) {
  __shared__ __align__(1024) uint8_t sB[64 * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int t = threadIdx.x, warp = t >> 5;
  // B: 64 rows (n) x 64 cols (k) bf16 -> K-major SW128: row n at n*128 B, 16-B chunk c at c ^ (n & 7)
  for (int idx = t; idx < 64 * 8; idx += 128) {
    const int n = idx / 8, c = idx % 8;
    *reinterpret_cast<uint4*>(sB + n * 128 + ((c ^ (n & 7)) << 4)) = *reinterpret_cast<const uint4*>(B + n * 64 + c * 8);
  }
  if (t == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(&slot, 128);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = slot;
  // A row t -> TMEM lane t, columns [64, 96): 64 bf16 packed in pairs
  {
    uint32_t r[16];
    for (int h = 0; h < 2; ++h) {
      for (int j = 0; j < 16; ++j) {
        __nv_bfloat162 v = __halves2bfloat162(A[t * 64 + h * 32 + 2 * j], A[t * 64 + h * 32 + 2 * j + 1]);
        r[j] = *reinterpret_cast<uint32_t*>(&v);
      }
      tmem_st16(tb + ((uint32_t)(warp * 32) << 16) + 64 + h * 16, r);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (t == 0) {
    constexpr uint32_t id = umma_idesc_bf16(128, 64, false, false);
    for (int kk = 0; kk < 4; ++kk)
      umma_f16_ts(tb, tb + 64 + kk * 8, umma_desc_sw128(smem_u32(sB) + kk * 32, 16, 1024), id, kk > 0);
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t u[32];
  for (int h = 0; h < 2; ++h) {
    tmem_ld32(tb + ((uint32_t)(warp * 32) << 16) + h * 32, u);
    tmem_wait_ld();
    for (int j = 0; j < 32; ++j) D[t * 64 + h * 32 + j] = __uint_as_float(u[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tb, 128); }
}

int main() {
  std::vector<__nv_bfloat16> A(128 * 64), B(64 * 64);
  std::vector<float> Af(128 * 64), Bf(64 * 64), D(128 * 64);
  unsigned s = 1;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return ((s >> 9) & 0xFFFF) / 32768.f - 1.f; };
  for (int i = 0; i < 128 * 64; ++i) { A[i] = __float2bfloat16(rnd()); Af[i] = __bfloat162float(A[i]); }
  for (int i = 0; i < 64 * 64; ++i) { B[i] = __float2bfloat16(rnd()); Bf[i] = __bfloat162float(B[i]); }
  __nv_bfloat16 *dA, *dB; float* dD;
  cudaMalloc(&dA, A.size() * 2); cudaMalloc(&dB, B.size() * 2); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  ts_kernel<<<1, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 64; ++n) {
      double r = 0;
      for (int k = 0; k < 64; ++k) r += (double)Af[m * 64 + k] * Bf[n * 64 + k];
      mx = fmax(mx, fabs(r - D[m * 64 + n]));
    }
  printf("ts MMA 128x64x64: max abs err %.3e (%s)\n", mx, mx < 1e-3 ? "OK" : "MISMATCH");
  return mx < 1e-3 ? 0 : 2;
}
