// Standalone NVLink peer-access probe (not part of the library): achievable SM-driven peer load /
// store bandwidth on this box, one direction and both directions at once, for a few launch shapes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o p2p_probe p2p_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void load_kernel(const float4* __restrict__ src, float4* __restrict__ dst, long long n, int unroll) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    float4 a = __ldcg(src + i), b = __ldcg(src + i + stride), c = __ldcg(src + i + 2 * stride), d = __ldcg(src + i + 3 * stride);
    dst[i] = a; dst[i + stride] = b; dst[i + 2 * stride] = c; dst[i + 3 * stride] = d;
  }
  for (; i < n; i += stride) dst[i] = __ldcg(src + i);
}
__global__ void store_kernel(const float4* __restrict__ src, float4* __restrict__ dst, long long n) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (; i < n; i += stride) __stcg(dst + i, src[i]);
}

int main() {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) { printf("needs 2 GPUs\n"); return 0; }
  const long long bytes = 64ll << 20, n = bytes / 16;
  float4 *a[2], *b[2];
  cudaStream_t st[2];
  cudaEvent_t e0[2], e1[2];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceEnablePeerAccess(1 - d, 0));
    CK(cudaMalloc(&a[d], bytes));
    CK(cudaMalloc(&b[d], bytes));
    CK(cudaMemset(a[d], 0, bytes));
    CK(cudaStreamCreate(&st[d]));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
  }
  struct Shape { int grid, threads; } shapes[] = {{148, 1024}, {296, 512}, {592, 256}, {1184, 256}, {148 * 8, 128}, {2368, 256}};
  for (int kind = 0; kind < 2; ++kind)
    for (int both = 0; both < 2; ++both)
      for (auto sh : shapes) {
        const int iters = 10;
        for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
        for (int d = 0; d < (both ? 2 : 1); ++d) {
          CK(cudaSetDevice(d));
          CK(cudaEventRecord(e0[d], st[d]));
          for (int it = 0; it < iters; ++it) {
            if (kind == 0) load_kernel<<<sh.grid, sh.threads, 0, st[d]>>>(a[1 - d], b[d], n, 4);  // remote -> local
            else store_kernel<<<sh.grid, sh.threads, 0, st[d]>>>(a[d], b[1 - d], n);            // local -> remote
          }
          CK(cudaEventRecord(e1[d], st[d]));
        }
        float ms = 0;
        for (int d = 0; d < (both ? 2 : 1); ++d) {
          CK(cudaSetDevice(d));
          CK(cudaEventSynchronize(e1[d]));
          float m;
          CK(cudaEventElapsedTime(&m, e0[d], e1[d]));
          ms = m > ms ? m : ms;
        }
        printf("%s %s grid %5d x %4d: %6.0f GB/s per GPU per direction\n", kind ? "peer STORE" : "peer LOAD ",
               both ? "both-dirs" : "one-dir  ", sh.grid, sh.threads, bytes * iters / (ms * 1e-3) / 1e9);
      }
  return 0;
}
