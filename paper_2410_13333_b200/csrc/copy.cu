// Multi-range copy: the migration pack / unpack kernel.
// Copies many (src, dst, bytes) ranges in one launch: gathers this rank's outgoing shard deltas
// into one contiguous buffer per destination peer (pack), scatters received buffers into the new
// layout (unpack), and performs the local keep-copies.  One block per <= 64 KB chunk, 16-byte
// vector path when aligned (4 loads in flight per thread).  HBM-bound: 2 x bytes moved.
#include "kernels.h"

namespace mls {

__global__ void __launch_bounds__(256) copy_ranges_kernel(const CopyDesc* __restrict__ d) {
  const CopyDesc c = d[blockIdx.x];
  const uintptr_t s = reinterpret_cast<uintptr_t>(c.src), t = reinterpret_cast<uintptr_t>(c.dst);
  if (((s | t | (uintptr_t)c.bytes) & 15) == 0) {
    // four 16-byte loads in flight per thread before their stores (hides NVLink / HBM latency on
    // the peer pulls of migration)
    const uint4* sp = reinterpret_cast<const uint4*>(c.src);
    uint4* tp = reinterpret_cast<uint4*>(c.dst);
    const long long n = c.bytes / 16, bd = blockDim.x;
    long long i = threadIdx.x;
    for (; i + 3 * bd < n; i += 4 * bd) {
      const uint4 a = sp[i], b = sp[i + bd], e = sp[i + 2 * bd], f = sp[i + 3 * bd];
      tp[i] = a; tp[i + bd] = b; tp[i + 2 * bd] = e; tp[i + 3 * bd] = f;
    }
    for (; i < n; i += bd) tp[i] = sp[i];
  } else if (((s | t | (uintptr_t)c.bytes) & 3) == 0) {
    const uint32_t* sp = reinterpret_cast<const uint32_t*>(c.src);
    uint32_t* tp = reinterpret_cast<uint32_t*>(c.dst);
    for (long long i = threadIdx.x; i < c.bytes / 4; i += blockDim.x) tp[i] = sp[i];
  } else {
    const uint16_t* sp = reinterpret_cast<const uint16_t*>(c.src);
    uint16_t* tp = reinterpret_cast<uint16_t*>(c.dst);
    for (long long i = threadIdx.x; i < c.bytes / 2; i += blockDim.x) tp[i] = sp[i];
  }
}

cudaError_t copy_ranges(int n, const CopyDesc* d_desc, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  for (int off = 0; off < n; off += 65535) {
    const int cnt = n - off < 65535 ? n - off : 65535;
    copy_ranges_kernel<<<cnt, 256, 0, st>>>(d_desc + off); count_launch();
  }
  return cudaGetLastError();
}

}  // namespace mls
