// Fused cross-layout batch-weighted gradient reduction + AdamW on owned ZeRO-1 pieces + bf16 cast
// (§5.1; readings R4, R5, R9).
//
// For every owned piece: G = sum_i w_i g_i over contributing pipelines in fixed pipeline order
// (w_i = m_i b / B), written to rgrad; then torch.optim.AdamW semantics:
//   theta *= 1 - lr*wd;  m = b1 m + (1-b1) G;  v = b2 v + (1-b2) G^2;
//   theta -= lr * (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps)
// and the owner's bf16 param copy = RNE(theta).  HBM-bound: (4 n_src + 16 read, 4 + 12 + 2 write)
// bytes per element.
#include <cuda_bf16.h>
#include "kernels.h"

namespace mls {

__global__ void __launch_bounds__(256) reduce_adam_kernel(const ChunkDesc* __restrict__ chunks,
                                                          const PieceDesc* __restrict__ pieces, AdamHyper hp) {
  const ChunkDesc ch = chunks[blockIdx.x];
  const PieceDesc& pd = pieces[ch.piece];
  const int ns = pd.n_src;
  for (long long i = ch.off + threadIdx.x; i < ch.off + ch.len; i += blockDim.x) {
    float g = 0.f;
    for (int s = 0; s < ns; ++s) g += pd.w[s] * pd.src[s][i];
    pd.rgrad[i] = g;
    if (hp.apply) {
      float th = pd.master[i];
      if (pd.decay) th *= 1.f - hp.lr * hp.wd;
      const float m = hp.b1 * pd.m[i] + (1.f - hp.b1) * g;
      const float v = hp.b2 * pd.v[i] + (1.f - hp.b2) * g * g;
      th -= hp.lr * (m / hp.bc1) / (sqrtf(v / hp.bc2) + hp.eps);
      pd.m[i] = m;
      pd.v[i] = v;
      pd.master[i] = th;
      __nv_bfloat16 b = __float2bfloat16_rn(th);
      pd.param[i] = *reinterpret_cast<uint16_t*>(&b);
    }
  }
}

cudaError_t reduce_adam(int n_chunks, const ChunkDesc* d_chunks, const PieceDesc* d_pieces, const AdamHyper& hp,
                        cudaStream_t st) {
  if (n_chunks <= 0) return cudaSuccess;
  reduce_adam_kernel<<<n_chunks, 256, 0, st>>>(d_chunks, d_pieces, hp); count_launch();
  return cudaGetLastError();
}

}  // namespace mls
