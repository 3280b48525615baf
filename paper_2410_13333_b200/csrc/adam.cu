// Fused cross-layout batch-weighted gradient reduction + AdamW on owned ZeRO-1 pieces + bf16 cast
// (§5.1; readings R4, R5, R9).
//
// For every owned piece: G = sum_i w_i g_i over contributing pipelines in fixed pipeline order
// (w_i = m_i b / B); optionally written to rgrad; then torch.optim.AdamW semantics:
//   theta *= 1 - lr*wd;  m = b1 m + (1-b1) G;  v = b2 v + (1-b2) G^2;
//   theta -= lr * (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps)
// and the owner's bf16 param copy = RNE(theta).  Optional global-norm clipping (torch
// clip_grad_norm_ semantics) runs as two passes: reduce (rgrad + per-chunk sum of G^2), world sum,
// coefficient, then AdamW on rgrad * coef (apply 3).  HBM-bound: per element (4 n_src + 12) B read and
// (12 + 2 [+ 4 rgrad]) B written; 128-bit accesses when the piece is 16-byte aligned.
#include <cuda_bf16.h>
#include "kernels.h"

namespace mls {

struct AdamEl {
  float th, m, v, g;
};

__device__ __forceinline__ float adam_one(float g, float& th, float& m, float& v, const AdamHyper& hp, int decay) {
  if (decay) th *= 1.f - hp.lr * hp.wd;
  m = hp.b1 * m + (1.f - hp.b1) * g;
  v = hp.b2 * v + (1.f - hp.b2) * g * g;
  th -= hp.lr * (m / hp.bc1) / (sqrtf(v / hp.bc2) + hp.eps);
  return th;
}

__global__ void __launch_bounds__(256) reduce_adam_kernel(const ChunkDesc* __restrict__ chunks,
                                                          const PieceDesc* __restrict__ pieces, AdamHyper hp) {
  const ChunkDesc ch = chunks[blockIdx.x];
  const PieceDesc& pd = pieces[ch.piece];
  const int ns = pd.n_src;
  const bool from_rgrad = hp.apply == 3;
  const bool keep_rgrad = hp.apply != 2 && !from_rgrad;
  const float cf = from_rgrad ? *hp.coef : 1.f;
  float sq = 0.f;
  if (pd.vec) {
    // 4 elements per thread per iteration
    for (long long i = ch.off + 4 * threadIdx.x; i < ch.off + ch.len; i += 4 * blockDim.x) {
      float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
      if (from_rgrad) {
        g = *reinterpret_cast<const float4*>(pd.rgrad + i);
        g.x *= cf; g.y *= cf; g.z *= cf; g.w *= cf;
      } else {
        for (int s = 0; s < ns; ++s) {
          const float4 x = *reinterpret_cast<const float4*>(pd.src[s] + i);
          const float w = pd.w[s];
          g.x += w * x.x; g.y += w * x.y; g.z += w * x.z; g.w += w * x.w;
        }
      }
      if (hp.sq) sq += g.x * g.x + g.y * g.y + g.z * g.z + g.w * g.w;
      if (keep_rgrad) *reinterpret_cast<float4*>(pd.rgrad + i) = g;
      if (hp.apply) {
        float4 th = *reinterpret_cast<const float4*>(pd.master + i);
        float4 m = *reinterpret_cast<const float4*>(pd.m + i);
        float4 v = *reinterpret_cast<const float4*>(pd.v + i);
        adam_one(g.x, th.x, m.x, v.x, hp, pd.decay);
        adam_one(g.y, th.y, m.y, v.y, hp, pd.decay);
        adam_one(g.z, th.z, m.z, v.z, hp, pd.decay);
        adam_one(g.w, th.w, m.w, v.w, hp, pd.decay);
        *reinterpret_cast<float4*>(pd.master + i) = th;
        *reinterpret_cast<float4*>(pd.m + i) = m;
        *reinterpret_cast<float4*>(pd.v + i) = v;
        if (pd.param_f32) {  // FP32 parity mode: the param copies are the fp32 master itself
          *reinterpret_cast<float4*>(reinterpret_cast<float*>(pd.param) + i) = th;
          for (int q = 0; q < pd.n_push; ++q) *reinterpret_cast<float4*>(reinterpret_cast<float*>(pd.push[q]) + i) = th;
          continue;
        }
        __nv_bfloat162 lo = __floats2bfloat162_rn(th.x, th.y), hi = __floats2bfloat162_rn(th.z, th.w);
        uint2 pk;
        pk.x = *reinterpret_cast<uint32_t*>(&lo);
        pk.y = *reinterpret_cast<uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(pd.param + i) = pk;
        for (int q = 0; q < pd.n_push; ++q) *reinterpret_cast<uint2*>(pd.push[q] + i) = pk;  // NVLink stores
      }
    }
  } else {
  for (long long i = ch.off + threadIdx.x; i < ch.off + ch.len; i += blockDim.x) {
    float g = 0.f;
    if (from_rgrad) g = pd.rgrad[i] * cf;
    else
      for (int s = 0; s < ns; ++s) g += pd.w[s] * pd.src[s][i];
    if (hp.sq) sq += g * g;
    if (keep_rgrad) pd.rgrad[i] = g;
    if (hp.apply) {
      float th = pd.master[i], m = pd.m[i], v = pd.v[i];
      adam_one(g, th, m, v, hp, pd.decay);
      pd.m[i] = m;
      pd.v[i] = v;
      pd.master[i] = th;
      if (pd.param_f32) {
        reinterpret_cast<float*>(pd.param)[i] = th;
        for (int q = 0; q < pd.n_push; ++q) reinterpret_cast<float*>(pd.push[q])[i] = th;
        continue;
      }
      __nv_bfloat16 b = __float2bfloat16_rn(th);
      pd.param[i] = *reinterpret_cast<uint16_t*>(&b);
      for (int q = 0; q < pd.n_push; ++q) pd.push[q][i] = *reinterpret_cast<uint16_t*>(&b);
    }
  }
  }
  if (hp.sq) {  // this chunk's sum of G^2, fixed-order block reduction (deterministic)
    __shared__ float red[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      float t = 0.f;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
      hp.sq[blockIdx.x] = t;
    }
  }
}

__global__ void __launch_bounds__(1024) sq_total_kernel(int n, const float* __restrict__ sq, double* __restrict__ out) {
  __shared__ double red[1024];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += sq[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

__global__ void clip_coef_kernel(const double* __restrict__ total, float max_norm, float* __restrict__ coef,
                                 float* __restrict__ norm) {
  const double t = sqrt(*total);
  const double c = (double)max_norm / (t + 1e-6);
  *coef = c < 1.0 ? (float)c : 1.f;
  *norm = (float)t;
}

cudaError_t sq_total(int n, const float* sq, double* local, cudaStream_t st) {
  sq_total_kernel<<<1, 1024, 0, st>>>(n, sq, local); count_launch();
  return cudaGetLastError();
}
cudaError_t clip_coef(const double* total, float max_norm, float* coef, float* norm, cudaStream_t st) {
  clip_coef_kernel<<<1, 1, 0, st>>>(total, max_norm, coef, norm); count_launch();
  return cudaGetLastError();
}

cudaError_t reduce_adam(int n_chunks, const ChunkDesc* d_chunks, const PieceDesc* d_pieces, const AdamHyper& hp,
                        cudaStream_t st) {
  if (n_chunks <= 0) return cudaSuccess;
  reduce_adam_kernel<<<n_chunks, 256, 0, st>>>(d_chunks, d_pieces, hp); count_launch();
  return cudaGetLastError();
}

}  // namespace mls
