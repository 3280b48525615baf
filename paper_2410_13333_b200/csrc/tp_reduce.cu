// TP partial-sum reduction over NVLink peer memory, fused with its consumer (SURVEY §8(a) S8 / K15:
// "TP reduce + residual + norm"; PAPER.md:262 row-parallel layers).  One kernel per reduction, no
// NCCL: reduce-scatter + all-gather through peer loads / stores.
//
// Member m of a TP group of k owns rows [m*T/k, (m+1)*T/k).  For each of its rows it reads the k
// fp32 partial rows (its own and the k-1 peers', in member order 0..k-1, so every row is summed in
// one fixed order) and pushes the finished row to every member:
//   TP_SUM        out = sum_j P_j                          (fp32; backward input gradients)
//   TP_RESID_NORM x1 = bf16(x + sum_j P_j), a = bf16(x1 * rsqrt(mean(x1^2) + eps) * g), rstd
//                 (attention output -> residual -> MLP RMSNorm, the same arithmetic as rmsnorm_fwd)
//   TP_RESID      x' = bf16(x + sum_j P_j)                 (MLP output -> residual)
// Per element NVLink traffic per member: (k-1)/k * 4 B in, (k-1)/k * {4, 4, 2} B out — half of a
// ring all-reduce's, and the residual / norm passes over HBM disappear.
//
// Synchronisation (one flag block of 64 u64 per member, in its work arena; epochs count the TP
// reductions of the current plan, identical on every member because they run the same schedule):
//   ready[j]  = epoch: member j's partial for this epoch is complete (written by every CTA of j's
//               kernel before it reads anything; the partial came from an earlier kernel on j's stream)
//   done[j]  += 1 per CTA of member j that finished pushing its rows into this member's buffers
//   ticket    local CTA counter: the last CTA to finish waits until done[j] == epoch * grid for all j,
//             so the kernel completes only when every row of this member's output has landed.
// Partials are double-buffered by epoch parity: member j overwrites P_j[e & 1] in epoch e + 2, after
// it has seen ready(e + 1) from every member, i.e. after every member finished reading epoch e.
// A member's output buffers (activations, or the fp32 sum) are written by peers in epoch e only
// after this member's ready(e), i.e. after all its earlier stream work (readers of the previous
// contents) completed.  A wait that exceeds 20 s traps (sticky CUDA error) instead of hanging.
#include <cuda_bf16.h>
#include "kernels.h"

namespace mls {
namespace {

constexpr int TPR_THREADS = 128;
constexpr int TPR_MAXV = 8;  // 8 vectors of 8 elements per thread: h <= 8192

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void wait_geq(const unsigned long long* p, unsigned long long target) {
  if (ld_acquire_sys(p) >= target) return;
  const unsigned long long t0 = now_ns();
  while (ld_acquire_sys(p) < target) {
    __nanosleep(64);
    if (now_ns() - t0 > 20000000000ull) __trap();  // a member never arrived: fail loudly
  }
}

__device__ __forceinline__ float4 ldcg4(const float* p) { return __ldcg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
  const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = __bfloat1622float2(b[i]);
    f[2 * i] = t.x; f[2 * i + 1] = t.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint4 u;
  __nv_bfloat162* b = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return u;
}
__device__ __forceinline__ float block_sum(float v, float* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  float r = 0.f;
#pragma unroll
  for (int i = 0; i < TPR_THREADS / 32; ++i) r += sh[i];
  return r;
}

template <int MODE>
__global__ void __launch_bounds__(TPR_THREADS) tp_reduce_kernel(const __grid_constant__ TpArgs a) {
  __shared__ float sh[TPR_THREADS / 32];
  __shared__ bool last;
  const int k = a.k, me = a.me, h = a.h, nv = h / 8;
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int j = 0; j < k; ++j) st_release_sys(a.flags[j] + TPF_READY + me, a.epoch);
    for (int j = 0; j < k; ++j) wait_geq(a.flags[me] + TPF_READY + j, a.epoch);
  }
  __syncthreads();
  const int r0 = (int)((long long)me * a.T / k), r1 = (int)((long long)(me + 1) * a.T / k);
  for (int row = r0 + blockIdx.x; row < r1; row += gridDim.x) {
    const long long rb = (long long)row * h;
    float v[TPR_MAXV][8];
#pragma unroll
    for (int i = 0; i < TPR_MAXV; ++i) {
      const int c = threadIdx.x + i * TPR_THREADS;
      if (c < nv) {
        float s[8];
        {
          const float4 p0 = ldcg4(a.part[0] + rb + 8 * c), p1 = ldcg4(a.part[0] + rb + 8 * c + 4);
          s[0] = p0.x; s[1] = p0.y; s[2] = p0.z; s[3] = p0.w; s[4] = p1.x; s[5] = p1.y; s[6] = p1.z; s[7] = p1.w;
        }
        for (int j = 1; j < k; ++j) {
          const float4 p0 = ldcg4(a.part[j] + rb + 8 * c), p1 = ldcg4(a.part[j] + rb + 8 * c + 4);
          s[0] += p0.x; s[1] += p0.y; s[2] += p0.z; s[3] += p0.w;
          s[4] += p1.x; s[5] += p1.y; s[6] += p1.z; s[7] += p1.w;
        }
        if (MODE == TP_SUM) {
#pragma unroll
          for (int t = 0; t < 8; ++t) v[i][t] = s[t];
        } else {
          float xv[8];
          unpack8(reinterpret_cast<const uint4*>(a.x)[(long long)row * nv + c], xv);
#pragma unroll
          for (int t = 0; t < 8; ++t) v[i][t] = xv[t] + s[t];
        }
      }
    }
    if (MODE == TP_SUM) {
#pragma unroll
      for (int i = 0; i < TPR_MAXV; ++i) {
        const int c = threadIdx.x + i * TPR_THREADS;
        if (c < nv) {
          const float4 o0 = make_float4(v[i][0], v[i][1], v[i][2], v[i][3]);
          const float4 o1 = make_float4(v[i][4], v[i][5], v[i][6], v[i][7]);
          for (int j = 0; j < k; ++j) {
            float4* d = reinterpret_cast<float4*>(static_cast<float*>(a.d0[j]) + rb + 8 * c);
            __stcg(d, o0);
            __stcg(d + 1, o1);
          }
        }
      }
    } else {
      float ss = 0.f;
#pragma unroll
      for (int i = 0; i < TPR_MAXV; ++i) {
        const int c = threadIdx.x + i * TPR_THREADS;
        if (c < nv) {
          const uint4 q = pack8(v[i]);  // residual stream is bf16 (reading R6)
          for (int j = 0; j < k; ++j) __stcg(static_cast<uint4*>(a.d0[j]) + (long long)row * nv + c, q);
          if (MODE == TP_RESID_NORM) {
            unpack8(q, v[i]);
#pragma unroll
            for (int t = 0; t < 8; ++t) ss += v[i][t] * v[i][t];
          }
        }
      }
      if (MODE == TP_RESID_NORM) {
        ss = block_sum(ss, sh);
        const float r = rsqrtf(ss / (float)h + a.eps);
        if (threadIdx.x == 0)
          for (int j = 0; j < k; ++j) __stcg(a.d2[j] + row, r);
#pragma unroll
        for (int i = 0; i < TPR_MAXV; ++i) {
          const int c = threadIdx.x + i * TPR_THREADS;
          if (c < nv) {
            float gg[8], o[8];
            unpack8(reinterpret_cast<const uint4*>(a.g)[c], gg);
#pragma unroll
            for (int t = 0; t < 8; ++t) o[t] = v[i][t] * r * gg[t];
            const uint4 q = pack8(o);
            for (int j = 0; j < k; ++j) __stcg(static_cast<uint4*>(a.d1[j]) + (long long)row * nv + c, q);
          }
        }
      }
    }
  }
  // completion: this CTA's pushes -> every member's done counter; the last local CTA waits for all
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int j = 0; j < k; ++j) red_release_sys(a.flags[j] + TPF_DONE + me, 1ull);
    const unsigned long long t = atomicAdd(a.flags[me] + TPF_TICKET, 1ull);
    last = t + 1 == a.epoch * (unsigned long long)gridDim.x;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    const unsigned long long target = a.epoch * (unsigned long long)gridDim.x;
    for (int j = 0; j < k; ++j) wait_geq(a.flags[me] + TPF_DONE + j, target);
    __threadfence_system();
  }
}

}  // namespace

cudaError_t tp_reduce(const TpArgs& a, cudaStream_t st) {
  if (a.k < 2 || a.k > MAX_TP || a.me < 0 || a.me >= a.k || a.h % 8 || a.h > 8 * TPR_MAXV * TPR_THREADS ||
      a.T <= 0 || a.epoch == 0)
    return cudaErrorInvalidValue;
  switch (a.mode) {
    case TP_SUM: tp_reduce_kernel<TP_SUM><<<TP_GRID, TPR_THREADS, 0, st>>>(a); break;
    case TP_RESID_NORM: tp_reduce_kernel<TP_RESID_NORM><<<TP_GRID, TPR_THREADS, 0, st>>>(a); break;
    case TP_RESID: tp_reduce_kernel<TP_RESID><<<TP_GRID, TPR_THREADS, 0, st>>>(a); break;
    default: return cudaErrorInvalidValue;
  }
  count_launch();
  return cudaGetLastError();
}

}  // namespace mls
