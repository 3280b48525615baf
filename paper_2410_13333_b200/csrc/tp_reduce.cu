// TP partial-sum reduction over NVLink peer memory, fused with its consumer (SURVEY §8(a) S8 / K15:
// "TP reduce + residual + norm"; PAPER.md:262 row-parallel layers).  One kernel per reduction, no
// NCCL: reduce-scatter + all-gather through peer loads / stores.
//
// Member m of a TP group of k owns rows [m*T/k, (m+1)*T/k), or an uneven range sized like its
// column share (TpArgs::row0) so that the replicated per-token work follows the member's speed.  For each of its rows it reads the k
// fp32 partial rows (its own and the k-1 peers', in member order 0..k-1, so every row is summed in
// one fixed order) and pushes the finished row to every member:
//   TP_SUM        out = sum_j P_j                          (fp32 or bf16; backward input gradients)
//   TP_RESID_NORM x1 = bf16(x + sum_j P_j), a = bf16(x1 * rsqrt(mean(x1^2) + eps) * g), rstd
//                 (attention output -> residual -> MLP RMSNorm, the same arithmetic as rmsnorm_fwd)
//   TP_RESID      x' = bf16(x + sum_j P_j)                 (MLP output -> residual)
// Per element NVLink traffic per member: (k-1)/k * 4 B in, (k-1)/k * {4, 4, 2} B out — half of a
// ring all-reduce's, and the residual / norm passes over HBM disappear.
//
// Synchronisation (one flag block of 64 u64 per member, in its work arena; epochs count the TP
// reductions of the current plan, identical on every member because they run the same schedule):
//   ready[j]  = epoch: member j's partial for this epoch is complete (written by CTA 0 of j's
//               kernel; the partial came from an earlier kernel on j's stream)
//   ticket    local CTA counter (each CTA fences its stores system-wide, then takes a ticket; the
//             last CTA resets it to 0 for the next call)
//   done[j]   = epoch: every CTA of member j finished pushing its rows (written by j's last CTA);
//             this member's last CTA waits for done[j] == epoch for all j, so the kernel completes
//             only when every row of this member's output has landed.
// Partials are double-buffered by epoch parity: member j overwrites P_j[e & 1] in epoch e + 2, after
// it has seen ready(e + 1) from every member, i.e. after every member finished reading epoch e.
// A member's output buffers (activations, or the fp32 sum) are written by peers in epoch e only
// after this member's ready(e), i.e. after all its earlier stream work (readers of the previous
// contents) completed.  A wait that exceeds the communication timeout, or sees the process-wide
// abort word (malleus_wait's failure path), gives up: it sets the status word and the
// kernel returns without completing the reduction (kernels.h CommGuard).
#include <cuda_bf16.h>
#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include "kernels.h"

namespace mls {
namespace {

constexpr int TPR_THREADS = 256;
constexpr int TPR_MAXV = 4;  // 4 vectors of 8 elements per thread: h <= 8192

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
// spin until *p >= target; false if the guard's abort word is set or the timeout passed (the status
// word records it).  The host words are read over PCIe only every 256 polls.
__device__ __forceinline__ bool wait_geq(const unsigned long long* p, unsigned long long target, const CommGuard& g) {
  if (ld_acquire_sys(p) >= target) return true;
  const unsigned long long t0 = now_ns();
  unsigned it = 0;
  while (ld_acquire_sys(p) < target) {
    __nanosleep(64);
    if ((++it & 255u) == 0u) {
      const bool ab = g.abort && *g.abort != 0u;
      if (ab || now_ns() - t0 > g.timeout_ns) {
        if (g.status) atomicOr(g.status, 1u);
        return false;
      }
    }
  }
  return true;
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

// K > 0: member count known at compile time, V = vectors of 8 per thread (h <= 8 * V * TPR_THREADS):
// the loads of up to KC members are issued before their adds.  K == 0: generic runtime k.
// MINB 4 (registers capped at 64 per thread): the co-resident variant that runs beside the weight-
// gradient GEMM (one CTA per SM fits next to the GEMM's 192 x 256 registers); MINB 2 otherwise
template <int MODE, int K, int V, bool PB, int MINB = 2>
__global__ void __launch_bounds__(TPR_THREADS, MINB) tp_reduce_kernel(const __grid_constant__ TpArgs a) {
  constexpr int KC = V >= 4 ? 2 : 3;
  __shared__ float sh[TPR_THREADS / 32];
  __shared__ bool last, gave_up;
  const int k = K > 0 ? K : a.k;
  const int me = a.me, h = a.h, nv = h / 8;
  // optional per-call stamps (debugging aid): [start of CTA 0, CTA 0 saw every ready, last CTA's
  // rows done, last CTA saw every done] at slot epoch % TP_TRACE_CALLS
  unsigned long long* tr = a.trace ? a.trace + 4 * (a.epoch % TP_TRACE_CALLS) : nullptr;
  if (tr && threadIdx.x == 0 && blockIdx.x == 0) tr[0] = now_ns();
  if (threadIdx.x == 0) {
    gave_up = false;
    // ready: only CTA 0 publishes (dispatched first, so it is resident whenever any CTA waits)
    if (blockIdx.x == 0) {
      __threadfence_system();
      for (int j = 0; j < k; ++j) st_release_sys(a.flags[j] + TPF_READY + me, a.epoch);
    }
    for (int j = 0; j < k && !gave_up; ++j) gave_up = !wait_geq(a.flags[me] + TPF_READY + j, a.epoch, a.guard);
    if (tr && blockIdx.x == 0) tr[1] = now_ns();
  }
  __syncthreads();
  if (gave_up) return;  // a member never arrived (failure path): the status word says so
  const int r0 = a.uneven ? a.row0[me] : (int)((long long)me * a.T / k);
  const int r1 = a.uneven ? a.row0[me + 1] : (int)((long long)(me + 1) * a.T / k);
  for (int row = r0 + blockIdx.x; row < r1; row += gridDim.x) {
    const long long rb = (long long)row * h;
    float4 acc[V][2];
    float4 t[KC][V][2];
    auto load = [&](float4 (&dst)[V][2], const void* base) {
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const int c = threadIdx.x + i * TPR_THREADS;
        if (c < nv) {
          if (PB) {
            float f[8];
            unpack8(__ldcg(reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(base) + rb) + c), f);
            dst[i][0] = make_float4(f[0], f[1], f[2], f[3]);
            dst[i][1] = make_float4(f[4], f[5], f[6], f[7]);
          } else {
            const float* b = static_cast<const float*>(base);
            dst[i][0] = ldcg4(b + rb + 8 * c);
            dst[i][1] = ldcg4(b + rb + 8 * c + 4);
          }
        }
      }
    };
    auto add = [&](const float4 (&src)[V][2]) {
#pragma unroll
      for (int i = 0; i < V; ++i)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          acc[i][q].x += src[i][q].x; acc[i][q].y += src[i][q].y;
          acc[i][q].z += src[i][q].z; acc[i][q].w += src[i][q].w;
        }
    };
    load(acc, a.part[0]);
    if (K > 0) {
#pragma unroll
      for (int j0 = 1; j0 < (K > 0 ? K : 1); j0 += KC) {  // members j0 .. j0+KC-1: loads, then adds in order
#pragma unroll
        for (int u = 0; u < KC; ++u)
          if (j0 + u < K) load(t[u], a.part[j0 + u]);
#pragma unroll
        for (int u = 0; u < KC; ++u)
          if (j0 + u < K) add(t[u]);
      }
    } else {
      for (int j = 1; j < k; ++j) {
        load(t[0], a.part[j]);
        add(t[0]);
      }
    }
    if (MODE == TP_SUM) {
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const int c = threadIdx.x + i * TPR_THREADS;
        if (c < nv) {
          if (a.sum_bf16) {  // bf16 sum (the activation-gradient dtype): half the push bytes
            const float f[8] = {acc[i][0].x, acc[i][0].y, acc[i][0].z, acc[i][0].w,
                                acc[i][1].x, acc[i][1].y, acc[i][1].z, acc[i][1].w};
            const uint4 q = pack8(f);
            for (int j = 0; j < k; ++j) __stcg(static_cast<uint4*>(a.d0[j]) + (long long)row * nv + c, q);
          } else {
            for (int j = 0; j < k; ++j) {
              float4* d = reinterpret_cast<float4*>(static_cast<float*>(a.d0[j]) + rb + 8 * c);
              __stcg(d, acc[i][0]);
              __stcg(d + 1, acc[i][1]);
            }
          }
        }
      }
    } else {
      float v[V][8];
      float ss = 0.f;
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const int c = threadIdx.x + i * TPR_THREADS;
        if (c < nv) {
          float xv[8];
          unpack8(reinterpret_cast<const uint4*>(a.x)[(long long)row * nv + c], xv);
          const float sv[8] = {acc[i][0].x, acc[i][0].y, acc[i][0].z, acc[i][0].w,
                               acc[i][1].x, acc[i][1].y, acc[i][1].z, acc[i][1].w};
#pragma unroll
          for (int t = 0; t < 8; ++t) v[i][t] = xv[t] + sv[t];
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
        for (int i = 0; i < V; ++i) {
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
  // completion: each CTA makes its stores visible system-wide and takes a local ticket; the last
  // CTA of this member tells every member "done" and waits for every member's "done"
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const unsigned long long t = atomicAdd(a.flags[me] + TPF_TICKET, 1ull);
    last = t + 1 == (unsigned long long)gridDim.x;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    // every CTA of this call has taken its ticket: reset the counter for the next call (ordered
    // before it by the stream), so a call that was rejected or replayed cannot desynchronise it
    a.flags[me][TPF_TICKET] = 0ull;
    if (tr) tr[2] = now_ns();
    __threadfence_system();
    for (int j = 0; j < k; ++j) st_release_sys(a.flags[j] + TPF_DONE + me, a.epoch);
    for (int j = 0; j < k; ++j)
      if (!wait_geq(a.flags[me] + TPF_DONE + j, a.epoch, a.guard)) break;
    __threadfence_system();
    if (tr) tr[3] = now_ns();
  }
}

}  // namespace

static unsigned* g_guard_host = nullptr;  // [abort, status], mapped pinned host memory

unsigned long long* tp_trace_buffer(int member) {
  static unsigned long long* buf = nullptr;
  if (!buf && cudaMallocManaged(&buf, (size_t)MAX_TP * TP_TRACE_CALLS * 4 * sizeof(unsigned long long)) != cudaSuccess) {
    cudaGetLastError();
    buf = nullptr;
  }
  return buf ? buf + (size_t)member * TP_TRACE_CALLS * 4 : nullptr;
}

int tp_grid(int rows) {
  const int waves = (rows + TP_GRID_MAX - 1) / TP_GRID_MAX;
  return std::max(1, waves > 0 ? (rows + waves - 1) / waves : 1);
}

void tp_rows(const TpArgs& a, int me, int* r0, int* r1) {
  *r0 = a.uneven ? a.row0[me] : (int)((long long)me * a.T / a.k);
  *r1 = a.uneven ? a.row0[me + 1] : (int)((long long)(me + 1) * a.T / a.k);
}

CommGuard comm_guard() {
  static CommGuard g{nullptr, nullptr, 0};
  static bool init = false;
  if (!init) {
    init = true;
    const char* e = getenv("MALLEUS_COMM_TIMEOUT_MS");
    g.timeout_ns = (unsigned long long)(e ? atof(e) : 20000.0) * 1000000ull;
    unsigned* h = nullptr;
    if (cudaHostAlloc((void**)&h, 2 * sizeof(unsigned), cudaHostAllocMapped | cudaHostAllocPortable) == cudaSuccess) {
      h[0] = h[1] = 0u;
      unsigned* d = nullptr;
      if (cudaHostGetDevicePointer((void**)&d, h, 0) == cudaSuccess) {
        g.abort = d;
        g.status = d + 1;
        g_guard_host = h;
      }
    }
    cudaGetLastError();
  }
  return g;
}
void comm_abort(unsigned v) {
  comm_guard();
  if (g_guard_host) reinterpret_cast<volatile unsigned*>(g_guard_host)[0] = v;
}
unsigned comm_status(bool clear) {
  comm_guard();
  if (!g_guard_host) return 0u;
  volatile unsigned* h = g_guard_host;
  const unsigned s = h[1];
  if (clear) h[1] = 0u;
  return s;
}

cudaError_t tp_reduce(const TpArgs& a0, cudaStream_t st) {
  TpArgs a = a0;
  a.guard = comm_guard();
  if (a.k < 2 || a.k > MAX_TP || a.me < 0 || a.me >= a.k || a.h % 8 || a.h > 8 * TPR_MAXV * TPR_THREADS ||
      a.T <= 0 || a.epoch == 0)
    return cudaErrorInvalidValue;
  if (a.uneven) {
    if (a.row0[0] != 0 || a.row0[a.k] != a.T) return cudaErrorInvalidValue;
    for (int j = 0; j < a.k; ++j)
      if (a.row0[j + 1] < a.row0[j]) return cudaErrorInvalidValue;
  }
  const int vpt = (a.h / 8 + TPR_THREADS - 1) / TPR_THREADS;
  int r0, r1;
  tp_rows(a, a.me, &r0, &r1);
  static int n_sms = 0;
  if (!n_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  // co-resident (beside the overlapped weight-gradient GEMM): at most one CTA per SM, 64 registers, so
  // the reduction never keeps the GEMM's CTAs off an SM while it waits for a slower peer (a waiting
  // 592-CTA reduction used to hold every SM's registers and serialise the GEMM behind the wait)
  const bool co = a.co_resident != 0 && a.mode == TP_SUM;
  const int grid = co ? std::min(tp_grid(r1 - r0), n_sms) : tp_grid(r1 - r0);
  if (co) {
    auto launch_co = [&](auto k_c) {
      constexpr int K = decltype(k_c)::value;
      if (a.part_bf16) {
        if (vpt <= 2) tp_reduce_kernel<TP_SUM, K, 2, true, 4><<<grid, TPR_THREADS, 0, st>>>(a);
        else tp_reduce_kernel<TP_SUM, K, TPR_MAXV, true, 4><<<grid, TPR_THREADS, 0, st>>>(a);
      } else {
        if (vpt <= 2) tp_reduce_kernel<TP_SUM, K, 2, false, 4><<<grid, TPR_THREADS, 0, st>>>(a);
        else tp_reduce_kernel<TP_SUM, K, TPR_MAXV, false, 4><<<grid, TPR_THREADS, 0, st>>>(a);
      }
    };
    switch (a.k) {
      case 2: launch_co(std::integral_constant<int, 2>{}); break;
      case 4: launch_co(std::integral_constant<int, 4>{}); break;
      default: launch_co(std::integral_constant<int, 0>{}); break;
    }
    count_launch();
    return cudaGetLastError();
  }
  auto launch_kv = [&](auto mode_c, auto k_c) {
    constexpr int M = decltype(mode_c)::value, K = decltype(k_c)::value;
    if (a.part_bf16) {
      if (vpt <= 2) tp_reduce_kernel<M, K, 2, true><<<grid, TPR_THREADS, 0, st>>>(a);
      else tp_reduce_kernel<M, K, TPR_MAXV, true><<<grid, TPR_THREADS, 0, st>>>(a);
    } else {
      if (vpt <= 2) tp_reduce_kernel<M, K, 2, false><<<grid, TPR_THREADS, 0, st>>>(a);
      else tp_reduce_kernel<M, K, TPR_MAXV, false><<<grid, TPR_THREADS, 0, st>>>(a);
    }
  };
  auto launch = [&](auto mode_c) {
    switch (a.k) {
      case 2: launch_kv(mode_c, std::integral_constant<int, 2>{}); break;
      case 3: launch_kv(mode_c, std::integral_constant<int, 3>{}); break;
      case 4: launch_kv(mode_c, std::integral_constant<int, 4>{}); break;
      case 8: launch_kv(mode_c, std::integral_constant<int, 8>{}); break;
      default: launch_kv(mode_c, std::integral_constant<int, 0>{}); break;
    }
  };
  switch (a.mode) {
    case TP_SUM: launch(std::integral_constant<int, TP_SUM>{}); break;
    case TP_RESID_NORM: launch(std::integral_constant<int, TP_RESID_NORM>{}); break;
    case TP_RESID: launch(std::integral_constant<int, TP_RESID>{}); break;
    default: return cudaErrorInvalidValue;
  }
  count_launch();
  return cudaGetLastError();
}

}  // namespace mls
