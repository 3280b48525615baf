// HBM-bound kernels of the hot path: RMSNorm fwd/bwd
// with fused residual add (the K15 epilogue once the TP partial sum is reduced), RoPE, SwiGLU,
// embedding gather / scatter-add, vocab-parallel cross-entropy.  128-bit loads/stores, fp32
// math, warp-shuffle reductions, deterministic column reductions (fixed order, no atomics) for
// the norm-gain gradients.  bf16 rounding points follow reading R6.
#include <cuda_bf16.h>
#include <algorithm>
#include <cstdlib>
#include "kernels.h"

namespace mls {

namespace {

constexpr int NORM_THREADS = 128;
constexpr int NORM_MAXV = 8;  // vectors of 8 bf16 per thread -> h <= 8 * 8 * 128 = 8192

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
template <int NT>
__device__ __forceinline__ float block_sum(float v, float* sh) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  float r = 0.f;
#pragma unroll
  for (int i = 0; i < NT / 32; ++i) r += sh[i];
  return r;
}
template <int NT>
__device__ __forceinline__ float block_max(float v, float* sh) {
  v = warp_max(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  float r = -INFINITY;
#pragma unroll
  for (int i = 0; i < NT / 32; ++i) r = fmaxf(r, sh[i]);
  return r;
}

__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
  const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = __bfloat1622float2(b[i]);
    f[2 * i] = t.x; f[2 * i + 1] = t.y;
  }
}
__device__ __forceinline__ uint32_t pack2_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint4 u;
  __nv_bfloat162* b = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return u;
}

// ---------------------------------------------------------------- RMSNorm forward
// y = x_new * r * g, r = rsqrt(mean(x_new^2) + eps), x_new = bf16(x + partial) if partial.
__global__ void __launch_bounds__(NORM_THREADS)
rmsnorm_fwd_kernel(int h, const uint4* __restrict__ x, const float4* __restrict__ partial,
                   uint4* __restrict__ x_out, const uint4* __restrict__ g, float eps,
                   uint4* __restrict__ y, float* __restrict__ rstd) {
  __shared__ float sh[NORM_THREADS / 32];
  const int row = blockIdx.x;
  const int nv = h / 8;
  const uint4* xr = x + (long long)row * nv;
  float v[NORM_MAXV][8];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < NORM_MAXV; ++i) {
    const int c = threadIdx.x + i * NORM_THREADS;
    if (c < nv) {
      unpack8(xr[c], v[i]);
      if (partial) {
        const float4* pr = partial + ((long long)row * nv + c) * 2;
        float4 p0 = pr[0], p1 = pr[1];
        v[i][0] += p0.x; v[i][1] += p0.y; v[i][2] += p0.z; v[i][3] += p0.w;
        v[i][4] += p1.x; v[i][5] += p1.y; v[i][6] += p1.z; v[i][7] += p1.w;
        uint4 q = pack8(v[i]);          // residual stream is bf16 (reading R6)
        x_out[(long long)row * nv + c] = q;
        unpack8(q, v[i]);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) ss += v[i][j] * v[i][j];
    }
  }
  ss = block_sum<NORM_THREADS>(ss, sh);
  const float r = rsqrtf(ss / (float)h + eps);
  if (threadIdx.x == 0) rstd[row] = r;
#pragma unroll
  for (int i = 0; i < NORM_MAXV; ++i) {
    const int c = threadIdx.x + i * NORM_THREADS;
    if (c < nv) {
      float gg[8];
      unpack8(g[c], gg);
      float o[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = v[i][j] * r * gg[j];
      y[(long long)row * nv + c] = pack8(o);
    }
  }
}

// Warp-per-row variant (no fused partial, h % 256 == 0): lane l holds columns 8 l + 256 i of its
// row (NV = h / 256 vectors), the sum of squares is a warp shuffle — no block barrier per row, 8 rows
// per CTA in flight.  Same arithmetic and rounding as rmsnorm_fwd_kernel.
template <int NV>
__global__ void __launch_bounds__(256) rmsnorm_fwd_warp_kernel(int T, int h, const uint4* __restrict__ x,
                                                               const uint4* __restrict__ g, float eps,
                                                               uint4* __restrict__ y, float* __restrict__ rstd) {
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= T) return;
  const int nv = h / 8;
  uint4 xq[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) xq[i] = x[(long long)row * nv + lane + 32 * i];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    float v[8];
    unpack8(xq[i], v);
#pragma unroll
    for (int j = 0; j < 8; ++j) ss += v[j] * v[j];
  }
  ss = warp_sum(ss);
  const float r = rsqrtf(ss / (float)h + eps);
  if (lane == 0) rstd[row] = r;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    float v[8], gg[8], o[8];
    unpack8(xq[i], v);
    unpack8(__ldg(g + lane + 32 * i), gg);
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = v[j] * r * gg[j];
    y[(long long)row * nv + lane + 32 * i] = pack8(o);
  }
}

// ---------------------------------------------------------------- RMSNorm backward
// dx = r*u - x*r^3*mean(x*u), u = g*dy; dx_out = bf16(dres + dx); dg partial per block.
// Two passes over each row (the second re-reads x / dy / g from L1) so that only the dg
// accumulators stay resident in registers.
__device__ __forceinline__ void load_f8(const float4* p, float (&f)[8]) {
  float4 a = p[0], b = p[1];
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}

template <int V, bool DY16>  // vectors of 8 columns per thread: h <= 8 * V * NORM_THREADS; dy bf16?
__global__ void __launch_bounds__(NORM_THREADS)
rmsnorm_bwd_kernel(int T, int h, int rows_per_block, const uint4* __restrict__ x,
                   const uint4* __restrict__ g, const float* __restrict__ rstd,
                   const void* __restrict__ dyv, const uint4* __restrict__ dres,
                   uint4* __restrict__ dx_out, float* __restrict__ dg_part) {
  const float4* dy = static_cast<const float4*>(dyv);
  const uint4* dy16 = static_cast<const uint4*>(dyv);
  __shared__ float sh[NORM_THREADS / 32];
  const int nv = h / 8;
  float dg[V][8];
#pragma unroll
  for (int i = 0; i < V; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) dg[i][j] = 0.f;
  const int r0 = blockIdx.x * rows_per_block;
  const int r1 = min(T, r0 + rows_per_block);
  for (int row = r0; row < r1; ++row) {
    const float r = rstd[row];
    float dot = 0.f;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int c = threadIdx.x + i * NORM_THREADS;
      if (c < nv) {
        float xv[8], dv[8], gg[8];
        unpack8(x[(long long)row * nv + c], xv);
        if (DY16) unpack8(dy16[(long long)row * nv + c], dv);
        else load_f8(dy + ((long long)row * nv + c) * 2, dv);
        unpack8(g[c], gg);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          dot += xv[j] * gg[j] * dv[j];
          dg[i][j] += dv[j] * xv[j] * r;
        }
      }
    }
    dot = block_sum<NORM_THREADS>(dot, sh);
    const float coef = r * r * r * dot / (float)h;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int c = threadIdx.x + i * NORM_THREADS;
      if (c < nv) {
        float xv[8], dv[8], gg[8], o[8], rs[8];
        unpack8(x[(long long)row * nv + c], xv);
        if (DY16) unpack8(dy16[(long long)row * nv + c], dv);
        else load_f8(dy + ((long long)row * nv + c) * 2, dv);
        unpack8(g[c], gg);
        if (dres) unpack8(dres[(long long)row * nv + c], rs);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          o[j] = r * gg[j] * dv[j] - xv[j] * coef;
          if (dres) o[j] += rs[j];
        }
        dx_out[(long long)row * nv + c] = pack8(o);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int c = threadIdx.x + i * NORM_THREADS;
    if (c < nv) {
      float4* out = reinterpret_cast<float4*>(dg_part + (long long)blockIdx.x * h + c * 8);
      out[0] = make_float4(dg[i][0], dg[i][1], dg[i][2], dg[i][3]);
      out[1] = make_float4(dg[i][4], dg[i][5], dg[i][6], dg[i][7]);
    }
  }
}

// dg[c] += sum_b part[b][c] in a fixed order (deterministic): block = 32 columns x 32 warps, warp w
// sums rows w, w+32, ... (lane = column, coalesced), then the 32 warp sums are added in warp order.
__global__ void __launch_bounds__(1024) colsum_accum_kernel(int nb, int h, const float* __restrict__ part,
                                                            float* __restrict__ dg) {
  __shared__ float sh[32][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  float s = 0.f;
  if (c < h)
    for (int b = w; b < nb; b += 32) s += part[(long long)b * h + c];
  sh[w][lane] = s;
  __syncthreads();
  if (w == 0 && c < h) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 32; ++i) t += sh[i][lane];
    dg[c] += t;
  }
}

// Warp-per-row variant for bf16 dy and h % 256 == 0 (every hot-path shape): lane l holds columns
// 8 l + 256 i of its row in registers (NV = h / 256 vectors of x and dy), so the row statistic is a
// warp shuffle (no block barrier per row) and many rows are in flight per SM.  The gain gradient
// sum_rows dy * x * r accumulates per warp in its own shared-memory slice (no atomics), the CTA adds
// its slices in warp order into part[blockIdx.x][h], and colsum_accum_kernel adds the CTA partials in
// CTA order: deterministic, and the partial array is grid x h (one CTA per SM) instead of a row band
// per 3 rows.
constexpr int BWDW_SMEM = 128 * 1024;
template <int NV>
__global__ void __launch_bounds__(256, 1)
rmsnorm_bwd_warp_kernel(int T, int h, const uint4* __restrict__ x, const uint4* __restrict__ g,
                        const float* __restrict__ rstd, const uint4* __restrict__ dy, const uint4* __restrict__ dres,
                        uint4* __restrict__ dx_out, float* __restrict__ dg_part) {
  extern __shared__ float4 sdg4[];  // [warps][h] fp32
  float* sdg = reinterpret_cast<float*>(sdg4);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nv = h / 8;
  float* my = sdg + (size_t)w * h;
  for (int c = lane; c < h / 4; c += 32) reinterpret_cast<float4*>(my)[c] = make_float4(0.f, 0.f, 0.f, 0.f);
  __syncwarp();
  for (int row = blockIdx.x * nw + w; row < T; row += gridDim.x * nw) {
    const float r = rstd[row];
    uint4 xq[NV], dq[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      xq[i] = x[(long long)row * nv + lane + 32 * i];
      dq[i] = dy[(long long)row * nv + lane + 32 * i];
    }
    float dot = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      float xv[8], dv[8];
      unpack8(xq[i], xv);
      unpack8(dq[i], dv);
      float4* d4 = reinterpret_cast<float4*>(my + (lane + 32 * i) * 8);
      float gv[8];
      unpack8(__ldg(g + lane + 32 * i), gv);
      float4 a = d4[0], b = d4[1];
      a.x += dv[0] * xv[0] * r; a.y += dv[1] * xv[1] * r; a.z += dv[2] * xv[2] * r; a.w += dv[3] * xv[3] * r;
      b.x += dv[4] * xv[4] * r; b.y += dv[5] * xv[5] * r; b.z += dv[6] * xv[6] * r; b.w += dv[7] * xv[7] * r;
      d4[0] = a;
      d4[1] = b;
#pragma unroll
      for (int j = 0; j < 8; ++j) dot += xv[j] * gv[j] * dv[j];
    }
    dot = warp_sum(dot);
    const float coef = r * r * r * dot / (float)h;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      float xv[8], dv[8], o[8], rs[8], gv[8];
      unpack8(xq[i], xv);
      unpack8(dq[i], dv);
      unpack8(__ldg(g + lane + 32 * i), gv);
      if (dres) unpack8(dres[(long long)row * nv + lane + 32 * i], rs);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        o[j] = r * gv[j] * dv[j] - xv[j] * coef;
        if (dres) o[j] += rs[j];
      }
      dx_out[(long long)row * nv + lane + 32 * i] = pack8(o);
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < h / 4; c += blockDim.x) {  // CTA partial: warp slices in warp order
    float4 acc = reinterpret_cast<const float4*>(sdg)[c];
    for (int k = 1; k < nw; ++k) {
      const float4 v = reinterpret_cast<const float4*>(sdg + (size_t)k * h)[c];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    reinterpret_cast<float4*>(dg_part + (long long)blockIdx.x * h)[c] = acc;
  }
}

// Row-group variant (h / 8 a multiple of 32, h / 8 <= 1024): TPR = h / 8 threads own one row, one
// 8-column vector each, RB = 1024 / TPR rows per 1024-thread CTA, two CTAs per SM.  Every load of a
// row (x, dy, dres) is issued one row ahead, before the row statistic's barrier of the current row,
// so the latency chain per row is one barrier, not two dependent global round trips.  The gain
// gradient stays in 8 registers per thread over all rows of the CTA; at the end the RB row groups'
// partials are added in group order into part[blockIdx.x][h] (grid = 148 x resident CTAs per SM, so
// the partial array and colsum_accum_kernel's pass are >= 3x smaller than the block kernel's).
// Deterministic (the row -> CTA assignment depends only on T and the grid).
constexpr int BWDR_THREADS = 1024;
template <bool DY16>
__global__ void __launch_bounds__(BWDR_THREADS, 1)
rmsnorm_bwd_rows_kernel(int T, int h, const uint4* __restrict__ x, const uint4* __restrict__ g,
                        const float* __restrict__ rstd, const void* __restrict__ dyv, const uint4* __restrict__ dres,
                        uint4* __restrict__ dx_out, float* __restrict__ dg_part) {
  __shared__ float sdot[2][32];
  __shared__ __align__(16) float sdg[BWDR_THREADS * 8];
  const int nv = h / 8, rb = blockDim.x / nv;  // threads per row, rows per CTA (blockDim = rb * nv)
  const int c = threadIdx.x % nv, grp = threadIdx.x / nv;
  const int w = threadIdx.x >> 5, wpr = nv >> 5;  // warps per row
  const int stride = gridDim.x * rb;
  const uint4* dyq = static_cast<const uint4*>(dyv);  // bf16: 1 vector of 8; fp32: 2 vectors of 4
  constexpr int DQ = DY16 ? 1 : 2;
  float dg[8];  // g is re-read per row (L1-resident): registers go to the rows in flight
#pragma unroll
  for (int j = 0; j < 8; ++j) dg[j] = 0.f;
  int row = blockIdx.x * rb + grp;
  const uint4* xc = x + c;
  const uint4* dyc = dyq + (size_t)c * DQ;
  const uint4* rc = dres ? dres + c : nullptr;
  // the current row's operands, packed as loaded, and the next row's (loaded one row ahead, so their
  // latency overlaps this row's barrier)
  uint4 cx = make_uint4(0, 0, 0, 0), cres = cx, cdy[DQ];
  float cr = 0.f;
#pragma unroll
  for (int k = 0; k < DQ; ++k) cdy[k] = cx;
  if (row < T) {
    const size_t o = (size_t)row * nv;
    cx = xc[o];
#pragma unroll
    for (int k = 0; k < DQ; ++k) cdy[k] = dyc[o * DQ + k];
    if (rc) cres = rc[o];
    cr = rstd[row];
  }
#pragma unroll 1
  for (int it = 0, base = blockIdx.x * rb; base < T; base += stride, row += stride, ++it) {
    const int nrow = row + stride;
    uint4 nx = cx, nres = cres, ndy[DQ];
    float nr = cr;
#pragma unroll
    for (int k = 0; k < DQ; ++k) ndy[k] = cdy[k];
    if (nrow < T) {
      const size_t o = (size_t)nrow * nv;
      nx = xc[o];
#pragma unroll
      for (int k = 0; k < DQ; ++k) ndy[k] = dyc[o * DQ + k];
      if (rc) nres = rc[o];
      nr = rstd[nrow];
    }
    // unpacked twice (before and after the barrier) so only the packed operands live across it
    auto unpack_row = [&](float (&xv)[8], float (&dv)[8], float (&gv)[8]) {
      unpack8(cx, xv);
      unpack8(__ldg(g + c), gv);
      if (DY16) {
        unpack8(cdy[0], dv);
      } else {
#pragma unroll
        for (int k = 0; k < DQ; ++k) {
          dv[4 * k] = __uint_as_float(cdy[k].x); dv[4 * k + 1] = __uint_as_float(cdy[k].y);
          dv[4 * k + 2] = __uint_as_float(cdy[k].z); dv[4 * k + 3] = __uint_as_float(cdy[k].w);
        }
      }
    };
    float dot = 0.f;
    if (row < T) {
      float xv[8], dv[8], gv[8];
      unpack_row(xv, dv, gv);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        dot += xv[j] * gv[j] * dv[j];
        dg[j] += dv[j] * xv[j] * cr;
      }
    }
    dot = warp_sum(dot);
    if ((threadIdx.x & 31) == 0) sdot[it & 1][w] = dot;
    __syncthreads();
    float tot = 0.f;
    for (int k = 0; k < wpr; ++k) tot += sdot[it & 1][grp * wpr + k];  // the row's warps in order
    if (row < T) {
      float xv[8], dv[8], gv[8];
      unpack_row(xv, dv, gv);
      const float coef = cr * cr * cr * tot / (float)h;
      float o[8], rs[8];
      if (dres) unpack8(cres, rs);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        o[j] = cr * gv[j] * dv[j] - xv[j] * coef;
        if (dres) o[j] += rs[j];
      }
      dx_out[(size_t)row * nv + c] = pack8(o);
    }
    cx = nx;
    cres = nres;
    cr = nr;
#pragma unroll
    for (int k = 0; k < DQ; ++k) cdy[k] = ndy[k];
  }
  float4* s4 = reinterpret_cast<float4*>(sdg + (size_t)threadIdx.x * 8);
  s4[0] = make_float4(dg[0], dg[1], dg[2], dg[3]);
  s4[1] = make_float4(dg[4], dg[5], dg[6], dg[7]);
  __syncthreads();
  for (int q = threadIdx.x; q < h / 4; q += blockDim.x) {  // column quad q: groups in order
    float4 acc = reinterpret_cast<const float4*>(sdg)[q];
    for (int k = 1; k < rb; ++k) {
      const float4 v = reinterpret_cast<const float4*>(sdg + (size_t)k * h)[q];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    reinterpret_cast<float4*>(dg_part + (long long)blockIdx.x * h)[q] = acc;
  }
}

constexpr int BWD_BLOCKS = 148 * 6;  // 6 per SM (80 registers at h = 4096): rows in flight to cover the per-row latency chain

// ---------------------------------------------------------------- residual add
__global__ void residual_add_kernel(long long nv, const uint4* __restrict__ x, const float4* __restrict__ p,
                                    uint4* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nv; i += (long long)gridDim.x * blockDim.x) {
    float v[8];
    unpack8(x[i], v);
    float4 a = p[2 * i], b = p[2 * i + 1];
    v[0] += a.x; v[1] += a.y; v[2] += a.z; v[3] += a.w; v[4] += b.x; v[5] += b.y; v[6] += b.z; v[7] += b.w;
    out[i] = pack8(v);
  }
}

// ---------------------------------------------------------------- RoPE (half-split, reading R3)
// buf row t: columns [col0 + j*d, col0 + (j+1)*d) is head j; pairs (i, i + d/2); pos = t % s.
// Applied to q (col0 = 0) and k (col0 = n*d) by blockIdx.y.
// One thread per (token, group of 8 consecutive pair indices i): the 8 angles are computed once and
// reused for every head of q and k (2n heads); 128-bit loads of both halves of each head.
__global__ void rope_kernel(int T, int s, int n, int d, __nv_bfloat16* __restrict__ buf, long long ld,
                            int col0, float log2_theta, float sign) {
  const int half = d / 2;
  const int groups = half / 8;
  const long long total = (long long)T * groups;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int gi = idx % groups;
    const long long t = idx / groups;
    const int pos = (int)(t % s);
    float cs[8], sn[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = gi * 8 + u;
      const float inv = exp2f(-(2.f * i / (float)d) * log2_theta);
      sincosf((float)pos * inv, &sn[u], &cs[u]);
      sn[u] *= sign;
    }
    __nv_bfloat16* row = buf + t * ld + col0;
    for (int j = 0; j < n; ++j) {  // the n rotated heads: q heads then k heads (GQA: fewer k heads)
      uint4* p1 = reinterpret_cast<uint4*>(row + j * d + gi * 8);
      uint4* p2 = reinterpret_cast<uint4*>(row + j * d + half + gi * 8);
      float a[8], b[8], o1[8], o2[8];
      unpack8(*p1, a);
      unpack8(*p2, b);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        o1[u] = a[u] * cs[u] - b[u] * sn[u];
        o2[u] = b[u] * cs[u] + a[u] * sn[u];
      }
      *p1 = pack8(o1);
      *p2 = pack8(o2);
    }
  }
}

// ---------------------------------------------------------------- SwiGLU
__device__ __forceinline__ float sigm(float x) { return 1.f / (1.f + __expf(-x)); }

__global__ void swiglu_fwd_kernel(int T, int F, const __nv_bfloat16* __restrict__ gu, __nv_bfloat16* __restrict__ u) {
  const int fv = F / 8;
  const long long total = (long long)T * fv;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long t = idx / fv;
    const int c = idx % fv;
    float G[8], U[8], o[8];
    unpack8(reinterpret_cast<const uint4*>(gu + t * 2 * F)[c], G);
    unpack8(reinterpret_cast<const uint4*>(gu + t * 2 * F + F)[c], U);
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = G[j] * sigm(G[j]) * U[j];
    reinterpret_cast<uint4*>(u + t * F)[c] = pack8(o);
  }
}

__global__ void swiglu_bwd_kernel(int T, int F, const __nv_bfloat16* __restrict__ gu,
                                  const __nv_bfloat16* __restrict__ du, __nv_bfloat16* __restrict__ dgu) {
  const int fv = F / 8;
  const long long total = (long long)T * fv;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long t = idx / fv;
    const int c = idx % fv;
    float G[8], U[8], D[8], dG[8], dU[8];
    unpack8(reinterpret_cast<const uint4*>(gu + t * 2 * F)[c], G);
    unpack8(reinterpret_cast<const uint4*>(gu + t * 2 * F + F)[c], U);
    unpack8(reinterpret_cast<const uint4*>(du + t * F)[c], D);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float sg = sigm(G[j]);
      dU[j] = D[j] * G[j] * sg;
      dG[j] = D[j] * U[j] * sg * (1.f + G[j] * (1.f - sg));
    }
    reinterpret_cast<uint4*>(dgu + t * 2 * F)[c] = pack8(dG);
    reinterpret_cast<uint4*>(dgu + t * 2 * F + F)[c] = pack8(dU);
  }
}

// ---------------------------------------------------------------- embedding
__global__ void embed_fwd_kernel(int T, int h, const int32_t* __restrict__ tok, const uint4* __restrict__ E,
                                 uint4* __restrict__ x) {
  const int nv = h / 8;
  const int t = blockIdx.x;
  const long long src = (long long)tok[t] * nv;
  for (int c = threadIdx.x; c < nv; c += blockDim.x) x[(long long)t * nv + c] = E[src + c];
}

// dE[v] += sum over positions t with tok[t] == v of dx[t], deterministic: the CTA of the first
// position of each distinct token sums all of that token's rows in position order and updates the
// dE row once (no atomics, so repeated tokens give run-to-run identical sums).  The CTA first
// compacts the later positions holding the same token into a shared list in position order
// (warp ballots, chunks of 256 positions), so the gather loop only visits the duplicates (few
// under uniform tokens).  Tokens staged in shared memory (T <= EMBED_MAX_T), 8 columns per thread.
constexpr int EMBED_MAX_T = 8192;
constexpr int EMBED_THREADS = 256;
__global__ void __launch_bounds__(EMBED_THREADS) embed_bwd_kernel(int T, int h, const int32_t* __restrict__ tok,
                                                                  const uint4* __restrict__ dx, float* __restrict__ dE) {
  extern __shared__ int32_t stok[];           // [T] tokens, then [T] duplicate positions
  int32_t* dup = stok + T;
  __shared__ int first, n_dup;
  __shared__ int wcnt[EMBED_THREADS / 32];
  const int t = blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < T; i += EMBED_THREADS) stok[i] = tok[i];
  if (threadIdx.x == 0) { first = 1; n_dup = 0; }
  __syncthreads();
  const int v = stok[t];
  for (int i = threadIdx.x; i < t; i += EMBED_THREADS)
    if (stok[i] == v) first = 0;  // benign race: every writer stores 0
  __syncthreads();
  if (!first) return;
  for (int base = t + 1; base < T; base += EMBED_THREADS) {  // ordered compaction of positions > t
    const int u = base + threadIdx.x;
    const bool hit = u < T && stok[u] == v;
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) wcnt[w] = __popc(m);
    __syncthreads();
    if (hit) {
      int off = n_dup + __popc(m & ((1u << lane) - 1u));
      for (int j = 0; j < w; ++j) off += wcnt[j];
      dup[off] = u;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int s = 0;
      for (int j = 0; j < EMBED_THREADS / 32; ++j) s += wcnt[j];
      n_dup += s;
    }
    __syncthreads();
  }
  const int nd = n_dup;
  const int nv = h / 8;
  float* dst = dE + (long long)v * h;
  for (int c = threadIdx.x; c < nv; c += EMBED_THREADS) {
    float acc[8];
    unpack8(dx[(long long)t * nv + c], acc);
    for (int k = 0; k < nd; ++k) {
      float x8[8];
      unpack8(dx[(long long)dup[k] * nv + c], x8);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += x8[j];
    }
    float4* d4 = reinterpret_cast<float4*>(dst + c * 8);
    float4 o0 = d4[0], o1 = d4[1];
    o0.x += acc[0]; o0.y += acc[1]; o0.z += acc[2]; o0.w += acc[3];
    o1.x += acc[4]; o1.y += acc[5]; o1.z += acc[6]; o1.w += acc[7];
    d4[0] = o0;
    d4[1] = o1;
  }
}

// ---------------------------------------------------------------- vocab-parallel cross-entropy
constexpr int CE_THREADS = 256;

// stats[t] = {local max, sum exp(z - local max), target logit or 0}.  One pass: each thread keeps
// a running (max, sum) over float4 chunks (rescaled when the max grows), then the block merges the
// pairs; V % 4 == 0 (vocab splits are multiples of 16).
__device__ __forceinline__ void ms_merge(float& m, float& s, float m2, float s2) {
  const float mn = fmaxf(m, m2);
  s = (m == -INFINITY ? 0.f : s * __expf(m - mn)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mn));
  m = mn;
}
__global__ void __launch_bounds__(CE_THREADS)
ce_stats_kernel(int V, const float* __restrict__ z, const int32_t* __restrict__ tgt, int v0,
                float* __restrict__ stats) {
  __shared__ float shm[CE_THREADS / 32], shs[CE_THREADS / 32];
  const int t = blockIdx.x;
  const float* zr = z + (long long)t * V;
  const float4* z4 = reinterpret_cast<const float4*>(zr);
  float m = -INFINITY, s = 0.f;
  for (int c = threadIdx.x; c < V / 4; c += CE_THREADS) {
    const float4 v = z4[c];
    const float cm = fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w));
    if (cm > m) {
      s = (m == -INFINITY) ? 0.f : s * __expf(m - cm);
      m = cm;
    }
    s += __expf(v.x - m) + __expf(v.y - m) + __expf(v.z - m) + __expf(v.w - m);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
    ms_merge(m, s, m2, s2);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { shm[w] = m; shs[w] = s; }
  __syncthreads();
  if (threadIdx.x == 0) {
    float M = shm[0], S = shs[0];
    for (int i = 1; i < CE_THREADS / 32; ++i) ms_merge(M, S, shm[i], shs[i]);
    const int y = tgt[t] - v0;
    stats[3 * t] = M;
    stats[3 * t + 1] = S;
    stats[3 * t + 2] = (y >= 0 && y < V) ? zr[y] : 0.f;
  }
}

// dz = (softmax - onehot) * scale (bf16, or fp32 in the FP32 parity mode), float4 in per thread step
template <bool F32>
__global__ void ce_grad_kernel(int V, const float* __restrict__ z, const int32_t* __restrict__ tgt, int v0,
                               const float* __restrict__ gmax, const float* __restrict__ gsum,
                               const float* __restrict__ gtgt, float scale, void* __restrict__ dzv,
                               float* __restrict__ loss_rows) {
  const int t = blockIdx.x;
  const float lse = gmax[t] + logf(gsum[t]);
  if (threadIdx.x == 0 && loss_rows) loss_rows[t] = lse - gtgt[t];
  const float4* z4 = reinterpret_cast<const float4*>(z + (long long)t * V);
  const int y = tgt[t] - v0;
  for (int c = threadIdx.x; c < V / 4; c += blockDim.x) {
    const float4 v = z4[c];
    float p[4];
    if (F32) {
      p[0] = expf(v.x - lse); p[1] = expf(v.y - lse); p[2] = expf(v.z - lse); p[3] = expf(v.w - lse);
    } else {
      p[0] = __expf(v.x - lse); p[1] = __expf(v.y - lse); p[2] = __expf(v.z - lse); p[3] = __expf(v.w - lse);
    }
    if ((y >> 2) == c) p[y & 3] -= 1.f;
    if (F32) {
      reinterpret_cast<float4*>(static_cast<float*>(dzv) + (long long)t * V)[c] =
          make_float4(p[0] * scale, p[1] * scale, p[2] * scale, p[3] * scale);
    } else {
      uint2 o;
      o.x = pack2_bf16(p[0] * scale, p[1] * scale);
      o.y = pack2_bf16(p[2] * scale, p[3] * scale);
      reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(dzv) + (long long)t * V)[c] = o;
    }
  }
}

// gmax[t] = stats max (before TP all-reduce MAX)
__global__ void ce_max_kernel(int T, const float* __restrict__ stats, float* __restrict__ gmax) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < T) gmax[t] = stats[3 * t];
}
// sum_tgt[2t] = local sumexp rescaled to the global max, sum_tgt[2t+1] = target logit
__global__ void ce_local_sum_kernel(int T, const float* __restrict__ stats, const float* __restrict__ gmax,
                                    float* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < T) {
    out[t] = stats[3 * t + 1] * __expf(stats[3 * t] - gmax[t]);
    out[T + t] = stats[3 * t + 2];
  }
}

__global__ void reduce_loss_kernel(int T, const float* __restrict__ rows, float scale, float* __restrict__ out,
                                   int accumulate) {
  __shared__ float sh[1024 / 32];
  float s = 0.f;
  for (int t = threadIdx.x; t < T; t += 1024) s += rows[t];
  s = block_sum<1024>(s, sh);
  if (threadIdx.x == 0) *out = accumulate ? *out + s * scale : s * scale;
}

__global__ void cast_kernel(long long n, const float* __restrict__ in, __nv_bfloat16* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = __float2bfloat16_rn(in[i]);
}
__global__ void fill_kernel(long long n, float* __restrict__ p, float v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = v;
}

struct CombinePtrs {
  float* p[MAX_TP];
};
__global__ void tp_combine_kernel(int k, int n, CombinePtrs b, int op) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    float v = b.p[0][i];
    for (int j = 1; j < k; ++j) v = op == 0 ? fmaxf(v, b.p[j][i]) : v + b.p[j][i];
    for (int j = 0; j < k; ++j) b.p[j][i] = v;
  }
}

inline int grid_for(long long n, int threads) {
  long long b = (n + threads - 1) / threads;
  return (int)(b < 148 * 16 ? (b < 1 ? 1 : b) : 148 * 16);
}

}  // namespace

cudaError_t rmsnorm_fwd(int T, int h, const void* x, const float* partial, void* x_out, const void* g,
                        float eps, void* y, float* rstd, cudaStream_t st) {
  if (h % 8 || h > 8 * NORM_MAXV * NORM_THREADS || T <= 0) return cudaErrorInvalidValue;
  if (partial && !x_out) return cudaErrorInvalidValue;
  if (!partial && h % 256 == 0) {  // warp per row
    using Fn = void (*)(int, int, const uint4*, const uint4*, float, uint4*, float*);
    Fn fn = nullptr;
    switch (h / 256) {
      case 1: fn = rmsnorm_fwd_warp_kernel<1>; break;
      case 2: fn = rmsnorm_fwd_warp_kernel<2>; break;
      case 4: fn = rmsnorm_fwd_warp_kernel<4>; break;
      case 8: fn = rmsnorm_fwd_warp_kernel<8>; break;
      case 12: fn = rmsnorm_fwd_warp_kernel<12>; break;
      case 16: fn = rmsnorm_fwd_warp_kernel<16>; break;
      default: break;
    }
    if (fn) {
      fn<<<(T + 7) / 8, 256, 0, st>>>(T, h, (const uint4*)x, (const uint4*)g, eps, (uint4*)y, rstd); count_launch();
      return cudaGetLastError();
    }
  }
  rmsnorm_fwd_kernel<<<T, NORM_THREADS, 0, st>>>(h, (const uint4*)x, (const float4*)partial, (uint4*)x_out,
                                                 (const uint4*)g, eps, (uint4*)y, rstd); count_launch();
  return cudaGetLastError();
}

size_t rmsnorm_bwd_scratch_floats(int T, int h) { return (size_t)BWD_BLOCKS * h; }

// warp-per-row kernel instance for h (NV = h / 256 vectors per lane), or nullptr
using BwdWarpFn = void (*)(int, int, const uint4*, const uint4*, const float*, const uint4*, const uint4*, uint4*,
                           float*);
static BwdWarpFn bwd_warp_fn(int h) {
  if (h % 256) return nullptr;
  switch (h / 256) {
    case 1: return rmsnorm_bwd_warp_kernel<1>;
    case 2: return rmsnorm_bwd_warp_kernel<2>;
    case 4: return rmsnorm_bwd_warp_kernel<4>;
    case 8: return rmsnorm_bwd_warp_kernel<8>;
    case 12: return rmsnorm_bwd_warp_kernel<12>;
    case 16: return rmsnorm_bwd_warp_kernel<16>;  // larger h: the block kernel (registers)
    default: return nullptr;
  }
}

cudaError_t rmsnorm_bwd(int T, int h, const void* x, const void* g, const float* rstd, const void* dy,
                        const void* dres, void* dx_out, float* dg_accum, float* scratch, cudaStream_t st,
                        bool dy_bf16) {
  if (h % 8 || h > 8 * NORM_MAXV * NORM_THREADS || T <= 0) return cudaErrorInvalidValue;
  // the warp-per-row kernel measured slower in the C2 step (31.8 + 4.7 us vs 24.9 + 7.1 us with the
  // block kernel on fp32 dy: one 128 KB-smem CTA per SM leaves too few rows in flight); opt-in only
  static const bool warp_kernel = getenv("MALLEUS_NORM_BWD_WARP") != nullptr;
  if (dy_bf16 && warp_kernel) {
    if (BwdWarpFn fn = bwd_warp_fn(h)) {
      const int warps = std::min(8, BWDW_SMEM / (h * 4));
      const int smem = warps * h * 4;
      static int attr_h = 0;
      if (attr_h != h) {  // opt in to > 48 KB of dynamic shared memory for this instance
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, BWDW_SMEM);
        if (e != cudaSuccess) return e;
        attr_h = h;
      }
      int nb = std::min(148, (T + warps - 1) / warps);
      fn<<<nb, warps * 32, smem, st>>>(T, h, (const uint4*)x, (const uint4*)g, rstd, (const uint4*)dy,
                                       (const uint4*)dres, (uint4*)dx_out, scratch); count_launch();
      colsum_accum_kernel<<<(h + 31) / 32, 1024, 0, st>>>(nb, h, scratch, dg_accum); count_launch();
      return cudaGetLastError();
    }
  }
  // row-group kernel (default where h / 8 is a multiple of 32 and at most 1024); MALLEUS_NORM_BWD_BLOCK=1
  // selects the block kernel below (A/B switch)
  static const bool block_kernel = getenv("MALLEUS_NORM_BWD_BLOCK") != nullptr;
  if (!block_kernel && (h / 8) % 32 == 0 && h / 8 <= BWDR_THREADS) {
    const int rb = BWDR_THREADS / (h / 8);
    auto kern = dy_bf16 ? rmsnorm_bwd_rows_kernel<true> : rmsnorm_bwd_rows_kernel<false>;
    static int per_sm[2][BWDR_THREADS / 32 + 1] = {};  // resident CTAs per SM per (instance, block size)
    int& occ = per_sm[dy_bf16 ? 1 : 0][rb * (h / 8) / 32];
    if (!occ) {
      cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, rb * (h / 8), 0);
      if (e != cudaSuccess) return e;
      occ = std::max(1, occ);
    }
    const int nb = std::min(148 * occ, (T + rb - 1) / rb);
    kern<<<nb, rb * (h / 8), 0, st>>>(T, h, (const uint4*)x, (const uint4*)g, rstd, dy, (const uint4*)dres,
                                      (uint4*)dx_out, scratch); count_launch();
    colsum_accum_kernel<<<(h + 31) / 32, 1024, 0, st>>>(nb, h, scratch, dg_accum); count_launch();
    return cudaGetLastError();
  }
  int rpb = (T + BWD_BLOCKS - 1) / BWD_BLOCKS;
  int nb = (T + rpb - 1) / rpb;
  const int vpt = (h / 8 + NORM_THREADS - 1) / NORM_THREADS;
  auto kern = dy_bf16 ? (vpt <= 1 ? rmsnorm_bwd_kernel<1, true> : vpt == 2 ? rmsnorm_bwd_kernel<2, true>
                          : vpt <= 4 ? rmsnorm_bwd_kernel<4, true> : rmsnorm_bwd_kernel<NORM_MAXV, true>)
                     : (vpt <= 1 ? rmsnorm_bwd_kernel<1, false> : vpt == 2 ? rmsnorm_bwd_kernel<2, false>
                          : vpt <= 4 ? rmsnorm_bwd_kernel<4, false> : rmsnorm_bwd_kernel<NORM_MAXV, false>);
  kern<<<nb, NORM_THREADS, 0, st>>>(T, h, rpb, (const uint4*)x, (const uint4*)g, rstd, dy,
                                    (const uint4*)dres, (uint4*)dx_out, scratch); count_launch();
  colsum_accum_kernel<<<(h + 31) / 32, 1024, 0, st>>>(nb, h, scratch, dg_accum); count_launch();
  return cudaGetLastError();
}

cudaError_t residual_add(long long n, const void* x, const float* partial, void* out, cudaStream_t st) {
  if (n % 8) return cudaErrorInvalidValue;
  residual_add_kernel<<<grid_for(n / 8, 256), 256, 0, st>>>(n / 8, (const uint4*)x, (const float4*)partial, (uint4*)out); count_launch();
  return cudaGetLastError();
}

cudaError_t rope_inplace(int T, int s, int n, int d, void* buf, long long ld, int col0, float theta,
                         bool inverse, cudaStream_t st) {
  if (d % 16 || ld % 8 || col0 % 8) return cudaErrorInvalidValue;
  long long total = (long long)T * (d / 16);
  rope_kernel<<<grid_for(total, 128), 128, 0, st>>>(T, s, n, d, (__nv_bfloat16*)buf, ld, col0, log2f(theta),
                                                    inverse ? -1.f : 1.f); count_launch();
  return cudaGetLastError();
}

cudaError_t swiglu_fwd(int T, int F, const void* gu, void* u, cudaStream_t st) {
  if (F % 8) return cudaErrorInvalidValue;
  swiglu_fwd_kernel<<<grid_for((long long)T * F / 8, 256), 256, 0, st>>>(T, F, (const __nv_bfloat16*)gu, (__nv_bfloat16*)u); count_launch();
  return cudaGetLastError();
}

cudaError_t swiglu_bwd(int T, int F, const void* gu, const void* du, void* dgu, cudaStream_t st) {
  if (F % 8) return cudaErrorInvalidValue;
  swiglu_bwd_kernel<<<grid_for((long long)T * F / 8, 256), 256, 0, st>>>(T, F, (const __nv_bfloat16*)gu,
                                                                       (const __nv_bfloat16*)du, (__nv_bfloat16*)dgu); count_launch();
  return cudaGetLastError();
}

cudaError_t embed_fwd(int T, int h, const int32_t* tok, const void* E, void* x, cudaStream_t st) {
  embed_fwd_kernel<<<T, 128, 0, st>>>(T, h, tok, (const uint4*)E, (uint4*)x); count_launch();
  return cudaGetLastError();
}

cudaError_t embed_bwd(int T, int h, const int32_t* tok, const void* dx, float* dE, cudaStream_t st) {
  if (T > EMBED_MAX_T || h % 8) return cudaErrorInvalidValue;
  static bool attr = false;  // 2 * T int32 of dynamic smem: up to 64 KB
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(embed_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         2 * EMBED_MAX_T * (int)sizeof(int32_t));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  embed_bwd_kernel<<<T, EMBED_THREADS, 2 * T * sizeof(int32_t), st>>>(T, h, tok, (const uint4*)dx, dE); count_launch();
  return cudaGetLastError();
}

cudaError_t ce_stats(int T, int V, const float* z, const int32_t* tgt, int v0, float* stats, cudaStream_t st) {
  if (V % 4) return cudaErrorInvalidValue;
  ce_stats_kernel<<<T, CE_THREADS, 0, st>>>(V, z, tgt, v0, stats); count_launch();
  return cudaGetLastError();
}

cudaError_t ce_combine_max(int T, const float* stats, float* gmax, cudaStream_t st) {
  ce_max_kernel<<<(T + 255) / 256, 256, 0, st>>>(T, stats, gmax); count_launch();
  return cudaGetLastError();
}

cudaError_t ce_local_sum(int T, const float* stats, const float* gmax, float* sum_tgt, cudaStream_t st) {
  ce_local_sum_kernel<<<(T + 255) / 256, 256, 0, st>>>(T, stats, gmax, sum_tgt); count_launch();
  return cudaGetLastError();
}

cudaError_t ce_grad(int T, int V, const float* z, const int32_t* tgt, int v0, const float* gmax, const float* gsum,
                    const float* gtgt, float scale, void* dz, float* loss_rows, cudaStream_t st, bool dz_f32) {
  if (V % 4) return cudaErrorInvalidValue;
  if (dz_f32) ce_grad_kernel<true><<<T, 256, 0, st>>>(V, z, tgt, v0, gmax, gsum, gtgt, scale, dz, loss_rows);
  else ce_grad_kernel<false><<<T, 256, 0, st>>>(V, z, tgt, v0, gmax, gsum, gtgt, scale, dz, loss_rows);
  count_launch();
  return cudaGetLastError();
}

cudaError_t reduce_loss(int T, const float* rows, float scale, float* out, int accumulate, cudaStream_t st) {
  reduce_loss_kernel<<<1, 1024, 0, st>>>(T, rows, scale, out, accumulate); count_launch();
  return cudaGetLastError();
}

cudaError_t cast_f32_bf16(long long n, const float* in, void* out, cudaStream_t st) {
  cast_kernel<<<grid_for(n, 256), 256, 0, st>>>(n, in, (__nv_bfloat16*)out); count_launch();
  return cudaGetLastError();
}

cudaError_t tp_combine_local(int k, int n, float* const* bufs, int op, cudaStream_t st) {
  if (k < 1 || k > MAX_TP || n < 0) return cudaErrorInvalidValue;
  CombinePtrs b{};
  for (int j = 0; j < k; ++j) b.p[j] = bufs[j];
  tp_combine_kernel<<<grid_for(n, 256), 256, 0, st>>>(k, n, b, op); count_launch();
  return cudaGetLastError();
}

cudaError_t fill_f32(long long n, float* p, float v, cudaStream_t st) {
  fill_kernel<<<grid_for(n, 256), 256, 0, st>>>(n, p, v); count_launch();
  return cudaGetLastError();
}

}  // namespace mls
