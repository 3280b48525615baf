// FP32 parity mode (north star: "<= 1e-4 in fp32 mode"; SURVEY §7 hard part (h), §8(d) "FP32 parity
// mode ... bound by the plain FP32 ALUs"): the hot path's activation kernels in IEEE fp32 with
// plain FFMA contractions — NO TF32 (its 10-bit mantissa would miss 1e-4) and no tensor cores.
// A correctness mode, not a performance configuration: simple tiled SIMT kernels, deterministic
// reductions (fixed order, no atomics), the same arithmetic as the bf16 path without its rounding
// points (reading R6: fp32 everywhere).
//   gemm_f32        C (op)= A B with the GemmDesc layouts (A [M][K] or [K][M], B [N][K] or [K][N])
//   rmsnorm / residual / RoPE / SwiGLU / embedding      elementwise, fp32 I/O
//   attention fwd / bwd                                 one warp per query (fwd, dQ) or key (dK, dV)
#include <cuda_runtime.h>
#include <cmath>

#include "kernels.h"

namespace mls {
namespace {

// ---------------------------------------------------------------- GEMM (SIMT fp32)
constexpr int FB = 64, FK = 16;  // 64 x 64 output tile, K slab of 16; 256 threads, 4 x 4 outputs each

template <bool AMN, bool BMN>
__global__ void __launch_bounds__(256) gemm_f32_kernel(int M, int N, int K, const float* __restrict__ A,
                                                       long long lda, const float* __restrict__ B, long long ldb,
                                                       float* __restrict__ C, long long ldc, int accum) {
  __shared__ float As[FK][FB + 1], Bs[FK][FB + 1];
  const int m0 = blockIdx.y * FB, n0 = blockIdx.x * FB;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += FK) {
    for (int i = threadIdx.x; i < FK * FB; i += 256) {
      // slab element (kk, r): consecutive threads walk the contiguous dimension of each layout
      const int kk = AMN ? i / FB : i % FK, r = AMN ? i % FB : i / FK;
      const int m = m0 + r, k = k0 + kk;
      As[kk][r] = (m < M && k < K) ? (AMN ? A[(long long)k * lda + m] : A[(long long)m * lda + k]) : 0.f;
      const int kb = BMN ? i / FB : i % FK, rb = BMN ? i % FB : i / FK;
      const int n = n0 + rb, k2 = k0 + kb;
      Bs[kb][rb] = (n < N && k2 < K) ? (BMN ? B[(long long)k2 * ldb + n] : B[(long long)n * ldb + k2]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < FK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { a[i] = As[kk][ty + 16 * i]; b[i] = Bs[kk][tx + 16 * i]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int m = m0 + ty + 16 * i, n = n0 + tx + 16 * j;
      if (m < M && n < N) {
        float* c = C + (long long)m * ldc + n;
        *c = accum ? *c + acc[i][j] : acc[i][j];
      }
    }
}

// ---------------------------------------------------------------- RMSNorm, residual
constexpr int FT = 256;
__device__ __forceinline__ float block_sum_f(float v, float* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  float r = 0.f;
  for (int i = 0; i < FT / 32; ++i) r += sh[i];
  return r;
}

// x_new = x + partial (if partial; written to x_out); y = x_new * r * g, r = rsqrt(mean(x_new^2) + eps)
__global__ void __launch_bounds__(FT) rmsnorm_fwd_f32_kernel(int h, const float* __restrict__ x,
                                                              const float* __restrict__ partial,
                                                              float* __restrict__ x_out, const float* __restrict__ g,
                                                              float eps, float* __restrict__ y, float* __restrict__ rstd) {
  __shared__ float sh[FT / 32];
  const long long row = blockIdx.x;
  float ss = 0.f;
  for (int c = threadIdx.x; c < h; c += FT) {
    float v = x[row * h + c];
    if (partial) {
      v += partial[row * h + c];
      x_out[row * h + c] = v;
    }
    ss += v * v;
  }
  ss = block_sum_f(ss, sh);
  const float r = 1.f / sqrtf(ss / (float)h + eps);
  if (threadIdx.x == 0) rstd[row] = r;
  for (int c = threadIdx.x; c < h; c += FT) {
    const float v = partial ? x_out[row * h + c] : x[row * h + c];
    y[row * h + c] = v * r * g[c];
  }
}

// u = g*dy; dx = r*u - x*r^3*mean(x*u); dx_out = dres + dx
__global__ void __launch_bounds__(FT) rmsnorm_bwd_f32_kernel(int h, const float* __restrict__ x,
                                                              const float* __restrict__ g, const float* __restrict__ rstd,
                                                              const float* __restrict__ dy, const float* __restrict__ dres,
                                                              float* __restrict__ dx_out) {
  __shared__ float sh[FT / 32];
  const long long row = blockIdx.x;
  const float r = rstd[row];
  float dot = 0.f;
  for (int c = threadIdx.x; c < h; c += FT) dot += x[row * h + c] * g[c] * dy[row * h + c];
  dot = block_sum_f(dot, sh);
  const float coef = r * r * r * dot / (float)h;
  for (int c = threadIdx.x; c < h; c += FT) {
    float o = r * g[c] * dy[row * h + c] - x[row * h + c] * coef;
    if (dres) o += dres[row * h + c];
    dx_out[row * h + c] = o;
  }
}

// dg[c] += sum_rows dy*x*r, one thread per column, rows in order (deterministic)
__global__ void rmsnorm_dg_f32_kernel(int T, int h, const float* __restrict__ x, const float* __restrict__ rstd,
                                      const float* __restrict__ dy, float* __restrict__ dg) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= h) return;
  float s = 0.f;
  for (int t = 0; t < T; ++t) s += dy[(long long)t * h + c] * x[(long long)t * h + c] * rstd[t];
  dg[c] += s;
}

__global__ void residual_add_f32_kernel(long long n, const float* __restrict__ x, const float* __restrict__ p,
                                        float* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = x[i] + p[i];
}

// ---------------------------------------------------------------- RoPE (half-split, reading R3)
__global__ void rope_f32_kernel(int T, int s, int n, int d, float* __restrict__ buf, long long ld, int col0,
                                float theta, float sign) {
  const int half = d / 2;
  const long long total = (long long)T * n * half;  // n rotated heads (q then k)
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = idx % half;
    const int j = (idx / half) % n;
    const long long t = idx / half / n;
    const double ang = (double)(t % s) * pow((double)theta, -2.0 * i / d);
    const float cs = (float)cos(ang), sn = sign * (float)sin(ang);
    float* p = buf + t * ld + col0 + (long long)j * d;
    const float a = p[i], b = p[i + half];
    p[i] = a * cs - b * sn;
    p[i + half] = b * cs + a * sn;
  }
}

// ---------------------------------------------------------------- SwiGLU, embedding
__device__ __forceinline__ float sig_f(float x) { return 1.f / (1.f + expf(-x)); }

__global__ void swiglu_fwd_f32_kernel(int T, int F, const float* __restrict__ gu, float* __restrict__ u) {
  const long long total = (long long)T * F;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long t = i / F;
    const int c = i % F;
    const float G = gu[t * 2 * F + c], U = gu[t * 2 * F + F + c];
    u[i] = G * sig_f(G) * U;
  }
}

__global__ void swiglu_bwd_f32_kernel(int T, int F, const float* __restrict__ gu, const float* __restrict__ du,
                                      float* __restrict__ dgu) {
  const long long total = (long long)T * F;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long t = i / F;
    const int c = i % F;
    const float G = gu[t * 2 * F + c], U = gu[t * 2 * F + F + c], D = du[i];
    const float sg = sig_f(G);
    dgu[t * 2 * F + c] = D * U * sg * (1.f + G * (1.f - sg));
    dgu[t * 2 * F + F + c] = D * G * sg;
  }
}

__global__ void embed_fwd_f32_kernel(int h, const int32_t* __restrict__ tok, const float* __restrict__ E,
                                     float* __restrict__ x) {
  const long long t = blockIdx.x;
  for (int c = threadIdx.x; c < h; c += blockDim.x) x[t * h + c] = E[(long long)tok[t] * h + c];
}

// dE[tok[t]] += dx[t]: one thread per column walks the tokens in order (deterministic, no atomics)
__global__ void embed_bwd_f32_kernel(int T, int h, const int32_t* __restrict__ tok, const float* __restrict__ dx,
                                     float* __restrict__ dE) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= h) return;
  for (int t = 0; t < T; ++t) dE[(long long)tok[t] * h + c] += dx[(long long)t * h + c];
}

// ---------------------------------------------------------------- attention (causal, fp32)
// qkv [T, 3 n d]: q | k | v column blocks, token t = b*s + position.  lse [nb][n][s].
// Forward: one warp per (query i, head, sequence); online softmax over keys j <= i; each lane
// holds d/32 dimensions (d <= 128).
constexpr int AD = 4;  // dims per lane (d <= 128)
// GQA: qkv = q (n heads) | k (n_kv) | v (n_kv); query head hd reads KV head hd / (n / n_kv).
__global__ void attn_fwd_f32_kernel(int s, int n, int n_kv, int d, int nb, const float* __restrict__ qkv,
                                    float* __restrict__ o, float* __restrict__ lse, float scale) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= nb * n * s) return;
  const int i = warp % s, hd = (warp / s) % n, b = warp / s / n, kvh = hd / (n / n_kv);
  const long long ld = (long long)(n + 2 * n_kv) * d, t0 = (long long)b * s;
  const float* q = qkv + (t0 + i) * ld + (long long)hd * d;
  float qv[AD], acc[AD];
#pragma unroll
  for (int u = 0; u < AD; ++u) {
    const int c = lane + 32 * u;
    qv[u] = c < d ? q[c] : 0.f;
    acc[u] = 0.f;
  }
  float m = -INFINITY, l = 0.f;
  for (int j = 0; j <= i; ++j) {
    const float* k = qkv + (t0 + j) * ld + (long long)(n + kvh) * d;
    const float* v = qkv + (t0 + j) * ld + (long long)(n + n_kv + kvh) * d;
    float sc = 0.f;
#pragma unroll
    for (int u = 0; u < AD; ++u) {
      const int c = lane + 32 * u;
      if (c < d) sc += qv[u] * k[c];
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sc += __shfl_xor_sync(0xffffffffu, sc, off);
    sc *= scale;
    const float mn = fmaxf(m, sc);
    const float alpha = expf(m - mn), p = expf(sc - mn);
    l = l * alpha + p;
#pragma unroll
    for (int u = 0; u < AD; ++u) {
      const int c = lane + 32 * u;
      acc[u] = acc[u] * alpha + (c < d ? p * v[c] : 0.f);
    }
    m = mn;
  }
  float* out = o + (t0 + i) * (long long)n * d + (long long)hd * d;
#pragma unroll
  for (int u = 0; u < AD; ++u) {
    const int c = lane + 32 * u;
    if (c < d) out[c] = acc[u] / l;
  }
  if (lane == 0) lse[((long long)b * n + hd) * s + i] = m + logf(l);
}

// dsum[(t) * n + hd] = sum_c dO * O  (per query row and head)
__global__ void attn_dsum_f32_kernel(long long T, int n, int d, const float* __restrict__ o,
                                     const float* __restrict__ dout, float* __restrict__ dsum) {
  const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= T * n) return;
  const long long base = w * d;  // row t, head hd are contiguous: (t * n + hd) * d
  float s = 0.f;
  for (int c = lane; c < d; c += 32) s += o[base + c] * dout[base + c];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) dsum[w] = s;
}

// dQ_i = scale * sum_{j<=i} dS_ij K_j,  dS_ij = P_ij (dO_i . V_j - D_i),  P_ij = exp(scale q_i.k_j - lse_i)
__global__ void attn_dq_f32_kernel(int s, int n, int n_kv, int d, int nb, const float* __restrict__ qkv,
                                   const float* __restrict__ dout, const float* __restrict__ lse,
                                   const float* __restrict__ dsum, float* __restrict__ dqkv, float scale) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= nb * n * s) return;
  const int i = warp % s, hd = (warp / s) % n, b = warp / s / n, kvh = hd / (n / n_kv);
  const long long ld = (long long)(n + 2 * n_kv) * d, t0 = (long long)b * s, ti = t0 + i;
  const float* q = qkv + ti * ld + (long long)hd * d;
  const float* dO = dout + ti * (long long)n * d + (long long)hd * d;
  float qv[AD], dov[AD], acc[AD];
#pragma unroll
  for (int u = 0; u < AD; ++u) {
    const int c = lane + 32 * u;
    qv[u] = c < d ? q[c] : 0.f;
    dov[u] = c < d ? dO[c] : 0.f;
    acc[u] = 0.f;
  }
  const float L = lse[((long long)b * n + hd) * s + i], D = dsum[ti * n + hd];
  for (int j = 0; j <= i; ++j) {
    const float* k = qkv + (t0 + j) * ld + (long long)(n + kvh) * d;
    const float* v = qkv + (t0 + j) * ld + (long long)(n + n_kv + kvh) * d;
    float sc = 0.f, dp = 0.f;
#pragma unroll
    for (int u = 0; u < AD; ++u) {
      const int c = lane + 32 * u;
      if (c < d) { sc += qv[u] * k[c]; dp += dov[u] * v[c]; }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      sc += __shfl_xor_sync(0xffffffffu, sc, off);
      dp += __shfl_xor_sync(0xffffffffu, dp, off);
    }
    const float p = expf(sc * scale - L), ds = p * (dp - D);
#pragma unroll
    for (int u = 0; u < AD; ++u) {
      const int c = lane + 32 * u;
      if (c < d) acc[u] += ds * k[c];
    }
  }
  float* dq = dqkv + ti * ld + (long long)hd * d;
#pragma unroll
  for (int u = 0; u < AD; ++u) {
    const int c = lane + 32 * u;
    if (c < d) dq[c] = acc[u] * scale;
  }
}

// dV_j = sum_{i>=j} P_ij dO_i;  dK_j = scale * sum_{i>=j} dS_ij Q_i   (one warp per key j and KV
// head; GQA: summed over the group's query heads in head order)
__global__ void attn_dkv_f32_kernel(int s, int n, int n_kv, int d, int nb, const float* __restrict__ qkv,
                                    const float* __restrict__ dout, const float* __restrict__ lse,
                                    const float* __restrict__ dsum, float* __restrict__ dqkv, float scale) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= nb * n_kv * s) return;
  const int j = warp % s, kvh = (warp / s) % n_kv, b = warp / s / n_kv, g = n / n_kv;
  const long long ld = (long long)(n + 2 * n_kv) * d, t0 = (long long)b * s, tj = t0 + j;
  const float* k = qkv + tj * ld + (long long)(n + kvh) * d;
  const float* v = qkv + tj * ld + (long long)(n + n_kv + kvh) * d;
  float kv[AD], vv[AD], dk[AD], dv[AD];
#pragma unroll
  for (int u = 0; u < AD; ++u) {
    const int c = lane + 32 * u;
    kv[u] = c < d ? k[c] : 0.f;
    vv[u] = c < d ? v[c] : 0.f;
    dk[u] = dv[u] = 0.f;
  }
  for (int hi = 0; hi < g * (s - j); ++hi) {
    const int hd = kvh * g + hi / (s - j), i = j + hi % (s - j);
    const long long ti = t0 + i;
    const float* q = qkv + ti * ld + (long long)hd * d;
    const float* dO = dout + ti * (long long)n * d + (long long)hd * d;
    float sc = 0.f, dp = 0.f;
#pragma unroll
    for (int u = 0; u < AD; ++u) {
      const int c = lane + 32 * u;
      if (c < d) { sc += q[c] * kv[u]; dp += dO[c] * vv[u]; }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      sc += __shfl_xor_sync(0xffffffffu, sc, off);
      dp += __shfl_xor_sync(0xffffffffu, dp, off);
    }
    const float p = expf(sc * scale - lse[((long long)b * n + hd) * s + i]);
    const float ds = p * (dp - dsum[ti * n + hd]);
#pragma unroll
    for (int u = 0; u < AD; ++u) {
      const int c = lane + 32 * u;
      if (c < d) { dv[u] += p * dO[c]; dk[u] += ds * q[c]; }
    }
  }
  float* dkp = dqkv + tj * ld + (long long)(n + kvh) * d;
  float* dvp = dqkv + tj * ld + (long long)(n + n_kv + kvh) * d;
#pragma unroll
  for (int u = 0; u < AD; ++u) {
    const int c = lane + 32 * u;
    if (c < d) { dkp[c] = dk[u] * scale; dvp[c] = dv[u]; }
  }
}

inline int grid_of(long long n, int threads) {
  long long b = (n + threads - 1) / threads;
  return (int)(b < 148 * 16 ? (b < 1 ? 1 : b) : 148 * 16);
}

}  // namespace

cudaError_t gemm_f32(const GemmDesc& g, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0 || g.K <= 0 || g.n_dst) return cudaErrorInvalidValue;
  if (g.rope_done) *g.rope_done = false;
  const dim3 grid((g.N + FB - 1) / FB, (g.M + FB - 1) / FB);
  const float* A = static_cast<const float*>(g.A);
  const float* B = static_cast<const float*>(g.B);
  float* C = static_cast<float*>(g.C);
  const int acc = g.mode == GEMM_ACCUM_F32;
  if (!g.a_mn && !g.b_mn) gemm_f32_kernel<false, false><<<grid, 256, 0, st>>>(g.M, g.N, g.K, A, g.lda, B, g.ldb, C, g.ldc, acc);
  else if (!g.a_mn && g.b_mn) gemm_f32_kernel<false, true><<<grid, 256, 0, st>>>(g.M, g.N, g.K, A, g.lda, B, g.ldb, C, g.ldc, acc);
  else if (g.a_mn && g.b_mn) gemm_f32_kernel<true, true><<<grid, 256, 0, st>>>(g.M, g.N, g.K, A, g.lda, B, g.ldb, C, g.ldc, acc);
  else gemm_f32_kernel<true, false><<<grid, 256, 0, st>>>(g.M, g.N, g.K, A, g.lda, B, g.ldb, C, g.ldc, acc);
  count_launch();
  return cudaGetLastError();
}

cudaError_t rmsnorm_fwd_f32(int T, int h, const float* x, const float* partial, float* x_out, const float* g,
                            float eps, float* y, float* rstd, cudaStream_t st) {
  if (T <= 0 || h <= 0 || (partial && !x_out)) return cudaErrorInvalidValue;
  rmsnorm_fwd_f32_kernel<<<T, FT, 0, st>>>(h, x, partial, x_out, g, eps, y, rstd); count_launch();
  return cudaGetLastError();
}

cudaError_t rmsnorm_bwd_f32(int T, int h, const float* x, const float* g, const float* rstd, const float* dy,
                            const float* dres, float* dx_out, float* dg_accum, cudaStream_t st) {
  if (T <= 0 || h <= 0) return cudaErrorInvalidValue;
  rmsnorm_dg_f32_kernel<<<(h + 127) / 128, 128, 0, st>>>(T, h, x, rstd, dy, dg_accum); count_launch();
  rmsnorm_bwd_f32_kernel<<<T, FT, 0, st>>>(h, x, g, rstd, dy, dres, dx_out); count_launch();
  return cudaGetLastError();
}

cudaError_t residual_add_f32(long long n, const float* x, const float* p, float* out, cudaStream_t st) {
  residual_add_f32_kernel<<<grid_of(n, 256), 256, 0, st>>>(n, x, p, out); count_launch();
  return cudaGetLastError();
}

cudaError_t rope_f32(int T, int s, int n, int d, float* buf, long long ld, int col0, float theta, bool inverse,
                     cudaStream_t st) {
  if (d % 2) return cudaErrorInvalidValue;
  rope_f32_kernel<<<grid_of((long long)T * n * d, 256), 256, 0, st>>>(T, s, n, d, buf, ld, col0, theta,
                                                                      inverse ? -1.f : 1.f); count_launch();
  return cudaGetLastError();
}

cudaError_t swiglu_fwd_f32(int T, int F, const float* gu, float* u, cudaStream_t st) {
  swiglu_fwd_f32_kernel<<<grid_of((long long)T * F, 256), 256, 0, st>>>(T, F, gu, u); count_launch();
  return cudaGetLastError();
}

cudaError_t swiglu_bwd_f32(int T, int F, const float* gu, const float* du, float* dgu, cudaStream_t st) {
  swiglu_bwd_f32_kernel<<<grid_of((long long)T * F, 256), 256, 0, st>>>(T, F, gu, du, dgu); count_launch();
  return cudaGetLastError();
}

cudaError_t embed_fwd_f32(int T, int h, const int32_t* tok, const float* E, float* x, cudaStream_t st) {
  embed_fwd_f32_kernel<<<T, 128, 0, st>>>(h, tok, E, x); count_launch();
  return cudaGetLastError();
}

cudaError_t embed_bwd_f32(int T, int h, const int32_t* tok, const float* dx, float* dE, cudaStream_t st) {
  embed_bwd_f32_kernel<<<(h + 127) / 128, 128, 0, st>>>(T, h, tok, dx, dE); count_launch();
  return cudaGetLastError();
}

cudaError_t attention_fwd_f32(int nb, int s, int n, int d, const float* qkv, float* o, float* lse, cudaStream_t st,
                              int n_kv) {
  if (n_kv <= 0) n_kv = n;
  if (d > 32 * AD || d < 1 || n % n_kv) return cudaErrorInvalidValue;
  const long long warps = (long long)nb * n * s;
  attn_fwd_f32_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(s, n, n_kv, d, nb, qkv, o, lse,
                                                                            1.f / sqrtf((float)d));
  count_launch();
  return cudaGetLastError();
}

cudaError_t attention_bwd_f32(int nb, int s, int n, int d, const float* qkv, const float* o, const float* lse,
                              const float* dout, float* dqkv, float* dsum, cudaStream_t st, int n_kv) {
  if (n_kv <= 0) n_kv = n;
  if (d > 32 * AD || d < 1 || n % n_kv) return cudaErrorInvalidValue;
  const long long T = (long long)nb * s, warps = T * n;
  const unsigned blocks = (unsigned)((warps * 32 + 255) / 256);
  const unsigned blocks_kv = (unsigned)((T * n_kv * 32 + 255) / 256);
  const float scale = 1.f / sqrtf((float)d);
  attn_dsum_f32_kernel<<<blocks, 256, 0, st>>>(T, n, d, o, dout, dsum); count_launch();
  attn_dq_f32_kernel<<<blocks, 256, 0, st>>>(s, n, n_kv, d, nb, qkv, dout, lse, dsum, dqkv, scale); count_launch();
  attn_dkv_f32_kernel<<<blocks_kv, 256, 0, st>>>(s, n, n_kv, d, nb, qkv, dout, lse, dsum, dqkv, scale); count_launch();
  return cudaGetLastError();
}

}  // namespace mls
