// Causal multi-head attention, forward and backward (PAPER.md:780 names
// FlashAttention).  FlashAttention-2-style tiling with warp-level mma.sync m16n8k16 bf16 tensor
// ops (fp32 accumulate), online softmax in registers, causal tile skipping.  Backward is split
// into a dK/dV kernel (one CTA per key block) and a dQ kernel (one CTA per query block) so that
// no atomics are needed and results are bitwise reproducible run to run.
//
// Layout: qkv [T, 3*n*d] bf16, T = nb * s; q | k | v column blocks, head j at columns j*d.
// RoPE has already been applied to q and k (elementwise.cu).  o [T, n*d]; lse [nb, n, s] fp32.
// Attention is 2-5% of step FLOPs; a tcgen05 version is future work
// (DESIGN.md §Attention).
#include <cuda_bf16.h>
#include "kernels.h"

namespace mls {
namespace {

constexpr int BQ = 64;   // queries per CTA (16 per warp)
constexpr int BKV = 64;  // keys per tile
constexpr float LOG2E = 1.4426950408889634f;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pk(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Tile in smem: rows x D bf16, row stride D + 8 elements (conflict-free ldmatrix).
template <int D>
struct Tile {
  static constexpr int LD = D + 8;
};

// Copy `rows` x D bf16 from global (row stride ld elements) to smem tile; zero rows >= valid.
template <int D>
__device__ __forceinline__ void load_tile(__nv_bfloat16* sm, const __nv_bfloat16* g, long long ld, int rows) {
  constexpr int CH = D / 8;  // 16-byte chunks per row
  for (int i = threadIdx.x; i < rows * CH; i += blockDim.x) {
    const int r = i / CH, c = i % CH;
    *reinterpret_cast<uint4*>(sm + r * Tile<D>::LD + c * 8) =
        *reinterpret_cast<const uint4*>(g + (long long)r * ld + c * 8);
  }
}

// A fragment (16x16) at (r0, c0) of a row-major smem tile.
template <int D>
__device__ __forceinline__ void frag_a(const __nv_bfloat16* sm, int r0, int c0, uint32_t (&a)[4]) {
  const int l = threadIdx.x & 31, mi = l >> 3;
  const int r = r0 + (mi & 1) * 8 + (l & 7), c = c0 + (mi >> 1) * 8;
  ldsm_x4(smem_addr(sm + r * Tile<D>::LD + c), a[0], a[1], a[2], a[3]);
}
// B fragments for two n-tiles [n0, n0+16) and k-step [k0, k0+16) from smem stored [n][k].
template <int D>
__device__ __forceinline__ void frag_b_nk(const __nv_bfloat16* sm, int n0, int k0, uint32_t& b00, uint32_t& b01,
                                          uint32_t& b10, uint32_t& b11) {
  const int l = threadIdx.x & 31, mi = l >> 3;
  const int n = n0 + (mi >> 1) * 8 + (l & 7), k = k0 + (mi & 1) * 8;
  ldsm_x4(smem_addr(sm + n * Tile<D>::LD + k), b00, b01, b10, b11);
}
// B fragments for k-step [k0, k0+16) and two n-tiles [n0, n0+16) from smem stored [k][n].
template <int D>
__device__ __forceinline__ void frag_b_kn(const __nv_bfloat16* sm, int k0, int n0, uint32_t& b00, uint32_t& b01,
                                          uint32_t& b10, uint32_t& b11) {
  const int l = threadIdx.x & 31, mi = l >> 3;
  const int k = k0 + (mi & 1) * 8 + (l & 7), n = n0 + (mi >> 1) * 8;
  ldsm_x4_t(smem_addr(sm + k * Tile<D>::LD + n), b00, b01, b10, b11);
}

// ------------------------------------------------------------------ forward
template <int D>
__global__ void __launch_bounds__(128)
attn_fwd_kernel(int s, int n, const __nv_bfloat16* __restrict__ qkv, __nv_bfloat16* __restrict__ o,
                float* __restrict__ lse, float scale) {
  extern __shared__ __align__(16) uint8_t sraw[];
  __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(sraw);
  __nv_bfloat16* sK = sQ + BQ * Tile<D>::LD;
  __nv_bfloat16* sV = sK + BKV * Tile<D>::LD;
  const int qb = blockIdx.x, head = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const long long ld = 3LL * n * D;
  const __nv_bfloat16* Qg = qkv + ((long long)b * s + qb * BQ) * ld + head * D;
  const __nv_bfloat16* Kg = qkv + (long long)b * s * ld + n * D + head * D;
  const __nv_bfloat16* Vg = qkv + (long long)b * s * ld + 2 * n * D + head * D;

  load_tile<D>(sQ, Qg, ld, BQ);
  __syncthreads();
  uint32_t qf[D / 16][4];
#pragma unroll
  for (int kk = 0; kk < D / 16; ++kk) frag_a<D>(sQ, warp * 16, kk * 16, qf[kk]);

  float acc[D / 8][4];
#pragma unroll
  for (int j = 0; j < D / 8; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  const float sl2 = scale * LOG2E;
  const int qrow0 = qb * BQ + warp * 16 + g;  // query index of rows g / g+8

  for (int kb = 0; kb <= qb; ++kb) {
    __syncthreads();
    load_tile<D>(sK, Kg + (long long)kb * BKV * ld, ld, BKV);
    load_tile<D>(sV, Vg + (long long)kb * BKV * ld, ld, BKV);
    __syncthreads();
    float S[BKV / 8][4];
#pragma unroll
    for (int j = 0; j < BKV / 8; ++j) S[j][0] = S[j][1] = S[j][2] = S[j][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
      for (int jj = 0; jj < BKV / 16; ++jj) {
        uint32_t b00, b01, b10, b11;
        frag_b_nk<D>(sK, jj * 16, kk * 16, b00, b01, b10, b11);
        mma16816(S[2 * jj], qf[kk], b00, b01);
        mma16816(S[2 * jj + 1], qf[kk], b10, b11);
      }
    }
    // causal mask on the diagonal tile, scaled row max
    float mx0 = m0, mx1 = m1;
#pragma unroll
    for (int j = 0; j < BKV / 8; ++j) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = kb * BKV + j * 8 + 2 * tq + (e & 1);
        const int q = qrow0 + (e >> 1) * 8;
        float v = S[j][e] * sl2;
        if (kb == qb && key > q) v = -INFINITY;
        S[j][e] = v;
      }
      mx0 = fmaxf(mx0, fmaxf(S[j][0], S[j][1]));
      mx1 = fmaxf(mx1, fmaxf(S[j][2], S[j][3]));
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float c0 = exp2f(m0 - mx0), c1 = exp2f(m1 - mx1);
    m0 = mx0; m1 = mx1;
    float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
    for (int j = 0; j < BKV / 8; ++j) {
      S[j][0] = exp2f(S[j][0] - m0); S[j][1] = exp2f(S[j][1] - m0);
      S[j][2] = exp2f(S[j][2] - m1); S[j][3] = exp2f(S[j][3] - m1);
      rs0 += S[j][0] + S[j][1];
      rs1 += S[j][2] + S[j][3];
    }
    l0 = l0 * c0 + rs0;
    l1 = l1 * c1 + rs1;
#pragma unroll
    for (int j = 0; j < D / 8; ++j) { acc[j][0] *= c0; acc[j][1] *= c0; acc[j][2] *= c1; acc[j][3] *= c1; }
#pragma unroll
    for (int kk = 0; kk < BKV / 16; ++kk) {
      uint32_t pa[4] = {pk(S[2 * kk][0], S[2 * kk][1]), pk(S[2 * kk][2], S[2 * kk][3]),
                        pk(S[2 * kk + 1][0], S[2 * kk + 1][1]), pk(S[2 * kk + 1][2], S[2 * kk + 1][3])};
#pragma unroll
      for (int jj = 0; jj < D / 16; ++jj) {
        uint32_t b00, b01, b10, b11;
        frag_b_kn<D>(sV, kk * 16, jj * 16, b00, b01, b10, b11);
        mma16816(acc[2 * jj], pa, b00, b01);
        mma16816(acc[2 * jj + 1], pa, b10, b11);
      }
    }
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float inv0 = 1.f / l0, inv1 = 1.f / l1;
  const long long ldo = (long long)n * D;
  __nv_bfloat16* O0 = o + ((long long)b * s + qrow0) * ldo + head * D;
  __nv_bfloat16* O1 = O0 + 8 * ldo;
#pragma unroll
  for (int j = 0; j < D / 8; ++j) {
    *reinterpret_cast<uint32_t*>(O0 + j * 8 + 2 * tq) = pk(acc[j][0] * inv0, acc[j][1] * inv0);
    *reinterpret_cast<uint32_t*>(O1 + j * 8 + 2 * tq) = pk(acc[j][2] * inv1, acc[j][3] * inv1);
  }
  if (tq == 0) {
    float* L = lse + ((long long)b * n + head) * s;
    L[qrow0] = (m0 + log2f(l0)) / LOG2E;       // natural-log LSE of the scaled scores
    L[qrow0 + 8] = (m1 + log2f(l1)) / LOG2E;
  }
}

// ------------------------------------------------------------------ backward preprocess
// dsum[b, head, i] = sum_dim dO[i] * O[i]
template <int D>
__global__ void attn_dsum_kernel(int s, int n, const __nv_bfloat16* __restrict__ o,
                                 const __nv_bfloat16* __restrict__ dout, float* __restrict__ dsum, long long T) {
  const long long idx = blockIdx.x * (long long)blockDim.y + threadIdx.y;  // (token, head)
  if (idx >= T * n) return;
  const long long t = idx / n;
  const int head = idx % n;
  const __nv_bfloat16* a = o + t * n * D + head * D;
  const __nv_bfloat16* c = dout + t * n * D + head * D;
  float acc = 0.f;
  for (int i = threadIdx.x * 2; i < D; i += 64) {
    float2 x = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(a + i));
    float2 y = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(c + i));
    acc += x.x * y.x + x.y * y.y;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (threadIdx.x == 0) {
    const long long b = t / s, i = t % s;
    dsum[(b * n + head) * s + i] = acc;
  }
}

// ------------------------------------------------------------------ backward dK, dV
template <int D>
__global__ void __launch_bounds__(128)
attn_bwd_dkv_kernel(int s, int n, const __nv_bfloat16* __restrict__ qkv, const __nv_bfloat16* __restrict__ dout,
                    const float* __restrict__ lse, const float* __restrict__ dsum,
                    __nv_bfloat16* __restrict__ dqkv, float scale) {
  extern __shared__ __align__(16) uint8_t sraw[];
  constexpr int LDT = Tile<D>::LD;
  __nv_bfloat16* sK = reinterpret_cast<__nv_bfloat16*>(sraw);
  __nv_bfloat16* sV = sK + BKV * LDT;
  __nv_bfloat16* sQ = sV + BKV * LDT;
  __nv_bfloat16* sO = sQ + BQ * LDT;  // dO tile
  float* sL = reinterpret_cast<float*>(sO + BQ * LDT);
  float* sD = sL + BQ;
  const int kb = blockIdx.x, head = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const long long ld = 3LL * n * D, ldo = (long long)n * D;
  const __nv_bfloat16* base = qkv + (long long)b * s * ld;
  load_tile<D>(sK, base + (long long)kb * BKV * ld + n * D + head * D, ld, BKV);
  load_tile<D>(sV, base + (long long)kb * BKV * ld + 2 * n * D + head * D, ld, BKV);

  float dK[D / 8][4], dV[D / 8][4];
#pragma unroll
  for (int j = 0; j < D / 8; ++j)
#pragma unroll
    for (int e = 0; e < 4; ++e) dK[j][e] = dV[j][e] = 0.f;
  const float sl2 = scale * LOG2E;
  const int key0 = kb * BKV + warp * 16 + g;  // key index of rows g / g+8
  const float* Lrow = lse + ((long long)b * n + head) * s;
  const float* Drow = dsum + ((long long)b * n + head) * s;

  for (int qb = kb; qb < s / BQ; ++qb) {
    __syncthreads();
    load_tile<D>(sQ, base + (long long)qb * BQ * ld + head * D, ld, BQ);
    load_tile<D>(sO, dout + ((long long)b * s + qb * BQ) * ldo + head * D, ldo, BQ);
    for (int i = threadIdx.x; i < BQ; i += blockDim.x) { sL[i] = Lrow[qb * BQ + i] * LOG2E; sD[i] = Drow[qb * BQ + i]; }
    __syncthreads();
    float S[BQ / 8][4], dP[BQ / 8][4];
#pragma unroll
    for (int j = 0; j < BQ / 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) S[j][e] = dP[j][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      uint32_t ka[4], va[4];
      frag_a<D>(sK, warp * 16, kk * 16, ka);
      frag_a<D>(sV, warp * 16, kk * 16, va);
#pragma unroll
      for (int jj = 0; jj < BQ / 16; ++jj) {
        uint32_t b00, b01, b10, b11;
        frag_b_nk<D>(sQ, jj * 16, kk * 16, b00, b01, b10, b11);
        mma16816(S[2 * jj], ka, b00, b01);
        mma16816(S[2 * jj + 1], ka, b10, b11);
        frag_b_nk<D>(sO, jj * 16, kk * 16, b00, b01, b10, b11);
        mma16816(dP[2 * jj], va, b00, b01);
        mma16816(dP[2 * jj + 1], va, b10, b11);
      }
    }
    // P^T = exp(S^T * scale - lse[q]); dS^T = P^T * (dP^T - D[q])
#pragma unroll
    for (int j = 0; j < BQ / 8; ++j) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int qi = j * 8 + 2 * tq + (e & 1);
        const int key = key0 + (e >> 1) * 8;
        float p = exp2f(S[j][e] * sl2 - sL[qi]);
        if (qb == kb && key > qb * BQ + qi) p = 0.f;
        S[j][e] = p;
        dP[j][e] = p * (dP[j][e] - sD[qi]);
      }
    }
#pragma unroll
    for (int kk = 0; kk < BQ / 16; ++kk) {
      uint32_t pa[4] = {pk(S[2 * kk][0], S[2 * kk][1]), pk(S[2 * kk][2], S[2 * kk][3]),
                        pk(S[2 * kk + 1][0], S[2 * kk + 1][1]), pk(S[2 * kk + 1][2], S[2 * kk + 1][3])};
      uint32_t da[4] = {pk(dP[2 * kk][0], dP[2 * kk][1]), pk(dP[2 * kk][2], dP[2 * kk][3]),
                        pk(dP[2 * kk + 1][0], dP[2 * kk + 1][1]), pk(dP[2 * kk + 1][2], dP[2 * kk + 1][3])};
#pragma unroll
      for (int jj = 0; jj < D / 16; ++jj) {
        uint32_t b00, b01, b10, b11;
        frag_b_kn<D>(sO, kk * 16, jj * 16, b00, b01, b10, b11);
        mma16816(dV[2 * jj], pa, b00, b01);
        mma16816(dV[2 * jj + 1], pa, b10, b11);
        frag_b_kn<D>(sQ, kk * 16, jj * 16, b00, b01, b10, b11);
        mma16816(dK[2 * jj], da, b00, b01);
        mma16816(dK[2 * jj + 1], da, b10, b11);
      }
    }
  }
  __nv_bfloat16* dK0 = dqkv + ((long long)b * s + key0) * ld + n * D + head * D;
  __nv_bfloat16* dV0 = dK0 + n * D;
#pragma unroll
  for (int j = 0; j < D / 8; ++j) {
    *reinterpret_cast<uint32_t*>(dK0 + j * 8 + 2 * tq) = pk(dK[j][0] * scale, dK[j][1] * scale);
    *reinterpret_cast<uint32_t*>(dK0 + 8 * ld + j * 8 + 2 * tq) = pk(dK[j][2] * scale, dK[j][3] * scale);
    *reinterpret_cast<uint32_t*>(dV0 + j * 8 + 2 * tq) = pk(dV[j][0], dV[j][1]);
    *reinterpret_cast<uint32_t*>(dV0 + 8 * ld + j * 8 + 2 * tq) = pk(dV[j][2], dV[j][3]);
  }
}

// ------------------------------------------------------------------ backward dQ
template <int D>
__global__ void __launch_bounds__(128)
attn_bwd_dq_kernel(int s, int n, const __nv_bfloat16* __restrict__ qkv, const __nv_bfloat16* __restrict__ dout,
                   const float* __restrict__ lse, const float* __restrict__ dsum,
                   __nv_bfloat16* __restrict__ dqkv, float scale) {
  extern __shared__ __align__(16) uint8_t sraw[];
  constexpr int LDT = Tile<D>::LD;
  __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(sraw);
  __nv_bfloat16* sO = sQ + BQ * LDT;
  __nv_bfloat16* sK = sO + BQ * LDT;
  __nv_bfloat16* sV = sK + BKV * LDT;
  const int qb = blockIdx.x, head = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const long long ld = 3LL * n * D, ldo = (long long)n * D;
  const __nv_bfloat16* base = qkv + (long long)b * s * ld;
  load_tile<D>(sQ, base + (long long)qb * BQ * ld + head * D, ld, BQ);
  load_tile<D>(sO, dout + ((long long)b * s + qb * BQ) * ldo + head * D, ldo, BQ);
  const float sl2 = scale * LOG2E;
  const int q0 = qb * BQ + warp * 16 + g;
  const float* Lrow = lse + ((long long)b * n + head) * s;
  const float* Drow = dsum + ((long long)b * n + head) * s;
  const float L0 = Lrow[q0] * LOG2E, L1 = Lrow[q0 + 8] * LOG2E;
  const float D0 = Drow[q0], D1 = Drow[q0 + 8];
  float dQ[D / 8][4];
#pragma unroll
  for (int j = 0; j < D / 8; ++j) dQ[j][0] = dQ[j][1] = dQ[j][2] = dQ[j][3] = 0.f;

  for (int kb = 0; kb <= qb; ++kb) {
    __syncthreads();
    load_tile<D>(sK, base + (long long)kb * BKV * ld + n * D + head * D, ld, BKV);
    load_tile<D>(sV, base + (long long)kb * BKV * ld + 2 * n * D + head * D, ld, BKV);
    __syncthreads();
    float S[BKV / 8][4], dP[BKV / 8][4];
#pragma unroll
    for (int j = 0; j < BKV / 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) S[j][e] = dP[j][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      uint32_t qa[4], oa[4];
      frag_a<D>(sQ, warp * 16, kk * 16, qa);
      frag_a<D>(sO, warp * 16, kk * 16, oa);
#pragma unroll
      for (int jj = 0; jj < BKV / 16; ++jj) {
        uint32_t b00, b01, b10, b11;
        frag_b_nk<D>(sK, jj * 16, kk * 16, b00, b01, b10, b11);
        mma16816(S[2 * jj], qa, b00, b01);
        mma16816(S[2 * jj + 1], qa, b10, b11);
        frag_b_nk<D>(sV, jj * 16, kk * 16, b00, b01, b10, b11);
        mma16816(dP[2 * jj], oa, b00, b01);
        mma16816(dP[2 * jj + 1], oa, b10, b11);
      }
    }
#pragma unroll
    for (int j = 0; j < BKV / 8; ++j) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = kb * BKV + j * 8 + 2 * tq + (e & 1);
        const int q = q0 + (e >> 1) * 8;
        float p = exp2f(S[j][e] * sl2 - ((e >> 1) ? L1 : L0));
        if (kb == qb && key > q) p = 0.f;
        dP[j][e] = p * (dP[j][e] - ((e >> 1) ? D1 : D0));
      }
    }
#pragma unroll
    for (int kk = 0; kk < BKV / 16; ++kk) {
      uint32_t da[4] = {pk(dP[2 * kk][0], dP[2 * kk][1]), pk(dP[2 * kk][2], dP[2 * kk][3]),
                        pk(dP[2 * kk + 1][0], dP[2 * kk + 1][1]), pk(dP[2 * kk + 1][2], dP[2 * kk + 1][3])};
#pragma unroll
      for (int jj = 0; jj < D / 16; ++jj) {
        uint32_t b00, b01, b10, b11;
        frag_b_kn<D>(sK, kk * 16, jj * 16, b00, b01, b10, b11);
        mma16816(dQ[2 * jj], da, b00, b01);
        mma16816(dQ[2 * jj + 1], da, b10, b11);
      }
    }
  }
  __nv_bfloat16* dQ0 = dqkv + ((long long)b * s + q0) * ld + head * D;
#pragma unroll
  for (int j = 0; j < D / 8; ++j) {
    *reinterpret_cast<uint32_t*>(dQ0 + j * 8 + 2 * tq) = pk(dQ[j][0] * scale, dQ[j][1] * scale);
    *reinterpret_cast<uint32_t*>(dQ0 + 8 * ld + j * 8 + 2 * tq) = pk(dQ[j][2] * scale, dQ[j][3] * scale);
  }
}

template <int D>
cudaError_t fwd_impl(int nb, int s, int n, const void* qkv, void* o, float* lse, cudaStream_t st) {
  const int smem = (BQ + 2 * BKV) * Tile<D>::LD * 2;
  auto k = attn_fwd_kernel<D>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  dim3 grid(s / BQ, n, nb);
  k<<<grid, 128, smem, st>>>(s, n, (const __nv_bfloat16*)qkv, (__nv_bfloat16*)o, lse, rsqrtf((float)D)); count_launch();
  return cudaGetLastError();
}

template <int D>
cudaError_t bwd_impl(int nb, int s, int n, const void* qkv, const void* o, const float* lse, const void* dout,
                     void* dqkv, float* dsum, cudaStream_t st) {
  const long long T = (long long)nb * s;
  dim3 pblk(32, 8);
  attn_dsum_kernel<D><<<(unsigned)((T * n + 7) / 8), pblk, 0, st>>>(s, n, (const __nv_bfloat16*)o,
                                                                     (const __nv_bfloat16*)dout, dsum, T); count_launch();
  const int smem = (BQ + BKV) * 2 * Tile<D>::LD * 2 + 2 * BQ * 4;
  auto k1 = attn_bwd_dkv_kernel<D>;
  auto k2 = attn_bwd_dq_kernel<D>;
  cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  dim3 grid(s / BQ, n, nb);
  const float scale = rsqrtf((float)D);
  k1<<<grid, 128, smem, st>>>(s, n, (const __nv_bfloat16*)qkv, (const __nv_bfloat16*)dout, lse, dsum,
                              (__nv_bfloat16*)dqkv, scale); count_launch();
  k2<<<grid, 128, smem, st>>>(s, n, (const __nv_bfloat16*)qkv, (const __nv_bfloat16*)dout, lse, dsum,
                              (__nv_bfloat16*)dqkv, scale); count_launch();
  return cudaGetLastError();
}

}  // namespace

cudaError_t attention_fwd(int nb, int s, int n, int d, const void* qkv, void* o, float* lse, cudaStream_t st) {
  if (s % BQ) return cudaErrorInvalidValue;
  switch (d) {
    case 32: return fwd_impl<32>(nb, s, n, qkv, o, lse, st);
    case 64: return fwd_impl<64>(nb, s, n, qkv, o, lse, st);
    case 128: return fwd_impl<128>(nb, s, n, qkv, o, lse, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t attention_bwd(int nb, int s, int n, int d, const void* qkv, const void* o, const float* lse,
                          const void* dout, void* dqkv, float* dsum, cudaStream_t st) {
  if (s % BQ) return cudaErrorInvalidValue;
  switch (d) {
    case 32: return bwd_impl<32>(nb, s, n, qkv, o, lse, dout, dqkv, dsum, st);
    case 64: return bwd_impl<64>(nb, s, n, qkv, o, lse, dout, dqkv, dsum, st);
    case 128: return bwd_impl<128>(nb, s, n, qkv, o, lse, dout, dqkv, dsum, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace mls
