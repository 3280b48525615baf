// Causal multi-head attention, forward and backward (PAPER.md:780 names
// FlashAttention).  FlashAttention-2-style tiling with warp-level mma.sync m16n8k16 bf16 tensor
// ops (fp32 accumulate), online softmax in registers, causal tile skipping, cp.async double
// buffering of the streamed tiles, heaviest causal blocks scheduled first.  Backward is split
// into a dK/dV kernel (one CTA per key block) and a dQ kernel (one CTA per query block) so that
// no atomics are needed and results are bitwise reproducible run to run.
//
// Layout: qkv [T, (n + 2 n_kv) d] bf16, T = nb * s; q | k | v column blocks, head j at columns j*d;
// GQA (n_kv < n): query head j reads KV head j / (n / n_kv), the dK/dV CTA of a KV head loops over its
// group's query heads.
// RoPE has already been applied to q and k (elementwise.cu).  o [T, n*d]; lse [nb, n, s] fp32.
// This mma.sync path serves the shapes the tcgen05 kernels (attention_tc.cu: d = 128, s % 128 == 0)
// do not cover, e.g. the tiny parity model C1 (d = 32).
#include <cuda_bf16.h>
#include "kernels.h"

namespace mls {
namespace {

constexpr int BKV = 64;  // keys per streamed tile / per dK-dV CTA
constexpr int BQB = 64;  // queries per streamed tile in the dK/dV kernel
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
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// smem tile: rows x D bf16, row stride D + 8 elements (conflict-free ldmatrix)
template <int D>
struct Tile {
  static constexpr int LD = D + 8;
  static constexpr int BYTES = LD * 2;
};

// async copy of `rows` x D bf16 (global row stride ld elements) into a smem tile
template <int D>
__device__ __forceinline__ void load_tile_async(__nv_bfloat16* sm, const __nv_bfloat16* g, long long ld, int rows) {
  constexpr int CH = D / 8;
  for (int i = threadIdx.x; i < rows * CH; i += blockDim.x) {
    const int r = i / CH, c = i % CH;
    cp_async16(sm + r * Tile<D>::LD + c * 8, g + (long long)r * ld + c * 8);
  }
}

template <int D>
__device__ __forceinline__ void frag_a(const __nv_bfloat16* sm, int r0, int c0, uint32_t (&a)[4]) {
  const int l = threadIdx.x & 31, mi = l >> 3;
  const int r = r0 + (mi & 1) * 8 + (l & 7), c = c0 + (mi >> 1) * 8;
  ldsm_x4(smem_addr(sm + r * Tile<D>::LD + c), a[0], a[1], a[2], a[3]);
}
// B fragments for two n-tiles [n0, n0+16) and k-step [k0, k0+16) from smem stored [n][k]
template <int D>
__device__ __forceinline__ void frag_b_nk(const __nv_bfloat16* sm, int n0, int k0, uint32_t& b00, uint32_t& b01,
                                          uint32_t& b10, uint32_t& b11) {
  const int l = threadIdx.x & 31, mi = l >> 3;
  const int n = n0 + (mi >> 1) * 8 + (l & 7), k = k0 + (mi & 1) * 8;
  ldsm_x4(smem_addr(sm + n * Tile<D>::LD + k), b00, b01, b10, b11);
}
// B fragments for k-step [k0, k0+16) and two n-tiles [n0, n0+16) from smem stored [k][n]
template <int D>
__device__ __forceinline__ void frag_b_kn(const __nv_bfloat16* sm, int k0, int n0, uint32_t& b00, uint32_t& b01,
                                          uint32_t& b10, uint32_t& b11) {
  const int l = threadIdx.x & 31, mi = l >> 3;
  const int k = k0 + (mi & 1) * 8 + (l & 7), n = n0 + (mi >> 1) * 8;
  ldsm_x4_t(smem_addr(sm + k * Tile<D>::LD + n), b00, b01, b10, b11);
}

// ------------------------------------------------------------------ forward
// CTA = NW warps x 16 queries; K/V tiles of 64 keys streamed with a 2-deep cp.async ring.
template <int D, int NW>
__global__ void __launch_bounds__(NW * 32)
attn_fwd_kernel(int s, int n, int n_kv, const __nv_bfloat16* __restrict__ qkv, __nv_bfloat16* __restrict__ o,
                float* __restrict__ lse, float scale) {
  constexpr int BQ = NW * 16;
  extern __shared__ __align__(16) uint8_t sraw[];
  __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(sraw);
  __nv_bfloat16* sKV = sQ + BQ * Tile<D>::LD;  // [2 stages][K | V][64][LD]
  const int nqb = s / BQ;
  const int qb = nqb - 1 - blockIdx.x;  // heaviest (most keys) first
  const int head = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const long long ld = (long long)(n + 2 * n_kv) * D;  // q | k | v (GQA: n_kv KV heads)
  const int kvh = head / (n / n_kv);
  const __nv_bfloat16* Qg = qkv + ((long long)b * s + qb * BQ) * ld + head * D;
  const __nv_bfloat16* Kg = qkv + (long long)b * s * ld + n * D + kvh * D;
  const __nv_bfloat16* Vg = Kg + n_kv * D;
  const int last_kb = ((qb + 1) * BQ - 1) / BKV;
  auto kv = [&](int stage, int which) { return sKV + (stage * 2 + which) * BKV * Tile<D>::LD; };

  load_tile_async<D>(sQ, Qg, ld, BQ);
  load_tile_async<D>(kv(0, 0), Kg, ld, BKV);
  load_tile_async<D>(kv(0, 1), Vg, ld, BKV);
  cp_commit();

  float acc[D / 8][4];
#pragma unroll
  for (int j = 0; j < D / 8; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  const float sl2 = scale * LOG2E;
  const int qrow0 = qb * BQ + warp * 16 + g;
  uint32_t qf[D / 16][4];

  for (int kb = 0; kb <= last_kb; ++kb) {
    const int stg = kb & 1;
    if (kb + 1 <= last_kb) {
      load_tile_async<D>(kv(stg ^ 1, 0), Kg + (long long)(kb + 1) * BKV * ld, ld, BKV);
      load_tile_async<D>(kv(stg ^ 1, 1), Vg + (long long)(kb + 1) * BKV * ld, ld, BKV);
    }
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    if (kb == 0) {
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) frag_a<D>(sQ, warp * 16, kk * 16, qf[kk]);
    }
    const __nv_bfloat16* sK = kv(stg, 0);
    const __nv_bfloat16* sV = kv(stg, 1);
    // warps whose 16 rows all precede this key tile skip it (causal)
    const bool active = kb * BKV <= qb * BQ + warp * 16 + 15;
    if (active) {
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
      const bool diag = (kb + 1) * BKV - 1 > qb * BQ + warp * 16;
      float mx0 = m0, mx1 = m1;
#pragma unroll
      for (int j = 0; j < BKV / 8; ++j) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int key = kb * BKV + j * 8 + 2 * tq + (e & 1);
          const int q = qrow0 + (e >> 1) * 8;
          float v = S[j][e] * sl2;
          if (diag && key > q) v = -INFINITY;
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
    __syncthreads();  // stage stg is refilled in the next iteration
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
    float* Lr = lse + ((long long)b * n + head) * s;
    Lr[qrow0] = (m0 + log2f(l0)) / LOG2E;  // natural-log LSE of the scaled scores
    Lr[qrow0 + 8] = (m1 + log2f(l1)) / LOG2E;
  }
}

// ------------------------------------------------------------------ backward preprocess
// dsum[b, head, i] = sum_dim dO[i] * O[i]
template <int D>
__global__ void attn_dsum_kernel(int s, int n, const __nv_bfloat16* __restrict__ o,
                                 const __nv_bfloat16* __restrict__ dout, float* __restrict__ dsum, long long T) {
  // D / 64 lanes x 128-bit loads per (token, head) row: 8 lanes per row at D = 128, 4 rows per warp
  constexpr int LPR = D / 16;  // lanes per row, 2 uint4 (16 elements) each
  const long long idx = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / LPR;  // (token, head)
  const int sub = threadIdx.x % LPR;
  float acc = 0.f;
  if (idx < T * n) {
    const uint4* a = reinterpret_cast<const uint4*>(o + idx * D) + sub * 2;
    const uint4* c = reinterpret_cast<const uint4*>(dout + idx * D) + sub * 2;
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const uint4 x = a[v], y = c[v];
      const __nv_bfloat162* xp = reinterpret_cast<const __nv_bfloat162*>(&x);
      const __nv_bfloat162* yp = reinterpret_cast<const __nv_bfloat162*>(&y);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 xf = __bfloat1622float2(xp[q]), yf = __bfloat1622float2(yp[q]);
        acc = fmaf(xf.x, yf.x, acc);
        acc = fmaf(xf.y, yf.y, acc);
      }
    }
  }
#pragma unroll
  for (int off = LPR / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (sub == 0 && idx < T * n) {
    const long long t = idx / n;
    const int head = (int)(idx % n);
    const long long b = t / s, i = t % s;
    dsum[(b * n + head) * s + i] = acc;
  }
}

// ------------------------------------------------------------------ backward dK, dV
// CTA = 4 warps x 16 keys (one 64-key block); Q / dO / lse / D tiles of 64 queries streamed with a
// 2-deep cp.async ring.
template <int D>
__global__ void __launch_bounds__(128)
attn_bwd_dkv_kernel(int s, int n, int n_kv, const __nv_bfloat16* __restrict__ qkv, const __nv_bfloat16* __restrict__ dout,
                    const float* __restrict__ lse, const float* __restrict__ dsum,
                    __nv_bfloat16* __restrict__ dqkv, float scale) {
  extern __shared__ __align__(16) uint8_t sraw[];
  constexpr int LDT = Tile<D>::LD;
  __nv_bfloat16* sK = reinterpret_cast<__nv_bfloat16*>(sraw);
  __nv_bfloat16* sV = sK + BKV * LDT;
  __nv_bfloat16* sQO = sV + BKV * LDT;  // [2 stages][Q | dO][64][LDT]
  float* sLD = reinterpret_cast<float*>(sQO + 4 * BQB * LDT);  // [2 stages][lse | D][64]
  const int nkb = s / BKV;
  const int kb = blockIdx.x;  // light blocks last: kb = 0 has the most query blocks
  const int kvh = blockIdx.y, b = blockIdx.z;  // KV head; GQA: its group's query heads one after another
  const int grp = n / n_kv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const long long ld = (long long)(n + 2 * n_kv) * D, ldo = (long long)n * D;
  const __nv_bfloat16* base = qkv + (long long)b * s * ld;
  auto qo = [&](int stage, int which) { return sQO + (stage * 2 + which) * BQB * LDT; };
  auto ldv = [&](int stage, int which) { return sLD + (stage * 2 + which) * BQB; };
  const int qb0 = (kb * BKV) / BQB;
  const int nqb_all = s / BQB, per_head = nqb_all - qb0;  // query blocks per query head
  auto issue = [&](int it, int stage) {  // iteration it = (query head of the group, query block)
    const int head = kvh * grp + it / per_head, qb = qb0 + it % per_head;
    const float* Lrow = lse + ((long long)b * n + head) * s;
    const float* Drow = dsum + ((long long)b * n + head) * s;
    load_tile_async<D>(qo(stage, 0), base + (long long)qb * BQB * ld + head * D, ld, BQB);
    load_tile_async<D>(qo(stage, 1), dout + ((long long)b * s + qb * BQB) * ldo + head * D, ldo, BQB);
    for (int i = threadIdx.x; i < BQB / 4; i += blockDim.x) {
      cp_async16(ldv(stage, 0) + 4 * i, Lrow + qb * BQB + 4 * i);
      cp_async16(ldv(stage, 1) + 4 * i, Drow + qb * BQB + 4 * i);
    }
  };
  load_tile_async<D>(sK, base + (long long)kb * BKV * ld + n * D + kvh * D, ld, BKV);
  load_tile_async<D>(sV, base + (long long)kb * BKV * ld + (n + n_kv) * D + kvh * D, ld, BKV);
  issue(0, 0);
  cp_commit();

  float dK[D / 8][4], dV[D / 8][4];
#pragma unroll
  for (int j = 0; j < D / 8; ++j)
#pragma unroll
    for (int e = 0; e < 4; ++e) dK[j][e] = dV[j][e] = 0.f;
  const float sl2 = scale * LOG2E;
  const int key0 = kb * BKV + warp * 16 + g;
  (void)nkb;
  const int n_it = grp * per_head;

  for (int it = 0; it < n_it; ++it) {
    const int qb = qb0 + it % per_head;
    const int stg = it & 1;
    if (it + 1 < n_it) issue(it + 1, stg ^ 1);
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    const __nv_bfloat16* sQ = qo(stg, 0);
    const __nv_bfloat16* sO = qo(stg, 1);
    const float* sL = ldv(stg, 0);
    const float* sD = ldv(stg, 1);
    float S[BQB / 8][4], dP[BQB / 8][4];
#pragma unroll
    for (int j = 0; j < BQB / 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) S[j][e] = dP[j][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      uint32_t ka[4], va[4];
      frag_a<D>(sK, warp * 16, kk * 16, ka);
      frag_a<D>(sV, warp * 16, kk * 16, va);
#pragma unroll
      for (int jj = 0; jj < BQB / 16; ++jj) {
        uint32_t b00, b01, b10, b11;
        frag_b_nk<D>(sQ, jj * 16, kk * 16, b00, b01, b10, b11);
        mma16816(S[2 * jj], ka, b00, b01);
        mma16816(S[2 * jj + 1], ka, b10, b11);
        frag_b_nk<D>(sO, jj * 16, kk * 16, b00, b01, b10, b11);
        mma16816(dP[2 * jj], va, b00, b01);
        mma16816(dP[2 * jj + 1], va, b10, b11);
      }
    }
    const bool diag = qb * BQB < kb * BKV + BKV;
#pragma unroll
    for (int j = 0; j < BQB / 8; ++j) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int qi = j * 8 + 2 * tq + (e & 1);
        const int key = key0 + (e >> 1) * 8;
        float p = exp2f(S[j][e] * sl2 - sL[qi] * LOG2E);
        if (diag && key > qb * BQB + qi) p = 0.f;
        S[j][e] = p;
        dP[j][e] = p * (dP[j][e] - sD[qi]);
      }
    }
#pragma unroll
    for (int kk = 0; kk < BQB / 16; ++kk) {
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
    __syncthreads();
  }
  __nv_bfloat16* dK0 = dqkv + ((long long)b * s + key0) * ld + n * D + kvh * D;
  __nv_bfloat16* dV0 = dK0 + n_kv * D;
#pragma unroll
  for (int j = 0; j < D / 8; ++j) {
    *reinterpret_cast<uint32_t*>(dK0 + j * 8 + 2 * tq) = pk(dK[j][0] * scale, dK[j][1] * scale);
    *reinterpret_cast<uint32_t*>(dK0 + 8 * ld + j * 8 + 2 * tq) = pk(dK[j][2] * scale, dK[j][3] * scale);
    *reinterpret_cast<uint32_t*>(dV0 + j * 8 + 2 * tq) = pk(dV[j][0], dV[j][1]);
    *reinterpret_cast<uint32_t*>(dV0 + 8 * ld + j * 8 + 2 * tq) = pk(dV[j][2], dV[j][3]);
  }
}

// ------------------------------------------------------------------ backward dQ
// CTA = 4 warps x 16 queries; K/V tiles streamed with a 2-deep cp.async ring.
template <int D>
__global__ void __launch_bounds__(128)
attn_bwd_dq_kernel(int s, int n, int n_kv, const __nv_bfloat16* __restrict__ qkv, const __nv_bfloat16* __restrict__ dout,
                   const float* __restrict__ lse, const float* __restrict__ dsum,
                   __nv_bfloat16* __restrict__ dqkv, float scale) {
  constexpr int BQ = 64;
  extern __shared__ __align__(16) uint8_t sraw[];
  constexpr int LDT = Tile<D>::LD;
  __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(sraw);
  __nv_bfloat16* sO = sQ + BQ * LDT;
  __nv_bfloat16* sKV = sO + BQ * LDT;  // [2 stages][K | V][64][LDT]
  const int nqb = s / BQ;
  const int qb = nqb - 1 - blockIdx.x;  // heaviest first
  const int head = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const long long ld = (long long)(n + 2 * n_kv) * D, ldo = (long long)n * D;
  const __nv_bfloat16* base = qkv + (long long)b * s * ld;
  const __nv_bfloat16* Kg = base + n * D + (head / (n / n_kv)) * D;  // GQA: the group's KV head
  const __nv_bfloat16* Vg = Kg + n_kv * D;
  auto kv = [&](int stage, int which) { return sKV + (stage * 2 + which) * BKV * LDT; };
  load_tile_async<D>(sQ, base + (long long)qb * BQ * ld + head * D, ld, BQ);
  load_tile_async<D>(sO, dout + ((long long)b * s + qb * BQ) * ldo + head * D, ldo, BQ);
  load_tile_async<D>(kv(0, 0), Kg, ld, BKV);
  load_tile_async<D>(kv(0, 1), Vg, ld, BKV);
  cp_commit();
  const float sl2 = scale * LOG2E;
  const int q0 = qb * BQ + warp * 16 + g;
  const float* Lrow = lse + ((long long)b * n + head) * s;
  const float* Drow = dsum + ((long long)b * n + head) * s;
  const float L0 = Lrow[q0] * LOG2E, L1 = Lrow[q0 + 8] * LOG2E;
  const float D0 = Drow[q0], D1 = Drow[q0 + 8];
  float dQ[D / 8][4];
#pragma unroll
  for (int j = 0; j < D / 8; ++j) dQ[j][0] = dQ[j][1] = dQ[j][2] = dQ[j][3] = 0.f;
  const int last_kb = ((qb + 1) * BQ - 1) / BKV;

  for (int kb = 0; kb <= last_kb; ++kb) {
    const int stg = kb & 1;
    if (kb + 1 <= last_kb) {
      load_tile_async<D>(kv(stg ^ 1, 0), Kg + (long long)(kb + 1) * BKV * ld, ld, BKV);
      load_tile_async<D>(kv(stg ^ 1, 1), Vg + (long long)(kb + 1) * BKV * ld, ld, BKV);
    }
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    const __nv_bfloat16* sK = kv(stg, 0);
    const __nv_bfloat16* sV = kv(stg, 1);
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
    const bool diag = kb == last_kb;
#pragma unroll
    for (int j = 0; j < BKV / 8; ++j) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = kb * BKV + j * 8 + 2 * tq + (e & 1);
        const int q = q0 + (e >> 1) * 8;
        float p = exp2f(S[j][e] * sl2 - ((e >> 1) ? L1 : L0));
        if (diag && key > q) p = 0.f;
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
    __syncthreads();
  }
  __nv_bfloat16* dQ0 = dqkv + ((long long)b * s + q0) * ld + head * D;
#pragma unroll
  for (int j = 0; j < D / 8; ++j) {
    *reinterpret_cast<uint32_t*>(dQ0 + j * 8 + 2 * tq) = pk(dQ[j][0] * scale, dQ[j][1] * scale);
    *reinterpret_cast<uint32_t*>(dQ0 + 8 * ld + j * 8 + 2 * tq) = pk(dQ[j][2] * scale, dQ[j][3] * scale);
  }
}

constexpr int FWD_NW = 8;  // 128 queries per forward CTA

template <int D>
cudaError_t fwd_impl(int nb, int s, int n, int n_kv, const void* qkv, void* o, float* lse, cudaStream_t st) {
  constexpr int BQ = FWD_NW * 16;
  if (s % BQ) {
    // short sequences: 64-query CTAs
    constexpr int smem = (64 + 4 * BKV) * Tile<D>::BYTES;
    auto k = attn_fwd_kernel<D, 4>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<dim3(s / 64, n, nb), 128, smem, st>>>(s, n, n_kv, (const __nv_bfloat16*)qkv, (__nv_bfloat16*)o, lse,
                                              rsqrtf((float)D)); count_launch();
    return cudaGetLastError();
  }
  constexpr int smem = (BQ + 4 * BKV) * Tile<D>::BYTES;
  auto k = attn_fwd_kernel<D, FWD_NW>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<<<dim3(s / BQ, n, nb), FWD_NW * 32, smem, st>>>(s, n, n_kv, (const __nv_bfloat16*)qkv, (__nv_bfloat16*)o, lse,
                                                    rsqrtf((float)D)); count_launch();
  return cudaGetLastError();
}

template <int D>
cudaError_t bwd_impl(int nb, int s, int n, int n_kv, const void* qkv, const void* o, const float* lse, const void* dout,
                     void* dqkv, float* dsum, cudaStream_t st) {
  const long long T = (long long)nb * s;
  {
    const long long threads = T * n * (D / 16);
    attn_dsum_kernel<D><<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(s, n, (const __nv_bfloat16*)o,
                                                                           (const __nv_bfloat16*)dout, dsum, T); count_launch();
  }
  const int smem1 = (2 * BKV + 4 * BQB) * Tile<D>::BYTES + 4 * BQB * 4;
  const int smem2 = (2 * 64 + 4 * BKV) * Tile<D>::BYTES;
  auto k1 = attn_bwd_dkv_kernel<D>;
  auto k2 = attn_bwd_dq_kernel<D>;
  cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, smem1);
  cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
  const float scale = rsqrtf((float)D);
  k1<<<dim3(s / BKV, n_kv, nb), 128, smem1, st>>>(s, n, n_kv, (const __nv_bfloat16*)qkv, (const __nv_bfloat16*)dout,
                                                  lse, dsum, (__nv_bfloat16*)dqkv, scale); count_launch();
  k2<<<dim3(s / 64, n, nb), 128, smem2, st>>>(s, n, n_kv, (const __nv_bfloat16*)qkv, (const __nv_bfloat16*)dout, lse,
                                              dsum, (__nv_bfloat16*)dqkv, scale); count_launch();
  return cudaGetLastError();
}

}  // namespace

static int g_attn_variant = 0;  // 0 auto (tcgen05 when supported), 1 mma.sync only
void attention_set_variant(int v) { g_attn_variant = v; }

cudaError_t attention_fwd(int nb, int s, int n, int d, const void* qkv, void* o, float* lse, cudaStream_t st,
                          int n_kv) {
  if (s % 64) return cudaErrorInvalidValue;
  if (n_kv <= 0) n_kv = n;
  if (n % n_kv) return cudaErrorInvalidValue;
  if (g_attn_variant == 0 && attention_fwd_tc_supported(s, d))
    return attention_fwd_tc(nb, s, n, qkv, o, lse, st, n_kv);
  switch (d) {
    case 32: return fwd_impl<32>(nb, s, n, n_kv, qkv, o, lse, st);
    case 64: return fwd_impl<64>(nb, s, n, n_kv, qkv, o, lse, st);
    case 128: return fwd_impl<128>(nb, s, n, n_kv, qkv, o, lse, st);
    default: return cudaErrorInvalidValue;
  }
}

bool attention_bwd_fuses_rope(int s, int d) { return g_attn_variant == 0 && attention_fwd_tc_supported(s, d); }

cudaError_t attention_bwd(int nb, int s, int n, int d, const void* qkv, const void* o, const float* lse,
                          const void* dout, void* dqkv, float* dsum, cudaStream_t st, const float2* rope_cs,
                          int n_kv) {
  if (s % 64) return cudaErrorInvalidValue;
  if (n_kv <= 0) n_kv = n;
  if (n % n_kv) return cudaErrorInvalidValue;
  if (g_attn_variant == 0 && attention_fwd_tc_supported(s, d)) {
    const long long T = (long long)nb * s;
    attn_dsum_kernel<128><<<(unsigned)((T * n * 8 + 255) / 256), 256, 0, st>>>(
        s, n, (const __nv_bfloat16*)o, (const __nv_bfloat16*)dout, dsum, T); count_launch();
    return attention_bwd_tc(nb, s, n, qkv, lse, dout, dqkv, dsum, rope_cs, st, n_kv);
  }
  switch (d) {
    case 32: return bwd_impl<32>(nb, s, n, n_kv, qkv, o, lse, dout, dqkv, dsum, st);
    case 64: return bwd_impl<64>(nb, s, n, n_kv, qkv, o, lse, dout, dqkv, dsum, st);
    case 128: return bwd_impl<128>(nb, s, n, n_kv, qkv, o, lse, dout, dqkv, dsum, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace mls
