// tcgen05 / TMEM / TMA bf16 GEMM for sm_100a: the uneven-split sharded GEMMs of the hot path
// (PAPER.md:262 Megatron TP column/row splits).
//
//   C[M,N] (op)= A[M,K] * B[K,N]      fp32 accumulation in TMEM, bf16 operands from HBM via TMA
//
// Operand storage (row-major in HBM):
//   A K-major : A stored [M][K]          A MN-major : A stored [K][M]   (i.e. A^T row-major)
//   B K-major : B stored [N][K] (Y=XW^T) B MN-major : B stored [K][N]
// The three combinations used by a transformer layer:
//   fwd / dgrad of K-major weights : (K, K)     x W^T
//   fwd of [in,out]-stored weights, dgrad of [out,in]-stored weights : (K, MN)
//   wgrad dW = dY^T X             : (MN, MN)
//
// Design: persistent, one CTA per SM, warp-specialised (warp 0 TMA producer, warp 1 MMA issuer +
// TMEM owner, warps 2..5 epilogue), 4-stage smem ring of 128x64 A + 256x64 B bf16 tiles with
// 128-byte swizzle, UMMA 128x256x16, double-buffered 2x256-column fp32 accumulators in TMEM so
// the epilogue of tile i overlaps the main loop of tile i+1.  Ragged M/N/K tails are handled by
// TMA out-of-bounds zero fill and masked epilogue stores (uneven TP shards produce ragged N).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <atomic>
#include <utility>
#include <vector>
#include <algorithm>
#include <cstring>
#include <cstdio>
#include <cstdlib>
#include "ptx.cuh"
#include "kernels.h"

namespace mls {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_TILE_BYTES = BM * BK * 2;   // 16 KB
constexpr int B_TILE_BYTES = BN * BK * 2;   // 32 KB
constexpr int STAGE_BYTES = A_TILE_BYTES + B_TILE_BYTES;
constexpr int GEMM_SMEM = STAGES * STAGE_BYTES + 1024 /*barriers*/ + 1024 /*align slack*/;
constexpr int GEMM_THREADS = 192;

struct GemmParams {
  int M, N, K;
  void* C;
  long long ldc;
  int mode;  // GEMM_STORE_BF16 / GEMM_STORE_F32 / GEMM_ACCUM_F32
  int vec_ok;  // rows of C are 16-byte aligned -> 128-bit stores
  int tma_epi; // C written by TMA store / reduce-add (CTA-pair kernel)
  const float2* rope_cs;  // fused RoPE (bf16 TMA epilogue only), see GemmDesc
  int rope_cols, rope_s;
  int n_dst, rows_per_dst;  // row-split destinations (GemmDesc::dst)
  void* dst[4];
  const void* res;          // fused residual (bf16, row stride ldr), GemmDesc::res
  long long ldr;
  int glu;                  // fused SwiGLU epilogue (GemmDesc::glu), CTA-pair TMA epilogue only
  const void* aux_in;       // glu 2: saved gu [M][2F] (row stride ld_aux_in)
  long long ld_aux_in;
  int dbg;                  // experiment switches of the glu 2 epilogue (MALLEUS_GLU2_DBG): 1 no smem
                            // reads of G/U, 2 no math, 4 no stores, 8 no G/U TMA loads (results are then wrong)
};
struct TmapSet {  // per-destination C maps of the row-split TMA epilogue
  CUtensorMap m[4];
};

__device__ __forceinline__ void tile_coords(int t, int tiles_m, int tiles_n, int& tm, int& tn) {
  constexpr int G = 8;  // group 8 M-tiles so consecutive CTAs share B tiles in L2
  int per_group = G * tiles_n;
  int g = t / per_group;
  int first_m = g * G;
  int gsz = min(tiles_m - first_m, G);
  int r = t % per_group;
  tm = first_m + r % gsz;
  tn = r / gsz;
}

// r[0..8) (fp32 bits) += the 8 bf16 values of q
__device__ __forceinline__ void add_bf16x8(uint32_t* r, uint4 q) {
  const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(b[i]);
    r[2 * i] = __float_as_uint(__uint_as_float(r[2 * i]) + f.x);
    r[2 * i + 1] = __float_as_uint(__uint_as_float(r[2 * i + 1]) + f.y);
  }
}
__device__ __forceinline__ float bf16r(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }
__device__ __forceinline__ float sigmoid_f(float x) { return 1.f / (1.f + __expf(-x)); }

// one 32-row x 64-column bf16 box of the TMA epilogue: lane = row, ra / rb = columns [0, 32) and
// [32, 64) as fp32 bits, packed to bf16 (RNE) into a 128B-swizzled 4 KB staging buffer and
// written by one TMA store (double-buffered: waits until the store issued two boxes ago has read
// its buffer)
__device__ __forceinline__ void stage_store_bf16(const CUtensorMap* tm, uint8_t* stg, int& sbuf,
                                                 const uint32_t (&ra)[32], const uint32_t (&rb)[32], int c0, int c1) {
  const int lane = threadIdx.x & 31;
  uint8_t* buf = stg + sbuf * 4096;
  if (lane == 0) bulk_wait_read<1>();
  __syncwarp();
#pragma unroll
  for (int ch = 0; ch < 8; ++ch) {
    const uint32_t* r = ch < 4 ? ra : rb;
    const int o = (ch & 3) * 8;
    uint4 w;
    w.x = pack_bf16(__uint_as_float(r[o + 0]), __uint_as_float(r[o + 1]));
    w.y = pack_bf16(__uint_as_float(r[o + 2]), __uint_as_float(r[o + 3]));
    w.z = pack_bf16(__uint_as_float(r[o + 4]), __uint_as_float(r[o + 5]));
    w.w = pack_bf16(__uint_as_float(r[o + 6]), __uint_as_float(r[o + 7]));
    *reinterpret_cast<uint4*>(buf + lane * 128 + ((ch ^ (lane & 7)) << 4)) = w;
  }
  fence_proxy_async();
  __syncwarp();
  if (lane == 0) {
    tma_store_2d(tm, buf, c0, c1);
    bulk_commit();
  }
  sbuf ^= 1;
}
// the same for a box already packed to bf16 (8 x 16 bytes per lane)
__device__ __forceinline__ void stage_store_packed(const CUtensorMap* tm, uint8_t* stg, int& sbuf,
                                                   const uint4 (&q)[8], int c0, int c1) {
  const int lane = threadIdx.x & 31;
  uint8_t* buf = stg + sbuf * 4096;
  if (lane == 0) bulk_wait_read<1>();
  __syncwarp();
#pragma unroll
  for (int ch = 0; ch < 8; ++ch) *reinterpret_cast<uint4*>(buf + lane * 128 + ((ch ^ (lane & 7)) << 4)) = q[ch];
  fence_proxy_async();
  __syncwarp();
  if (lane == 0) {
    tma_store_2d(tm, buf, c0, c1);
    bulk_commit();
  }
  sbuf ^= 1;
}

// SwiGLU forward epilogue (glu 1): the accumulator holds gate columns [j0, j0 + 128) in TMEM
// columns [0, 128) and the matching up columns in [128, 256).  G and U are rounded to bf16 (the
// saved pre-activations, reading R6) and stored into gu's two halves; u = silu(G) * U (fp32 math on
// the bf16 values, as the standalone kernel) is stored into u.  Maps: tmC = gu[:, :F], tmD->m[0] =
// gu[:, F:], tmD->m[1] = u (each F columns wide, so ragged F is clipped by TMA).
__device__ __forceinline__ void epilogue_glu_fwd(const GemmParams& p, const CUtensorMap* tmC, const TmapSet* tmD,
                                                 uint32_t taddr, int crow, int j0, uint8_t* stg, int& sbuf) {
  const int F = p.N >> 1;
#pragma unroll 1
  for (int c = 0; c < 2; ++c) {
    const int col0 = j0 + c * 64;
    uint32_t g0[32], g1[32], u0[32], u1[32];
    tmem_ld32(taddr + c * 64, g0);
    tmem_ld32(taddr + c * 64 + 32, g1);
    tmem_ld32(taddr + 128 + c * 64, u0);
    tmem_ld32(taddr + 128 + c * 64 + 32, u1);
    tmem_wait_ld();
    if (col0 >= F) continue;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      g0[j] = __float_as_uint(bf16r(__uint_as_float(g0[j])));
      g1[j] = __float_as_uint(bf16r(__uint_as_float(g1[j])));
      u0[j] = __float_as_uint(bf16r(__uint_as_float(u0[j])));
      u1[j] = __float_as_uint(bf16r(__uint_as_float(u1[j])));
    }
    stage_store_bf16(tmC, stg, sbuf, g0, g1, col0, crow);
    stage_store_bf16(&tmD->m[0], stg, sbuf, u0, u1, col0, crow);
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float a = __uint_as_float(g0[j]), b = __uint_as_float(g1[j]);
      u0[j] = __float_as_uint(a * sigmoid_f(a) * __uint_as_float(u0[j]));
      u1[j] = __float_as_uint(b * sigmoid_f(b) * __uint_as_float(u1[j]));
    }
    stage_store_bf16(&tmD->m[1], stg, sbuf, u0, u1, col0, crow);
  }
}

// Epilogue operand boxes read from HBM (the saved gu of glu 2, the residual) are staged by TMA into
// the warp's own two 4 KB staging buffers (the same 128B-swizzled 32-row x 64-column layout the
// output boxes use; lane = row), completing on the warp's mbarrier: per-lane row loads from global
// memory (32 rows per instruction) measured ~60 us slower per C2 du GEMM.
__device__ __forceinline__ void epi_load_boxes(uint8_t* buf, uint64_t* ebar, const CUtensorMap* m0,
                                               const CUtensorMap* m1, int c0, int c1) {
  mbar_arrive_expect_tx(ebar, m1 ? 8192 : 4096);
  tma_load_2d(buf, m0, ebar, c0, c1);
  if (m1) tma_load_2d(buf + 4096, m1, ebar, c0, c1);
}
__device__ __forceinline__ void epi_read_box(const uint8_t* buf, uint4 (&q)[8]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int v = 0; v < 8; ++v) q[v] = *reinterpret_cast<const uint4*>(buf + lane * 128 + ((v ^ (lane & 7)) << 4));
}

// SwiGLU backward epilogue (glu 2) of the down-projection dgrad du = dy W_d: D = bf16(du) (reading
// R6), G / U from the saved gu (tmD->m[2] / m[3]), dU = D * G * s, dG = D * U * s * (1 + G (1 - s)),
// s = sigmoid(G), stored into dgu's halves (tmD->m[0] = dgu[:, :F], tmD->m[1] = dgu[:, F:]); du
// itself is not stored.  Staging per warp: [0, 8K) G | U load boxes (chunk 0's issued by the caller
// before the accumulator wait, chunk c + 1's as soon as chunk c is in registers), [8K, 16K) dG | dU.
__device__ __forceinline__ void epilogue_glu_bwd(const GemmParams& p, const TmapSet* tmD, uint32_t taddr,
                                                 int row_box0, int crow, int col_base, uint8_t* stg, uint64_t* ebar,
                                                 uint32_t& ephase) {
  const int lane = threadIdx.x & 31;
  const int F = p.N;
  uint8_t* out = stg + 8192;
#pragma unroll 1
  for (int c = 0; c < 4; ++c) {
    const int col0 = col_base + c * 64;
    if (col0 >= F) break;  // warp-uniform: the remaining chunks are past the edge too
    uint32_t d0[32], d1[32];
    tmem_ld32(taddr + c * 64, d0);
    tmem_ld32(taddr + c * 64 + 32, d1);
    tmem_wait_ld();
    if (!(p.dbg & 8)) {
      mbar_wait(ebar, ephase);
      ephase ^= 1;
    }
    uint4 gq[8], uq[8];
    if (!(p.dbg & 1)) {
      epi_read_box(stg, gq);
      epi_read_box(stg + 4096, uq);
    } else {
#pragma unroll
      for (int v = 0; v < 8; ++v) { gq[v] = make_uint4(0x3f803f80u, 0, 0, 0); uq[v] = gq[v]; }
    }
    fence_proxy_async();  // these generic reads before the async-proxy (TMA) write of the next chunk
    __syncwarp();  // every lane has its rows: the load buffers may take the next chunk
    if (lane == 0 && c + 1 < 4 && col0 + 64 < F && !(p.dbg & 8))
      epi_load_boxes(stg, ebar, &tmD->m[2], &tmD->m[3], col0 + 64, row_box0);
#pragma unroll
    for (int v = 0; v < 8 && !(p.dbg & 2); ++v) {
      uint32_t* d = v < 4 ? d0 + 8 * v : d1 + 8 * (v - 4);
      const __nv_bfloat162* gb = reinterpret_cast<const __nv_bfloat162*>(&gq[v]);
      const __nv_bfloat162* ub = reinterpret_cast<const __nv_bfloat162*>(&uq[v]);
      float dU[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 G = __bfloat1622float2(gb[i]), U = __bfloat1622float2(ub[i]);
        const float D0 = bf16r(__uint_as_float(d[2 * i])), D1 = bf16r(__uint_as_float(d[2 * i + 1]));
        const float s0 = sigmoid_f(G.x), s1 = sigmoid_f(G.y);
        dU[2 * i] = D0 * G.x * s0;
        dU[2 * i + 1] = D1 * G.y * s1;
        d[2 * i] = __float_as_uint(D0 * U.x * s0 * (1.f + G.x * (1.f - s0)));
        d[2 * i + 1] = __float_as_uint(D1 * U.y * s1 * (1.f + G.y * (1.f - s1)));
      }
      uq[v].x = pack_bf16(dU[0], dU[1]);
      uq[v].y = pack_bf16(dU[2], dU[3]);
      uq[v].z = pack_bf16(dU[4], dU[5]);
      uq[v].w = pack_bf16(dU[6], dU[7]);
    }
    if (lane == 0) bulk_wait_read<0>();  // the previous chunk's stores have read the output buffers
    __syncwarp();
#pragma unroll
    for (int ch = 0; ch < 8; ++ch) {
      const uint32_t* r = ch < 4 ? d0 : d1;
      const int o = (ch & 3) * 8;
      uint4 w;
      w.x = pack_bf16(__uint_as_float(r[o + 0]), __uint_as_float(r[o + 1]));
      w.y = pack_bf16(__uint_as_float(r[o + 2]), __uint_as_float(r[o + 3]));
      w.z = pack_bf16(__uint_as_float(r[o + 4]), __uint_as_float(r[o + 5]));
      w.w = pack_bf16(__uint_as_float(r[o + 6]), __uint_as_float(r[o + 7]));
      *reinterpret_cast<uint4*>(out + lane * 128 + ((ch ^ (lane & 7)) << 4)) = w;
      *reinterpret_cast<uint4*>(out + 4096 + lane * 128 + ((ch ^ (lane & 7)) << 4)) = uq[ch];
    }
    fence_proxy_async();
    __syncwarp();
    if (lane == 0 && !(p.dbg & 4)) {
      tma_store_2d(&tmD->m[0], out, col0, crow);
      tma_store_2d(&tmD->m[1], out + 4096, col0, crow);
      bulk_commit();
    }
  }
}

// Residual epilogue (bf16 store of acc + res): staging per warp [0, 4K) the residual box (chunk 0's
// issued by the caller before the accumulator wait, chunk c + 1's once chunk c is in registers),
// [4K, 8K) the output box (tmD->m[0] = res).
__device__ __forceinline__ void epilogue_residual(const GemmParams& p, const CUtensorMap* tmC, const TmapSet* tmD,
                                                  uint32_t taddr, int row_box0, int col_base, uint8_t* stg,
                                                  uint64_t* ebar, uint32_t& ephase) {
  const int lane = threadIdx.x & 31;
  uint8_t* out = stg + 4096;
#pragma unroll 1
  for (int c = 0; c < 4; ++c) {
    const int col0 = col_base + c * 64;
    if (col0 >= p.N) break;
    uint32_t r0[32], r1[32];
    tmem_ld32(taddr + c * 64, r0);
    tmem_ld32(taddr + c * 64 + 32, r1);
    tmem_wait_ld();
    mbar_wait(ebar, ephase);
    ephase ^= 1;
    uint4 q[8];
    epi_read_box(stg, q);
    fence_proxy_async();
    __syncwarp();
    if (lane == 0 && c + 1 < 4 && col0 + 64 < p.N) epi_load_boxes(stg, ebar, &tmD->m[0], nullptr, col0 + 64, row_box0);
#pragma unroll
    for (int v = 0; v < 8; ++v) add_bf16x8(v < 4 ? r0 + 8 * v : r1 + 8 * (v - 4), q[v]);
    if (lane == 0) bulk_wait_read<0>();
    __syncwarp();
#pragma unroll
    for (int ch = 0; ch < 8; ++ch) {
      const uint32_t* r = ch < 4 ? r0 : r1;
      const int o = (ch & 3) * 8;
      uint4 w;
      w.x = pack_bf16(__uint_as_float(r[o + 0]), __uint_as_float(r[o + 1]));
      w.y = pack_bf16(__uint_as_float(r[o + 2]), __uint_as_float(r[o + 3]));
      w.z = pack_bf16(__uint_as_float(r[o + 4]), __uint_as_float(r[o + 5]));
      w.w = pack_bf16(__uint_as_float(r[o + 6]), __uint_as_float(r[o + 7]));
      *reinterpret_cast<uint4*>(out + lane * 128 + ((ch ^ (lane & 7)) << 4)) = w;
    }
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
      tma_store_2d(tmC, out, col0, row_box0);
      bulk_commit();
    }
  }
}

// Epilogue of one 256-column accumulator for one row per thread: TMEM (32 lanes x 32 columns per
// tcgen05.ld) -> registers -> bf16 / fp32 store or fp32 read-add-write (wgrad accumulation).
__device__ __forceinline__ void epilogue_tile(const GemmParams& p, uint32_t taddr, int row, int col_base) {
  const bool row_ok = row < p.M;
  void* Cb = p.C;
  long long crow = row;
  if (p.n_dst && row_ok) {
    const int d = row / p.rows_per_dst;
    Cb = d == 0 ? p.dst[0] : d == 1 ? p.dst[1] : d == 2 ? p.dst[2] : p.dst[3];  // no local-memory indexing
    crow = row - (long long)d * p.rows_per_dst;
  }
#pragma unroll 1
  for (int c = 0; c < 256 / 32; ++c) {
    const int col0 = col_base + c * 32;
    uint32_t r[32];
    tmem_ld32(taddr + c * 32, r);
    tmem_wait_ld();
    if (!row_ok || col0 >= p.N) continue;
    const bool full_chunk = p.vec_ok && col0 + 32 <= p.N;
    if (p.mode == GEMM_STORE_BF16) {
      __nv_bfloat16* C = reinterpret_cast<__nv_bfloat16*>(Cb) + crow * p.ldc + col0;
      if (p.res) {  // fused residual: C = bf16(acc + res), res rows 16-byte aligned, N % 8 == 0
        const uint4* rp = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(p.res) +
                                                         (long long)row * p.ldr + col0);
#pragma unroll
        for (int v = 0; v < 4; ++v)
          if (col0 + 8 * v < p.N) add_bf16x8(r + 8 * v, __ldg(rp + v));
      }
      if (full_chunk) {
        uint4* dst = reinterpret_cast<uint4*>(C);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          uint4 w;
          w.x = pack_bf16(__uint_as_float(r[8 * v + 0]), __uint_as_float(r[8 * v + 1]));
          w.y = pack_bf16(__uint_as_float(r[8 * v + 2]), __uint_as_float(r[8 * v + 3]));
          w.z = pack_bf16(__uint_as_float(r[8 * v + 4]), __uint_as_float(r[8 * v + 5]));
          w.w = pack_bf16(__uint_as_float(r[8 * v + 6]), __uint_as_float(r[8 * v + 7]));
          dst[v] = w;
        }
      } else {
        for (int j = 0; j < 32 && col0 + j < p.N; ++j) C[j] = __float2bfloat16_rn(__uint_as_float(r[j]));
      }
    } else {
      float* C = reinterpret_cast<float*>(Cb) + crow * p.ldc + col0;
      const bool accum = p.mode == GEMM_ACCUM_F32;
      if (full_chunk) {
        float4* dst = reinterpret_cast<float4*>(C);
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          float4 w = make_float4(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1]),
                                 __uint_as_float(r[4 * v + 2]), __uint_as_float(r[4 * v + 3]));
          if (accum) {
            float4 o = dst[v];
            w.x += o.x; w.y += o.y; w.z += o.z; w.w += o.w;
          }
          dst[v] = w;
        }
      } else {
        for (int j = 0; j < 32 && col0 + j < p.N; ++j)
          C[j] = accum ? C[j] + __uint_as_float(r[j]) : __uint_as_float(r[j]);
      }
    }
  }
}

// TMA epilogue: per warp, 32 rows x 128 bytes (32 fp32 or 64 bf16 columns) are staged in a
// 128B-swizzled smem box (double buffered) and written with one TMA store, or, for the fp32
// wgrad accumulation, with one TMA reduce-add (the add happens in L2; the SM never reads C).
// Out-of-bounds rows / columns are clipped by TMA, so ragged uneven-split shapes need no masks.
template <int GLU>
__device__ __forceinline__ void epilogue_tile_tma(const GemmParams& p, const CUtensorMap* tmC, const TmapSet* tmD,
                                                  uint32_t taddr, int row_box0, int col_base, uint8_t* stg,
                                                  int& sbuf, uint64_t* ebar, uint32_t& ephase) {
  const int lane = threadIdx.x & 31;
  if (row_box0 >= p.M) return;
  int crow = row_box0;  // store coordinate: in C, or in this box's destination (rows_per_dst % 32 == 0)
  if (p.n_dst) {
    const int d = row_box0 / p.rows_per_dst;
    tmC = &tmD->m[d];
    crow = row_box0 - d * p.rows_per_dst;
  }
  if constexpr (GLU == 1) { epilogue_glu_fwd(p, tmC, tmD, taddr, crow, col_base, stg, sbuf); return; }
  if constexpr (GLU == 2) { epilogue_glu_bwd(p, tmD, taddr, row_box0, crow, col_base, stg, ebar, ephase); return; }
  if constexpr (GLU == 3) { epilogue_residual(p, tmC, tmD, taddr, row_box0, col_base, stg, ebar, ephase); return; }
  if (p.mode == GEMM_STORE_BF16 && p.rope_cs != nullptr && col_base < p.rope_cols) {
    // QKV projection with RoPE fused (half-split pairs (i, i+64) of each 128-column head, reading
    // R3): the two heads of this 256-column tile are rotated in registers before the bf16 store.
    const int row = min(row_box0 + lane, p.M - 1);
    const float2* cs = p.rope_cs + (long long)(row % p.rope_s) * 64;
#pragma unroll 1
    for (int h2 = 0; h2 < 2; ++h2) {
      const int hc0 = col_base + h2 * 128;
      uint32_t r0[32], r1[32], r2[32], r3[32];
      tmem_ld32(taddr + h2 * 128, r0);
      tmem_ld32(taddr + h2 * 128 + 32, r1);
      tmem_ld32(taddr + h2 * 128 + 64, r2);
      tmem_ld32(taddr + h2 * 128 + 96, r3);
      tmem_wait_ld();
      if (hc0 >= p.N) continue;
      if (hc0 < p.rope_cols) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float2 c0 = cs[j], c1 = cs[32 + j];
          const float a0 = __uint_as_float(r0[j]), b0 = __uint_as_float(r2[j]);
          const float a1 = __uint_as_float(r1[j]), b1 = __uint_as_float(r3[j]);
          r0[j] = __float_as_uint(a0 * c0.x - b0 * c0.y);
          r2[j] = __float_as_uint(b0 * c0.x + a0 * c0.y);
          r1[j] = __float_as_uint(a1 * c1.x - b1 * c1.y);
          r3[j] = __float_as_uint(b1 * c1.x + a1 * c1.y);
        }
      }
#pragma unroll
      for (int half = 0; half < 2; ++half) {  // unrolled: register arrays are selected statically
        const uint32_t* ra = half ? r2 : r0;
        const uint32_t* rb = half ? r3 : r1;
        uint8_t* buf = stg + sbuf * 4096;
        if (lane == 0) bulk_wait_read<1>();
        __syncwarp();
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          const uint32_t* r = ch < 4 ? ra : rb;
          const int o = (ch & 3) * 8;
          uint4 w;
          w.x = pack_bf16(__uint_as_float(r[o + 0]), __uint_as_float(r[o + 1]));
          w.y = pack_bf16(__uint_as_float(r[o + 2]), __uint_as_float(r[o + 3]));
          w.z = pack_bf16(__uint_as_float(r[o + 4]), __uint_as_float(r[o + 5]));
          w.w = pack_bf16(__uint_as_float(r[o + 6]), __uint_as_float(r[o + 7]));
          *reinterpret_cast<uint4*>(buf + lane * 128 + ((ch ^ (lane & 7)) << 4)) = w;
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(tmC, buf, hc0 + half * 64, crow);
          bulk_commit();
        }
        sbuf ^= 1;
      }
    }
    return;
  }
  if (p.mode == GEMM_STORE_BF16) {
#pragma unroll 1
    for (int c = 0; c < 256 / 64; ++c) {
      const int col0 = col_base + c * 64;
      uint32_t r0[32], r1[32];
      tmem_ld32(taddr + c * 64, r0);
      tmem_ld32(taddr + c * 64 + 32, r1);
      tmem_wait_ld();
      if (col0 >= p.N) continue;
      uint8_t* buf = stg + sbuf * 4096;
      if (lane == 0) bulk_wait_read<1>();
      __syncwarp();
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) {
        const uint32_t* r = ch < 4 ? r0 : r1;
        const int o = (ch & 3) * 8;
        uint4 w;
        w.x = pack_bf16(__uint_as_float(r[o + 0]), __uint_as_float(r[o + 1]));
        w.y = pack_bf16(__uint_as_float(r[o + 2]), __uint_as_float(r[o + 3]));
        w.z = pack_bf16(__uint_as_float(r[o + 4]), __uint_as_float(r[o + 5]));
        w.w = pack_bf16(__uint_as_float(r[o + 6]), __uint_as_float(r[o + 7]));
        *reinterpret_cast<uint4*>(buf + lane * 128 + ((ch ^ (lane & 7)) << 4)) = w;
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(tmC, buf, col0, crow);
        bulk_commit();
      }
      sbuf ^= 1;
    }
  } else {
#pragma unroll 1
    for (int c = 0; c < 256 / 32; ++c) {
      const int col0 = col_base + c * 32;
      uint32_t r[32];
      tmem_ld32(taddr + c * 32, r);
      tmem_wait_ld();
      if (col0 >= p.N) continue;
      uint8_t* buf = stg + sbuf * 4096;
      if (lane == 0) bulk_wait_read<1>();
      __syncwarp();
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) {
        uint4 w = make_uint4(r[4 * ch], r[4 * ch + 1], r[4 * ch + 2], r[4 * ch + 3]);
        *reinterpret_cast<uint4*>(buf + lane * 128 + ((ch ^ (lane & 7)) << 4)) = w;
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        if (p.mode == GEMM_ACCUM_F32) tma_reduce_add_2d(tmC, buf, col0, crow);
        else tma_store_2d(tmC, buf, col0, crow);
        bulk_commit();
      }
      sbuf ^= 1;
    }
  }
}

template <bool A_MN, bool B_MN>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
gemm_tcgen05_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    GemmParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;   // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int tiles_m = (p.M + BM - 1) / BM;
  const int tiles_n = (p.N + BN - 1) / BN;
  const int n_tiles = tiles_m * tiles_n;
  const int n_kb = (p.K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 128); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      int stage = 0; uint32_t phase = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        int tm, tn; tile_coords(t, tiles_m, tiles_n, tm, tn);
        const int m0 = tm * BM, n0 = tn * BN;
        for (int kb = 0; kb < n_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_TILE_BYTES;
          mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
          const int k0 = kb * BK;
          if (!A_MN) {
            tma_load_2d(sa, &tmA, &full[stage], k0, m0);
          } else {
            tma_load_2d(sa, &tmA, &full[stage], m0, k0);
            tma_load_2d(sa + 8192, &tmA, &full[stage], m0 + 64, k0);
          }
          if (!B_MN) {
            tma_load_2d(sb, &tmB, &full[stage], k0, n0);
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) tma_load_2d(sb + j * 8192, &tmB, &full[stage], n0 + 64 * j, k0);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (single thread)
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(BM, BN, A_MN, B_MN);
      int stage = 0; uint32_t phase = 0; int it = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < n_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t sb = sa + A_TILE_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            uint64_t ad, bd;
            if (!A_MN) ad = umma_desc_sw128(sa + k * 32, 16, 1024);
            else       ad = umma_desc_sw128(sa + k * 2048, 8192, 1024);
            if (!B_MN) bd = umma_desc_sw128(sb + k * 32, 16, 1024);
            else       bd = umma_desc_sw128(sb + k * 2048, 8192, 1024);
            umma_f16(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          umma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else {
    // ---------------- epilogue: TMEM -> registers -> HBM
    const int quarter = warp & 3;  // TMEM lane quarter accessible by this warp
    int it = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
      int tm, tn; tile_coords(t, tiles_m, tiles_n, tm, tn);
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = tm * BM + quarter * 32 + lane;
      epilogue_tile(p, tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN, row, tn * BN);
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
    if (p.n_dst) __threadfence_system();  // row-split stores (possibly peer memory) visible system-wide
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

// ------------------------------------------------------------------ CTA-pair variant (cta_group::2)
// A cluster of 2 CTAs on one TPC computes a 256 x 256 tile with UMMA M=256 (tcgen05.mma.cta_group::2
// issued by the even CTA): each CTA stages its own 128 rows of A and 128 rows (N) of B, so per SM the
// smem operand traffic per MMA drops by a third and each B tile is fetched from L2 once per pair.
// Both CTAs' TMA loads complete on the leader's full barrier; the leader's commits multicast to
// both CTAs' empty / TMEM-full barriers; both epilogues arrive on the leader's TMEM-empty barrier.
constexpr int BM2 = 128, BN2 = 256, STAGES2 = 6;
constexpr int A2_BYTES = BM2 * BK * 2;            // 16 KB
constexpr int B2_BYTES = (BN2 / 2) * BK * 2;      // 16 KB (this CTA's half of N)
constexpr int STAGE2_BYTES = A2_BYTES + B2_BYTES;
constexpr int EPI_STAGE_BYTES = 4 * 2 * 4096;  // 4 epilogue warps x 2 swizzled 4 KB boxes
// per-warp staging: 8 KB, or 16 KB for the SwiGLU backward (8 KB of prefetched G | U boxes + 8 KB of
// dG | dU output boxes; that variant runs a 5-stage operand ring to make room)
constexpr int epi_warp_bytes(int glu) { return glu == 2 ? 16384 : 8192; }
constexpr int gemm2_smem(int stages, int glu = 0) {
  return stages * STAGE2_BYTES + 4 * epi_warp_bytes(glu) + 1024 + 1024;
}

// ST: smem ring depth (6 by default; 5 leaves room on each SM for a concurrently running
// communication kernel, see GemmDesc::co_resident)
template <bool A_MN, bool B_MN, int ST, int GLU>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GEMM_THREADS, 1)
gemm_tcgen05_2sm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const __grid_constant__ CUtensorMap tmB2, const __grid_constant__ CUtensorMap tmC,
                        const __grid_constant__ TmapSet tmD, GemmParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* epi_stage = smem + ST * STAGE2_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(epi_stage + 4 * epi_warp_bytes(GLU));
  uint64_t* empty = full + ST;
  uint64_t* tfull = empty + ST;  // [2]
  uint64_t* tempty = tfull + 2;       // [2] (leader's copy is the one used)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint64_t* ebar = tempty + 3;        // [4] epilogue warps' operand-box barriers (GLU 2 / 3)

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int tiles_m = (p.M + 2 * BM2 - 1) / (2 * BM2);
  // glu 1: a tile is 128 gate columns (B rows from tmB, staged by the even CTA) next to the same
  // 128 up columns (tmB2, odd CTA), so the pair's 256-column accumulator holds both halves
  const int tiles_n = GLU == 1 ? ((p.N >> 1) + BN2 / 2 - 1) / (BN2 / 2) : (p.N + BN2 - 1) / BN2;
  const int n_tiles = tiles_m * tiles_n;
  const int n_kb = (p.K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    if (GLU == 1) tma_prefetch(&tmB2);
    for (int s = 0; s < ST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 8); }
    if (GLU >= 2)
      for (int w = 0; w < 4; ++w) mbar_init(&ebar[w], 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc2(tmem_slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0; uint32_t phase = 0;
      for (int t = cid; t < n_tiles; t += ncl) {
        int tm, tn; tile_coords(t, tiles_m, tiles_n, tm, tn);
        const int m0 = tm * 2 * BM2 + rank * BM2;
        const int n0 = GLU == 1 ? tn * (BN2 / 2) : tn * BN2 + rank * (BN2 / 2);
        const CUtensorMap* mB = GLU == 1 && rank ? &tmB2 : &tmB;
        for (int kb = 0; kb < n_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE2_BYTES;
          uint8_t* sb = sa + A2_BYTES;
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * STAGE2_BYTES);
          const int k0 = kb * BK;
          if (!A_MN) {
            tma_load_2d_2sm(sa, &tmA, &full[stage], k0, m0);
          } else {
            tma_load_2d_2sm(sa, &tmA, &full[stage], m0, k0);
            tma_load_2d_2sm(sa + 8192, &tmA, &full[stage], m0 + 64, k0);
          }
          if (!B_MN) {
            tma_load_2d_2sm(sb, mB, &full[stage], k0, n0);
          } else {
            tma_load_2d_2sm(sb, mB, &full[stage], n0, k0);
            tma_load_2d_2sm(sb + 8192, mB, &full[stage], n0 + 64, k0);
          }
          if (++stage == ST) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(2 * BM2, BN2, A_MN, B_MN);
      int stage = 0; uint32_t phase = 0; int it = 0;
      for (int t = cid; t < n_tiles; t += ncl, ++it) {
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN2;
        for (int kb = 0; kb < n_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * STAGE2_BYTES);
          const uint32_t sb = sa + A2_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            uint64_t ad, bd;
            if (!A_MN) ad = umma_desc_sw128(sa + k * 32, 16, 1024);
            else       ad = umma_desc_sw128(sa + k * 2048, 8192, 1024);
            if (!B_MN) bd = umma_desc_sw128(sb + k * 32, 16, 1024);
            else       bd = umma_desc_sw128(sb + k * 2048, 8192, 1024);
            umma_f16_2sm(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          umma_commit_2sm_mc(&empty[stage]);
          if (++stage == ST) { stage = 0; phase ^= 1; }
        }
        umma_commit_2sm_mc(&tfull[acc]);
      }
    }
  } else {
    const int quarter = warp & 3;
    uint8_t* stg = epi_stage + (warp - 2) * epi_warp_bytes(GLU);
    int sbuf = 0;
    uint32_t ephase = 0;
    int it = 0;
    for (int t = cid; t < n_tiles; t += ncl, ++it) {
      int tm, tn; tile_coords(t, tiles_m, tiles_n, tm, tn);
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int row_box0 = tm * 2 * BM2 + rank * BM2 + quarter * 32;
      if constexpr (GLU == 2) {  // G | U boxes of the tile's first chunk: independent of the accumulator
        if (lane == 0 && !(p.dbg & 8)) epi_load_boxes(stg, &ebar[warp - 2], &tmD.m[2], &tmD.m[3], tn * BN2, row_box0);
      } else if constexpr (GLU == 3) {
        if (lane == 0) epi_load_boxes(stg, &ebar[warp - 2], &tmD.m[0], nullptr, tn * BN2, row_box0);
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN2;
      if (GLU || p.tma_epi)
        epilogue_tile_tma<GLU>(p, &tmC, &tmD, taddr, row_box0, GLU == 1 ? tn * (BN2 / 2) : tn * BN2, stg, sbuf,
                               &ebar[warp - 2], ephase);
      else epilogue_tile(p, taddr, row_box0 + lane, tn * BN2);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_leader(&tempty[acc]);
    }
    if (lane == 0) bulk_wait_all();
    if (p.n_dst) __threadfence_system();  // row-split stores (possibly peer memory) visible system-wide
    __syncwarp();
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc2(tmem_base, 512);
  }
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static cudaError_t get_encoder() {
  if (g_encode) return cudaSuccess;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) return cudaErrorNotSupported;
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return cudaSuccess;
}

// 2-D bf16 row-major tensor [outer][inner] with row stride ld (elements); box = {64, box_outer}.
static bool make_map(CUtensorMap* m, const void* ptr, long long inner, long long outer, long long ld,
                     int box_outer) {
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                        box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// C map for the TMA epilogue: [M][N] row stride ldc, box {128 bytes, 32 rows}, 128B swizzle.
static bool make_map_c(CUtensorMap* m, void* ptr, long long N, long long M, long long ldc, bool f32) {
  cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)M};
  cuuint64_t strides[1] = {(cuuint64_t)ldc * (f32 ? 4 : 2)};
  cuuint32_t box[2] = {f32 ? 32u : 64u, 32u};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, ptr, dims,
                        strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

static int g_num_sms = 0;

static std::atomic<long long> g_launches{0};
void count_launch(int n) { g_launches += n; }
long long launches_total() { return g_launches.load(); }

// Optional per-launch CUDA-event timing of this GEMM (bench.py roofline of the dominant kernel).
struct GemmProf {
  bool on = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
  std::vector<double> flops;
  size_t used = 0;
};
static GemmProf g_prof;

// MALLEUS_GEMM_LOG=<path>: append "M N K a_mn b_mn mode epi kernel" per launch (measurement aid: the
// n-th line is the n-th gemm_tcgen05 launch of an ncu launch list of the same program)
static void gemm_log(const GemmParams& p, bool a_mn, bool b_mn, const char* kern) {
  static FILE* f = [] {
    const char* e = getenv("MALLEUS_GEMM_LOG");
    return e ? fopen(e, "a") : nullptr;
  }();
  if (f) {
    fprintf(f, "%d %d %d %d %d %d %d %s\n", p.M, p.N, p.K, (int)a_mn, (int)b_mn, p.mode, p.glu, kern);
    fflush(f);
  }
}

void gemm_profile_enable(bool on) {
  g_prof.on = on;
  g_prof.used = 0;
  g_prof.flops.clear();
}
// ms = the length of the union of the launches' [start, end] intervals (GEMM-busy wall time): the sum of
// their durations when they run one after another on one stream; when weight-gradient GEMMs run on a
// side stream beside the dgrad chain (pair mode) overlapping intervals are counted once
cudaError_t gemm_profile_query(long long* launches, double* flops, double* ms) {
  double f = 0;
  std::vector<std::pair<double, double>> iv;
  iv.reserve(g_prof.used);
  for (size_t i = 0; i < g_prof.used; ++i) {
    cudaError_t e = cudaEventSynchronize(g_prof.ev[i].second);
    if (e != cudaSuccess) return e;
    float a = 0.f, b = 0.f;
    cudaEventElapsedTime(&a, g_prof.ev[0].first, g_prof.ev[i].first);
    cudaEventElapsedTime(&b, g_prof.ev[0].first, g_prof.ev[i].second);
    iv.push_back({a, b});
    f += g_prof.flops[i];
  }
  std::sort(iv.begin(), iv.end());
  double t = 0, cur_a = 0, cur_b = -1;
  for (const auto& x : iv) {
    if (x.first > cur_b) {
      if (cur_b > cur_a) t += cur_b - cur_a;
      cur_a = x.first;
      cur_b = x.second;
    } else {
      cur_b = std::max(cur_b, x.second);
    }
  }
  if (cur_b > cur_a) t += cur_b - cur_a;
  *launches = (long long)g_prof.used;
  *flops = f;
  *ms = t;
  return cudaSuccess;
}

template <bool A_MN, bool B_MN>
static cudaError_t launch(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p,
                          cudaStream_t st) {
  static bool attr_set = false;
  auto kern = gemm_tcgen05_kernel<A_MN, B_MN>;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  if (!g_num_sms) {
    int dev; cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  gemm_log(p, A_MN, B_MN, "cta1");
  int tiles = ((p.M + BM - 1) / BM) * ((p.N + BN - 1) / BN);
  const int sms = g_num_sms;
  int grid = tiles < sms ? tiles : sms;
  if (g_prof.on) {
    if (g_prof.used == g_prof.ev.size()) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      g_prof.ev.push_back({a, b});
    }
    cudaEventRecord(g_prof.ev[g_prof.used].first, st);
    kern<<<grid, GEMM_THREADS, GEMM_SMEM, st>>>(ta, tb, p);
    count_launch();
    cudaEventRecord(g_prof.ev[g_prof.used].second, st);
    g_prof.flops.push_back(2.0 * p.M * (double)p.N * p.K);
    g_prof.used++;
    return cudaGetLastError();
  }
  kern<<<grid, GEMM_THREADS, GEMM_SMEM, st>>>(ta, tb, p); count_launch();
  return cudaGetLastError();
}

static int g_variant = 0;  // 0 auto, 1 single-CTA, 2 CTA pair (TMA epilogue), 3 CTA pair (direct stores)
static int g_tma_epi = 1;
void gemm_set_variant(int v) {
  g_variant = v == 3 ? 2 : v;
  g_tma_epi = v == 3 ? 0 : 1;
}

template <bool A_MN, bool B_MN, int ST, int GLU = 0>
static cudaError_t launch2(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tb2, const CUtensorMap& tc,
                           const TmapSet& td, const GemmParams& p, cudaStream_t st) {
  static bool attr_set = false;
  auto kern = gemm_tcgen05_2sm_kernel<A_MN, B_MN, ST, GLU>;
  constexpr int SMEM2 = gemm2_smem(ST, GLU);
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM2);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  if (!g_num_sms) {
    int dev; cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  gemm_log(p, A_MN, B_MN, "cta2");
  const int tiles_n = p.glu == 1 ? ((p.N >> 1) + BN2 / 2 - 1) / (BN2 / 2) : (p.N + BN2 - 1) / BN2;
  const int tiles = ((p.M + 2 * BM2 - 1) / (2 * BM2)) * tiles_n;
  const int sms = g_num_sms;
  const int clusters = tiles < sms / 2 ? tiles : sms / 2;
  const int grid = 2 * (clusters > 0 ? clusters : 1);
  const bool prof = g_prof.on;
  if (prof) {
    if (g_prof.used == g_prof.ev.size()) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      g_prof.ev.push_back({a, b});
    }
    cudaEventRecord(g_prof.ev[g_prof.used].first, st);
  }
  kern<<<grid, GEMM_THREADS, SMEM2, st>>>(ta, tb, tb2, tc, td, p); count_launch();
  if (prof) {
    cudaEventRecord(g_prof.ev[g_prof.used].second, st);
    g_prof.flops.push_back(2.0 * p.M * (double)p.N * p.K);
    g_prof.used++;
  }
  return cudaGetLastError();
}

cudaError_t gemm_bf16(const GemmDesc& g, cudaStream_t st) {
  if (g.glu_done) *g.glu_done = false;
  if (g.f32) return (g.res || g.glu) ? cudaErrorInvalidValue : gemm_f32(g, st);
  if (g.M <= 0 || g.N <= 0 || g.K <= 0) return cudaErrorInvalidValue;
  cudaError_t e = get_encoder();
  if (e != cudaSuccess) return e;
  if ((g.lda % 8) || (g.ldb % 8) || (g.ldc % 4) ||
      (reinterpret_cast<uintptr_t>(g.A) & 15) || (reinterpret_cast<uintptr_t>(g.B) & 15))
    return cudaErrorInvalidValue;
  if (g.n_dst < 0 || g.n_dst > 4 || (g.n_dst > 0 && (g.rows_per_dst <= 0 || g.n_dst * g.rows_per_dst != g.M ||
                                                     g.mode == GEMM_ACCUM_F32 || g.rope_cs)))
    return cudaErrorInvalidValue;
  if (g.res && (g.mode != GEMM_STORE_BF16 || g.n_dst || g.rope_cs || g.glu || (g.ldr % 8) || (g.N % 8) ||
                (reinterpret_cast<uintptr_t>(g.res) & 15)))
    return cudaErrorInvalidValue;
  if (g.glu < 0 || g.glu > 2 || (g.glu && (g.mode != GEMM_STORE_BF16 || g.n_dst || g.rope_cs || g.b_mn || !g.aux)))
    return cudaErrorInvalidValue;
  if (g.glu == 1 && (g.N % 32)) return cudaErrorInvalidValue;  // F = N / 2, F % 16 == 0
  if (g.glu == 2 && ((g.N % 16) || !g.aux_in || (reinterpret_cast<uintptr_t>(g.aux_in) & 15))) return cudaErrorInvalidValue;
  const int esz = g.mode == GEMM_STORE_BF16 ? 2 : 4;
  int vec_ok = (g.ldc * esz) % 16 == 0;
  if (g.n_dst)
    for (int d = 0; d < g.n_dst; ++d) vec_ok &= (reinterpret_cast<uintptr_t>(g.dst[d]) & 15) == 0;
  else
    vec_ok &= (reinterpret_cast<uintptr_t>(g.C) & 15) == 0;
  GemmParams p{g.M, g.N, g.K, g.C, g.ldc, g.mode, vec_ok, 0, nullptr, 0, 0, g.n_dst, g.rows_per_dst,
               {g.dst[0], g.dst[1], g.dst[2], g.dst[3]}, g.res, g.ldr, 0, nullptr, 0, 0};
  const bool pair = g_variant == 2 || (g_variant == 0 && g.M >= 256);
  if (pair) {
    CUtensorMap ta, tb, tb2;
    memset(&tb2, 0, sizeof(tb2));
    bool ok = g.a_mn ? make_map(&ta, g.A, g.M, g.K, g.lda, 64) : make_map(&ta, g.A, g.K, g.M, g.lda, BM2);
    ok = ok && (g.b_mn ? make_map(&tb, g.B, g.N, g.K, g.ldb, 64) : make_map(&tb, g.B, g.K, g.N, g.ldb, BN2 / 2));
    if (!ok) return cudaErrorInvalidValue;
    CUtensorMap tc;
    TmapSet td;
    memset(&tc, 0, sizeof(tc));
    memset(&td, 0, sizeof(td));
    int tma_epi = vec_ok && g_tma_epi;
    if (tma_epi && g.n_dst) {  // one C map per destination; 32-row boxes must not straddle two
      tma_epi = g.rows_per_dst % 32 == 0;
      for (int d = 0; d < g.n_dst && tma_epi; ++d)
        tma_epi = make_map_c(&td.m[d], g.dst[d], g.N, g.rows_per_dst, g.ldc, g.mode != GEMM_STORE_BF16);
    } else if (tma_epi) {
      tma_epi = make_map_c(&tc, g.C, g.N, g.M, g.ldc, g.mode != GEMM_STORE_BF16);
    }
    // fused SwiGLU (TMA epilogue only): per-half B maps (glu 1) and per-half output maps, each F
    // columns wide so that TMA clips a ragged F at the half's own edge
    if (tma_epi && g.glu == 1) {
      const int F = g.N / 2;
      const char* B = static_cast<const char*>(g.B);
      bool gok = make_map(&tb, B, g.K, F, g.ldb, BN2 / 2) &&
                 make_map(&tb2, B + (size_t)F * g.ldb * 2, g.K, F, g.ldb, BN2 / 2) &&
                 make_map_c(&tc, g.C, F, g.M, g.ldc, false) &&
                 make_map_c(&td.m[0], static_cast<char*>(g.C) + (size_t)F * 2, F, g.M, g.ldc, false) &&
                 make_map_c(&td.m[1], g.aux, F, g.M, F, false) && (reinterpret_cast<uintptr_t>(g.aux) & 15) == 0;
      if (!gok) {  // plain GEMM (the caller runs the standalone SwiGLU)
        make_map(&tb, g.B, g.K, g.N, g.ldb, BN2 / 2);
        make_map_c(&tc, g.C, g.N, g.M, g.ldc, false);
      } else {
        p.glu = 1;
      }
    } else if (tma_epi && g.glu == 2) {
      const int F = g.N;
      char* gin = static_cast<char*>(const_cast<void*>(g.aux_in));
      bool gok = make_map_c(&td.m[0], g.aux, F, g.M, 2LL * F, false) &&
                 make_map_c(&td.m[1], static_cast<char*>(g.aux) + (size_t)F * 2, F, g.M, 2LL * F, false) &&
                 make_map_c(&td.m[2], gin, F, g.M, 2LL * F, false) &&
                 make_map_c(&td.m[3], gin + (size_t)F * 2, F, g.M, 2LL * F, false) &&
                 (reinterpret_cast<uintptr_t>(g.aux) & 15) == 0;
      if (gok) {
        p.glu = 2;
        p.aux_in = g.aux_in;
        p.ld_aux_in = 2LL * F;
        static const int dbg = getenv("MALLEUS_GLU2_DBG") ? atoi(getenv("MALLEUS_GLU2_DBG")) : 0;
        p.dbg = dbg;
      }
    } else if (tma_epi && g.res) {  // residual staged by TMA (EPI 3); the direct epilogues read it per row
      if (make_map_c(&td.m[0], const_cast<void*>(g.res), g.N, g.M, g.ldr, false)) p.glu = 3;
    }
    if (g.glu_done) *g.glu_done = p.glu == 1 || p.glu == 2;
    const bool rope = tma_epi && g.rope_cs && g.mode == GEMM_STORE_BF16 && g.rope_cols % 128 == 0;
    if (g.rope_done) *g.rope_done = rope;
    p.tma_epi = tma_epi;
    p.rope_cs = rope ? g.rope_cs : nullptr;
    p.rope_cols = g.rope_cols;
    p.rope_s = g.rope_s;
    if (p.glu == 1) return launch2<false, false, STAGES2, 1>(ta, tb, tb2, tc, td, p, st);
    if (p.glu == 2) {
      if (g.a_mn) return launch2<true, false, 5, 2>(ta, tb, tb2, tc, td, p, st);
      return launch2<false, false, 5, 2>(ta, tb, tb2, tc, td, p, st);
    }
    if (p.glu == 3) {
      if (!g.a_mn && g.b_mn) return launch2<false, true, STAGES2, 3>(ta, tb, tb2, tc, td, p, st);
      if (!g.a_mn && !g.b_mn) return launch2<false, false, STAGES2, 3>(ta, tb, tb2, tc, td, p, st);
      if (g.a_mn && g.b_mn) return launch2<true, true, STAGES2, 3>(ta, tb, tb2, tc, td, p, st);
      return launch2<true, false, STAGES2, 3>(ta, tb, tb2, tc, td, p, st);
    }
    if (g.co_resident) {  // 5-stage ring: ~32 KB of smem per SM left for a concurrent kernel
      if (!g.a_mn && !g.b_mn) return launch2<false, false, 5>(ta, tb, tb2, tc, td, p, st);
      if (!g.a_mn && g.b_mn) return launch2<false, true, 5>(ta, tb, tb2, tc, td, p, st);
      if (g.a_mn && g.b_mn) return launch2<true, true, 5>(ta, tb, tb2, tc, td, p, st);
      return launch2<true, false, 5>(ta, tb, tb2, tc, td, p, st);
    }
    if (!g.a_mn && !g.b_mn) return launch2<false, false, STAGES2>(ta, tb, tb2, tc, td, p, st);
    if (!g.a_mn && g.b_mn) return launch2<false, true, STAGES2>(ta, tb, tb2, tc, td, p, st);
    if (g.a_mn && g.b_mn) return launch2<true, true, STAGES2>(ta, tb, tb2, tc, td, p, st);
    return launch2<true, false, STAGES2>(ta, tb, tb2, tc, td, p, st);
  }
  CUtensorMap ta, tb;
  bool ok = g.a_mn ? make_map(&ta, g.A, g.M, g.K, g.lda, 64) : make_map(&ta, g.A, g.K, g.M, g.lda, BM);
  ok = ok && (g.b_mn ? make_map(&tb, g.B, g.N, g.K, g.ldb, 64) : make_map(&tb, g.B, g.K, g.N, g.ldb, BN));
  if (!ok) return cudaErrorInvalidValue;
  if (g.rope_done) *g.rope_done = false;
  if (!g.a_mn && !g.b_mn) return launch<false, false>(ta, tb, p, st);
  if (!g.a_mn && g.b_mn) return launch<false, true>(ta, tb, p, st);
  if (g.a_mn && g.b_mn) return launch<true, true>(ta, tb, p, st);
  return launch<true, false>(ta, tb, p, st);
}

}  // namespace mls
