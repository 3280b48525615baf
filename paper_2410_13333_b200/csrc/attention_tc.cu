// Causal attention forward on the 5th-gen tensor cores (tcgen05 / TMEM / TMA) for head_dim 128
// and sequence lengths that are multiples of 128 (PAPER.md:780 FlashAttention).
//
// One CTA = 128 queries of one (sequence, query head); GQA: K / V of the head's KV group.  Warp roles:
//   warp 0      TMA producer: Q once; K and V tiles of 128 keys through separate 3-stage rings
//               (K_i is released when S_i is done, a full tile before V_i, so its reload is hidden);
//   warp 1      MMA issuer (one thread) + TMEM owner: S_i = Q K_i^T into one of two TMEM S buffers,
//               then O += P_{i-1} V_{i-1} once the softmax warps have written P_{i-1};
//   warps 2..9  softmax (two warps per query row, 64 keys each): S row from TMEM, online max with lazy
//               rescaling (O in TMEM is rescaled only when the running max grows by > 2^8, FA4
//               style; exact since numerator and denominator share the stale max), P (bf16) written
//               over the row's own S columns in TMEM; final O / l, LSE.
// Both A operands come from TMEM ("ts" MMAs: Q copied once by the softmax warps, P in place), so the
// only shared-memory operand traffic is K and V: measured on the previous version (Q and P as smem
// operands) the tile loop was bound by shared-memory bandwidth (A + B of every MMA, P stores, TMA).
// TMEM: S0 cols [0,128), S1 [128,256), O [256,384), row-max exchange [384,388), Q [448,512).
// smem: Q 32 KB (TMA landing), 3 x K 32 KB, 3 x V 32 KB.
// Output identical in layout to attention.cu: o [T, n*d] bf16, lse [nb, n, s] (natural log).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdlib>
#include "kernels.h"
#include "ptx.cuh"

namespace mls {
namespace {

constexpr int TQ = 128, TK = 128, DH = 128;
constexpr int PANEL = 128 * 64 * 2;            // one 128-row x 64-col bf16 swizzled panel (16 KB)
constexpr int Q_BYTES = 2 * PANEL;             // 32 KB
constexpr int K_BYTES = 2 * PANEL;             // one K (or V) tile of 128 keys
constexpr float LOG2E = 1.4426950408889634f;

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// MUFU exp2 without the non-ftz fix-up sequence (inputs are <= 0 after max subtraction; ex2(-inf) = 0)
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x for x <= 0 on the FMA pipe (FA4's trick to offload the MUFU unit, 16 ex2 / clk / SM, i.e.
// 1024 cycles per 128 x 128 tile; off by default: measured slower here, see the launcher).
// Round-to-nearest split x = j + f with the 1.5 * 2^23 magic constant, near-minimax cubic for 2^f
// on [-0.5, 0.5] (max rel. error 7.5e-5, far below bf16's 2^-9), exponent added in the integer
// domain; x < -126 (incl. -inf) gives 0.
__device__ __forceinline__ float ex2_poly(float x) {
  const float xc = fmaxf(x, -127.f);
  const float t = xc + 12582912.f;
  const float f = xc - (t - 12582912.f);
  const float p = fmaf(fmaf(fmaf(0.05517147f, f, 0.24261111f), f, 0.693261f), f, 0.99992806f);
  const float r = __int_as_float(__float_as_int(p) + ((__float_as_int(t) - 0x4B400000) << 23));
  return x < -126.f ? 0.f : r;
}

constexpr int FWD_STAGES = 3;
constexpr int SMEM_FWD = Q_BYTES + 2 * FWD_STAGES * K_BYTES + 1024 + 1024;

// NPOLY of every 8 consecutive P elements take ex2_poly, the rest the MUFU ex2
template <int NPOLY>
__global__ void __launch_bounds__(320, 1)
attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tm, int s, int n, int n_kv, __nv_bfloat16* __restrict__ o,
                   float* __restrict__ lse, float scale, unsigned long long* __restrict__ trace, int order) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + Q_BYTES;                  // [FWD_STAGES] K tiles
  uint8_t* sV = sK + FWD_STAGES * K_BYTES;     // [FWD_STAGES] V tiles
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + FWD_STAGES * K_BYTES);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;                 // [3]
  uint64_t* k_empty = bars + 4;                // [3] K_i free once S_i = Q K_i^T is done
  uint64_t* v_full = bars + 7;                 // [3]
  uint64_t* v_empty = bars + 10;               // [3] V_j free once O += P_j V_j is done
  uint64_t* s_full = bars + 13;                // [2]
  uint64_t* s_empty = bars + 15;               // [2]
  uint64_t* p_full = bars + 17;                // [2] P_j (in S_j's TMEM columns) written
  uint64_t* o_done = bars + 19;                // [2] (PV of tile j completes on o_done[j & 1])
  uint64_t* q_tmem = bars + 21;                // Q copied into TMEM by the softmax warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 22);
  constexpr uint32_t COL_O = 256, COL_X = 384, COL_Q = 448;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = s / TQ;
  // grid (heads, query blocks, sequences): CTAs are dispatched x-fastest, so every head's heaviest
  // query block goes first and the last wave holds the lightest (longest-processing-time-first order)
  // (order = 1: the previous head-major grid (query blocks, heads, sequences), MALLEUS_ATTN_GRID_HEADMAJOR=1)
  const int qb = nqb - 1 - (order ? blockIdx.x : blockIdx.y);
  const int head = order ? blockIdx.y : blockIdx.x, b = blockIdx.z;
  const int n_tiles = qb + 1;           // causal: key tiles 0..qb
  const int row0 = b * s + qb * TQ;     // first query row in qkv
  const int nd = n * DH;
  // qkv = q (n heads) | k (n_kv heads) | v (n_kv heads); GQA: this query head reads KV head head / g
  const int kcol = nd + (head / (n / n_kv)) * DH, vcol = nd + n_kv * DH + (head / (n / n_kv)) * DH;
  // debugging aid (MALLEUS_ATTN_TRACE): globaltimer stamps of CTAs (0, 0..1, 0), [event][tile]
  unsigned long long* tr = (trace && blockIdx.y == 0 && blockIdx.x < 2 && blockIdx.z == 0)
                               ? trace + blockIdx.x * 8 * 64 : nullptr;
  auto stamp = [&](int ev, int i) {
    if (tr && i < 64) { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); tr[ev * 64 + i] = t; }
  };
  if (threadIdx.x == 0) stamp(7, 0);

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm);
    mbar_init(q_full, 1);
    for (int i = 0; i < FWD_STAGES; ++i) {
      mbar_init(&k_full[i], 1); mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1); mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1); mbar_init(&s_empty[i], 8);
      mbar_init(&p_full[i], 8); mbar_init(&o_done[i], 1);
    }
    mbar_init(q_tmem, 8);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, Q_BYTES);
      tma_load_2d(sQ, &tm, q_full, head * DH, row0);
      tma_load_2d(sQ + PANEL, &tm, q_full, head * DH + 64, row0);
      // K runs one tile ahead of V in this thread's program order: K_{i+1} is requested as soon as
      // its slot frees (S_{i+1-3} done) instead of queueing behind V_i (measured: that ordering put
      // the load latency on the critical path of every tile)
      auto load_k = [&](int i) {
        const int st = i % FWD_STAGES;
        uint8_t* k = sK + st * K_BYTES;
        mbar_wait(&k_empty[st], ((i / FWD_STAGES) & 1) ^ 1);
        stamp(0, i);
        mbar_arrive_expect_tx(&k_full[st], K_BYTES);
        tma_load_2d(k, &tm, &k_full[st], kcol, b * s + i * TK);
        tma_load_2d(k + PANEL, &tm, &k_full[st], kcol + 64, b * s + i * TK);
      };
      auto load_v = [&](int i) {
        const int st = i % FWD_STAGES;
        uint8_t* v = sV + st * K_BYTES;
        mbar_wait(&v_empty[st], ((i / FWD_STAGES) & 1) ^ 1);
        stamp(1, i);
        mbar_arrive_expect_tx(&v_full[st], K_BYTES);
        tma_load_2d(v, &tm, &v_full[st], vcol, b * s + i * TK);
        tma_load_2d(v + PANEL, &tm, &v_full[st], vcol + 64, b * s + i * TK);
      };
      load_k(0);
      for (int i = 0; i < n_tiles; ++i) {
        if (i + 1 < n_tiles) load_k(i + 1);
        load_v(i);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id_qk = umma_idesc_bf16(128, 128, false, false);
      constexpr uint32_t id_pv = umma_idesc_bf16(128, 128, false, true);
      auto issue_pv = [&](int j) {  // O += P_j V_j, P_j from TMEM (S_j's columns)
        const int st = j % FWD_STAGES;
        mbar_wait(&v_full[st], (j / FWD_STAGES) & 1);
        mbar_wait(&p_full[j & 1], (j >> 1) & 1);
        stamp(3, j);
        tc_fence_after();
        const uint32_t v = smem_u32(sV + st * K_BYTES);
#pragma unroll
        for (int kk = 0; kk < TK / 16; ++kk)
          umma_f16_ts(tbase + COL_O, tbase + 128 * (j & 1) + (kk >> 2) * 64 + (kk & 3) * 8,
                      umma_desc_sw128(v + kk * 2048, PANEL, 1024), id_pv, (j > 0 || kk > 0) ? 1u : 0u);
        umma_commit(&o_done[j & 1]);
        umma_commit(&v_empty[st]);
      };
      mbar_wait(q_tmem, 0);
      for (int i = 0; i < n_tiles; ++i) {
        const int st = i % FWD_STAGES, sb = i & 1;
        mbar_wait(&k_full[st], (i / FWD_STAGES) & 1);
        mbar_wait(&s_empty[sb], ((i >> 1) & 1) ^ 1);
        stamp(2, i);
        tc_fence_after();
        const uint32_t k = smem_u32(sK + st * K_BYTES);
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk)  // S_i = Q K_i^T, Q from TMEM
          umma_f16_ts(tbase + 128 * sb, tbase + COL_Q + kk * 8,
                      umma_desc_sw128(k + (kk >> 2) * PANEL + (kk & 3) * 32, 16, 1024), id_qk, kk > 0 ? 1u : 0u);
        umma_commit(&s_full[sb]);
        umma_commit(&k_empty[st]);
        if (i > 0) issue_pv(i - 1);
      }
      issue_pv(n_tiles - 1);
    }
  } else {
    // ---------------- softmax: 8 warps, two per TMEM lane quarter; thread = half a query row
    // (64 of the 128 keys of a tile).  The pair exchanges its partial row maxima through spare TMEM
    // columns and a named barrier; each half writes its 64 P values (bf16) over its own S columns
    // and owns half of the O columns for rescaling and the epilogue.
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    const int r = quarter * 32 + lane;            // row within the 128-query block
    const int q = qb * TQ + r;                    // query position in the sequence
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const float sl2 = scale * LOG2E;
    float m_used = -INFINITY, l = 0.f;
    {  // Q row -> TMEM (A operand of S = Q K^T): this half's 64 dims = 32 packed columns
      mbar_wait(q_full, 0);
      const uint8_t* qrow = sQ + half * PANEL + r * 128;
      uint32_t u[32];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint4 w = *reinterpret_cast<const uint4*>(qrow + ((c ^ (r & 7)) << 4));
        u[4 * c] = w.x; u[4 * c + 1] = w.y; u[4 * c + 2] = w.z; u[4 * c + 3] = w.w;
      }
      tmem_st32(tbase + lane_off + COL_Q + 32 * half, u);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(q_tmem);
    }
    auto pair_sync = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(1 + quarter) : "memory"); };
    // the pair exchanges its partial row statistics through spare TMEM columns (measured: an smem
    // exchange through the free Q landing buffer made the forward slower, 65.8 -> 70.0 us at C2)
    auto exchange = [&](float mine, int slot) -> float {  // returns the partner's value
      uint32_t v = __float_as_uint(mine);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tbase + lane_off + COL_X + slot * 2 + half),
                   "r"(v) : "memory");
      tmem_wait_st();
      tc_fence_before();
      pair_sync();
      tc_fence_after();
      uint32_t o;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(o)
                   : "r"(tbase + lane_off + COL_X + slot * 2 + (half ^ 1)) : "memory");
      tmem_wait_ld();
      return __uint_as_float(o);
    };
    for (int i = 0; i < n_tiles; ++i) {
      const int sb = i & 1;
      mbar_wait(&s_full[sb], (i >> 1) & 1);
      if (warp == 2 && lane == 0) stamp(4, i);
      tc_fence_after();
      const uint32_t cs = tbase + lane_off + 128 * sb + half * 64;
      float sv[TK / 2];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t u[32];
        tmem_ld32(cs + c * 32, u);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) sv[c * 32 + j] = __uint_as_float(u[j]);  // raw S; scaled in the exp FFMA
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[sb]);
      float mt = -INFINITY;
      if (i == n_tiles - 1) {  // diagonal tile: keys > query masked
#pragma unroll
        for (int j = 0; j < TK / 2; ++j)
          if (i * TK + half * 64 + j > q) sv[j] = -INFINITY;
      }
#pragma unroll
      for (int j = 0; j < TK / 2; ++j) mt = fmaxf(mt, sv[j]);
      mt = fmaxf(mt, exchange(mt, i & 1)) * sl2;  // full-row max of this tile, log2 units (sl2 > 0)
      if (warp == 2 && lane == 0) stamp(5, i);
      // tcgen05.ld / st are warp-collective: the rescale decision is warp-uniform (and identical
      // in both warps of the pair: same rows, same maxima); lanes whose max did not grow scale by 1
      if (__any_sync(0xffffffffu, mt > m_used + 8.f)) {
        const float m_new = fmaxf(m_used, mt);
        if (i > 0) {
          mbar_wait(&o_done[(i - 1) & 1], ((i - 1) >> 1) & 1);  // O stable: PV_{i-1} done
          tc_fence_after();
          const float f = ex2(m_used - m_new);
          l *= f;
#pragma unroll 1
          for (int c = 0; c < 2; ++c) {
            uint32_t u[32];
            tmem_ld32(tbase + lane_off + COL_O + half * 64 + c * 32, u);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j) u[j] = __float_as_uint(__uint_as_float(u[j]) * f);
            tmem_st32(tbase + lane_off + COL_O + half * 64 + c * 32, u);
          }
          tmem_wait_st();
        }
        m_used = m_new;
      }
      // P = exp2(s - m_used) -> bf16 pairs over this half's own S columns (A operand of PV; the
      // MMA that overwrites them, S_{i+2}, is issued after O += P_i V_i)
      uint32_t pk[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int e0 = (2 * j) & 7, e1 = (2 * j + 1) & 7;  // position within each group of 8
        const float x0 = fmaf(sv[2 * j], sl2, -m_used), x1 = fmaf(sv[2 * j + 1], sl2, -m_used);
        const float p0 = ((e0 * NPOLY) % 8 < NPOLY && NPOLY > 0) ? ex2_poly(x0) : ex2(x0);
        const float p1 = ((e1 * NPOLY) % 8 < NPOLY && NPOLY > 0) ? ex2_poly(x1) : ex2(x1);
        l += p0 + p1;
        pk[j] = pack_bf16(p0, p1);
      }
      tmem_st32(cs, pk);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[sb]);
      if (warp == 2 && lane == 0) stamp(6, i);
    }
    // epilogue: O / l (MMAs complete in issue order: the last PV implies all)
    mbar_wait(&o_done[(n_tiles - 1) & 1], ((n_tiles - 1) >> 1) & 1);
    if (warp == 2 && lane == 0) stamp(7, 1);
    tc_fence_after();
    l += exchange(l, n_tiles & 1);  // the slot the last tile did not use
    const float inv = 1.f / l;
    __nv_bfloat16* orow = o + (long long)(b * s + q) * nd + head * DH + half * 64;
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      uint32_t u[32];
      tmem_ld32(tbase + lane_off + COL_O + half * 64 + c * 32, u);
      tmem_wait_ld();
      uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        uint4 w;
        w.x = pack_bf16(__uint_as_float(u[8 * v + 0]) * inv, __uint_as_float(u[8 * v + 1]) * inv);
        w.y = pack_bf16(__uint_as_float(u[8 * v + 2]) * inv, __uint_as_float(u[8 * v + 3]) * inv);
        w.z = pack_bf16(__uint_as_float(u[8 * v + 4]) * inv, __uint_as_float(u[8 * v + 5]) * inv);
        w.w = pack_bf16(__uint_as_float(u[8 * v + 6]) * inv, __uint_as_float(u[8 * v + 7]) * inv);
        dst[v] = w;
      }
    }
    if (half == 0) lse[((long long)b * n + head) * s + q] = (m_used + log2f(l)) / LOG2E;
    if (warp == 2 && lane == 0) stamp(7, 2);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
}

// ------------------------------------------------------------------ backward (tcgen05)
// 1-D bulk copy global -> shared completing on an mbarrier (lse / D rows of a query tile)
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// The (cos, sin) pairs of one 32-column chunk of this thread's row, loaded before the accumulator is
// final so their latency overlaps the last MMAs (the epilogue then only waits for TMEM).
__device__ __forceinline__ void load_cs32(const float2* cs_row, int c, float2 (&cs)[32]) {
  const float4* p = reinterpret_cast<const float4*>(cs_row + c * 32);
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const float4 v = __ldg(p + q);
    cs[2 * q] = make_float2(v.x, v.y);
    cs[2 * q + 1] = make_float2(v.z, v.w);
  }
}
// store_row_rope for the single chunk c with preloaded (cos, sin) (rope = false: no rotation)
__device__ __forceinline__ void store_row_rope_pre(__nv_bfloat16* dst, uint32_t taddr, float scale, bool rope,
                                                   const float2 (&cs)[32], int c) {
  uint32_t ua[32], ub[32];
  tmem_ld32(taddr + c * 32, ua);
  tmem_ld32(taddr + 64 + c * 32, ub);
  tmem_wait_ld();
  float a[32], bb[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    float x = __uint_as_float(ua[j]) * scale, y = __uint_as_float(ub[j]) * scale;
    if (rope) {
      const float x2 = x * cs[j].x + y * cs[j].y;
      y = y * cs[j].x - x * cs[j].y;
      x = x2;
    }
    a[j] = x;
    bb[j] = y;
  }
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    uint4 wa, wb;
    wa.x = pack_bf16(a[8 * v], a[8 * v + 1]); wa.y = pack_bf16(a[8 * v + 2], a[8 * v + 3]);
    wa.z = pack_bf16(a[8 * v + 4], a[8 * v + 5]); wa.w = pack_bf16(a[8 * v + 6], a[8 * v + 7]);
    wb.x = pack_bf16(bb[8 * v], bb[8 * v + 1]); wb.y = pack_bf16(bb[8 * v + 2], bb[8 * v + 3]);
    wb.z = pack_bf16(bb[8 * v + 4], bb[8 * v + 5]); wb.w = pack_bf16(bb[8 * v + 6], bb[8 * v + 7]);
    reinterpret_cast<uint4*>(dst + c * 32)[v] = wa;
    reinterpret_cast<uint4*>(dst + 64 + c * 32)[v] = wb;
  }
}

// ---- backward: 64-wide sub-tiles, P^T / dS^T (and dS) kept in TMEM as the A operand of the second
// pair of MMAs ("ts" form), S / dP double-buffered in TMEM, 3-stage TMA rings.  Measured on the
// 128-wide version: shared-memory bandwidth (A and B of every MMA plus P / dS round trips through
// smem) and exposed TMA latency (single-buffered Q / dO) bounded the loop; here the only smem
// operands are the TMA-loaded tiles and every load has two sub-tiles of slack.
constexpr int HPANEL = 64 * 128;          // 64 rows x 128 B (one 64-column half of a 64-row tile)
constexpr int SUB_STAGE = 4 * HPANEL;     // two 64-row x 128-col bf16 tiles (Q | dO or K | V)
constexpr int NSUB1 = 4;                  // Q | dO ring depth (dK / dV kernel)
// measured (tools/attn_trace.py): a 32 KB TMA sub-tile load takes ~1.4 us under full load, so the ring
// must cover load latency + MMA + compute: with 3 stages the loop ran at (that chain) / 3 per sub-tile

// dK / dV: CTA = 128 keys of one (sequence, KV head); loop over the 64-query sub-tiles j >= 2 kb of
// each query head that reads this KV head (MHA: one; GQA: the g heads of the group, one after another,
// all accumulating into the same dK / dV in TMEM — the group sum of the GQA backward).
//   TMEM: S^T[b] cols [64b, 64b+64), dP^T[b] [128+64b, ..), dV [256,384), dK [384,512); warp half h
//   overwrites its own 32 S^T / dP^T columns with 16 columns of packed bf16 P^T / dS^T at 32h.
//   S^T = K Q_j^T and dP^T = V dO_j^T (M = 128 keys, N = 64 queries, A = K / V from smem);
//   dV += P^T dO_j and dK += dS^T Q_j (A from TMEM, K = 64 queries; Q_j / dO_j MN-major B).
constexpr int BWD1_SMEM = 2 * 2 * PANEL + NSUB1 * SUB_STAGE + NSUB1 * 512 + 256 + 1024;

__global__ void __launch_bounds__(320, 1)
attn_bwd_dkv_tc_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tm64,
                       const __grid_constant__ CUtensorMap tmo64, int s, int n, int n_kv, const float* __restrict__ lse,
                       const float* __restrict__ dsum, __nv_bfloat16* __restrict__ dqkv, float scale,
                       const float2* __restrict__ rope_cs, unsigned long long* __restrict__ trace, int order) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // debugging aid (MALLEUS_ATTN_TRACE): stamps of CTAs (0, 0..1, 0), [event][iteration]
  unsigned long long* tr = (trace && blockIdx.y == 0 && blockIdx.x < 2 && blockIdx.z == 0)
                               ? trace + blockIdx.x * 16 * 64 : nullptr;
  auto stamp = [&](int ev, int i) {
    if (tr && i < 64) { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); tr[ev * 64 + i] = t; }
  };
  if (threadIdx.x == 0) stamp(7, 0);
  uint8_t* sK = smem;
  uint8_t* sV = sK + 2 * PANEL;
  uint8_t* ring = sV + 2 * PANEL;                                       // [NSUB1][Q | dO]
  float* sLD = reinterpret_cast<float*>(ring + NSUB1 * SUB_STAGE);      // [NSUB1][lse 64 | D 64]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sLD + NSUB1 * 128);
  uint64_t* kv_full = bars;
  uint64_t* qd_full = bars + 1;            // [NSUB1]
  uint64_t* qd_empty = bars + 1 + NSUB1;   // [NSUB1]
  uint64_t* sd_full = bars + 1 + 2 * NSUB1;  // [2]
  uint64_t* pd_full = sd_full + 2;         // [2]
  uint64_t* done = pd_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // grid (KV heads, key blocks, sequences), dispatched x-fastest: kb = 0 (the most query sub-tiles) of
  // every KV head first, the lightest key blocks in the last wave
  const int kb = order ? blockIdx.x : blockIdx.y;
  const int kvh = order ? blockIdx.y : blockIdx.x, b = blockIdx.z;  // KV head (GQA: shared by the g query heads of its group)
  const int nd = n * DH, g = n / n_kv, ldq = nd + 2 * n_kv * DH;
  const int j0 = 2 * kb, n_sub = s / 64 - j0;  // query sub-tiles per query head
  const int n_it = g * n_sub;                   // iterations: the group's query heads one after another
  auto head_of = [&](int it) { return kvh * g + it / n_sub; };
  auto sub_of = [&](int it) { return j0 + it % n_sub; };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm);
    tma_prefetch(&tm64);
    tma_prefetch(&tmo64);
    mbar_init(kv_full, 1);
    for (int i = 0; i < NSUB1; ++i) { mbar_init(&qd_full[i], 1); mbar_init(&qd_empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&sd_full[i], 1); mbar_init(&pd_full[i], 8); }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const int krow = b * s + kb * TK;
      mbar_arrive_expect_tx(kv_full, 4 * PANEL);
      tma_load_2d(sK, &tm, kv_full, nd + kvh * DH, krow);
      tma_load_2d(sK + PANEL, &tm, kv_full, nd + kvh * DH + 64, krow);
      tma_load_2d(sV, &tm, kv_full, nd + (n_kv + kvh) * DH, krow);
      tma_load_2d(sV + PANEL, &tm, kv_full, nd + (n_kv + kvh) * DH + 64, krow);
      for (int it = 0; it < n_it; ++it) {
        const int st = it % NSUB1, j = sub_of(it), head = head_of(it);
        const long long lrow = ((long long)b * n + head) * s;
        mbar_wait(&qd_empty[st], ((it / NSUB1) & 1) ^ 1);
        stamp(0, it);
        uint8_t* q = ring + st * SUB_STAGE;
        const int qrow = b * s + j * 64;
        mbar_arrive_expect_tx(&qd_full[st], SUB_STAGE + 512);
        tma_load_2d(q, &tm64, &qd_full[st], head * DH, qrow);
        tma_load_2d(q + HPANEL, &tm64, &qd_full[st], head * DH + 64, qrow);
        tma_load_2d(q + 2 * HPANEL, &tmo64, &qd_full[st], head * DH, qrow);
        tma_load_2d(q + 3 * HPANEL, &tmo64, &qd_full[st], head * DH + 64, qrow);
        bulk_load(sLD + st * 128, lse + lrow + j * 64, 256, &qd_full[st]);
        bulk_load(sLD + st * 128 + 64, dsum + lrow + j * 64, 256, &qd_full[st]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id_s = umma_idesc_bf16(128, 64, false, false);
      constexpr uint32_t id_d = umma_idesc_bf16(128, 128, false, true);
      const uint32_t ak = smem_u32(sK), av = smem_u32(sV);
      auto issue_dvdk = [&](int i) {
        const int bb = i & 1, st = i % NSUB1;
        mbar_wait(&pd_full[bb], (i >> 1) & 1);
        stamp(3, i);
        tc_fence_after();
        const uint32_t q = smem_u32(ring + st * SUB_STAGE), o = q + 2 * HPANEL;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint32_t acol = bb * 64 + (kk >> 1) * 32 + (kk & 1) * 8;
          const uint32_t acc = (i > 0 || kk > 0) ? 1u : 0u;
          umma_f16_ts(tbase + 256, tbase + acol, umma_desc_sw128(o + kk * 2048, HPANEL, 1024), id_d, acc);
          umma_f16_ts(tbase + 384, tbase + 128 + acol, umma_desc_sw128(q + kk * 2048, HPANEL, 1024), id_d, acc);
        }
        umma_commit(&qd_empty[st]);
      };
      mbar_wait(kv_full, 0);
      for (int it = 0; it < n_it; ++it) {
        const int bb = it & 1, st = it % NSUB1;
        mbar_wait(&qd_full[st], (it / NSUB1) & 1);
        stamp(2, it);
        tc_fence_after();
        const uint32_t q = smem_u32(ring + st * SUB_STAGE), o = q + 2 * HPANEL;
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const uint32_t aoff = (kk >> 2) * PANEL + (kk & 3) * 32, boff = (kk >> 2) * HPANEL + (kk & 3) * 32;
          umma_f16(tbase + bb * 64, umma_desc_sw128(ak + aoff, 16, 1024), umma_desc_sw128(q + boff, 16, 1024), id_s,
                   kk > 0 ? 1u : 0u);
          umma_f16(tbase + 128 + bb * 64, umma_desc_sw128(av + aoff, 16, 1024), umma_desc_sw128(o + boff, 16, 1024),
                   id_s, kk > 0 ? 1u : 0u);
        }
        umma_commit(&sd_full[bb]);
        if (it > 0) issue_dvdk(it - 1);
      }
      issue_dvdk(n_it - 1);
      umma_commit(done);
    }
  } else {
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;   // this warp's 32 query columns of each sub-tile
    const int r = quarter * 32 + lane;  // key row within the tile
    const int key = kb * TK + r;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const float sl2 = scale * LOG2E;
    for (int it = 0; it < n_it; ++it) {
      const int bb = it & 1, st = it % NSUB1, j = sub_of(it);
      mbar_wait(&sd_full[bb], (it >> 1) & 1);
      if (warp == 2 && lane == 0) stamp(4, it);
      tc_fence_after();
      const uint32_t cs = tbase + lane_off + bb * 64 + half * 32;  // S^T columns; dP^T at +128
      uint32_t us[32], ud[32];
      tmem_ld32(cs, us);
      tmem_ld32(cs + 128, ud);
      // this warp's 32 (lse, D) pairs: broadcast 128-bit shared loads while the TMEM loads fly
      float Lv[32], Dv[32];
      {
        const float4* L4 = reinterpret_cast<const float4*>(sLD + st * 128 + half * 32);
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const float4 a = L4[t], d = L4[t + 16];
          Lv[4 * t] = a.x * LOG2E; Lv[4 * t + 1] = a.y * LOG2E; Lv[4 * t + 2] = a.z * LOG2E; Lv[4 * t + 3] = a.w * LOG2E;
          Dv[4 * t] = d.x; Dv[4 * t + 1] = d.y; Dv[4 * t + 2] = d.z; Dv[4 * t + 3] = d.w;
        }
      }
      tmem_wait_ld();
      if (warp == 2 && lane == 0) stamp(1, it);
      const bool diag = j * 64 + half * 32 < key + 32;  // some query column of this warp may precede the key
      uint32_t pp[16], dd[16];
#pragma unroll
      for (int t = 0; t < 32; t += 2) {
        float p0 = ex2(fmaf(__uint_as_float(us[t]), sl2, -Lv[t]));
        float p1 = ex2(fmaf(__uint_as_float(us[t + 1]), sl2, -Lv[t + 1]));
        if (diag) {
          const int qi = j * 64 + half * 32 + t;
          if (key > qi) p0 = 0.f;
          if (key > qi + 1) p1 = 0.f;
        }
        pp[t / 2] = pack_bf16(p0, p1);
        dd[t / 2] = pack_bf16(p0 * (__uint_as_float(ud[t]) - Dv[t]), p1 * (__uint_as_float(ud[t + 1]) - Dv[t + 1]));
      }
      if (warp == 2 && lane == 0) stamp(5, it);
      tmem_st16(cs, pp);
      tmem_st16(cs + 128, dd);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&pd_full[bb]);
      if (warp == 2 && lane == 0) stamp(6, it);
      if (lane == 0) stamp(8 + warp - 2, it);  // every compute warp's finish
    }
    float2 csr[32];
    if (rope_cs) load_cs32(rope_cs + (long long)key * 64, half, csr);
    mbar_wait(done, 0);
    if (warp == 2 && lane == 0) stamp(7, 1);
    tc_fence_after();
    __nv_bfloat16* dk = dqkv + (long long)(b * s + key) * ldq + nd + kvh * DH;
    __nv_bfloat16* dv = dk + n_kv * DH;
    store_row_rope_pre(dk, tbase + lane_off + 384, scale, rope_cs != nullptr, csr, half);
    store_row_rope_pre(dv, tbase + lane_off + 256, 1.f, false, csr, half);
    if (warp == 2 && lane == 0) stamp(7, 2);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
}

// dQ: CTA = 128 queries; loop over 128-key tiles i <= qb (2-stage K | V ring, 64 KB per stage).
//   TMEM: S[b] cols [128b, 128b+128) (double-buffered), dP [256,384), dQ [384,512).  Warp half h
//   overwrites its own 64 dP columns with 32 columns of packed bf16 dS, the A operand of
//   dQ += dS K_i (K = 128 keys, K_i MN-major B).  MMA order per tile: S_i (overlaps the softmax-
//   gradient math of tile i-1), then dQ_{i-1} (reads dS_{i-1}), then dP_i (overwrites it; the tensor
//   pipe runs in order).  All MMAs are N = 128 (full rate; N = 64 runs at 2/3, profiles/r01_mma_probe.log).
constexpr int KV2_STAGE = 4 * PANEL;  // K (2 panels of 128 rows) | V (2 panels)
constexpr int BWD2_SMEM = 2 * 2 * PANEL + 2 * KV2_STAGE + 256 + 1024;

__global__ void __launch_bounds__(320, 1)
attn_bwd_dq_tc_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tmo, int s, int n,
                      int n_kv,
                      const float* __restrict__ lse, const float* __restrict__ dsum, __nv_bfloat16* __restrict__ dqkv,
                      float scale, const float2* __restrict__ rope_cs, unsigned long long* __restrict__ trace,
                      int order) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  unsigned long long* tr = (trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) ? trace : nullptr;
  auto stamp = [&](int ev, int i) {
    if (tr && i < 64) { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); tr[ev * 64 + i] = t; }
  };
  if (threadIdx.x == 0) stamp(7, 0);
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sO = sQ + 2 * PANEL;
  uint8_t* ring = sO + 2 * PANEL;  // [2][K | V]
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + 2 * KV2_STAGE);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;   // [2]
  uint64_t* kv_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;    // [2]
  uint64_t* s_free = bars + 7;    // [2] (8 warp arrivals: S_i read into registers)
  uint64_t* dp_full = bars + 9;
  uint64_t* ds_full = bars + 10;  // 8 warp arrivals
  uint64_t* done = bars + 11;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = s / TQ;
  // grid (heads, query blocks, sequences): heaviest first overall (order = 1: head-major, as before)
  const int qb = nqb - 1 - (order ? blockIdx.x : blockIdx.y);
  const int head = order ? blockIdx.y : blockIdx.x, b = blockIdx.z;
  const int n_it = qb + 1;              // key tiles up to the diagonal
  const int nd = n * DH;
  const int row0 = b * s + qb * TQ;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm);
    tma_prefetch(&tmo);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1); mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1); mbar_init(&s_free[i], 8);
    }
    mbar_init(dp_full, 1);
    mbar_init(ds_full, 8);
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, 4 * PANEL);
      tma_load_2d(sQ, &tm, q_full, head * DH, row0);
      tma_load_2d(sQ + PANEL, &tm, q_full, head * DH + 64, row0);
      tma_load_2d(sO, &tmo, q_full, head * DH, row0);
      tma_load_2d(sO + PANEL, &tmo, q_full, head * DH + 64, row0);
      for (int i = 0; i < n_it; ++i) {
        const int st = i & 1;
        mbar_wait(&kv_empty[st], ((i >> 1) & 1) ^ 1);
        stamp(0, i);
        uint8_t* k = ring + st * KV2_STAGE;
        const int krow = b * s + i * TK;
        mbar_arrive_expect_tx(&kv_full[st], KV2_STAGE);
        const int kvh = head / (n / n_kv);  // GQA: the group's KV head
        tma_load_2d(k, &tm, &kv_full[st], nd + kvh * DH, krow);
        tma_load_2d(k + PANEL, &tm, &kv_full[st], nd + kvh * DH + 64, krow);
        tma_load_2d(k + 2 * PANEL, &tm, &kv_full[st], nd + (n_kv + kvh) * DH, krow);
        tma_load_2d(k + 3 * PANEL, &tm, &kv_full[st], nd + (n_kv + kvh) * DH + 64, krow);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id_s = umma_idesc_bf16(128, 128, false, false);
      constexpr uint32_t id_q = umma_idesc_bf16(128, 128, false, true);
      const uint32_t aq = smem_u32(sQ), ao = smem_u32(sO);
      auto issue_dq = [&](int i) {  // dQ += dS_i K_i
        mbar_wait(ds_full, i & 1);
        stamp(3, i);
        tc_fence_after();
        const uint32_t k = smem_u32(ring + (i & 1) * KV2_STAGE);
#pragma unroll
        for (int kk = 0; kk < TK / 16; ++kk)
          umma_f16_ts(tbase + 384, tbase + 256 + (kk >> 2) * 64 + (kk & 3) * 8,
                      umma_desc_sw128(k + kk * 2048, PANEL, 1024), id_q, (i > 0 || kk > 0) ? 1u : 0u);
        umma_commit(&kv_empty[i & 1]);
      };
      mbar_wait(q_full, 0);
      for (int i = 0; i < n_it; ++i) {
        const int sb = i & 1;
        mbar_wait(&kv_full[sb], (i >> 1) & 1);
        mbar_wait(&s_free[sb], ((i >> 1) & 1) ^ 1);  // S_{i-2} read by the math warps
        stamp(2, i);
        tc_fence_after();
        const uint32_t k = smem_u32(ring + sb * KV2_STAGE), v = k + 2 * PANEL;
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const uint32_t off = (kk >> 2) * PANEL + (kk & 3) * 32;
          umma_f16(tbase + sb * 128, umma_desc_sw128(aq + off, 16, 1024), umma_desc_sw128(k + off, 16, 1024), id_s,
                   kk > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[sb]);
        if (i > 0) issue_dq(i - 1);
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const uint32_t off = (kk >> 2) * PANEL + (kk & 3) * 32;
          umma_f16(tbase + 256, umma_desc_sw128(ao + off, 16, 1024), umma_desc_sw128(v + off, 16, 1024), id_s,
                   kk > 0 ? 1u : 0u);
        }
        umma_commit(dp_full);
      }
      issue_dq(n_it - 1);
      umma_commit(done);
    }
  } else {
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;  // this warp's 64 key columns of each tile
    const int r = quarter * 32 + lane;
    const int q = qb * TQ + r;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const float sl2 = scale * LOG2E;
    const long long lrow = ((long long)b * n + head) * s;
    const float L2 = lse[lrow + q] * LOG2E, Dq = dsum[lrow + q];
    for (int i = 0; i < n_it; ++i) {
      const int sb = i & 1;
      mbar_wait(&s_full[sb], (i >> 1) & 1);
      if (warp == 2 && lane == 0) stamp(1, i);
      mbar_wait(dp_full, i & 1);
      if (warp == 2 && lane == 0) stamp(4, i);
      tc_fence_after();
      const uint32_t cs = tbase + lane_off + sb * 128 + half * 64, cd = tbase + lane_off + 256 + half * 64;
      const bool diag = i == n_it - 1;
      uint32_t dd[2][16];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t us[32], ud[32];
        tmem_ld32(cs + c * 32, us);
        tmem_ld32(cd + c * 32, ud);
        tmem_wait_ld();
        if (c == 1) {  // S_i fully in registers: its TMEM buffer may take S_{i+2}
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&s_free[sb]);
        }
        const int k0 = i * TK + half * 64 + c * 32;
#pragma unroll
        for (int t = 0; t < 32; t += 2) {
          float p0 = ex2(fmaf(__uint_as_float(us[t]), sl2, -L2));
          float p1 = ex2(fmaf(__uint_as_float(us[t + 1]), sl2, -L2));
          if (diag) {
            if (k0 + t > q) p0 = 0.f;
            if (k0 + t + 1 > q) p1 = 0.f;
          }
          dd[c][t / 2] = pack_bf16(p0 * (__uint_as_float(ud[t]) - Dq), p1 * (__uint_as_float(ud[t + 1]) - Dq));
        }
      }
      // dS over this warp's own dP columns (both 32-column chunks already read)
      if (warp == 2 && lane == 0) stamp(5, i);
      tmem_st16(cd, dd[0]);
      tmem_st16(cd + 16, dd[1]);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(ds_full);
      if (warp == 2 && lane == 0) stamp(6, i);
    }
    float2 csr[32];
    if (rope_cs) load_cs32(rope_cs + (long long)q * 64, half, csr);
    mbar_wait(done, 0);
    tc_fence_after();
    __nv_bfloat16* dq = dqkv + (long long)(b * s + q) * (nd + 2 * n_kv * DH) + head * DH;
    store_row_rope_pre(dq, tbase + lane_off + 384, scale, rope_cs != nullptr, csr, half);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 f = nullptr;
  if (!f) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      f = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  return f;
}

}  // namespace

bool attention_fwd_tc_supported(int s, int d) { return d == DH && s % TQ == 0; }
unsigned long long* attn_trace_buffer = nullptr;
unsigned long long* attn_bwd_trace_buffer = nullptr;
unsigned long long* attn_dq_trace_buffer = nullptr;

// CTA order of the attention grids: 0 = (heads, blocks, sequences) — dispatched x-fastest, so the heaviest
// block of every head goes first and the last wave holds the lightest (longest-processing-time first);
// 1 = the earlier head-major (blocks, heads, sequences) order (MALLEUS_ATTN_GRID_HEADMAJOR=1, A/B switch)
static int grid_order() {
  static const int o = getenv("MALLEUS_ATTN_GRID_HEADMAJOR") ? 1 : 0;
  return o;
}
static dim3 grid_of(int heads, int blocks, int nb) { return grid_order() ? dim3(blocks, heads, nb) : dim3(heads, blocks, nb); }

static bool map_rows(CUtensorMap* m, const void* base, long long cols, long long rows, int box_rows = 128) {
  auto enc = encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// dsum (= rowsum(dO * O)) must already be in `dsum`; writes dq, dk, dv column blocks of dqkv.
cudaError_t attention_bwd_tc(int nb, int s, int n, const void* qkv, const float* lse, const void* dout,
                             void* dqkv, const float* dsum, const float2* rope_cs, cudaStream_t st, int n_kv) {
  CUtensorMap tm, tmo, tm64, tmo64;
  const long long T = (long long)nb * s, cols = (long long)(n + 2 * n_kv) * DH;
  if (n_kv < 1 || n % n_kv) return cudaErrorInvalidValue;
  if (!map_rows(&tm, qkv, cols, T) || !map_rows(&tmo, dout, (long long)n * DH, T) ||
      !map_rows(&tm64, qkv, cols, T, 64) || !map_rows(&tmo64, dout, (long long)n * DH, T, 64))
    return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_bwd_dkv_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, BWD1_SMEM);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(attn_bwd_dq_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, BWD2_SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const float scale = rsqrtf((float)DH);
  static unsigned long long* trace = nullptr;
  if (getenv("MALLEUS_ATTN_TRACE") && !trace) {
    if (cudaMallocManaged(&trace, 2 * 16 * 64 * sizeof(unsigned long long)) != cudaSuccess) trace = nullptr;
    attn_bwd_trace_buffer = trace;
  }
  // dK/dV and dQ are independent (same inputs, disjoint column blocks of dqkv): dQ runs on a side
  // stream forked from `st` and joined back, so its CTAs fill the SMs the dK/dV grid's last wave
  // leaves idle (one CTA of either kernel per SM: ~190 KB of shared memory each).
  // MALLEUS_ATTN_BWD_SERIAL=1 launches both on `st`.
  static const bool serial = getenv("MALLEUS_ATTN_BWD_SERIAL") != nullptr;
  cudaStream_t side = st;
  cudaEvent_t fork = nullptr, join = nullptr;
  if (!serial) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    static cudaStream_t sides[64] = {};
    static cudaEvent_t forks[64] = {}, joins[64] = {};
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    if (!sides[dev]) {
      if ((e = cudaStreamCreateWithFlags(&sides[dev], cudaStreamNonBlocking)) != cudaSuccess) return e;
      if ((e = cudaEventCreateWithFlags(&forks[dev], cudaEventDisableTiming)) != cudaSuccess) return e;
      if ((e = cudaEventCreateWithFlags(&joins[dev], cudaEventDisableTiming)) != cudaSuccess) return e;
    }
    side = sides[dev];
    fork = forks[dev];
    join = joins[dev];
    if ((e = cudaEventRecord(fork, st)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(side, fork, 0)) != cudaSuccess) return e;
  }
  attn_bwd_dkv_tc_kernel<<<grid_of(n_kv, s / TK, nb), 320, BWD1_SMEM, st>>>(tm, tm64, tmo64, s, n, n_kv, lse, dsum,
                                                                         (__nv_bfloat16*)dqkv, scale, rope_cs, trace,
                                                                         grid_order()); count_launch();
  static unsigned long long* trace2 = nullptr;
  if (getenv("MALLEUS_ATTN_TRACE") && !trace2) {
    if (cudaMallocManaged(&trace2, 8 * 64 * sizeof(unsigned long long)) != cudaSuccess) trace2 = nullptr;
    attn_dq_trace_buffer = trace2;
  }
  attn_bwd_dq_tc_kernel<<<grid_of(n, s / TQ, nb), 320, BWD2_SMEM, side>>>(tm, tmo, s, n, n_kv, lse, dsum,
                                                                          (__nv_bfloat16*)dqkv, scale, rope_cs, trace2,
                                                                          grid_order()); count_launch();
  if (!serial) {
    cudaError_t e = cudaEventRecord(join, side);
    if (e != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(st, join, 0)) != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

cudaError_t attention_fwd_tc(int nb, int s, int n, const void* qkv, void* o, float* lse, cudaStream_t st,
                             int n_kv) {
  auto enc = encoder();
  if (!enc) return cudaErrorNotSupported;
  if (n_kv < 1 || n % n_kv) return cudaErrorInvalidValue;
  CUtensorMap tm;
  const long long T = (long long)nb * s, cols = (long long)(n + 2 * n_kv) * DH;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)T};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(qkv), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    for (auto fn : {attn_fwd_tc_kernel<0>, attn_fwd_tc_kernel<1>, attn_fwd_tc_kernel<2>, attn_fwd_tc_kernel<3>}) {
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_FWD);
      if (e != cudaSuccess) return e;
    }
    attr = true;
  }
  static unsigned long long* trace = nullptr;
  if (getenv("MALLEUS_ATTN_TRACE") && !trace) {
    if (cudaMallocManaged(&trace, 2 * 8 * 64 * sizeof(unsigned long long)) != cudaSuccess) trace = nullptr;
    attn_trace_buffer = trace;
  }
  static const int npoly = [] {  // exps per 8 on the FMA pipe (MALLEUS_ATTN_POLY); measured C2 forward:
    const char* e = getenv("MALLEUS_ATTN_POLY");  // 0: 67.8 us, 1: 70.7, 2: 73.3, 3: 76.7 -> off
    return e ? atoi(e) : 0;
  }();
  auto fn = npoly <= 0 ? attn_fwd_tc_kernel<0> : npoly == 1 ? attn_fwd_tc_kernel<1>
          : npoly == 2 ? attn_fwd_tc_kernel<2> : attn_fwd_tc_kernel<3>;
  fn<<<grid_of(n, s / TQ, nb), 320, SMEM_FWD, st>>>(tm, s, n, n_kv, (__nv_bfloat16*)o, lse, rsqrtf((float)DH), trace,
                                                    grid_order());
  count_launch();
  return cudaGetLastError();
}

}  // namespace mls
