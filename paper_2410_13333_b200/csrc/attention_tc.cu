// Causal attention forward on the 5th-gen tensor cores (tcgen05 / TMEM / TMA) for head_dim 128
// and sequence lengths that are multiples of 128 (PAPER.md:780 FlashAttention).
//
// One CTA = 128 queries of one (sequence, head).  Warp roles:
//   warp 0      TMA producer: Q once; K and V tiles of 128 keys through a 2-stage ring;
//   warp 1      MMA issuer (one thread) + TMEM owner: S_i = Q K_i^T into one of two TMEM S buffers,
//               then O += P_{i-1} V_{i-1} once the softmax warps have written P_{i-1};
//   warps 2..5  softmax (one query row per thread): S row from TMEM, online max with lazy
//               rescaling (O in TMEM is rescaled only when the running max grows by > 2^8, FA4
//               style; exact since numerator and denominator share the stale max), P (bf16) into
//               a 128B-swizzled smem tile that is the A operand of the PV MMA; final O / l, LSE.
// TMEM: S0 cols [0,128), S1 [128,256), O [256,384).  smem: Q 32 KB, 2 x (K 32 KB + V 32 KB), P 32 KB.
// Output identical in layout to attention.cu: o [T, n*d] bf16, lse [nb, n, s] (natural log).
#include <cuda.h>
#include <cudaTypedefs.h>
#include "kernels.h"
#include "ptx.cuh"

namespace mls {
namespace {

constexpr int TQ = 128, TK = 128, DH = 128;
constexpr int PANEL = 128 * 64 * 2;            // one 128-row x 64-col bf16 swizzled panel (16 KB)
constexpr int Q_BYTES = 2 * PANEL;             // 32 KB
constexpr int KV_STAGE = 4 * PANEL;            // K (2 panels) + V (2 panels)
constexpr int P_BYTES = 2 * PANEL;
constexpr int KV_STAGES = 2;
constexpr int SMEM_TC = Q_BYTES + KV_STAGES * KV_STAGE + P_BYTES + 1024 + 1024;
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

__global__ void __launch_bounds__(192, 1)
attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tm, int s, int n, __nv_bfloat16* __restrict__ o,
                   float* __restrict__ lse, float scale) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sKV = sQ + Q_BYTES;
  uint8_t* sP = sKV + KV_STAGES * KV_STAGE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + P_BYTES);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;              // [2]
  uint64_t* kv_empty = bars + 3;             // [2]
  uint64_t* s_full = bars + 5;               // [2]
  uint64_t* s_empty = bars + 7;              // [2]
  uint64_t* p_full = bars + 9;
  uint64_t* o_done = bars + 10;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = s / TQ;
  const int qb = nqb - 1 - blockIdx.x;  // heaviest first
  const int head = blockIdx.y, b = blockIdx.z;
  const int n_tiles = qb + 1;           // causal: key tiles 0..qb
  const int row0 = b * s + qb * TQ;     // first query row in qkv
  const int nd = n * DH;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1); mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1); mbar_init(&s_empty[i], 4);
    }
    mbar_init(p_full, 4);
    mbar_init(o_done, 1);
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
      for (int i = 0; i < n_tiles; ++i) {
        const int st = i & 1;
        const uint32_t ph = (i >> 1) & 1;
        mbar_wait(&kv_empty[st], ph ^ 1);
        uint8_t* k = sKV + st * KV_STAGE;
        uint8_t* v = k + 2 * PANEL;
        const int krow = b * s + i * TK;
        mbar_arrive_expect_tx(&kv_full[st], KV_STAGE);
        tma_load_2d(k, &tm, &kv_full[st], nd + head * DH, krow);
        tma_load_2d(k + PANEL, &tm, &kv_full[st], nd + head * DH + 64, krow);
        tma_load_2d(v, &tm, &kv_full[st], 2 * nd + head * DH, krow);
        tma_load_2d(v + PANEL, &tm, &kv_full[st], 2 * nd + head * DH + 64, krow);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id_qk = umma_idesc_bf16(128, 128, false, false);
      constexpr uint32_t id_pv = umma_idesc_bf16(128, 128, false, true);
      const uint32_t aq = smem_u32(sQ), ap = smem_u32(sP);
      auto issue_pv = [&](int j) {
        const int st = j & 1;
        mbar_wait(p_full, j & 1);
        tc_fence_after();
        const uint32_t v = smem_u32(sKV + st * KV_STAGE + 2 * PANEL);
#pragma unroll
        for (int kk = 0; kk < TK / 16; ++kk) {
          const uint64_t ad = umma_desc_sw128(ap + (kk >> 2) * PANEL + (kk & 3) * 32, 16, 1024);
          const uint64_t bd = umma_desc_sw128(v + kk * 2048, PANEL, 1024);
          umma_f16(tbase + 256, ad, bd, id_pv, (j > 0 || kk > 0) ? 1u : 0u);
        }
        umma_commit(o_done);
        umma_commit(&kv_empty[st]);
      };
      mbar_wait(q_full, 0);
      for (int i = 0; i < n_tiles; ++i) {
        const int st = i & 1, sb = i & 1;
        mbar_wait(&kv_full[st], (i >> 1) & 1);
        mbar_wait(&s_empty[sb], ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t k = smem_u32(sKV + st * KV_STAGE);
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const uint64_t ad = umma_desc_sw128(aq + (kk >> 2) * PANEL + (kk & 3) * 32, 16, 1024);
          const uint64_t bd = umma_desc_sw128(k + (kk >> 2) * PANEL + (kk & 3) * 32, 16, 1024);
          umma_f16(tbase + 128 * sb, ad, bd, id_qk, kk > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[sb]);
        if (i > 0) issue_pv(i - 1);
      }
      issue_pv(n_tiles - 1);
    }
  } else {
    // ---------------- softmax warps: thread = one query row
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;            // row within the 128-query block
    const int q = qb * TQ + r;                    // query position in the sequence
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const float sl2 = scale * LOG2E;
    float m_used = -INFINITY, l = 0.f;
    uint8_t* prow = sP + r * 128;  // this row inside each 64-col panel (128 B per row)
    for (int i = 0; i < n_tiles; ++i) {
      const int sb = i & 1;
      mbar_wait(&s_full[sb], (i >> 1) & 1);
      tc_fence_after();
      float sv[TK];
#pragma unroll
      for (int c = 0; c < TK / 32; ++c) {
        uint32_t u[32];
        tmem_ld32(tbase + lane_off + 128 * sb + c * 32, u);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) sv[c * 32 + j] = __uint_as_float(u[j]) * sl2;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[sb]);
      float mt = -INFINITY;
      if (i == n_tiles - 1) {  // diagonal tile: keys > query masked
#pragma unroll
        for (int j = 0; j < TK; ++j)
          if (i * TK + j > q) sv[j] = -INFINITY;
      }
#pragma unroll
      for (int j = 0; j < TK; ++j) mt = fmaxf(mt, sv[j]);
      // previous PV must be done before O may be rescaled and before P is overwritten
      if (i > 0) {
        mbar_wait(o_done, (i - 1) & 1);
        tc_fence_after();
      }
      if (mt > m_used + 8.f) {
        if (i > 0) {
          const float f = exp2f(m_used - mt);
          l *= f;
#pragma unroll 1
          for (int c = 0; c < DH / 32; ++c) {
            uint32_t u[32];
            tmem_ld32(tbase + lane_off + 256 + c * 32, u);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j) u[j] = __float_as_uint(__uint_as_float(u[j]) * f);
            tmem_st32(tbase + lane_off + 256 + c * 32, u);
          }
          tmem_wait_st();
        }
        m_used = mt;
      }
      // P = exp2(s - m_used) -> bf16 into the swizzled A tile (2 panels of 64 keys)
#pragma unroll
      for (int ch = 0; ch < TK / 8; ++ch) {
        float p[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          p[j] = exp2f(sv[ch * 8 + j] - m_used);
          l += p[j];
        }
        uint4 w;
        w.x = pack_bf16(p[0], p[1]); w.y = pack_bf16(p[2], p[3]);
        w.z = pack_bf16(p[4], p[5]); w.w = pack_bf16(p[6], p[7]);
        const int panel = ch >> 3, c16 = ch & 7;
        *reinterpret_cast<uint4*>(prow + panel * PANEL + ((c16 ^ (r & 7)) << 4)) = w;
      }
      fence_proxy_async();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
    }
    // epilogue: O / l
    mbar_wait(o_done, (n_tiles - 1) & 1);
    tc_fence_after();
    const float inv = 1.f / l;
    __nv_bfloat16* orow = o + (long long)(b * s + q) * nd + head * DH;
#pragma unroll 1
    for (int c = 0; c < DH / 32; ++c) {
      uint32_t u[32];
      tmem_ld32(tbase + lane_off + 256 + c * 32, u);
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
    lse[((long long)b * n + head) * s + q] = (m_used + log2f(l)) / LOG2E;
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

cudaError_t attention_fwd_tc(int nb, int s, int n, const void* qkv, void* o, float* lse, cudaStream_t st) {
  auto enc = encoder();
  if (!enc) return cudaErrorNotSupported;
  CUtensorMap tm;
  const long long T = (long long)nb * s, cols = 3LL * n * DH;
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
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_TC);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  attn_fwd_tc_kernel<<<dim3(s / TQ, n, nb), 192, SMEM_TC, st>>>(tm, s, n, (__nv_bfloat16*)o, lse,
                                                                rsqrtf((float)DH)); count_launch();
  return cudaGetLastError();
}

}  // namespace mls
