// Kernel-level C-ABI entry points (include/malleus.h, "kernel-level entry points").
#include "malleus.h"
#include "kernels.h"

using namespace mls;

static malleus_status cu(cudaError_t e) { return e == cudaSuccess ? MALLEUS_OK : (e == cudaErrorInvalidValue ? MALLEUS_E_ARG : MALLEUS_E_CUDA); }

extern "C" malleus_status malleus_k_gemm(int32_t M, int32_t N, int32_t K, const void* A, int64_t lda,
                                         int32_t a_mn, const void* B, int64_t ldb, int32_t b_mn,
                                         void* C, int64_t ldc, int32_t mode, void* stream) {
  if (!A || !B || !C || mode < 0 || mode > 2) return MALLEUS_E_ARG;
  GemmDesc g{M, N, K, A, lda, a_mn != 0, B, ldb, b_mn != 0, C, ldc, mode};
  return cu(gemm_bf16(g, (cudaStream_t)stream));
}

extern "C" malleus_status malleus_k_rmsnorm_fwd(int32_t T, int32_t h, const void* x, const float* partial,
                                                void* x_out, const void* g, float eps, void* y, float* rstd,
                                                void* stream) {
  if (!x || !g || !y || !rstd) return MALLEUS_E_ARG;
  return cu(rmsnorm_fwd(T, h, x, partial, x_out, g, eps, y, rstd, (cudaStream_t)stream));
}

extern "C" malleus_status malleus_k_rmsnorm_bwd(int32_t T, int32_t h, const void* x, const void* g,
                                                const float* rstd, const float* dy, const void* dres,
                                                void* dx_out, float* dg_accum, void* stream) {
  if (!x || !g || !rstd || !dy || !dx_out || !dg_accum) return MALLEUS_E_ARG;
  float* scratch = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&scratch, rmsnorm_bwd_scratch_floats(T, h) * sizeof(float),
                                  (cudaStream_t)stream);
  if (e != cudaSuccess) return MALLEUS_E_CUDA;
  e = rmsnorm_bwd(T, h, x, g, rstd, dy, dres, dx_out, dg_accum, scratch, (cudaStream_t)stream);
  cudaFreeAsync(scratch, (cudaStream_t)stream);
  return cu(e);
}

extern "C" malleus_status malleus_k_attention_fwd(int32_t nb, int32_t s, int32_t n, int32_t d, void* qkv,
                                                  void* o, float* lse, float rope_theta, void* stream) {
  if (!qkv || !o || !lse) return MALLEUS_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = rope_inplace(nb * s, s, n, d, qkv, 3LL * n * d, 0, rope_theta, false, st);
  if (e == cudaSuccess) e = attention_fwd(nb, s, n, d, qkv, o, lse, st);
  return cu(e);
}

extern "C" malleus_status malleus_k_attention_bwd(int32_t nb, int32_t s, int32_t n, int32_t d, const void* qkv,
                                                  const void* o, const float* lse, const void* dout, void* dqkv,
                                                  float rope_theta, void* stream) {
  if (!qkv || !o || !lse || !dout || !dqkv) return MALLEUS_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  float* dsum = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&dsum, (size_t)nb * s * n * sizeof(float), st);
  if (e != cudaSuccess) return MALLEUS_E_CUDA;
  e = attention_bwd(nb, s, n, d, qkv, o, lse, dout, dqkv, dsum, st);
  if (e == cudaSuccess) e = rope_inplace(nb * s, s, n, d, dqkv, 3LL * n * d, 0, rope_theta, true, st);
  cudaFreeAsync(dsum, st);
  return cu(e);
}

extern "C" int64_t malleus_kernel_launches(void) { return (int64_t)launches_total(); }

extern "C" malleus_status malleus_gemm_profile(int32_t enable, int64_t* launches, double* flops, double* ms) {
  if (enable >= 0) {
    gemm_profile_enable(enable != 0);
    return MALLEUS_OK;
  }
  if (!launches || !flops || !ms) return MALLEUS_E_ARG;
  long long l = 0;
  cudaError_t e = gemm_profile_query(&l, flops, ms);
  *launches = l;
  return cu(e);
}

extern "C" malleus_status malleus_k_gemm_variant(int32_t variant) {
  if (variant < 0 || variant > 3) return MALLEUS_E_ARG;
  gemm_set_variant(variant);
  return MALLEUS_OK;
}

extern "C" malleus_status malleus_k_attention_variant(int32_t variant) {
  if (variant < 0 || variant > 1) return MALLEUS_E_ARG;
  attention_set_variant(variant);
  return MALLEUS_OK;
}

extern "C" malleus_status malleus_k_tp_reduce(int32_t k, int32_t me, int32_t T, int32_t h, int32_t mode,
                                              int32_t part_dtype, float eps, uint64_t epoch, const void* const* part,
                                              uint64_t* const* flags,
                                              void* const* d0, void* const* d1, float* const* d2, const void* x,
                                              const void* g, void* stream) {
  if (k < 2 || k > MAX_TP || !part || !flags || !d0) return MALLEUS_E_ARG;
  if (mode == TP_RESID_NORM && (!d1 || !d2 || !g)) return MALLEUS_E_ARG;
  if (mode != TP_SUM && !x) return MALLEUS_E_ARG;
  TpArgs a{};
  if (getenv("MALLEUS_TP_TRACE")) a.trace = tp_trace_buffer(me);
  if (part_dtype < 0 || part_dtype > 3) return MALLEUS_E_ARG;
  a.part_bf16 = part_dtype & 1;
  a.sum_bf16 = (part_dtype >> 1) & 1;
  a.k = k; a.me = me; a.T = T; a.h = h; a.mode = mode; a.eps = eps; a.epoch = epoch;
  a.x = x; a.g = g;
  for (int j = 0; j < k; ++j) {
    if (!part[j] || !flags[j] || !d0[j]) return MALLEUS_E_ARG;
    a.part[j] = part[j];
    a.flags[j] = reinterpret_cast<unsigned long long*>(flags[j]);
    a.d0[j] = d0[j];
    if (mode == TP_RESID_NORM) { a.d1[j] = d1[j]; a.d2[j] = d2[j]; }
  }
  return cu(tp_reduce(a, (cudaStream_t)stream));
}

// debugging aid for tools/tp_bench.py: the globaltimer stamps of the last traced call per member
extern "C" const unsigned long long* malleus_k_tp_trace_buffer() { return tp_trace_buffer(0); }
extern "C" const unsigned long long* malleus_k_attn_trace_buffer() { return attn_trace_buffer; }
extern "C" const unsigned long long* malleus_k_attn_bwd_trace_buffer() { return attn_bwd_trace_buffer; }
extern "C" const unsigned long long* malleus_k_attn_dq_trace_buffer() { return attn_dq_trace_buffer; }
