// Kernel-level C-ABI entry points (include/malleus.h, "kernel-level entry points").
#include <algorithm>
#include <cmath>
#include <vector>

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

extern "C" malleus_status malleus_k_gemm_fused(int32_t M, int32_t N, int32_t K, const void* A, int64_t lda,
                                               const void* B, int64_t ldb, void* C, int64_t ldc, const void* res,
                                               int64_t ldr, int32_t glu, void* aux, const void* aux_in,
                                               int32_t* fused, void* stream) {
  if (!A || !B || !C || glu < 0 || glu > 2 || (glu && res) || (glu && !aux) || (glu == 2 && !aux_in))
    return MALLEUS_E_ARG;
  GemmDesc g{M, N, K, A, lda, false, B, ldb, false, C, ldc, GEMM_STORE_BF16};
  g.res = res;
  g.ldr = ldr;
  g.glu = glu;
  g.aux = aux;
  g.aux_in = aux_in;
  bool done = false;
  g.glu_done = &done;
  malleus_status s = cu(gemm_bf16(g, (cudaStream_t)stream));
  if (fused) *fused = done ? 1 : 0;
  return s;
}

extern "C" malleus_status malleus_k_rmsnorm_bwd16(int32_t T, int32_t h, const void* x, const void* g,
                                                  const float* rstd, const void* dy, const void* dres, void* dx_out,
                                                  float* dg_accum, void* stream) {
  if (!x || !g || !rstd || !dy || !dx_out || !dg_accum) return MALLEUS_E_ARG;
  float* scratch = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&scratch, rmsnorm_bwd_scratch_floats(T, h) * sizeof(float),
                                  (cudaStream_t)stream);
  if (e != cudaSuccess) return MALLEUS_E_CUDA;
  e = rmsnorm_bwd(T, h, x, g, rstd, dy, dres, dx_out, dg_accum, scratch, (cudaStream_t)stream, true);
  cudaFreeAsync(scratch, (cudaStream_t)stream);
  return cu(e);
}

extern "C" malleus_status malleus_k_comm_abort(int32_t value) {
  comm_abort(value ? 1u : 0u);
  return MALLEUS_OK;
}
extern "C" int32_t malleus_k_comm_status(int32_t clear) { return (int32_t)comm_status(clear != 0); }

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
  cudaError_t e = rope_inplace(nb * s, s, 2 * n, d, qkv, 3LL * n * d, 0, rope_theta, false, st);
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
  if (e == cudaSuccess) e = rope_inplace(nb * s, s, 2 * n, d, dqkv, 3LL * n * d, 0, rope_theta, true, st);
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
                                              const void* g, const int32_t* row_split, void* stream) {
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
  if (row_split) {
    a.uneven = 1;
    for (int j = 0; j <= k; ++j) a.row0[j] = row_split[j];
  }
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

// ---------------------------------------------------------------- single-device drivers of the
// multi-GPU rows (include/malleus.h): same kernels as the runtime, descriptors built here

extern "C" malleus_status malleus_k_reduce_adam(int32_t n, const malleus_piece* pieces, const malleus_adam_cfg* adam,
                                                float* norm_coef, void* stream) {
  if (n < 0 || (n > 0 && !pieces) || !adam || adam->step < 1) return MALLEUS_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<PieceDesc> pd(n);
  std::vector<ChunkDesc> ch;
  const long long CH = 8192;  // the runtime's chunk (runtime.cu build_sync)
  for (int i = 0; i < n; ++i) {
    const malleus_piece& p = pieces[i];
    if (p.n_src < 1 || p.n_src > MAX_DP || p.n_push < 0 || p.n_push > 15 || p.len < 0 || !p.master || !p.m ||
        !p.v || !p.rgrad || !p.param)
      return MALLEUS_E_ARG;
    PieceDesc& d = pd[i];
    d = PieceDesc{};
    d.len = p.len;
    d.n_src = p.n_src;
    bool vec = p.len % 4 == 0 && ((uintptr_t)p.param % 8 == 0);
    for (int k = 0; k < p.n_src; ++k) {
      if (!p.src[k]) return MALLEUS_E_ARG;
      d.src[k] = p.src[k];
      d.w[k] = p.w[k];
      vec &= (uintptr_t)p.src[k] % 16 == 0;
    }
    d.decay = p.decay ? 1 : 0;
    d.master = p.master; d.m = p.m; d.v = p.v; d.rgrad = p.rgrad; d.param = p.param;
    for (uintptr_t q : {(uintptr_t)p.master, (uintptr_t)p.m, (uintptr_t)p.v, (uintptr_t)p.rgrad}) vec &= q % 16 == 0;
    d.n_push = p.n_push;
    for (int q = 0; q < p.n_push; ++q) {
      if (!p.push[q]) return MALLEUS_E_ARG;
      d.push[q] = p.push[q];
      vec &= (uintptr_t)p.push[q] % 8 == 0;
    }
    d.vec = vec ? 1 : 0;
    for (long long o = 0; o < p.len; o += CH) ch.push_back({i, 0, o, std::min(CH, p.len - o)});
  }
  const int nc = (int)ch.size();
  if (nc == 0) return MALLEUS_OK;
  PieceDesc* dpd = nullptr;
  ChunkDesc* dch = nullptr;
  float *sq = nullptr, *coef = nullptr;
  double* tot = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&dpd, pd.size() * sizeof(PieceDesc), st);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&dch, ch.size() * sizeof(ChunkDesc), st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dpd, pd.data(), pd.size() * sizeof(PieceDesc), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dch, ch.data(), ch.size() * sizeof(ChunkDesc), cudaMemcpyHostToDevice, st);
  AdamHyper hp{adam->lr, adam->beta1, adam->beta2, adam->eps, adam->weight_decay,
               (float)(1.0 - std::pow((double)adam->beta1, adam->step)),
               (float)(1.0 - std::pow((double)adam->beta2, adam->step)), adam->apply_update};
  const bool clip = adam->apply_update && adam->max_grad_norm > 0.f;
  if (e == cudaSuccess && !clip) e = reduce_adam(nc, dch, dpd, hp, st);
  if (e == cudaSuccess && clip) {  // the runtime's two passes around the (here: local) norm
    e = cudaMallocAsync((void**)&sq, nc * sizeof(float), st);
    if (e == cudaSuccess) e = cudaMallocAsync((void**)&tot, sizeof(double), st);
    if (e == cudaSuccess) e = cudaMallocAsync((void**)&coef, 2 * sizeof(float), st);
    AdamHyper h1 = hp;
    h1.apply = 0;
    h1.sq = sq;
    if (e == cudaSuccess) e = reduce_adam(nc, dch, dpd, h1, st);
    if (e == cudaSuccess) e = sq_total(nc, sq, tot, st);
    if (e == cudaSuccess) e = clip_coef(tot, adam->max_grad_norm, coef, coef + 1, st);
    AdamHyper h2 = hp;
    h2.apply = 3;
    h2.coef = coef;
    if (e == cudaSuccess) e = reduce_adam(nc, dch, dpd, h2, st);
    if (e == cudaSuccess && norm_coef) e = cudaMemcpyAsync(norm_coef, coef, 2 * sizeof(float), cudaMemcpyDeviceToDevice, st);
  }
  for (void* q : {(void*)dpd, (void*)dch, (void*)sq, (void*)tot, (void*)coef})
    if (q) cudaFreeAsync(q, st);
  return cu(e);
}

extern "C" malleus_status malleus_k_copy_ranges(int32_t n, const malleus_copy* copies, void* stream) {
  if (n < 0 || (n > 0 && !copies)) return MALLEUS_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<CopyDesc> d;
  const long long CHUNK = COPY_CHUNK;
  for (int i = 0; i < n; ++i) {
    const malleus_copy& c = copies[i];
    if (c.bytes < 0 || c.bytes % 2 || (c.bytes && (!c.src || !c.dst))) return MALLEUS_E_ARG;
    for (long long o = 0; o < c.bytes; o += CHUNK)
      d.push_back({static_cast<const char*>(c.src) + o, static_cast<char*>(c.dst) + o, std::min(CHUNK, c.bytes - o)});
  }
  if (d.empty()) return MALLEUS_OK;
  CopyDesc* dd = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&dd, d.size() * sizeof(CopyDesc), st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dd, d.data(), d.size() * sizeof(CopyDesc), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = copy_ranges((int)d.size(), dd, st);
  if (dd) cudaFreeAsync(dd, st);
  return cu(e);
}

extern "C" malleus_status malleus_k_vocab_ce(int32_t k, int32_t T, const int32_t* V, const float* const* z,
                                             const int32_t* tgt, float scale, void* const* dz, float* loss_rows,
                                             void* stream) {
  if (k < 1 || k > MAX_TP || T < 1 || !V || !z || !tgt || !dz || !loss_rows) return MALLEUS_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  // per member: stats [3T] (local max, sum exp, target logit), gmax [T], sum_tgt [2T], loss rows [T]
  float* buf = nullptr;
  const size_t per = 7 * (size_t)T;
  cudaError_t e = cudaMallocAsync((void**)&buf, per * k * sizeof(float), st);
  int v0 = 0;
  std::vector<float*> gm(k), sm(k);
  for (int j = 0; j < k && e == cudaSuccess; ++j) {
    if (!z[j] || !dz[j] || V[j] < 4) { e = cudaErrorInvalidValue; break; }
    float* b = buf + per * j;
    e = ce_stats(T, V[j], z[j], tgt, v0, b, st);
    if (e == cudaSuccess) e = ce_combine_max(T, b, b + 3 * T, st);
    gm[j] = b + 3 * T;
    v0 += V[j];
  }
  // the TP all-reduce (max) of the runtime (NCCL there), k-way in member order on this device
  if (e == cudaSuccess) e = tp_combine_local(k, T, gm.data(), 0, st);
  for (int j = 0; j < k && e == cudaSuccess; ++j) {
    float* b = buf + per * j;
    e = ce_local_sum(T, b, b + 3 * T, b + 4 * T, st);
    sm[j] = b + 4 * T;
  }
  if (e == cudaSuccess) e = tp_combine_local(k, 2 * T, sm.data(), 1, st);  // ... and the sum
  v0 = 0;
  for (int j = 0; j < k && e == cudaSuccess; ++j) {
    float* b = buf + per * j;
    e = ce_grad(T, V[j], z[j], tgt, v0, b + 3 * T, b + 4 * T, b + 5 * T, scale, dz[j], j == 0 ? loss_rows : b + 6 * T, st);
    v0 += V[j];
  }
  if (buf) cudaFreeAsync(buf, st);
  return cu(e);
}
