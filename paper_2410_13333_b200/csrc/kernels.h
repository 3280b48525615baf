// Internal launcher interface between the C++ runtime and the sm_100a kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mls {

// instrumentation: library-wide kernel launch counter (gpu_launches in bench.py)
void count_launch(int n = 1);
long long launches_total();
void gemm_profile_enable(bool on);
void gemm_set_variant(int v);
cudaError_t gemm_profile_query(long long* launches, double* flops, double* ms);

enum { GEMM_STORE_BF16 = 0, GEMM_STORE_F32 = 1, GEMM_ACCUM_F32 = 2 };

struct GemmDesc {
  int M, N, K;
  const void* A; long long lda; bool a_mn;
  const void* B; long long ldb; bool b_mn;
  void* C; long long ldc;
  int mode;
  // optional RoPE fused into the bf16 epilogue (QKV projection): columns [0, rope_cols) are heads
  // of 128; row r is position r % rope_s; rope_cs = [rope_s][64] (cos, sin).  *rope_done tells the
  // caller whether the kernel applied it (only the CTA-pair TMA epilogue does).
  const float2* rope_cs = nullptr;
  int rope_cols = 0, rope_s = 0;
  bool* rope_done = nullptr;
  // optional row-split destination (reduce-scatter fused into the epilogue, TP partials): row r
  // goes to dst[r / rows_per_dst] + (r % rows_per_dst) * ldc instead of C (M == n_dst * rows_per_dst;
  // dst may be peer memory).  The kernel makes its stores visible system-wide before it ends.
  int n_dst = 0, rows_per_dst = 0;
  void* dst[4] = {nullptr, nullptr, nullptr, nullptr};
  // leave shared memory on every SM for a kernel running concurrently on another stream (the
  // backward TP reduction overlapping the weight-gradient GEMM): 5-stage instead of 6-stage ring
  bool co_resident = false;
  // FP32 parity mode: A, B, C fp32 (GEMM_STORE_BF16 then stores the fp32 activation), SIMT kernel
  bool f32 = false;
  // optional residual add fused into the bf16 epilogue (TP-1 row-parallel GEMMs, S7 / S10 + the
  // residual of S8): C = bf16(acc + res[row][col]), res bf16 with row stride ldr.  Every bf16 kernel.
  const void* res = nullptr;
  long long ldr = 0;
  // optional SwiGLU fused into the epilogue; CTA-pair TMA epilogue only,
  // *glu_done reports whether the kernel applied it (else C holds the plain GEMM result):
  //   glu = 1 (forward, gate/up GEMM): N = 2F, B rows [0, F) = W_g and [F, 2F) = W_u (K-major);
  //           C = gu [M][2F] (bf16 pre-activations, ldc = 2F) and aux = u = silu(G) * U [M][F].
  //   glu = 2 (backward, down dgrad): N = F, the GEMM result is du; aux_in = gu [M][2F] (saved
  //           pre-activations) and aux = dgu [M][2F] = [dG | dU]; C is not written when fused.
  int glu = 0;
  void* aux = nullptr;
  const void* aux_in = nullptr;
  bool* glu_done = nullptr;
};
cudaError_t gemm_bf16(const GemmDesc& g, cudaStream_t st);  // dispatches to gemm_f32 when g.f32

// ---- FP32 parity mode (fp32.cu): IEEE fp32 activations, plain FFMA (no TF32), deterministic
cudaError_t gemm_f32(const GemmDesc& g, cudaStream_t st);
cudaError_t rmsnorm_fwd_f32(int T, int h, const float* x, const float* partial, float* x_out, const float* g,
                            float eps, float* y, float* rstd, cudaStream_t st);
cudaError_t rmsnorm_bwd_f32(int T, int h, const float* x, const float* g, const float* rstd, const float* dy,
                            const float* dres, float* dx_out, float* dg_accum, cudaStream_t st);
cudaError_t residual_add_f32(long long n, const float* x, const float* p, float* out, cudaStream_t st);
cudaError_t rope_f32(int T, int s, int n, int d, float* buf, long long ld, int col0, float theta, bool inverse,
                     cudaStream_t st);
cudaError_t swiglu_fwd_f32(int T, int F, const float* gu, float* u, cudaStream_t st);
cudaError_t swiglu_bwd_f32(int T, int F, const float* gu, const float* du, float* dgu, cudaStream_t st);
cudaError_t embed_fwd_f32(int T, int h, const int32_t* tok, const float* E, float* x, cudaStream_t st);
cudaError_t embed_bwd_f32(int T, int h, const int32_t* tok, const float* dx, float* dE, cudaStream_t st);
cudaError_t attention_fwd_f32(int nb, int s, int n, int d, const float* qkv, float* o, float* lse, cudaStream_t st,
                              int n_kv = 0);  // n_kv <= 0: MHA
cudaError_t attention_bwd_f32(int nb, int s, int n, int d, const float* qkv, const float* o, const float* lse,
                              const float* dout, float* dqkv, float* dsum, cudaStream_t st, int n_kv = 0);

// ---- elementwise / normalisation (elementwise.cu)
cudaError_t rmsnorm_fwd(int T, int h, const void* x, const float* partial, void* x_out,
                        const void* g, float eps, void* y, float* rstd, cudaStream_t st);
cudaError_t rmsnorm_bwd(int T, int h, const void* x, const void* g, const float* rstd,
                        const void* dy, const void* dres, void* dx_out, float* dg_accum,
                        float* scratch, cudaStream_t st, bool dy_bf16 = false);
size_t rmsnorm_bwd_scratch_floats(int T, int h);
cudaError_t residual_add(long long n, const void* x, const float* partial, void* out,
                         cudaStream_t st);
cudaError_t rope_inplace(int T, int s, int n, int d, void* buf, long long ld, int col0,
                         float theta, bool inverse, cudaStream_t st);
cudaError_t swiglu_fwd(int T, int F, const void* gu, void* u, cudaStream_t st);
cudaError_t swiglu_bwd(int T, int F, const void* gu, const void* du, void* dgu, cudaStream_t st);
cudaError_t embed_fwd(int T, int h, const int32_t* tok, const void* E, void* x, cudaStream_t st);
cudaError_t embed_bwd(int T, int h, const int32_t* tok, const void* dx, float* dE, cudaStream_t st);
// vocab-parallel CE, step 1: per-row local max, sum exp(z - max), target logit (0 if not local)
cudaError_t ce_stats(int T, int V, const float* z, const int32_t* tgt, int v0, float* stats,
                     cudaStream_t st);
// step 2 (after TP reduction of stats): loss rows and dz = (softmax - onehot) * scale (bf16)
cudaError_t ce_grad(int T, int V, const float* z, const int32_t* tgt, int v0, const float* gmax,
                    const float* gsum, const float* gtgt, float scale, void* dz, float* loss_rows,
                    cudaStream_t st, bool dz_f32 = false);
cudaError_t ce_combine_max(int T, const float* stats, float* gmax, cudaStream_t st);
cudaError_t ce_local_sum(int T, const float* stats, const float* gmax, float* sum_tgt,
                         cudaStream_t st);
cudaError_t reduce_loss(int T, const float* loss_rows, float scale, float* out, int accumulate,
                        cudaStream_t st);
cudaError_t cast_f32_bf16(long long n, const float* in, void* out, cudaStream_t st);
// k-way elementwise combine of k device buffers of n floats (op 0 max, 1 sum in buffer order), the
// result written back to every buffer: the single-device stand-in of a TP all-reduce (tests)
cudaError_t tp_combine_local(int k, int n, float* const* bufs, int op, cudaStream_t st);
cudaError_t fill_f32(long long n, float* p, float v, cudaStream_t st);

// ---- optimizer: fused batch-weighted reduce + AdamW on owned pieces (adam.cu)
constexpr int MAX_DP = 8;
struct PieceDesc {
  long long len;
  const float* src[MAX_DP];  // contributions in pipeline order (local grad or receive staging)
  float w[MAX_DP];           // w_i = m_i b / B
  int n_src;
  int decay;                 // apply weight decay (2-D tensors)
  int vec;                   // all pointers 16-byte aligned (param 8-byte), len % 4 == 0
  int param_f32;             // FP32 parity mode: param / push copies are fp32 (= master)
  float* master;
  float* m;
  float* v;
  float* rgrad;              // reduced gradient out (sum_i w_i g_i)
  uint16_t* param;           // owner's bf16 copy of the piece
  int n_push;                // peer-memory param push (fused ZeRO-1 all-gather): other holders' copies
  int pad2_;
  uint16_t* push[15];
};
struct ChunkDesc {
  int piece;
  int pad;
  long long off, len;
};
struct AdamHyper {
  float lr, b1, b2, eps, wd;
  float bc1, bc2;  // 1 - b1^t, 1 - b2^t
  int apply;       // 0 reduce only, 1 reduce + AdamW (+ rgrad), 2 AdamW without storing rgrad,
                   // 3 AdamW on rgrad * (*coef) (second pass of a clipped step; no reduction)
  float* sq = nullptr;          // optional: per-chunk sum of G^2 (deterministic, one float per chunk)
  const float* coef = nullptr;  // apply 3: clipping coefficient (device)
};
cudaError_t reduce_adam(int n_chunks, const ChunkDesc* d_chunks, const PieceDesc* d_pieces,
                        const AdamHyper& hp, cudaStream_t st);
// global-norm clipping helpers: local = sum of the n per-chunk squares (fixed order, fp64) ->
// (world all-reduce by the caller) -> coef = min(1, max_norm / (sqrt(total) + 1e-6)), norm = sqrt(total)
cudaError_t sq_total(int n, const float* sq, double* local, cudaStream_t st);
cudaError_t clip_coef(const double* total, float max_norm, float* coef, float* norm, cudaStream_t st);

// ---- attention (attention.cu): qkv [T, (n + 2 n_kv) d] bf16 = q | k | v column blocks (rope already
// applied to q, k); GQA (n_kv < n, query head j reads KV head j / (n / n_kv)) runs on the tcgen05
// kernels only (head_dim 128); n_kv <= 0 means n (MHA)
cudaError_t attention_fwd(int nb, int s, int n, int d, const void* qkv, void* o, float* lse,
                          cudaStream_t st, int n_kv = 0);
cudaError_t attention_bwd(int nb, int s, int n, int d, const void* qkv, const void* o,
                          const float* lse, const void* dout, void* dqkv, float* dsum,
                          cudaStream_t st, const float2* rope_cs = nullptr, int n_kv = 0);

// tcgen05/TMEM/TMA forward for d = 128, s % 128 == 0 (attention_tc.cu)
bool attention_fwd_tc_supported(int s, int d);
cudaError_t attention_fwd_tc(int nb, int s, int n, const void* qkv, void* o, float* lse, cudaStream_t st,
                             int n_kv);
void attention_set_variant(int v);
cudaError_t attention_bwd_tc(int nb, int s, int n, const void* qkv, const float* lse, const void* dout,
                             void* dqkv, const float* dsum, const float2* rope_cs, cudaStream_t st, int n_kv);
// true when attention_bwd with this (s, d) runs the tcgen05 kernels, which apply the RoPE backward
// rotation to dq / dk in their epilogues when given a (cos, sin) table
bool attention_bwd_fuses_rope(int s, int d);
extern unsigned long long* attn_trace_buffer;      // MALLEUS_ATTN_TRACE stamps of the last forward
extern unsigned long long* attn_bwd_trace_buffer;  // ... and of the last dK / dV kernel
extern unsigned long long* attn_dq_trace_buffer;   // ... and of the last dQ kernel

// ---- failure detection ("we add a threshold for communication calls during training
// in order to detect failures"): a process-wide abort word and status word in mapped pinned host
// memory, polled by every device-side communication wait (the peer-memory TP reduction).  A wait
// that exceeds the timeout (MALLEUS_COMM_TIMEOUT_MS, default 20000) or sees the abort word gives up:
// it sets the status word and the kernel returns (no trap: the context stays usable for teardown).
struct CommGuard {
  const volatile unsigned* abort;  // device alias of the host abort word
  unsigned* status;                // device alias of the host status word (1 = a wait gave up)
  unsigned long long timeout_ns;
};
CommGuard comm_guard();        // lazily allocated; zero pointers if mapped memory is unavailable
void comm_abort(unsigned v);   // host: set / clear the abort word
unsigned comm_status(bool clear);

// ---- TP partial-sum reduction over NVLink peer memory, fused with residual / RMSNorm (tp_reduce.cu)
constexpr int MAX_TP = 16;
constexpr int TP_GRID_MAX = 592;  // 4 CTAs of 256 threads per SM; the grid is a function of (T, k) only
enum { TP_SUM = 0, TP_RESID_NORM = 1, TP_RESID = 2 };
enum { TPF_READY = 0, TPF_DONE = 16, TPF_TICKET = 32, TPF_WORDS = 64 };  // u64 flag block layout
struct TpArgs {
  int k, me, T, h, mode;
  float eps;
  unsigned long long epoch;              // 1, 2, ... per reduction under the current plan
  const void* part[MAX_TP];              // member j's partial [T, h] for this epoch (fp32 or bf16)
  int part_bf16;                         // partials are bf16 (summed in fp32, member order)
  int sum_bf16;                          // TP_SUM writes a bf16 sum (else fp32)
  unsigned long long* flags[MAX_TP];     // member j's flag block (TPF_WORDS u64)
  void* d0[MAX_TP];                      // member j's out: fp32 sum | bf16 x1 | bf16 x'
  void* d1[MAX_TP];                      // member j's normalised bf16 a (TP_RESID_NORM)
  float* d2[MAX_TP];                     // member j's rstd [T] (TP_RESID_NORM)
  const void* x;                         // local bf16 residual input [T, h] (RESID modes)
  const void* g;                         // local bf16 RMSNorm gain [h] (RESID_NORM)
  int uneven;                            // rows of member j are [row0[j], row0[j+1]) (else even)
  int row0[MAX_TP + 1];
  unsigned long long* trace;             // optional: per-call globaltimer stamps (MALLEUS_TP_TRACE)
  CommGuard guard;                       // filled by tp_reduce()
  int co_resident;                       // TP_SUM beside the overlapped wgrad GEMM: <= 1 CTA / SM, 64 regs
};
constexpr int TP_TRACE_CALLS = 4096;
unsigned long long* tp_trace_buffer(int member);  // managed [TP_TRACE_CALLS][4] per member, lazily allocated
cudaError_t tp_reduce(const TpArgs& a, cudaStream_t st);
int tp_grid(int rows);  // CTAs for one member's rows: spread evenly over <= TP_GRID_MAX CTAs
// rows [*r0, *r1) reduced by member me (even split, or a.row0 when a.uneven)
void tp_rows(const TpArgs& a, int me, int* r0, int* r1);

// ---- multi-range copy (copy.cu): migration pack / unpack / keep-copies
struct CopyDesc {
  const char* src;
  char* dst;
  long long bytes;  // <= 64 KB per descriptor (host splits longer ranges)
};
constexpr long long COPY_CHUNK = 64 * 1024;  // bytes per descriptor (one CTA)
cudaError_t copy_ranges(int n, const CopyDesc* d_desc, cudaStream_t st);

// ---- probe / straggler emulation (probe.cu)
cudaError_t spin_ns(long long ns, cudaStream_t st);
cudaError_t probe_copy(long long n, const float* src, float* dst, cudaStream_t st);

}  // namespace mls
