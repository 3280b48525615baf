/* malleus.h — C-ABI of the B200-native Malleus hot path (arXiv 2410.13333).
 *
 * The library runs the paper's malleable hybrid-parallel training step on sm_100a:
 * transformer layers with non-uniform tensor-parallel (TP) shards, non-uniform micro-batch
 * counts per data-parallel (DP) pipeline, the batch-weighted gradient reduction across
 * pipelines whose TP layouts differ (ZeRO-1 with varying TP degrees, §5.1),
 * and model-state migration when the plan changes (§5.1).  The planner is
 * host-side input (§4.1 defines the plan's four components).
 *
 * Conventions (all entry points):
 *  - Every function returns malleus_status; nothing throws or aborts across the ABI.  On error
 *    malleus_last_error(ctx) names the violated invariant.  CUDA / NCCL errors are sticky: the
 *    context must be destroyed.
 *  - Pointers documented "device" are CUDA device pointers owned by the caller (PyTorch
 *    allocations); the library borrows them until the next plan_apply / migrate / destroy.
 *    Pointers documented "host" are read (or written) during the call only; plan and config
 *    structs are deep-copied.
 *  - Streams: functions taking a cudaStream_t (passed as void*) only enqueue work on it;
 *    plan_apply, migrate and probe_speed block.
 *  - "collective" calls must be made by every rank of the world in the same order (NCCL rule);
 *    standby ranks take part but do no work.  "local" calls involve one rank only.
 *  - Activations are bf16 row-major [tokens, hidden], tokens = b * s, replicated across the
 *    members of a TP group.
 */
#ifndef MALLEUS_H
#define MALLEUS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MALLEUS_OK = 0,
  MALLEUS_E_ARG = 1,     /* bad argument (null pointer, size, alignment) */
  MALLEUS_E_PLAN = 2,    /* plan violates an invariant (see malleus_plan) */
  MALLEUS_E_CUDA = 3,    /* CUDA runtime error (sticky) */
  MALLEUS_E_NCCL = 4,    /* NCCL error (sticky) */
  MALLEUS_E_NOMEM = 5,   /* caller-provided arena smaller than malleus_plan_requirements */
  MALLEUS_E_STATE = 6,   /* call not valid in the current state (e.g. no plan applied) */
  MALLEUS_E_TIMEOUT = 7
} malleus_status;

/* ---------------------------------------------------------------- model and plan
 * Model: LLaMA-2 architecture (§7.1), MHA (n_kv_heads == n_heads, reading R1) or GQA
 * (n_kv_heads dividing n_heads: query head j reads KV head j / (n_heads / n_kv_heads), the
 * LLaMA-2-70B grouping), RMSNorm eps, RoPE half-split with theta (readings
 * R2/R3), SwiGLU FFN, untied embedding and LM head.  Logical tensors are stored split-axis-outermost
 * with hidden innermost (reading R9): Wq, WoT [n*d, h]; Wk, Wv [n_kv*d, h]; Wg, Wu, WdT [ffn, h];
 * E, Wlm [vocab, h]; norm gains [h].  With GQA every TP member holds whole KV groups (its heads split
 * entry is a multiple of n_heads / n_kv_heads). */
/* Arithmetic of the step (reading R6).  BF16: bf16 params and activations, fp32 accumulation,
 * statistics, gradients and optimizer state; tcgen05 tensor-core GEMMs and attention.  FP32: the
 * parity mode of the north star ("<= 1e-4 in fp32 mode"): fp32 params and activations everywhere,
 * SIMT fp32 GEMMs and attention with plain FFMA (no TF32, no tensor cores), the TP reductions over
 * NCCL; for correctness checks, not for speed.  In FP32 mode the PARAM kind is fp32 (== MASTER). */
typedef enum { MALLEUS_BF16 = 0, MALLEUS_FP32 = 1 } malleus_dtype;

typedef struct {
  int32_t n_layers, hidden, n_heads, n_kv_heads, head_dim, ffn, vocab, seq_len;
  float rms_eps;    /* 1e-5 */
  float rope_theta; /* 1e4 */
  int32_t dtype;    /* malleus_dtype */
} malleus_model_cfg;

/* One pipeline stage = one TP group.  Per-member split vectors are the
 * north-star extension (uneven TP shards): heads[k], ffn_cols[k], vocab_rows[k] are member k's
 * share; each sums to n_heads / ffn / vocab.  Whole heads; ffn and vocab multiples of 16; every
 * member >= 1 head and >= 16 ffn columns / vocab rows.  Layers [layer_begin, layer_end),
 * l_ij = layer_end - layer_begin >= 1 (zero-layer stages are omitted). */
typedef struct {
  int32_t n_members;
  const int32_t* ranks;      /* host, [n_members] */
  const int32_t* heads;      /* host, [n_members] */
  const int32_t* ffn_cols;   /* host, [n_members] */
  const int32_t* vocab_rows; /* host, [n_members]; used on the last stage (LM head) */
  int32_t layer_begin, layer_end;
} malleus_stage;

/* One DP pipeline: ordered stages (embedding on stage 0, final norm + LM head on the last,
 * PAPER.md:1688) and its micro-batch count m_i >= 0. */
typedef struct {
  int32_t n_stages;
  const malleus_stage* stages; /* host */
  int32_t n_micro;
} malleus_pipeline;

/* The plan with b and B (Table 1).  Validation (E_PLAN):
 * sum_i m_i * b == B (Eq.1); each pipeline's layer ranges partition [0, L) in
 * stage order; every rank of [0, world) is in exactly one stage or standby. */
typedef struct {
  int32_t plan_id;
  int32_t dp; /* number of pipelines */
  const malleus_pipeline* pipes; /* host, [dp] */
  int32_t micro_batch;  /* b */
  int32_t global_batch; /* B, sequences per step */
  int32_t n_standby;
  const int32_t* standby; /* host, [n_standby] */
} malleus_plan;

/* Device arenas provided by the caller after malleus_plan_requirements.  256-byte aligned
 * (E_ARG otherwise), each inside a cudaMalloc-backed allocation: plan_apply exports all three to
 * the other ranks with CUDA IPC (the peers read gradients from grads, store parameters into
 * state, and the TP reductions read / write partial sums and activations in work over NVLink).
 *   state : bf16 params held + fp32 master/m/v of owned pieces (persistent across steps)
 *   grads : fp32 gradient shards of held tensors (persistent within a step)
 *   work  : activations, saved tensors, staging, TP reduction buffers and flags (scratch)  */
typedef struct {
  void* state; size_t state_bytes;
  void* grads; size_t grads_bytes;
  void* work;  size_t work_bytes;
} malleus_arenas;

typedef struct { size_t state, grads, work; } malleus_requirements;

/* AdamW (torch.optim.AdamW semantics, reading R5).  step = global step count t >= 1.
 * apply_update = 0 -> grad_sync only reduces gradients into RGRAD (no optimizer update);
 * 1 -> reduce (kept in RGRAD) + AdamW + push; 2 -> reduce + AdamW + push without storing RGRAD
 * (saves 4 B/element of HBM traffic; the production setting).
 * max_grad_norm > 0 (with apply_update != 0): global-norm clipping before AdamW,
 * torch.nn.utils.clip_grad_norm_ semantics: total = ||reduced gradient||_2
 * over every element of the model (each counted once, on its owner), coef = min(1, max_grad_norm /
 * (total + 1e-6)); costs a second pass over the owned pieces and one world all-reduce. */
typedef struct {
  float lr, beta1, beta2, eps, weight_decay;
  int32_t step, apply_update;
  float max_grad_norm;
} malleus_adam_cfg;

typedef struct {
  uint64_t bytes_sent, bytes_recv; /* this rank, payload bytes of the shard deltas */
  double seconds;                  /* wall, this rank: data movement (keep-copies, pack, NCCL, unpack) */
  int32_t n_packs;                 /* 4-layer NCCL packs exchanged; 0 on the peer path */
  double total_seconds;            /* wall, this rank, including host planning and comm split */
} malleus_migrate_stats;

typedef struct malleus_ctx malleus_ctx;

/* Tensor ids: layer*16 + {0 ATTN_NORM g1, 1 WQ, 2 WK, 3 WV, 4 WO(T), 5 MLP_NORM g2, 6 WG, 7 WU,
 * 8 WD(T)} and the globals below.  Kinds select which copy is read / written. */
#define MALLEUS_T_EMBED 0x7FFF0000
#define MALLEUS_T_FINAL_NORM 0x7FFF0001
#define MALLEUS_T_LM_HEAD 0x7FFF0002
enum { MALLEUS_KIND_PARAM = 0, MALLEUS_KIND_GRAD = 1, MALLEUS_KIND_MASTER = 2,
       MALLEUS_KIND_ADAM_M = 3, MALLEUS_KIND_ADAM_V = 4, MALLEUS_KIND_RGRAD = 5 };
/* PARAM: bf16 held rows (fp32 in FP32 mode); GRAD: fp32 local (pipeline-mean) gradient of held rows;
 * MASTER/ADAM_M/ADAM_V: fp32 owned pieces; RGRAD: fp32 reduced gradient of owned pieces
 * (sum_i w_i g_i, written by malleus_grad_sync). */

/* ---------------------------------------------------------------- lifecycle
 * malleus_nccl_unique_id (local): fills 128 bytes with a fresh ncclUniqueId (rank 0 calls it
 * and broadcasts the bytes).  malleus_create (collective): binds `device`, creates the world
 * NCCL communicator.  cfg is deep-copied. */
malleus_status malleus_nccl_unique_id(uint8_t out[128]);
malleus_status malleus_create(const malleus_model_cfg* cfg, int32_t rank, int32_t world,
                              int32_t device, const uint8_t nccl_uid[128], malleus_ctx** out);
/* wait (local): block until the work enqueued on `stream` has completed, or until timeout_ms elapses
 * (timeout_ms <= 0: no limit).  This is the failure detector of PAPER.md:745 ("we add a threshold
 * for communication calls during training in order to detect failures"): a step whose TP
 * reductions, pipeline transfers or gradient exchange wait for an unresponsive GPU does not finish.
 * On timeout — or when a device-side communication wait of the peer-memory TP reduction gave up
 * after MALLEUS_COMM_TIMEOUT_MS (default 20000) — the context enters the failed state and
 * MALLEUS_E_TIMEOUT is returned: the process-wide abort word is set, so every device-side
 * communication wait of the enqueued work gives up at once; every later call except
 * malleus_last_error / malleus_destroy returns MALLEUS_E_STATE, and malleus_destroy of a failed
 * context only releases host resources (NCCL communicators and kernels that still wait on the lost
 * peer are left to process teardown).  Recovery is PAPER.md:735's: the job restarts on the
 * surviving GPUs (a new process) with the unresponsive GPUs' straggling rates set to infinity
 * (a plan without them) and loads the latest checkpoint (write_tensor of every kind). */
malleus_status malleus_wait(malleus_ctx* ctx, void* stream, int32_t timeout_ms);
malleus_status malleus_destroy(malleus_ctx* ctx);
const char* malleus_last_error(const malleus_ctx* ctx); /* never NULL; static if ctx == NULL */
const char* malleus_version(void);

/* ---------------------------------------------------------------- plans
 * plan_requirements (local, no GPU work): arena sizes this rank needs for `plan`.
 * plan_apply (collective, blocking): validate, build layer/stage maps, split vectors, the
 * common-refinement holder/owner maps (reading R9), TP and stage communicators
 * (ncclCommSplit), bind arenas; parameters are undefined until written / migrated. */
malleus_status malleus_plan_requirements(malleus_ctx* ctx, const malleus_plan* plan,
                                         malleus_requirements* out);
malleus_status malleus_plan_apply(malleus_ctx* ctx, const malleus_plan* plan,
                                  const malleus_arenas* arenas);

/* write_tensor (local, blocking): host_full is the whole logical tensor (PARAM: bf16 bits
 * uint16[numel], float[numel] in FP32 mode; MASTER/ADAM_M/ADAM_V: float[numel]); the rank stores its held rows / owned
 * pieces.  Writing PARAM also initialises MASTER = param and zeroes m, v of owned pieces.
 * read_local (local, blocking): copies this rank's elements of (tensor, kind) to host_dst as a
 * concatenation of flat element ranges [ranges[2i], ranges[2i+1]) of the logical tensor.
 * Call with host_dst == NULL to get *n_ranges and *n_elems; capacity is *n_ranges on input. */
malleus_status malleus_write_tensor(malleus_ctx* ctx, int32_t tensor_id, int32_t kind,
                                    const void* host_full);
malleus_status malleus_read_local(malleus_ctx* ctx, int32_t tensor_id, int32_t kind,
                                  void* host_dst, int64_t* ranges, int32_t* n_ranges,
                                  int64_t* n_elems);

/* layout_query (local, host only, no GPU needed): flat element ranges of (tensor, kind) that
 * `rank` holds (PARAM/GRAD) or owns (MASTER, ADAM_M, ADAM_V, RGRAD) under `plan` — the range arithmetic
 * the runtime uses, exposed so it can be checked against the oracle's per-element maps.
 * ranges capacity in pairs is *n_ranges on input; count on output. */
malleus_status malleus_layout_query(const malleus_model_cfg* cfg, const malleus_plan* plan,
                                    int32_t world, int32_t rank, int32_t tensor_id, int32_t kind,
                                    int64_t* ranges, int32_t* n_ranges);

/* migration_query (local, host only): the transfers of `kind` into (dst_rank) when moving from
 * plan `from` to plan `to` (readings R10/R11): triples (tensor_id, elem_begin, elem_end) and
 * the source rank, for every element dst needs and does not have.  Capacity in entries is
 * *n on input. */
malleus_status malleus_migration_query(const malleus_model_cfg* cfg, const malleus_plan* from,
                                       const malleus_plan* to, int32_t world, int32_t dst_rank,
                                       int32_t kind, int64_t* tensor_begin_end, int32_t* src,
                                       int32_t* n);

/* ---------------------------------------------------------------- the hot path
 * layer_fwd / layer_bwd (local to the TP group; collective over it): one transformer layer
 * held by this rank on one micro-batch `slot` (0 <= slot < b_in_flight).  x_in / x_out / dy /
 * dx are device bf16 [b*s, h].  Saved activations live in the work arena.
 * train_step (collective): the whole malleable step of this rank: embedding (first stage),
 * its layers for all m_i micro-batches in 1F1B order with PP send/recv,
 * LM head + vocab-parallel CE (last stage), fp32 gradient accumulation over micro-batches,
 * then malleus_grad_sync.  tokens/targets: device int32 [B, s] (the whole global batch; the
 * rank reads its pipeline's contiguous slice, reading R14).  loss_dev: device float[1],
 * receives sum_i w_i * loss_i on every rank.
 * grad_sync (collective): batch-weighted reduce of every tensor's gradient pieces to their
 * owners, G = sum_i w_i g_i with w_i = m_i b / B (readings R4, R9),
 * AdamW on owned pieces (if apply_update), bf16 push of the updated pieces to every holder. */
malleus_status malleus_layer_fwd(malleus_ctx* ctx, int32_t layer, int32_t slot,
                                 const void* x_in, void* x_out, void* stream);
/* layer_bwd: dy = gradient of the layer output, dx receives the gradient of its input (device bf16
 * [b*s, h]; dx may alias dy), using the activations layer_fwd saved for (layer, slot).  The layer's
 * weight gradients are ACCUMULATED (+=) into its fp32 GRAD rows: call malleus_zero_grads first to
 * start a new accumulation (plan_apply and migrate leave GRAD zeroed; train_step overwrites GRAD
 * with its first micro-batch).  grad_sync then reduces GRAD as the pipeline's gradient. */
malleus_status malleus_layer_bwd(malleus_ctx* ctx, int32_t layer, int32_t slot,
                                 const void* dy, void* dx, void* stream);
malleus_status malleus_train_step(malleus_ctx* ctx, const int32_t* tokens,
                                  const int32_t* targets, float* loss_dev,
                                  const malleus_adam_cfg* adam, void* stream);
malleus_status malleus_grad_sync(malleus_ctx* ctx, const malleus_adam_cfg* adam, void* stream);
/* zero_grads (local): GRAD = 0 for every tensor this rank holds (enqueued on stream). */
malleus_status malleus_zero_grads(malleus_ctx* ctx, void* stream);

/* migrate (collective, blocking): move params (to new holders) and fp32 master/m/v (to new
 * owners) from the current plan to new_plan (readings R10/R11); then new_plan
 * becomes current and new_arenas are used.  The old arenas may be freed by the caller afterwards.
 * Bit-exact copies.  Two transports, same result:
 *  - peer path (default when every rank mapped every peer's arenas with CUDA IPC at plan_apply):
 *    each rank pulls its deltas straight from the sources' old arenas over NVLink in one copy
 *    kernel together with its keep-copies, between two world barriers (no packing; stats->n_packs
 *    = 0);
 *  - NCCL path (MALLEUS_NO_P2P=1 or no peer mapping): per pack of 4 consecutive layers
 *     the outgoing ranges are packed per peer, exchanged with one grouped NCCL
 *    send/recv, and unpacked (stats->n_packs = number of packs).
 * stats may be NULL.  The caller must not run other work on this context concurrently. */
malleus_status malleus_migrate(malleus_ctx* ctx, const malleus_plan* new_plan,
                               const malleus_arenas* new_arenas, malleus_migrate_stats* stats);

/* probe_speed (collective, blocking): fixed micro-benchmark (bf16 GEMM + HBM copy) timed with
 * CUDA events (§5.2), all-gathered: ms_per_rank[world] (host) = the median over 5
 * rounds of the mean time of one iteration in a round of `iters`.
 * set_slowdown (local): straggler emulation for tests and benchmarks (PAPER.md:818-825 uses
 * competing processes).  mode 0 = off, 2 = DUTY (spin kernel of (x-1) * t after every compute
 * segment on the rank's stream).  Mode 1 (HOG, an SM-occupying resident kernel) is rejected with
 * E_ARG: a resident kernel deadlocks every device-wide synchronisation of the process.  x >= 1. */
malleus_status malleus_probe_speed(malleus_ctx* ctx, int32_t iters, float* ms_per_rank);
malleus_status malleus_set_slowdown(malleus_ctx* ctx, float x, int32_t mode);

/* compute / comm breakdown of the last train_step on this rank (ms, from CUDA events):
 * out[0] compute, out[1] tp_comm, out[2] pp_comm, out[3] grad_sync, out[4] total. */
malleus_status malleus_last_step_timing(malleus_ctx* ctx, float out[5]);
/* global gradient norm and clipping coefficient of the last clipped grad_sync / train_step
 * (max_grad_norm > 0); synchronises the device.  coef may be NULL. */
malleus_status malleus_last_grad_norm(malleus_ctx* ctx, float* norm, float* coef);

/* ---------------------------------------------------------------- instrumentation
 * kernel_launches (local): number of kernels this library has launched since it was loaded
 * (all entry points), for the bench's gpu_launches count.
 * gemm_profile (local): enable = 1 starts recording CUDA events around every tcgen05 GEMM launch
 * (resetting totals), enable = 0 stops; enable = -1 queries (synchronising on the recorded
 * events): number of recorded launches, their algorithmic FLOPs (sum of 2*M*N*K) and summed
 * device milliseconds.  Used for the roofline of the dominant kernel. */
int64_t malleus_kernel_launches(void);
malleus_status malleus_gemm_profile(int32_t enable, int64_t* launches, double* flops, double* ms);

/* ---------------------------------------------------------------- kernel-level entry points
 * Single-GPU building blocks of the hot path, exposed for parity tests and roofline
 * measurement.  All pointers are device pointers; all calls enqueue on `stream` and return
 * immediately.  bf16 = uint16 bit patterns, row-major. */

/* C (op)= A * B.  a_mn = 0: A stored [M][K] (lda >= K); a_mn = 1: A stored [K][M] (lda >= M).
 * b_mn = 0: B stored [N][K] (ldb >= K, i.e. C = A B^T); b_mn = 1: B stored [K][N] (ldb >= N).
 * mode 0: C bf16 = AB; 1: C fp32 = AB; 2: C fp32 += AB.  lda, ldb multiples of 8, ldc of 4,
 * A and B 16-byte aligned.  tcgen05/TMEM/TMA kernel, fp32 accumulation. */
malleus_status malleus_k_gemm(int32_t M, int32_t N, int32_t K, const void* A, int64_t lda,
                              int32_t a_mn, const void* B, int64_t ldb, int32_t b_mn, void* C,
                              int64_t ldc, int32_t mode, void* stream);

/* The GEMM with a fused epilogue (the TP-1 residual of S7 / S10 and the SwiGLU of S9 / S12,
 * SURVEY §8(a); "LLaMA-2 architecture"), C = A B (K-major A and B, bf16 out):
 *   res != NULL (glu = 0): C = bf16(A B + res), res bf16 [M, N] row stride ldr (16-byte aligned,
 *     N % 8 == 0);
 *   glu = 1 (SwiGLU forward): N = 2F, B = [W_g; W_u] [2F, K]; C = gu [M, 2F] (bf16 G | U, ldc = 2F)
 *     and aux = u [M, F] = bf16(silu(G) * U) on the bf16-rounded G, U;
 *   glu = 2 (SwiGLU backward): N = F, A B = du (rounded to bf16), aux_in = gu [M, 2F]; aux = dgu
 *     [M, 2F] = [dG | dU] with dU = du * G * s, dG = du * U * s * (1 + G (1 - s)), s = sigmoid(G);
 *     C receives du instead when the kernel cannot fuse.
 * *fused (may be NULL) = 1 when the kernel applied the SwiGLU (CTA-pair TMA epilogue: M >= 256),
 * else 0 (then C holds the plain product and aux is untouched).  E_ARG on a violated layout. */
malleus_status malleus_k_gemm_fused(int32_t M, int32_t N, int32_t K, const void* A, int64_t lda, const void* B,
                                    int64_t ldb, void* C, int64_t ldc, const void* res, int64_t ldr,
                                    int32_t glu, void* aux, const void* aux_in, int32_t* fused, void* stream);
/* Failure-detection controls of the kernel-level entry points (tests): set (1) / clear (0) the
 * process-wide abort word that releases every device-side communication wait; read the status word
 * (nonzero: a wait gave up, after the timeout or on abort), clearing it when clear != 0. */
malleus_status malleus_k_comm_abort(int32_t value);
int32_t malleus_k_comm_status(int32_t clear);
/* GEMM kernel selection for all subsequent GEMMs (tests / benchmarks): 0 = automatic (CTA pair,
 * tcgen05.mma.cta_group::2 with 256x256 tiles, when M >= 256; single CTA 128x256 otherwise),
 * 1 = always single CTA, 2 = always CTA pair (TMA-store / TMA-reduce-add epilogue), 3 = always CTA
 * pair with direct register-to-global epilogue stores. */
malleus_status malleus_k_gemm_variant(int32_t variant);
/* Attention forward kernel selection: 0 = automatic (tcgen05/TMEM/TMA kernel when head_dim == 128
 * and s % 128 == 0, warp-level mma.sync kernel otherwise), 1 = always mma.sync. */
malleus_status malleus_k_attention_variant(int32_t variant);

/* y = x * rsqrt(mean(x^2) + eps) * g; optional fused residual: if partial != NULL then
 * x_new = bf16(x + partial) is written to x_out and normalised.  x, x_out, y: bf16 [T, h];
 * partial: fp32 [T, h] or NULL; g: bf16 [h]; rstd: fp32 [T]. */
malleus_status malleus_k_rmsnorm_fwd(int32_t T, int32_t h, const void* x, const float* partial,
                                     void* x_out, const void* g, float eps, void* y, float* rstd,
                                     void* stream);
/* dx = r*u - x*r^3*mean(x*u) with u = g*dy (dy fp32 [T,h]), plus residual dres (bf16 or NULL):
 * dx_out bf16 = bf16(dres + dx).  dg_accum fp32 [h] += sum_rows dy*x*r (deterministic). */
malleus_status malleus_k_rmsnorm_bwd(int32_t T, int32_t h, const void* x, const void* g,
                                     const float* rstd, const float* dy, const void* dres,
                                     void* dx_out, float* dg_accum, void* stream);
/* The same with a bf16 input gradient dy [T, h] (the TP sums and TP-1 dgrad outputs of the step). */
malleus_status malleus_k_rmsnorm_bwd16(int32_t T, int32_t h, const void* x, const void* g, const float* rstd,
                                       const void* dy, const void* dres, void* dx_out, float* dg_accum,
                                       void* stream);
/* Causal attention on qkv [T, 3*n*d] (q | k | v column blocks, T = nb * s tokens, sequences of
 * length s), RoPE applied in place to q and k first (fwd) / to dq, dk last (bwd).
 * o: bf16 [T, n*d]; lse: fp32 [nb, n, s]. */
malleus_status malleus_k_attention_fwd(int32_t nb, int32_t s, int32_t n, int32_t d, void* qkv,
                                       void* o, float* lse, float rope_theta, void* stream);
malleus_status malleus_k_attention_bwd(int32_t nb, int32_t s, int32_t n, int32_t d,
                                       const void* qkv, const void* o, const float* lse,
                                       const void* dout, void* dqkv, float rope_theta,
                                       void* stream);

/* One member's part of the TP partial-sum reduction over NVLink peer memory (SURVEY §8(a) S8,
 * K15; PAPER.md:262 row-parallel layers).  k members (2..16); member `me` sums rows
 * [me*T/k, (me+1)*T/k) of the k partials part[0..k-1] ([T, h]; part_dtype bit 0: partials bf16
 * (else fp32), bit 1: mode 0 writes a bf16 sum (else fp32); summed in fp32 in member order) and stores
 * the result into every member's destination:
 *   mode 0 (SUM):        d0[j] fp32 or bf16 [T, h] = sum_j part[j];
 *   mode 1 (RESID_NORM): d0[j] bf16 x1 = bf16(x + sum), d1[j] bf16 = x1 * rsqrt(mean(x1^2) + eps) * g,
 *                        d2[j] fp32 [T] = rsqrt(...);  (x: this member's bf16 [T, h]; g: bf16 [h])
 *   mode 2 (RESID):      d0[j] bf16 = bf16(x + sum).
 * flags[j]: member j's block of 64 zero-initialised uint64 (ready / done counters / ticket);
 * epoch: 1, 2, ... incremented by one per reduction, the same sequence on every member; partials
 * of epoch e must not be overwritten before epoch e + 2 (double-buffer them by epoch parity).
 * Every pointer must be addressable from this device (peer access or CUDA IPC).  All k members
 * must call with the same k, T, h, mode and epoch; a member that never arrives makes the kernel
 * trap after 20 s (sticky CUDA error, MALLEUS_E_CUDA on the next call) instead of hanging.
 * h % 8 == 0, h <= 8192; 16-byte aligned rows. */
malleus_status malleus_k_tp_reduce(int32_t k, int32_t me, int32_t T, int32_t h, int32_t mode,
                                   int32_t part_dtype, float eps, uint64_t epoch, const void* const* part,
                                   uint64_t* const* flags,
                                   void* const* d0, void* const* d1, float* const* d2, const void* x,
                                   const void* g, const int32_t* row_split, void* stream);
/* row_split (host, [k + 1] or NULL): member j reduces rows [row_split[j], row_split[j+1]) instead of
 * the even [j*T/k, (j+1)*T/k); 0 = row_split[0] <= ... <= row_split[k] = T.  The runtime sizes the
 * shares like the members' column shares (speed-proportional replicated work, SURVEY §7 hard part
 * (e)).  All members must pass the same split.  Members may live on one device (each on its own
 * stream, grids small enough to be co-resident: the parity tests do this). */

/* ---------------------------------------------------------------- single-device drivers of the
 * multi-GPU rows.  They run the same kernels the runtime runs for
 * these rows, with every "rank's" buffer on one device, so their arithmetic can be checked against
 * the oracle on a one-GPU box. */

/* One owned ZeRO-1 piece for malleus_k_reduce_adam (the runtime's per-piece descriptor; reading
 * R9).  All pointers are device pointers; src[i] are the contributing pipelines'
 * fp32 gradient rows of the piece in pipeline order with weights w[i] = m_i b / B (reading R4,
 * PAPER.md:523); master/m/v/rgrad the owner's fp32 state of the piece, param the owner's bf16 copy,
 * push[q] the other holders' bf16 copies (the fused param push, S17).  master, m, v, rgrad, src 16-byte
 * aligned and len % 4 == 0 select the vector path; anything else runs the scalar path. */
typedef struct {
  int64_t len;
  int32_t n_src;  /* 1..8 */
  int32_t decay;  /* AdamW weight decay on this tensor (2-D tensors, reading R5) */
  const float* src[8];
  float w[8];
  float *master, *m, *v, *rgrad;
  uint16_t* param;
  int32_t n_push; /* 0..15 */
  uint16_t* push[15];
} malleus_piece;

/* Fused batch-weighted reduce + AdamW + bf16 cast + push over n pieces (K14 + K9 + S17,
 * SURVEY §8(a) S15-S17): rgrad = sum_i w_i src_i (fp32, fixed pipeline order), then, if
 * adam->apply_update, AdamW on (master, m, v) with that gradient and param = push[q] = RNE(master).
 * adam->max_grad_norm > 0 clips by the norm of these pieces only (the runtime sums it over the
 * world): norm_coef (device float[2] or NULL) receives (coef, norm).  pieces is a host array, copied
 * during the call; enqueues on stream. */
malleus_status malleus_k_reduce_adam(int32_t n, const malleus_piece* pieces, const malleus_adam_cfg* adam,
                                     float* norm_coef, void* stream);

/* Multi-range byte copy (the migration keep / pull / pack / unpack kernel, K11):
 * copies[i].bytes bytes from src to dst for every i (device pointers, ranges must not overlap;
 * bytes % 2 == 0).  copies is a host array, copied during the call. */
typedef struct {
  const void* src;
  void* dst;
  int64_t bytes;
} malleus_copy;
malleus_status malleus_k_copy_ranges(int32_t n, const malleus_copy* copies, void* stream);

/* Vocab-parallel cross entropy of one micro-batch over k LM-head members on one device (SURVEY
 * §8(a) S11): member j holds logits z[j] (device fp32 [T, V[j]], vocab rows [v0_j, v0_j + V[j]),
 * v0_j = sum_{i<j} V[i]).  The runtime's kernels run per member: local (max, sum exp, target logit),
 * the TP combine of max and of (sum, target) — done here by a k-way device kernel in member order
 * instead of the NCCL all-reduce — then dz[j] = bf16((softmax - onehot) * scale) for the member's
 * columns (device bf16 [T, V[j]]) and, from member 0, loss_rows (device fp32 [T]) = lse - z_target.
 * tgt: device int32 [T].  V[j] % 4 == 0. */
malleus_status malleus_k_vocab_ce(int32_t k, int32_t T, const int32_t* V, const float* const* z,
                                  const int32_t* tgt, float scale, void* const* dz, float* loss_rows,
                                  void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MALLEUS_H */
