// The malleable hybrid-parallel training step behind include/malleus.h.
//
// One context per process == per GPU.  A plan fixes this rank's pipeline,
// stage and TP member; the runtime owns:
//   * state placement (layout.cpp, reading R9): bf16 params of held rows, fp32 master/m/v of
//     owned ZeRO-1 pieces, fp32 grads of held rows;
//   * the layer forward / backward with uneven TP shards (Megatron column / row parallel,
//     PAPER.md:262, with per-member split vectors) on the sm_100a kernels;
//   * 1F1B pipelining over this pipeline's m_i micro-batches with NCCL P2P
//     between stages whose TP degrees may differ (receiver r <- sender r mod TP_prev);
//   * the batch-weighted cross-layout gradient reduction to owners + AdamW + bf16 push
//     (readings R4, R9): owners read the other pipelines' gradient rows over
//     NVLink (CUDA IPC) and push the updated bf16 rows from the optimizer kernel (NCCL P2P per
//     refined piece is the fallback without peer mapping);
//   * migration to a new plan: peer pulls of the deltas over NVLink, or 4-layer
//     packs with one grouped NCCL send/recv each as the fallback;
//   * probe and straggler emulation.
#include <cuda.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "kernels.h"
#include "layout.h"
#include "malleus.h"

using namespace mls;

namespace {

struct LayerPtrs {
  uint16_t *g1 = nullptr, *wqkv = nullptr, *wo = nullptr, *g2 = nullptr, *wgu = nullptr, *wd = nullptr;
  float *dg1 = nullptr, *dwqkv = nullptr, *dwo = nullptr, *dg2 = nullptr, *dwgu = nullptr, *dwd = nullptr;
};

struct SlotLayer {
  uint16_t *a1, *qkv, *o, *x1, *a2, *gu, *u;
  float *r1, *r2, *lse;
};

struct Slot {
  std::vector<uint16_t*> x;  // n_local + 1 activations [T, h]
  std::vector<SlotLayer> L;
  uint16_t *xf = nullptr, *dlast = nullptr;
  float* rf = nullptr;
};

struct TState {
  TensorInfo t;
  bool held = false;
  Range rows{0, 0};
  uint16_t* param = nullptr;
  float* grad = nullptr;
  std::vector<Piece> owned;
  std::vector<int64_t> owned_off;  // element offset of each owned piece in master/m/v/rgrad
  int64_t owned_elems = 0;
  float *master = nullptr, *m = nullptr, *v = nullptr, *rgrad = nullptr;
};

struct P2POp {
  void* ptr;
  size_t count;
  ncclDataType_t type;
  int peer;
  bool send;
};

struct Layout {
  PlanInfo plan;
  int pipe = -1, stage = -1, member = -1;
  bool standby = true;
  int T = 0, n_loc = 0, kv_loc = 0, F_loc = 0, V_loc = 0, v0 = 0;  // kv_loc: KV heads (GQA groups)
  int lb = 0, le = 0, n_local = 0, PP = 0, TP = 0, slots = 0;
  bool first = false, last = false;
  std::vector<TState> ts;
  std::map<int32_t, int> tix;
  std::vector<LayerPtrs> lp;
  uint16_t *E = nullptr, *gf = nullptr, *Wlm = nullptr;
  float *dE = nullptr, *dgf = nullptr, *dWlm = nullptr;
  std::vector<Slot> slot;
  // transient
  float *part = nullptr, *scratch = nullptr, *dsum = nullptr, *logits = nullptr, *stats = nullptr;
  float2* rope_cs = nullptr;  // [seq_len][64] (cos, sin) for the fused RoPE (head_dim 128)
  float *gmax = nullptr, *sumtgt = nullptr, *loss_rows = nullptr, *loss_acc = nullptr;
  uint16_t *dxa = nullptr, *dxb = nullptr, *dxc = nullptr, *dyrecv = nullptr, *dqkv = nullptr, *dout = nullptr;
  uint16_t *dgu = nullptr, *du = nullptr, *dlogits = nullptr;
  float* staging = nullptr;
  int64_t staging_elems = 0;
  // grad sync
  std::vector<P2POp> gops, pops;
  std::vector<PieceDesc> pieces;
  std::vector<ChunkDesc> chunks;
  PieceDesc* d_pieces = nullptr;
  ChunkDesc* d_chunks = nullptr;
  float* d_sq = nullptr;      // clipping: per-chunk sum of G^2
  double* d_norm = nullptr;   // clipping: local, then world, sum of G^2
  float* d_coef = nullptr;    // clipping: [coef, global norm]
  size_t state_bytes = 0, grads_bytes = 0, work_bytes = 0;
  ncclComm_t tp_comm = nullptr;
  std::vector<int> prev_ranks, next_ranks;  // adjacent stages' members
  // peer memory (CUDA IPC over NVLink): every other rank's layout with its state / grads arena
  // pointers mapped into this process; p2p == true when every rank mapped every peer.
  std::vector<std::unique_ptr<Layout>> peer;
  std::vector<void*> ipc_opened;
  bool p2p = false;
  // TP reduction over peer memory (tp_reduce.cu): double-buffered fp32 partials + flag block
  float* tpp[2] = {nullptr, nullptr};
  unsigned long long* tpflags = nullptr;
  unsigned long long tp_epoch = 0;
  bool tp_bf16 = true;   // partials in bf16 (default; MALLEUS_TP_PARTIAL=fp32 for fp32)
  bool tp_uneven = false; // K15 rows follow the members' column shares (MALLEUS_TP_ROWS=speed)
  // FP32 parity mode (malleus_model_cfg.dtype == MALLEUS_FP32): params and activations fp32,
  // SIMT fp32 kernels (fp32.cu); aes = bytes per param / activation element (2 bf16, 4 fp32)
  bool f32 = false;
  int aes = 2;
  int tp_row0[MAX_TP + 1] = {};
  // weight gradients of micro-batch pairs as one GEMM with K = 2T (single-stage pipelines, bf16, m >= 2):
  // the pair's activations sit in two adjacent slots and its output gradients in per-layer [2][T]
  // stashes, so every weight-gradient operand is one [2T, cols] matrix; the fp32 accumulator is read
  // and written once per pair instead of once per micro-batch
  bool pair = false;
  std::vector<uint16_t*> pdy, pdgu, pdx1, pdqkv;  // per local layer, [2][T][cols]
  uint16_t* pdlogits = nullptr;                   // [2][T][V_loc]
};

// bump allocator over an arena whose base may be 0 (sizing pass)
struct Bump {
  uintptr_t base;
  size_t off = 0;
  explicit Bump(uintptr_t b) : base(b) {}
  template <class T>
  T* take(size_t n, size_t align = 256) {
    off = (off + align - 1) / align * align;
    T* p = reinterpret_cast<T*>(base + off);
    off += n * sizeof(T);
    return p;
  }
};

constexpr int kDutySegs = 16, kDutyRing = 64;
constexpr int kDutyLearn = 4;  // segment durations measured (without spin) before the spin starts
struct DutyTimer {
  bool init = false;
  cudaEvent_t b[kDutyRing], e[kDutyRing];
  long long head = 0, tail = 0;
  double ms = -1.0;   // mean duration of the segment at full speed (frozen after kDutyLearn samples)
  int n = 0;          // samples taken since set_slowdown
};

}  // namespace

struct malleus_ctx {
  malleus_model_cfg cfg{};
  int rank = 0, world = 1, device = 0;
  ncclComm_t world_comm = nullptr;
  std::unique_ptr<Layout> L;
  std::string err;
  bool sticky = false;
  bool failed = false;                        // malleus_wait timed out: communicators aborted
  cudaStream_t tp_side = nullptr;             // backward TP reductions overlapping the wgrad GEMM
  cudaEvent_t tp_ev_a = nullptr, tp_ev_b = nullptr;
  cudaStream_t wg_side = nullptr;             // pair-flush weight-gradient GEMMs beside the dgrad chain
  cudaEvent_t wg_fork_ev = nullptr, wg_join_ev = nullptr;
  bool wg_pending = false;
  float slowdown = 1.f;
  int slow_mode = 0;
  DutyTimer duty[kDutySegs];
  int cur_seg = -1;
  // timing
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pool;
  std::vector<int> ev_cat;
  size_t ev_used = 0;
  cudaEvent_t step_beg = nullptr, step_end = nullptr;
  bool have_timing = false;
};

static const char* kNoCtx = "no context";

#define CK(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess) {                                                          \
      ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);                  \
      ctx->sticky = e_ != cudaErrorInvalidValue;                                      \
      return e_ == cudaErrorInvalidValue ? MALLEUS_E_ARG : MALLEUS_E_CUDA;            \
    }                                                                                 \
  } while (0)
#define NK(call)                                                                      \
  do {                                                                                \
    ncclResult_t r_ = (call);                                                         \
    if (r_ != ncclSuccess) {                                                          \
      ctx->err = std::string(#call) + ": " + ncclGetErrorString(r_);                  \
      ctx->sticky = true;                                                             \
      return MALLEUS_E_NCCL;                                                          \
    }                                                                                 \
  } while (0)
#define RET(st)                                 \
  do {                                          \
    malleus_status s_ = (st);                   \
    if (s_ != MALLEUS_OK) return s_;            \
  } while (0)

static malleus_status fail(malleus_ctx* ctx, malleus_status s, const std::string& m) {
  ctx->err = m;
  return s;
}

// ------------------------------------------------------------------ layout construction
static void build_shape(const malleus_model_cfg& cfg, const PlanInfo& p, int rank, Layout& L) {
  L.plan = p;
  L.f32 = cfg.dtype == MALLEUS_FP32;
  L.aes = L.f32 ? 4 : 2;
  locate(p, rank, &L.pipe, &L.stage, &L.member);
  L.standby = L.pipe < 0;
  L.T = p.b * cfg.seq_len;
  if (L.standby) return;
  const PipeInfo& pp = p.pipes[L.pipe];
  const StageInfo& st = pp.stages[L.stage];
  L.PP = (int)pp.stages.size();
  L.TP = (int)st.ranks.size();
  L.lb = st.lb;
  L.le = st.le;
  L.n_local = st.le - st.lb;
  L.first = L.stage == 0;
  L.last = L.stage == L.PP - 1;
  L.n_loc = st.heads[L.member];
  L.kv_loc = L.n_loc * cfg.n_kv_heads / cfg.n_heads;
  L.F_loc = st.ffn[L.member];
  L.V_loc = st.vocab[L.member];
  L.v0 = 0;
  for (int k = 0; k < L.member; ++k) L.v0 += st.vocab[k];
  L.slots = std::max(1, std::min(L.PP - L.stage, std::max(pp.n_micro, 1)));
  // pair mode on TP-1 single-stage pipelines: on a TP > 1 stage the deferring micro-batch has no
  // weight-gradient GEMM for the backward TP sums to overlap, so its waits for a slower member are
  // exposed (C2 N = 2, rank 1 at 2x: 176.5 K tokens/s paired vs 208.4 K unpaired, profiles/r02);
  // MALLEUS_WGRAD_PAIR_TP=1 allows it there too (tests), MALLEUS_WGRAD_PAIR_OFF=1 disables it
  static const bool pair_off = getenv("MALLEUS_WGRAD_PAIR_OFF") != nullptr;
  static const bool pair_tp = getenv("MALLEUS_WGRAD_PAIR_TP") != nullptr;
  L.pair = !pair_off && L.PP == 1 && !L.f32 && pp.n_micro >= 2 && (L.TP == 1 || pair_tp);
  if (L.pair) L.slots = 2;
  L.prev_ranks.clear();
  L.next_ranks.clear();
  if (!L.first) L.prev_ranks = pp.stages[L.stage - 1].ranks;
  if (!L.last) L.next_ranks = pp.stages[L.stage + 1].ranks;
}

// Assign every buffer.  With zero bases this only computes sizes.
static void assign(const malleus_model_cfg& cfg, int rank, Layout& L, uintptr_t sb, uintptr_t gb, uintptr_t wb) {
  Bump S(sb), G(gb), W(wb);
  L.ts.clear();
  L.tix.clear();
  L.lp.assign(std::max(L.n_local, 0), LayerPtrs{});
  const int64_t h = cfg.hidden, d = cfg.head_dim;
  for (const TensorInfo& t : all_tensors(cfg)) {
    TState s;
    s.t = t;
    s.held = held_rows(cfg, L.plan, t, rank, &s.rows);
    L.tix[t.id] = (int)L.ts.size();
    L.ts.push_back(s);
  }
  // params / grads: per layer the 9 tensors back to back (fused Wqkv, Wgu views), 16-byte units
  for (TState& s : L.ts) {
    if (!s.held) continue;
    const bool group_start = s.t.layer < 0 || s.t.idx == LT_G1;
    const int64_t n = (s.rows.e - s.rows.b) * s.t.cols;
    const size_t al = group_start ? 256 : 16;
    s.param = L.f32 ? reinterpret_cast<uint16_t*>(S.take<float>((size_t)((n + 3) / 4 * 4), al))
                    : S.take<uint16_t>((size_t)((n + 7) / 8 * 8), al);
    s.grad = G.take<float>((size_t)((n + 3) / 4 * 4), al);
  }
  // owned pieces: master, m, v in state; rgrad in grads
  for (TState& s : L.ts) {
    s.owned.clear();
    s.owned_off.clear();
    s.owned_elems = 0;
    for (const Piece& pc : pieces(cfg, L.plan, s.t))
      if (pc.owner == rank) {
        s.owned.push_back(pc);
        s.owned_off.push_back(s.owned_elems);
        s.owned_elems += pc.e1 - pc.e0;
      }
    if (s.owned_elems) {
      s.master = S.take<float>(s.owned_elems);
      s.m = S.take<float>(s.owned_elems);
      s.v = S.take<float>(s.owned_elems);
      s.rgrad = G.take<float>(s.owned_elems);
    }
  }
  // grad-sync receive staging: one fp32 slot per (owned piece, remote contributing pipeline);
  // standby ranks own nothing, so this sizes to zero for them
  int64_t stage_elems = 0;
  for (TState& s : L.ts)
    for (const Piece& pc : s.owned)
      for (size_t i = 0; i < L.plan.pipes.size(); ++i) {
        if (L.plan.pipes[i].n_micro <= 0) continue;
        if (sync_holder(cfg, L.plan.pipes[i], s.t, pc.row0) != rank) stage_elems += (pc.e1 - pc.e0 + 3) / 4 * 4;
      }
  L.staging_elems = stage_elems;
  L.staging = G.take<float>(std::max<int64_t>(stage_elems, 1));

  if (!L.standby) {
    // per-layer fused views
    for (int li = 0; li < L.n_local; ++li) {
      const int l = L.lb + li;
      auto ts = [&](int k) -> TState& { return L.ts[L.tix[l * 16 + k]]; };
      LayerPtrs& P = L.lp[li];
      P.g1 = ts(LT_G1).param; P.dg1 = ts(LT_G1).grad;
      P.wqkv = ts(LT_WQ).param; P.dwqkv = ts(LT_WQ).grad;
      P.wo = ts(LT_WO).param; P.dwo = ts(LT_WO).grad;
      P.g2 = ts(LT_G2).param; P.dg2 = ts(LT_G2).grad;
      P.wgu = ts(LT_WG).param; P.dwgu = ts(LT_WG).grad;
      P.wd = ts(LT_WD).param; P.dwd = ts(LT_WD).grad;
    }
    if (L.first) { auto& s = L.ts[L.tix[MALLEUS_T_EMBED]]; L.E = s.param; L.dE = s.grad; }
    if (L.last) {
      auto& a = L.ts[L.tix[MALLEUS_T_FINAL_NORM]]; L.gf = a.param; L.dgf = a.grad;
      auto& b = L.ts[L.tix[MALLEUS_T_LM_HEAD]]; L.Wlm = b.param; L.dWlm = b.grad;
    }
    // activations
    const int64_t T = L.T, nd = (int64_t)L.n_loc * d, F = L.F_loc;
    // activation buffers: bf16, or fp32 in the parity mode
    auto act = [&](int64_t n) { return L.f32 ? reinterpret_cast<uint16_t*>(W.take<float>(n)) : W.take<uint16_t>(n); };
    L.slot.assign(L.slots, Slot{});
    for (Slot& sl : L.slot) {
      sl.x.resize(L.n_local + 1);
      for (auto& x : sl.x) x = act(T * h);
      sl.L.resize(L.n_local);
    }
    // per-layer activations with the slots adjacent ([slots][T][cols]): in pair mode the two
    // micro-batches of a pair are one [2T, cols] operand of the weight-gradient GEMMs
    auto at = [&](uint16_t* p, int64_t elems) {
      return reinterpret_cast<uint16_t*>(reinterpret_cast<char*>(p) + elems * L.aes);
    };
    const int64_t qkvw = (int64_t)(L.n_loc + 2 * L.kv_loc) * d;
    for (int li = 0; li < L.n_local; ++li) {
      auto adj = [&](int64_t cols, uint16_t* SlotLayer::*f) {
        uint16_t* base = act(T * cols * L.slots);
        for (int sidx = 0; sidx < L.slots; ++sidx) L.slot[sidx].L[li].*f = at(base, sidx * T * cols);
      };
      adj(h, &SlotLayer::a1);
      adj(qkvw, &SlotLayer::qkv);
      adj(nd, &SlotLayer::o);
      adj(h, &SlotLayer::x1);
      adj(h, &SlotLayer::a2);
      adj(2 * F, &SlotLayer::gu);
      adj(F, &SlotLayer::u);
      for (Slot& sl : L.slot) {
        SlotLayer& y = sl.L[li];
        y.r1 = W.take<float>(T);
        y.r2 = W.take<float>(T);
        y.lse = W.take<float>(T * L.n_loc);
      }
    }
    L.pdy.assign(L.n_local, nullptr);
    L.pdgu.assign(L.n_local, nullptr);
    L.pdx1.assign(L.n_local, nullptr);
    L.pdqkv.assign(L.n_local, nullptr);
    if (L.pair)
      for (int li = 0; li < L.n_local; ++li) {
        L.pdy[li] = act(2 * T * h);
        L.pdgu[li] = act(2 * T * 2 * F);
        L.pdx1[li] = act(2 * T * h);
        L.pdqkv[li] = act(2 * T * qkvw);
      }
    if (L.last) {
      uint16_t* xf = act(T * h * L.slots);
      for (int sidx = 0; sidx < L.slots; ++sidx) {
        Slot& sl = L.slot[sidx];
        sl.xf = at(xf, sidx * T * h);
        // pair mode: the head's output gradient lands in the top layer's dy stash
        sl.dlast = (L.pair && L.n_local > 0) ? at(L.pdy[L.n_local - 1], sidx * T * h) : act(T * h);
        sl.rf = W.take<float>(T);
      }
      if (L.pair) L.pdlogits = act(2 * T * L.V_loc);
    }
    L.part = W.take<float>(T * h);
    if (L.TP > 1) {
      L.tpp[0] = W.take<float>(T * h);
      L.tpp[1] = W.take<float>(T * h);
      L.tpflags = W.take<unsigned long long>(TPF_WORDS);
    }
    L.scratch = W.take<float>(rmsnorm_bwd_scratch_floats((int)T, (int)h));
    L.dsum = W.take<float>(T * L.n_loc);
    if (cfg.head_dim == 128 && !L.f32) L.rope_cs = W.take<float2>((size_t)cfg.seq_len * 64);
    L.dxa = act(T * h);
    L.dxb = act(T * h);
    L.dxc = act(T * h);
    L.dyrecv = act(T * h);
    L.dqkv = act(T * qkvw);
    L.dout = act(T * nd);
    L.dgu = act(T * 2 * F);
    L.du = act(T * F);
    if (L.last) {
      L.logits = W.take<float>(T * L.V_loc);
      L.dlogits = act(T * L.V_loc);
      L.stats = W.take<float>(3 * T);
      L.gmax = W.take<float>(T);
      L.sumtgt = W.take<float>(2 * T);
      L.loss_rows = W.take<float>(T);
    }
  }
  L.loss_acc = W.take<float>(4);
  L.state_bytes = S.off + 256;
  L.grads_bytes = G.off + 256;
  L.work_bytes = W.off + 256;
}

// address of flat element e of tensor s's held parameter rows (bf16 or fp32 storage)
static uint16_t* param_at(const Layout& L, const TState& s, int64_t e) {
  return reinterpret_cast<uint16_t*>(reinterpret_cast<char*>(s.param) + (e - s.rows.b * s.t.cols) * L.aes);
}

// grad-sync op lists and the reduce/Adam piece table (needs bound pointers)
static bool build_sync(const malleus_model_cfg& cfg, int rank, Layout& L) {
  L.gops.clear();
  L.pops.clear();
  L.pieces.clear();
  L.chunks.clear();
  const PlanInfo& p = L.plan;
  const int DP = (int)p.pipes.size();
  int64_t stage_off = 0;
  for (TState& s : L.ts) {
    const int64_t c = s.t.cols;
    const size_t ti = &s - &L.ts[0];
    // pointer to element e of tensor ti in rank r's grad / param buffer (own or peer-mapped)
    auto peer_grad = [&](int r, int64_t e) {
      TState& q = r == rank ? s : L.peer[r]->ts[ti];
      return q.grad + (e - q.rows.b * c);
    };
    auto peer_param = [&](int r, int64_t e) {
      TState& q = r == rank ? s : L.peer[r]->ts[ti];
      return param_at(L, q, e);
    };
    for (const Piece& pc : pieces(cfg, p, s.t)) {
      const int64_t len = pc.e1 - pc.e0;
      // contributions
      PieceDesc pd{};
      pd.len = len;
      pd.n_src = 0;
      for (int i = 0; i < DP; ++i) {
        if (p.pipes[i].n_micro <= 0) continue;
        const int hld = sync_holder(cfg, p.pipes[i], s.t, pc.row0);
        const float w = (float)((double)p.pipes[i].n_micro * p.b / p.B);
        if (hld == rank && pc.owner != rank && !L.p2p) {
          L.gops.push_back({s.grad + (pc.e0 - s.rows.b * c), (size_t)len, ncclFloat, pc.owner, true});
        }
        if (pc.owner == rank) {
          if (hld == rank) {
            pd.src[pd.n_src] = s.grad + (pc.e0 - s.rows.b * c);
          } else if (L.p2p) {
            pd.src[pd.n_src] = peer_grad(hld, pc.e0);  // read the holder's gradient over NVLink
          } else {
            float* dst = L.staging + stage_off;
            stage_off += (len + 3) / 4 * 4;  // keep every slot 16-byte aligned
            L.gops.push_back({dst, (size_t)len, ncclFloat, hld, false});
            pd.src[pd.n_src] = dst;
          }
          pd.w[pd.n_src] = w;
          pd.n_src++;
        }
      }
      // param push: owner -> every other holder of the segment
      std::vector<int> holders;
      for (int i = 0; i < DP; ++i) {
        const PipeInfo& pp = p.pipes[i];
        const StageInfo& st = pp.stages[stage_of(cfg, pp, s.t)];
        for (size_t k = 0; k < st.ranks.size(); ++k) {
          Range r = member_rows(cfg, st, s.t, (int)k);
          if (r.b <= pc.row0 && pc.row0 < r.e) holders.push_back(st.ranks[k]);
        }
      }
      for (int hr : holders) {
        if (hr == pc.owner) continue;
        if (L.p2p) {
          if (rank == pc.owner) {  // NVLink store in the Adam kernel
            if (pd.n_push >= (int)(sizeof(pd.push) / sizeof(pd.push[0]))) return false;
            pd.push[pd.n_push++] = peer_param(hr, pc.e0);
          }
        } else if (rank == pc.owner) {
          L.pops.push_back({param_at(L, s, pc.e0), (size_t)len, L.f32 ? ncclFloat : ncclBfloat16, hr, true});
        } else if (rank == hr) {
          L.pops.push_back({param_at(L, s, pc.e0), (size_t)len, L.f32 ? ncclFloat : ncclBfloat16, pc.owner, false});
        }
      }
      if (pc.owner == rank) {
        size_t idx = 0;
        while (s.owned[idx].e0 != pc.e0) ++idx;
        const int64_t off = s.owned_off[idx];
        pd.decay = s.t.decay ? 1 : 0;
        pd.master = s.master + off;
        pd.m = s.m + off;
        pd.v = s.v + off;
        pd.rgrad = s.rgrad + off;
        pd.param = param_at(L, s, pc.e0);
        pd.param_f32 = L.f32 ? 1 : 0;
        const uintptr_t pal = L.f32 ? 16 : 8;  // param / push copies: float4 or 4 x bf16 stores
        bool vec = (len % 4 == 0) && ((uintptr_t)pd.param % pal == 0);
        for (uintptr_t q : {(uintptr_t)pd.master, (uintptr_t)pd.m, (uintptr_t)pd.v, (uintptr_t)pd.rgrad}) vec &= q % 16 == 0;
        for (int k = 0; k < pd.n_src; ++k) vec &= (uintptr_t)pd.src[k] % 16 == 0;
        for (int k = 0; k < pd.n_push; ++k) vec &= (uintptr_t)pd.push[k] % pal == 0;
        pd.vec = vec ? 1 : 0;
        const int pid = (int)L.pieces.size();
        L.pieces.push_back(pd);
        const int64_t CH = 8192;
        for (int64_t o = 0; o < len; o += CH) L.chunks.push_back({pid, 0, o, std::min(CH, len - o)});
      }
    }
  }
  return true;
}

static malleus_status free_layout(malleus_ctx* ctx, Layout* L) {
  if (!L) return MALLEUS_OK;
  for (void* p : L->ipc_opened) cudaIpcCloseMemHandle(p);
  L->ipc_opened.clear();
  L->peer.clear();
  L->p2p = false;
  if (L->d_pieces) cudaFree(L->d_pieces);
  if (L->d_chunks) cudaFree(L->d_chunks);
  if (L->d_sq) cudaFree(L->d_sq);
  if (L->d_norm) cudaFree(L->d_norm);
  if (L->d_coef) cudaFree(L->d_coef);
  L->d_sq = nullptr;
  L->d_norm = nullptr;
  L->d_coef = nullptr;
  if (L->tp_comm) ncclCommDestroy(L->tp_comm);
  L->d_pieces = nullptr;
  L->d_chunks = nullptr;
  L->tp_comm = nullptr;
  return MALLEUS_OK;
}

// CUDA IPC exchange of the state and grads arenas (collective).  Each rank publishes, per arena,
// an IPC handle of the enclosing allocation and the arena's offset in it; every rank opens the
// others' handles and rebuilds their layouts (the bump-allocator arithmetic is deterministic) so
// it can address any peer's parameter / gradient rows directly over NVLink.  If any rank fails
// to map any peer, all ranks fall back to the NCCL point-to-point path (p2p = false).
struct IpcInfo {
  cudaIpcMemHandle_t h[3];
  unsigned long long off[3];
  int ok, pad;
};
typedef CUresult (*PFN_getAddrRange)(CUdeviceptr*, size_t*, CUdeviceptr);

static malleus_status map_peers(malleus_ctx* ctx, Layout& L, const malleus_arenas* a) {
  L.peer.clear();
  L.peer.resize(ctx->world);
  L.p2p = false;
  if (ctx->world == 1 || getenv("MALLEUS_NO_P2P")) return MALLEUS_OK;
  static PFN_getAddrRange get_range = nullptr;
  if (!get_range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      get_range = reinterpret_cast<PFN_getAddrRange>(fn);
  }
  IpcInfo mine{};
  mine.ok = get_range != nullptr;
  void* bases[3] = {a->state, a->grads, a->work};
  for (int i = 0; i < 3 && mine.ok; ++i) {
    CUdeviceptr base = 0;
    size_t size = 0;
    if (get_range(&base, &size, (CUdeviceptr)bases[i]) != CUDA_SUCCESS ||
        cudaIpcGetMemHandle(&mine.h[i], (void*)base) != cudaSuccess) {
      mine.ok = 0;
      cudaGetLastError();
      break;
    }
    mine.off[i] = (unsigned long long)((uintptr_t)bases[i] - (uintptr_t)base);
  }
  IpcInfo* dbuf = nullptr;
  CK(cudaMalloc(&dbuf, sizeof(IpcInfo) * ctx->world));
  CK(cudaMemcpy(dbuf + ctx->rank, &mine, sizeof(IpcInfo), cudaMemcpyHostToDevice));
  NK(ncclAllGather(dbuf + ctx->rank, dbuf, sizeof(IpcInfo), ncclUint8, ctx->world_comm, 0));
  std::vector<IpcInfo> all(ctx->world);
  CK(cudaMemcpy(all.data(), dbuf, sizeof(IpcInfo) * ctx->world, cudaMemcpyDeviceToHost));
  cudaFree(dbuf);
  bool ok = true;
  for (auto& x : all) ok &= x.ok != 0;
  for (int r = 0; r < ctx->world && ok; ++r) {
    if (r == ctx->rank) continue;
    char* ptrs[3] = {nullptr, nullptr, nullptr};
    for (int i = 0; i < 3; ++i) {
      int same = -1;  // arenas inside one allocation share its mapping
      for (int q = 0; q < i; ++q)
        if (memcmp(&all[r].h[i], &all[r].h[q], sizeof(cudaIpcMemHandle_t)) == 0) same = q;
      if (same >= 0) {
        ptrs[i] = ptrs[same] - all[r].off[same];
      } else {
        void* p = nullptr;
        if (cudaIpcOpenMemHandle(&p, all[r].h[i], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
          cudaGetLastError();
          ok = false;
          break;
        }
        L.ipc_opened.push_back(p);
        ptrs[i] = static_cast<char*>(p);
      }
      ptrs[i] += all[r].off[i];
    }
    if (!ok) break;
    auto P = std::make_unique<Layout>();
    build_shape(ctx->cfg, L.plan, r, *P);
    assign(ctx->cfg, r, *P, (uintptr_t)ptrs[0], (uintptr_t)ptrs[1], (uintptr_t)ptrs[2]);
    L.peer[r] = std::move(P);
  }
  // every rank must agree on the path
  int* dok = nullptr;
  int flag = ok ? 1 : 0;
  CK(cudaMalloc(&dok, sizeof(int)));
  CK(cudaMemcpy(dok, &flag, sizeof(int), cudaMemcpyHostToDevice));
  NK(ncclAllReduce(dok, dok, 1, ncclInt32, ncclMin, ctx->world_comm, 0));
  CK(cudaMemcpy(&flag, dok, sizeof(int), cudaMemcpyDeviceToHost));
  cudaFree(dok);
  L.p2p = flag == 1;
  if (!L.p2p) {
    for (void* p : L.ipc_opened) cudaIpcCloseMemHandle(p);
    L.ipc_opened.clear();
    L.peer.clear();
    L.peer.resize(ctx->world);
  }
  return MALLEUS_OK;
}

static malleus_status check_plan(malleus_ctx* ctx, const malleus_plan* plan, PlanInfo* out) {
  if (!plan) return fail(ctx, MALLEUS_E_ARG, "plan is NULL");
  *out = plan_from_c(plan);
  std::string e = validate_plan(ctx->cfg, *out, ctx->world);
  if (e.empty()) e = check_kernel_limits(ctx->cfg, *out);
  if (!e.empty()) return fail(ctx, MALLEUS_E_PLAN, e);
  return MALLEUS_OK;
}

// K15 row shares.  Even by default.  MALLEUS_TP_ROWS=speed sizes member j's rows like its share of
// the stage's work, w_j = l * (8 h n_j d + 2 s n_j d + 6 h F_j) (+ 2 h V_j on the last stage): a plan
// made for rates x_j gives w_j ~ 1/x_j, so the replicated per-token work of the reduction, residual
// and norm follows the member's speed like its columns do (SURVEY §7 hard part (e)).  Rows in units
// of 32 (largest remainder).  Under DUTY emulation the reduction is communication, not stretched
// compute, so even rows are the faster choice there.
static void tp_row_split(const malleus_model_cfg& c, Layout& L) {
  L.tp_uneven = false;
  if (L.standby || L.TP <= 1) return;
  static const bool speed = [] {
    const char* e = getenv("MALLEUS_TP_ROWS");
    return e && strcmp(e, "speed") == 0;
  }();
  if (!speed) return;
  const StageInfo& st = L.plan.pipes[L.pipe].stages[L.stage];
  const int k = L.TP, T = L.T, unit = T % 32 == 0 && T / 32 >= k ? 32 : 1, units = T / unit;
  std::vector<double> w(k);
  double tot = 0;
  for (int j = 0; j < k; ++j) {
    const double n = st.heads[j], f = st.ffn[j];
    w[j] = L.n_local * (8.0 * c.hidden * n * c.head_dim + 2.0 * c.seq_len * n * c.head_dim + 6.0 * c.hidden * f) +
           (L.last ? 2.0 * c.hidden * st.vocab[j] : 0.0);
    tot += w[j];
  }
  std::vector<int> cnt(k);
  std::vector<std::pair<double, int>> rem;
  int used = 0;
  for (int j = 0; j < k; ++j) {
    const double q = units * w[j] / tot;
    cnt[j] = (int)q;
    used += cnt[j];
    rem.push_back({-(q - cnt[j]), j});
  }
  std::sort(rem.begin(), rem.end());
  for (int i = 0; used < units; ++i, ++used) cnt[rem[i % k].second]++;
  L.tp_row0[0] = 0;
  for (int j = 0; j < k; ++j) L.tp_row0[j + 1] = L.tp_row0[j] + cnt[j] * unit;
  L.tp_row0[k] = T;  // the ragged tail (T % unit) goes to the last member
  L.tp_uneven = true;
}

// bind arenas, split communicators, upload the piece table (collective: ncclCommSplit)
static malleus_status bind_layout(malleus_ctx* ctx, Layout& L, const malleus_arenas* a) {
  if (!a) return fail(ctx, MALLEUS_E_ARG, "arenas is NULL");
  if (a->state_bytes < L.state_bytes || a->grads_bytes < L.grads_bytes || a->work_bytes < L.work_bytes)
    return fail(ctx, MALLEUS_E_NOMEM, "arena smaller than malleus_plan_requirements");
  if (((uintptr_t)a->state | (uintptr_t)a->grads | (uintptr_t)a->work) & 255)
    return fail(ctx, MALLEUS_E_ARG, "arenas must be 256-byte aligned");
  assign(ctx->cfg, ctx->rank, L, (uintptr_t)a->state, (uintptr_t)a->grads, (uintptr_t)a->work);
  // TP flag blocks start at zero on every member before any peer can signal (map_peers ends
  // with a world all-reduce, which orders this memset before every later kernel of every rank)
  L.tp_epoch = 0;
  {
    // bf16 partials by default (the row-parallel output dtype of Megatron-style TP, half the
    // NVLink bytes); MALLEUS_TP_PARTIAL=fp32 keeps them fp32 (bitwise equal to the NCCL path at TP 2)
    const char* e = getenv("MALLEUS_TP_PARTIAL");
    L.tp_bf16 = !(e && strcmp(e, "fp32") == 0);
  }
  tp_row_split(ctx->cfg, L);
  if (L.tpflags) CK(cudaMemset(L.tpflags, 0, TPF_WORDS * sizeof(unsigned long long)));
  CK(cudaDeviceSynchronize());
  RET(map_peers(ctx, L, a));
  if (L.rope_cs) {  // (cos, sin)(pos * theta^(-2i/d)) in double precision (readings R2/R3)
    const int d = ctx->cfg.head_dim, S = ctx->cfg.seq_len;
    std::vector<float2> cs((size_t)S * 64);
    for (int pos = 0; pos < S; ++pos)
      for (int i = 0; i < 64; ++i) {
        const double ang = pos * std::pow((double)ctx->cfg.rope_theta, -2.0 * i / d);
        cs[(size_t)pos * 64 + i] = make_float2((float)std::cos(ang), (float)std::sin(ang));
      }
    CK(cudaMemcpy(L.rope_cs, cs.data(), cs.size() * sizeof(float2), cudaMemcpyHostToDevice));
  }
  if (!build_sync(ctx->cfg, ctx->rank, L))
    return fail(ctx, MALLEUS_E_PLAN, "more than 15 other holders of one piece (world <= 16)");
  // TP communicator: color = global stage index
  int color = NCCL_SPLIT_NOCOLOR, key = 0;
  if (!L.standby) {
    color = 0;
    for (int i = 0; i < L.pipe; ++i) color += (int)L.plan.pipes[i].stages.size();
    color += L.stage;
    key = L.member;
  }
  NK(ncclCommSplit(ctx->world_comm, color, key, &L.tp_comm, nullptr));
  CK(cudaMalloc(&L.d_norm, sizeof(double)));
  CK(cudaMalloc(&L.d_coef, 2 * sizeof(float)));
  CK(cudaMemset(L.d_coef, 0, 2 * sizeof(float)));
  if (!L.chunks.empty()) CK(cudaMalloc(&L.d_sq, L.chunks.size() * sizeof(float)));
  if (!L.pieces.empty()) {
    CK(cudaMalloc(&L.d_pieces, L.pieces.size() * sizeof(PieceDesc)));
    CK(cudaMemcpy(L.d_pieces, L.pieces.data(), L.pieces.size() * sizeof(PieceDesc), cudaMemcpyHostToDevice));
    CK(cudaMalloc(&L.d_chunks, L.chunks.size() * sizeof(ChunkDesc)));
    CK(cudaMemcpy(L.d_chunks, L.chunks.data(), L.chunks.size() * sizeof(ChunkDesc), cudaMemcpyHostToDevice));
  }
  return MALLEUS_OK;
}

// ------------------------------------------------------------------ timing helpers
enum { CAT_TP = 1, CAT_PP = 2, CAT_SYNC = 3 };
static void ev_begin(malleus_ctx* ctx, cudaStream_t st, int cat) {
  if (ctx->ev_used == ctx->ev_pool.size()) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    ctx->ev_pool.push_back({a, b});
    ctx->ev_cat.push_back(0);
  }
  ctx->ev_cat[ctx->ev_used] = cat;
  cudaEventRecord(ctx->ev_pool[ctx->ev_used].first, st);
}
static void ev_end(malleus_ctx* ctx, cudaStream_t st) {
  cudaEventRecord(ctx->ev_pool[ctx->ev_used].second, st);
  ctx->ev_used++;
}

// ------------------------------------------------------------------ compute pieces
// debugging aid (MALLEUS_DEBUG_SYNC=1): serialise and trace every GEMM / attention call; read once
static bool debug_sync() {
  static const bool on = getenv("MALLEUS_DEBUG_SYNC") != nullptr;
  return on;
}
static malleus_status gemm(malleus_ctx* ctx, int M, int N, int K, const void* A, long long lda, bool amn,
                           const void* B, long long ldb, bool bmn, void* C, long long ldc, int mode,
                           cudaStream_t st) {
  GemmDesc g{M, N, K, A, lda, amn, B, ldb, bmn, C, ldc, mode};
  g.f32 = ctx->L && ctx->L->f32;
  CK(gemm_bf16(g, st));
  if (debug_sync()) {
    fprintf(stderr, "[malleus] gemm M=%d N=%d K=%d amn=%d bmn=%d mode=%d ...", M, N, K, amn, bmn, mode);
    CK(cudaStreamSynchronize(st));
    fprintf(stderr, " ok\n");
  }
  return MALLEUS_OK;
}

static malleus_status gemm_co(malleus_ctx* ctx, int M, int N, int K, const void* A, long long lda, bool amn,
                              const void* B, long long ldb, bool bmn, void* C, long long ldc, int mode,
                              cudaStream_t st) {  // GEMM leaving room for a concurrent kernel (GemmDesc::co_resident)
  GemmDesc g{M, N, K, A, lda, amn, B, ldb, bmn, C, ldc, mode};
  g.co_resident = true;
  g.f32 = ctx->L && ctx->L->f32;
  CK(gemm_bf16(g, st));
  return MALLEUS_OK;
}

static void duty_begin(malleus_ctx* ctx, int seg, cudaStream_t st);
static void duty_end(malleus_ctx* ctx, cudaStream_t st);
static void duty_relearn(malleus_ctx* ctx);

// Weight-gradient GEMMs of a pair's flush micro-batch on a side stream (TP-1 stages, pair mode): they
// read only saved activations of the pair's two slots and the per-layer gradient stashes, which
// nothing overwrites before the next micro-batch's forward, so they run beside the dgrad chain and
// fill the SMs its GEMM tails, norms and attention leave idle (the persistent GEMM grids take every
// SM, so this is tail filling, not sharing).  Each is forked from the main stream once its inputs
// are enqueued; the side stream is joined before the next forward and before the gradient sync.
// Not under DUTY emulation (its segment timers live on the main stream); MALLEUS_WGRAD_SIDE_OFF=1.
static bool wg_side_on(const malleus_ctx* ctx, int pair) {
  static const bool off = getenv("MALLEUS_WGRAD_SIDE_OFF") != nullptr;
  const Layout& L = *ctx->L;
  return !off && pair == 1 && L.pair && L.TP == 1 && !(ctx->slow_mode == 2 && ctx->slowdown > 1.f);
}
static malleus_status wg_stream(malleus_ctx* ctx, int pair, cudaStream_t st, cudaStream_t* out) {
  *out = st;
  if (!wg_side_on(ctx, pair)) return MALLEUS_OK;
  if (!ctx->wg_side) {
    CK(cudaStreamCreateWithFlags(&ctx->wg_side, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ctx->wg_fork_ev, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ctx->wg_join_ev, cudaEventDisableTiming));
  }
  CK(cudaEventRecord(ctx->wg_fork_ev, st));
  CK(cudaStreamWaitEvent(ctx->wg_side, ctx->wg_fork_ev, 0));
  ctx->wg_pending = true;
  *out = ctx->wg_side;
  return MALLEUS_OK;
}
static malleus_status wg_join(malleus_ctx* ctx, cudaStream_t st) {
  if (!ctx->wg_pending) return MALLEUS_OK;
  CK(cudaEventRecord(ctx->wg_join_ev, ctx->wg_side));
  CK(cudaStreamWaitEvent(st, ctx->wg_join_ev, 0));
  ctx->wg_pending = false;
  return MALLEUS_OK;
}

static malleus_status tp_allreduce(malleus_ctx* ctx, float* buf, size_t n, ncclRedOp_t op, cudaStream_t st) {
  Layout& L = *ctx->L;
  duty_end(ctx, st);
  if (L.TP <= 1) return MALLEUS_OK;
  ev_begin(ctx, st, CAT_TP);
  NK(ncclAllReduce(buf, buf, n, ncclFloat, op, L.tp_comm, st));
  ev_end(ctx, st);
  return MALLEUS_OK;
}

// ---- TP reduction over NVLink peer memory (tp_reduce.cu), fused with residual / RMSNorm
static bool tp_peer(const Layout& L) { return L.TP > 1 && L.p2p && L.tpflags != nullptr && !L.f32; }
// where the next row-parallel GEMM writes its fp32 partial
static float* tp_part(Layout& L) { return tp_peer(L) ? L.tpp[(L.tp_epoch + 1) & 1] : L.part; }
// the row-parallel GEMM's store mode for that buffer
// (TP 1: the row-parallel dgrad output is the full sum, stored in bf16 like every activation gradient
// between kernels, reading R6; the forward fuses its residual into the GEMM epilogue instead)
static int tp_part_mode(const Layout& L) {
  return (tp_peer(L) && L.tp_bf16) || (L.TP == 1 && !L.f32) ? GEMM_STORE_BF16 : GEMM_STORE_F32;
}
// the backward TP sums (input gradients of the norms) are bf16 when the partials are
static bool tp_sum_bf16(const Layout& L) { return (tp_peer(L) && L.tp_bf16) || (L.TP == 1 && !L.f32); }
// reduce-scatter fused into the GEMM epilogue: each member's GEMM stores the rows owned by member d
// straight into d's receive slot (its own index) over NVLink, overlapping the transfer with the
// GEMM; the reduction kernel then reads only local slots.  Needs bf16 partials and T / k rows per
// member in whole 32-row boxes.  Used for k = 2 only: measured at TP 4 (3/4 of the rows remote) the
// epilogue's remote stores slowed the GEMMs by more than the reduction gained (C2: N = 2 T0 258 ->
// 263 K tokens/s, N = 4 DP2 x TP2 502 -> 514 K, TP 4 stage 355 -> 351 K).  MALLEUS_TP_NO_SCATTER=1
// disables it, MALLEUS_TP_SCATTER_K=4 allows it up to k = 4.
static bool tp_scatter(const Layout& L) {
  static const bool off = getenv("MALLEUS_TP_NO_SCATTER") != nullptr;
  static const int kmax = getenv("MALLEUS_TP_SCATTER_K") ? atoi(getenv("MALLEUS_TP_SCATTER_K")) : 2;
  return !off && tp_peer(L) && L.tp_bf16 && !L.tp_uneven && L.TP <= std::min(kmax, 4) && L.T % L.TP == 0 &&
         (L.T / L.TP) % 32 == 0;
}
static Layout& member_layout(Layout& L, int j) {
  const int r = L.plan.pipes[L.pipe].stages[L.stage].ranks[j];
  return L.peer[r] ? *L.peer[r] : L;
}
// sel(M, a, j) fills member j's destinations a.d0/d1/d2[j] from its layout M
template <class Sel>
static malleus_status tp_reduce_peer(malleus_ctx* ctx, int mode, const void* x, const void* g, Sel sel,
                                     cudaStream_t st, bool async = false) {  // async: beside the wgrad GEMM
  Layout& L = *ctx->L;
  if (!async) {  // async: the caller handles DUTY and times only the exposed wait
    duty_end(ctx, st);
    ev_begin(ctx, st, CAT_TP);
  }
  TpArgs a{};
  a.k = L.TP;
  a.me = L.member;
  a.T = L.T;
  a.h = ctx->cfg.hidden;
  a.mode = mode;
  a.eps = ctx->cfg.rms_eps;
  a.epoch = L.tp_epoch + 1;  // committed below once the launch was accepted
  a.x = x;
  a.g = g;
  a.part_bf16 = L.tp_bf16 ? 1 : 0;
  a.sum_bf16 = L.tp_bf16 ? 1 : 0;  // bf16 partials => the backward sums go out in bf16 too
  a.uneven = L.tp_uneven ? 1 : 0;
  a.co_resident = async ? 1 : 0;
  for (int j = 0; j <= L.TP; ++j) a.row0[j] = L.tp_row0[j];
  static const bool trace = getenv("MALLEUS_TP_TRACE") != nullptr;  // debugging aid (tools/tp_step_trace.py)
  if (trace) a.trace = tp_trace_buffer(0);
  const int buf = (int)(a.epoch & 1);
  const bool scatter = tp_scatter(L);
  const size_t slot = (size_t)(L.T / L.TP) * a.h;  // elements per receive slot (scatter layout)
  for (int j = 0; j < L.TP; ++j) {
    Layout& M = member_layout(L, j);
    // the kernel reads part[j] + row * h for its own rows [me*T/k, ...): with the scatter layout
    // that is local slot j, addressed relative to this member's first row
    a.part[j] = scatter ? reinterpret_cast<const void*>(reinterpret_cast<uintptr_t>(L.tpp[buf]) +
                                                         ((size_t)j - (size_t)L.member) * slot * 2)
                        : M.tpp[buf];
    a.flags[j] = M.tpflags;
    sel(M, a, j);
  }
  CK(tp_reduce(a, st));
  L.tp_epoch = a.epoch;
  if (!async) ev_end(ctx, st);
  return MALLEUS_OK;
}

// backward input gradients: L.part = sum_j P_j on every member (peer kernel, else NCCL in place)
static malleus_status tp_sum(malleus_ctx* ctx, cudaStream_t st) {
  Layout& L = *ctx->L;
  if (!tp_peer(L)) return tp_allreduce(ctx, L.part, (size_t)L.T * ctx->cfg.hidden, ncclSum, st);
  return tp_reduce_peer(ctx, TP_SUM, nullptr, nullptr, [&](Layout& M, TpArgs& a, int j) { a.d0[j] = M.part; }, st);
}

// Backward TP sums overlap the weight-gradient GEMM that follows the row-parallel dgrad GEMM: the
// reduction runs on a side stream (it only reads the partial slots and writes the members' sum
// buffers; the wgrad GEMM touches neither) while the GEMM, given a 5-stage ring so the reduction's
// CTAs fit beside it on every SM, runs on the main stream; the main stream joins before the norm's
// backward reads the sum.  MALLEUS_TP_NO_OVERLAP=1 serialises them.
static bool duty_learning(const malleus_ctx* ctx);
static bool tp_overlap(const malleus_ctx* ctx) {
  static const bool off = getenv("MALLEUS_TP_NO_OVERLAP") != nullptr;
  // while the DUTY emulation learns the current segment's full-speed duration the reduction is
  // not overlapped: the learned time is the segment's compute alone, without the interference of
  // a reduction spinning beside the weight-gradient GEMM while it waits for a slower peer
  return !off && tp_peer(*ctx->L) && !duty_learning(ctx);
}
static malleus_status tp_sum_begin(malleus_ctx* ctx, cudaStream_t st) {
  if (!ctx->tp_side) {
    CK(cudaStreamCreateWithFlags(&ctx->tp_side, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ctx->tp_ev_a, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ctx->tp_ev_b, cudaEventDisableTiming));
  }
  // the DUTY segment stays open: the wgrad GEMM that overlaps the reduction is compute of this
  // segment and is stretched with it (tp_sum_end closes the segment before joining)
  CK(cudaEventRecord(ctx->tp_ev_a, st));
  CK(cudaStreamWaitEvent(ctx->tp_side, ctx->tp_ev_a, 0));
  RET(tp_reduce_peer(ctx, TP_SUM, nullptr, nullptr, [&](Layout& M, TpArgs& a, int j) { a.d0[j] = M.part; },
                     ctx->tp_side, true));
  CK(cudaEventRecord(ctx->tp_ev_b, ctx->tp_side));
  return MALLEUS_OK;
}
static malleus_status tp_sum_end(malleus_ctx* ctx, cudaStream_t st) {
  duty_end(ctx, st);
  ev_begin(ctx, st, CAT_TP);  // the exposed part of the reduction
  CK(cudaStreamWaitEvent(st, ctx->tp_ev_b, 0));
  ev_end(ctx, st);
  return MALLEUS_OK;
}

// row-parallel GEMM producing this member's partial sum of a TP reduction (C = A B, [M = T, N = h]):
// into L.part (no peer path), this member's full partial buffer, or scattered by rows to the members'
// receive slots (tp_scatter)
static malleus_status part_gemm(malleus_ctx* ctx, int M, int N, int K, const void* A, long long lda, bool amn,
                                const void* B, long long ldb, bool bmn, cudaStream_t st) {
  Layout& L = *ctx->L;
  if (!tp_scatter(L)) return gemm(ctx, M, N, K, A, lda, amn, B, ldb, bmn, tp_part(L), N, tp_part_mode(L), st);
  const int buf = (int)((L.tp_epoch + 1) & 1);
  const int rows = L.T / L.TP;
  GemmDesc g{M, N, K, A, lda, amn, B, ldb, bmn, nullptr, N, GEMM_STORE_BF16};
  g.n_dst = L.TP;
  g.rows_per_dst = rows;
  for (int d = 0; d < L.TP; ++d)
    g.dst[d] = reinterpret_cast<uint16_t*>(member_layout(L, d).tpp[buf]) + (size_t)L.member * rows * N;
  CK(gemm_bf16(g, st));
  return MALLEUS_OK;
}

// DUTY straggler emulation: every compute segment (the kernels between two TP collectives) is
// bracketed by CUDA events; after it a spin kernel of (x - 1) * t_segment is enqueued on the same
// stream, where t_segment is a moving average of that segment's own measured duration (events are
// polled without blocking).  Only compute is stretched, not communication, as with a GPU that is
// x times slower (PAPER.md:400-401 defines x as the slowdown vs a normal GPU).
static bool duty_learning(const malleus_ctx* ctx) {
  return ctx->slow_mode == 2 && ctx->slowdown > 1.f && ctx->cur_seg >= 0 &&
         ctx->duty[ctx->cur_seg % kDutySegs].n < kDutyLearn;
}
// a new plan changes every segment's work: the full-speed durations are learned again
static void duty_relearn(malleus_ctx* ctx) {
  for (auto& d : ctx->duty) { d.ms = -1.0; d.n = 0; }
}
static void duty_begin(malleus_ctx* ctx, int seg, cudaStream_t st) {
  if (ctx->slow_mode != 2 || ctx->slowdown <= 1.f) return;
  DutyTimer& d = ctx->duty[seg % kDutySegs];
  if (!d.init) {
    for (int i = 0; i < kDutyRing; ++i) { cudaEventCreate(&d.b[i]); cudaEventCreate(&d.e[i]); }
    d.init = true;
  }
  if (d.head - d.tail >= kDutyRing) {  // ring full: wait for the oldest
    cudaEventSynchronize(d.e[d.tail % kDutyRing]);
  }
  cudaEventRecord(d.b[d.head % kDutyRing], st);
  ctx->cur_seg = seg;
}
static void duty_end(malleus_ctx* ctx, cudaStream_t st) {
  if (ctx->slow_mode != 2 || ctx->slowdown <= 1.f || ctx->cur_seg < 0) return;
  DutyTimer& d = ctx->duty[ctx->cur_seg % kDutySegs];
  cudaEventRecord(d.e[d.head % kDutyRing], st);
  d.head++;
  // the segment's full-speed duration is learned from its first kDutyLearn executions after
  // set_slowdown (no spin yet) and then frozen: a spin proportional to a duration that already
  // contains earlier spins' side effects (a peer's TP reduction spinning beside the overlapped
  // weight-gradient GEMM while it waits for this rank) would feed back and over-slow the rank
  while (d.tail < d.head && cudaEventQuery(d.e[d.tail % kDutyRing]) == cudaSuccess) {
    if (d.n < kDutyLearn) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, d.b[d.tail % kDutyRing], d.e[d.tail % kDutyRing]);
      d.ms = d.n == 0 ? ms : (d.ms * d.n + ms) / (d.n + 1);
      d.n++;
      static const bool dbg = getenv("MALLEUS_DUTY_DEBUG") != nullptr;  // measurement aid
      if (dbg && d.n == kDutyLearn)
        fprintf(stderr, "[duty] rank %d seg %d learned %.3f ms (last %.3f)\n", ctx->rank, ctx->cur_seg, d.ms, ms);
    }
    d.tail++;
  }
  if (d.n >= kDutyLearn) spin_ns((long long)((ctx->slowdown - 1.0) * d.ms * 1e6), st);
  ctx->cur_seg = -1;
}

// activation kernels: bf16 path, or the fp32 parity kernels (fp32.cu) when L.f32
#define F(p) reinterpret_cast<float*>(const_cast<void*>(static_cast<const void*>(p)))
static cudaError_t k_norm_fwd(const Layout& L, int T, int h, const void* x, const float* part, void* x_out,
                              const void* g, float eps, void* y, float* rstd, cudaStream_t st) {
  if (L.f32) return rmsnorm_fwd_f32(T, h, F(x), part, F(x_out), F(g), eps, F(y), rstd, st);
  return rmsnorm_fwd(T, h, x, part, x_out, g, eps, y, rstd, st);
}
static cudaError_t k_norm_bwd(const Layout& L, int T, int h, const void* x, const void* g, const float* rstd,
                              const void* dy, const void* dres, void* dx, float* dg, float* scratch, cudaStream_t st,
                              bool dy_bf16) {
  if (L.f32) return rmsnorm_bwd_f32(T, h, F(x), F(g), rstd, F(dy), dres ? F(dres) : nullptr, F(dx), dg, st);
  return rmsnorm_bwd(T, h, x, g, rstd, dy, dres, dx, dg, scratch, st, dy_bf16);
}
static cudaError_t k_rope(const Layout& L, int T, int s, int n, int d, void* buf, long long ld, float theta,
                          bool inverse, cudaStream_t st) {
  if (L.f32) return rope_f32(T, s, n, d, F(buf), ld, 0, theta, inverse, st);
  return rope_inplace(T, s, n, d, buf, ld, 0, theta, inverse, st);
}
static cudaError_t k_attn_fwd(const Layout& L, int nb, int s, int n, int d, const void* qkv, void* o, float* lse,
                              cudaStream_t st) {
  if (L.f32) return attention_fwd_f32(nb, s, n, d, F(qkv), F(o), lse, st, L.kv_loc);
  return attention_fwd(nb, s, n, d, qkv, o, lse, st, L.kv_loc);
}
static cudaError_t k_attn_bwd(const Layout& L, int nb, int s, int n, int d, const void* qkv, const void* o,
                              const float* lse, const void* dout, void* dqkv, float* dsum, cudaStream_t st,
                              const float2* rope_cs) {
  if (L.f32) return attention_bwd_f32(nb, s, n, d, F(qkv), F(o), lse, F(dout), F(dqkv), dsum, st, L.kv_loc);
  return attention_bwd(nb, s, n, d, qkv, o, lse, dout, dqkv, dsum, st, rope_cs, L.kv_loc);
}
static cudaError_t k_swiglu_fwd(const Layout& L, int T, int Fc, const void* gu, void* u, cudaStream_t st) {
  if (L.f32) return swiglu_fwd_f32(T, Fc, F(gu), F(u), st);
  return swiglu_fwd(T, Fc, gu, u, st);
}
static cudaError_t k_swiglu_bwd(const Layout& L, int T, int Fc, const void* gu, const void* du, void* dgu,
                                cudaStream_t st) {
  if (L.f32) return swiglu_bwd_f32(T, Fc, F(gu), F(du), F(dgu), st);
  return swiglu_bwd(T, Fc, gu, du, dgu, st);
}
static cudaError_t k_residual(const Layout& L, long long n, const void* x, const float* part, void* out,
                              cudaStream_t st) {
  if (L.f32) return residual_add_f32(n, F(x), part, F(out), st);
  return residual_add(n, x, part, out, st);
}
static cudaError_t k_embed_fwd(const Layout& L, int T, int h, const int32_t* tok, const void* E, void* x,
                               cudaStream_t st) {
  if (L.f32) return embed_fwd_f32(T, h, tok, F(E), F(x), st);
  return embed_fwd(T, h, tok, E, x, st);
}
static cudaError_t k_embed_bwd(const Layout& L, int T, int h, const int32_t* tok, const void* dx, float* dE,
                               cudaStream_t st) {
  if (L.f32) return embed_bwd_f32(T, h, tok, F(dx), dE, st);
  return embed_bwd(T, h, tok, dx, dE, st);
}
#undef F

static malleus_status layer_fwd_impl(malleus_ctx* ctx, int li, int si, cudaStream_t st) {
  Layout& L = *ctx->L;
  const malleus_model_cfg& c = ctx->cfg;
  const int T = L.T, h = c.hidden, d = c.head_dim, nd = L.n_loc * d, F = L.F_loc;
  Slot& S = L.slot[si];
  SlotLayer& Y = S.L[li];
  LayerPtrs& P = L.lp[li];
  duty_begin(ctx, 0, st);
  CK(k_norm_fwd(L, T, h, S.x[li], nullptr, nullptr, P.g1, c.rms_eps, Y.a1, Y.r1, st));
  {  // QKV projection; RoPE fused into the epilogue when the kernel supports it
    bool rope_done = false;
    const int qkvw = (L.n_loc + 2 * L.kv_loc) * d, nrot = L.n_loc + L.kv_loc;  // q | k | v; RoPE on q and k
    GemmDesc g{T, qkvw, h, Y.a1, h, false, P.wqkv, h, false, Y.qkv, qkvw, GEMM_STORE_BF16};
    g.f32 = L.f32;
    g.rope_cs = L.rope_cs;
    g.rope_cols = nrot * d;
    g.rope_s = c.seq_len;
    g.rope_done = &rope_done;
    CK(gemm_bf16(g, st));
    if (!rope_done) CK(k_rope(L, T, c.seq_len, nrot, d, Y.qkv, qkvw, c.rope_theta, false, st));
  }
  CK(k_attn_fwd(L, L.plan.b, c.seq_len, L.n_loc, d, Y.qkv, Y.o, Y.lse, st));
  if (debug_sync()) { fprintf(stderr, "[malleus] attn fwd ..."); CK(cudaStreamSynchronize(st)); fprintf(stderr, " ok\n"); }
  // TP 1: the residual add is fused into the row-parallel GEMM's epilogue (x1 = bf16(x + o W_o^T),
  // no fp32 partial round trip); the norm then reads x1
  const bool fuse_res = L.TP == 1 && !L.f32;
  if (fuse_res) {
    GemmDesc g{T, h, nd, Y.o, nd, false, P.wo, h, true, Y.x1, h, GEMM_STORE_BF16};
    g.res = S.x[li];
    g.ldr = h;
    CK(gemm_bf16(g, st));
  } else {
    RET(part_gemm(ctx, T, h, nd, Y.o, nd, false, P.wo, h, true, st));
  }
  if (tp_peer(L)) {  // x1 = x + sum P, a2 = RMSNorm(x1) in one peer-memory kernel
    RET(tp_reduce_peer(ctx, TP_RESID_NORM, S.x[li], P.g2, [&](Layout& M, TpArgs& a, int j) {
      const SlotLayer& Z = M.slot[si].L[li];
      a.d0[j] = Z.x1; a.d1[j] = Z.a2; a.d2[j] = Z.r2;
    }, st));
    duty_begin(ctx, 1, st);
  } else if (fuse_res) {
    duty_end(ctx, st);
    duty_begin(ctx, 1, st);
    CK(k_norm_fwd(L, T, h, Y.x1, nullptr, nullptr, P.g2, c.rms_eps, Y.a2, Y.r2, st));
  } else {
    RET(tp_allreduce(ctx, L.part, (size_t)T * h, ncclSum, st));
    duty_begin(ctx, 1, st);
    CK(k_norm_fwd(L, T, h, S.x[li], L.part, Y.x1, P.g2, c.rms_eps, Y.a2, Y.r2, st));
  }
  {  // gate/up projection; SwiGLU fused into the epilogue when the kernel supports it
    bool glu_done = false;
    GemmDesc g{T, 2 * F, h, Y.a2, h, false, P.wgu, h, false, Y.gu, 2 * F, GEMM_STORE_BF16};
    g.f32 = L.f32;
    if (!L.f32) {
      g.glu = 1;
      g.aux = Y.u;
      g.glu_done = &glu_done;
    }
    CK(gemm_bf16(g, st));
    if (!glu_done) CK(k_swiglu_fwd(L, T, F, Y.gu, Y.u, st));
  }
  if (fuse_res) {  // x[l+1] = bf16(x1 + u W_d^T) in the epilogue
    GemmDesc g{T, h, F, Y.u, F, false, P.wd, h, true, S.x[li + 1], h, GEMM_STORE_BF16};
    g.res = Y.x1;
    g.ldr = h;
    CK(gemm_bf16(g, st));
    duty_end(ctx, st);
  } else {
    RET(part_gemm(ctx, T, h, F, Y.u, F, false, P.wd, h, true, st));
    if (tp_peer(L)) {  // x[l+1] = x1 + sum P
      RET(tp_reduce_peer(ctx, TP_RESID, Y.x1, nullptr, [&](Layout& M, TpArgs& a, int j) {
        a.d0[j] = M.slot[si].x[li + 1];
      }, st));
    } else {
      RET(tp_allreduce(ctx, L.part, (size_t)T * h, ncclSum, st));
      duty_begin(ctx, 2, st);
      CK(k_residual(L, (long long)T * h, Y.x1, L.part, S.x[li + 1], st));
      duty_end(ctx, st);
    }
  }
  return MALLEUS_OK;
}

// dy: grad of x[li+1]; writes grad of x[li] to dx.  first: STORE into wgrad (first micro-batch, or the
// first pair).  pair: -1 = this micro-batch's weight gradients now (K = T); 0 = the first micro-batch of
// a pair (slot 0): output gradients into the stash, weight gradients deferred; 1 = the second (slot 1):
// the pair's weight gradients as one GEMM each with K = 2T over the adjacent slots / stash halves.
static malleus_status layer_bwd_impl(malleus_ctx* ctx, int li, int si, const uint16_t* dy, uint16_t* dx,
                                     bool first, cudaStream_t st, int pair = -1) {
  Layout& L = *ctx->L;
  const malleus_model_cfg& c = ctx->cfg;
  const int T = L.T, h = c.hidden, d = c.head_dim, nd = L.n_loc * d, F = L.F_loc;
  const int qkvw = (L.n_loc + 2 * L.kv_loc) * d;
  Slot& S = L.slot[si];
  SlotLayer& Y = S.L[li];
  LayerPtrs& P = L.lp[li];
  const int wm = first ? GEMM_STORE_F32 : GEMM_ACCUM_F32;
  const bool stash = pair >= 0;
  const int half = stash ? si : 0;
  uint16_t* dgu = stash ? L.pdgu[li] + (size_t)half * T * 2 * F : L.dgu;
  uint16_t* dx1 = stash ? L.pdx1[li] + (size_t)half * T * h : L.dxc;
  uint16_t* dqkv = stash ? L.pdqkv[li] + (size_t)half * T * qkvw : L.dqkv;
  // weight-gradient operands: this micro-batch (K = T) or the pair (K = 2T, slot 0 / stash half 0 base)
  const bool wg = pair != 0;
  const int Kw = pair == 1 ? 2 * T : T;
  const SlotLayer& Y0 = pair == 1 ? L.slot[0].L[li] : Y;
  const uint16_t* w_dy = pair == 1 ? L.pdy[li] : dy;
  const uint16_t* w_dgu = pair == 1 ? L.pdgu[li] : dgu;
  const uint16_t* w_dx1 = pair == 1 ? L.pdx1[li] : dx1;
  const uint16_t* w_dqkv = pair == 1 ? L.pdqkv[li] : dqkv;
  // overlap decided inside each segment (tp_overlap: not while DUTY learns that segment's duration)
  // MLP
  duty_begin(ctx, 3, st);
  {  // du = dy W_d with the SwiGLU backward fused into the epilogue (dgu straight from the GEMM)
    bool glu_done = false;
    GemmDesc g{T, F, h, dy, h, false, P.wd, h, false, L.du, F, GEMM_STORE_BF16};
    g.f32 = L.f32;
    if (!L.f32) {
      g.glu = 2;
      g.aux = dgu;
      g.aux_in = Y.gu;
      g.glu_done = &glu_done;
    }
    CK(gemm_bf16(g, st));
    if (wg) {
      cudaStream_t ws;
      RET(wg_stream(ctx, pair, st, &ws));
      RET(gemm(ctx, F, h, Kw, Y0.u, F, true, w_dy, h, true, P.dwd, h, wm, ws));
    }
    if (!glu_done) CK(k_swiglu_bwd(L, T, F, Y.gu, L.du, dgu, st));
  }
  RET(part_gemm(ctx, T, h, 2 * F, dgu, 2 * F, false, P.wgu, h, true, st));
  if (wg && tp_overlap(ctx)) {
    RET(tp_sum_begin(ctx, st));
    RET(gemm_co(ctx, 2 * F, h, Kw, w_dgu, 2 * F, true, Y0.a2, h, true, P.dwgu, h, wm, st));
    RET(tp_sum_end(ctx, st));
  } else {
    if (wg) {
      cudaStream_t ws;
      RET(wg_stream(ctx, pair, st, &ws));
      RET(gemm(ctx, 2 * F, h, Kw, w_dgu, 2 * F, true, Y0.a2, h, true, P.dwgu, h, wm, ws));
    }
    RET(tp_sum(ctx, st));
  }
  duty_begin(ctx, 4, st);
  CK(k_norm_bwd(L, T, h, Y.x1, P.g2, Y.r2, L.part, dy, dx1, P.dg2, L.scratch, st, tp_sum_bf16(L)));
  // attention
  RET(gemm(ctx, T, nd, h, dx1, h, false, P.wo, h, false, L.dout, nd, GEMM_STORE_BF16, st));
  if (wg) {
    cudaStream_t ws;
    RET(wg_stream(ctx, pair, st, &ws));
    RET(gemm(ctx, nd, h, Kw, Y0.o, nd, true, w_dx1, h, true, P.dwo, h, wm, ws));
  }
  CK(k_attn_bwd(L, L.plan.b, c.seq_len, L.n_loc, d, Y.qkv, Y.o, Y.lse, L.dout, dqkv, L.dsum, st, L.rope_cs));
  if (debug_sync()) { fprintf(stderr, "[malleus] attn bwd ..."); CK(cudaStreamSynchronize(st)); fprintf(stderr, " ok\n"); }
  if (!(L.rope_cs && attention_bwd_fuses_rope(c.seq_len, d)))
    CK(k_rope(L, T, c.seq_len, L.n_loc + L.kv_loc, d, dqkv, qkvw, c.rope_theta, true, st));
  RET(part_gemm(ctx, T, h, qkvw, dqkv, qkvw, false, P.wqkv, h, true, st));
  if (wg && tp_overlap(ctx)) {
    RET(tp_sum_begin(ctx, st));
    RET(gemm_co(ctx, qkvw, h, Kw, w_dqkv, qkvw, true, Y0.a1, h, true, P.dwqkv, h, wm, st));
    RET(tp_sum_end(ctx, st));
  } else {
    if (wg) {
      cudaStream_t ws;
      RET(wg_stream(ctx, pair, st, &ws));
      RET(gemm(ctx, qkvw, h, Kw, w_dqkv, qkvw, true, Y0.a1, h, true, P.dwqkv, h, wm, ws));
    }
    RET(tp_sum(ctx, st));
  }
  duty_begin(ctx, 5, st);
  CK(k_norm_bwd(L, T, h, S.x[li], P.g1, Y.r1, L.part, dx1, dx, P.dg1, L.scratch, st, tp_sum_bf16(L)));
  duty_end(ctx, st);
  return MALLEUS_OK;
}

// last stage: final norm, LM head, vocab-parallel CE, and the head's backward (dlast).
static malleus_status head_fwd_bwd(malleus_ctx* ctx, int si, const int32_t* tgt, bool first, cudaStream_t st,
                                   int pair = -1) {  // pair: as layer_bwd_impl (LM-head weight gradient)
  Layout& L = *ctx->L;
  const malleus_model_cfg& c = ctx->cfg;
  const int T = L.T, h = c.hidden, V = L.V_loc;
  Slot& S = L.slot[si];
  uint16_t* dlogits = pair >= 0 ? L.pdlogits + (size_t)si * T * V : L.dlogits;
  const bool wg = pair != 0;
  const int Kw = pair == 1 ? 2 * T : T;
  const uint16_t* w_dl = pair == 1 ? L.pdlogits : dlogits;
  const uint16_t* w_xf = pair == 1 ? L.slot[0].xf : S.xf;
  const PipeInfo& pp = L.plan.pipes[L.pipe];
  duty_begin(ctx, 6, st);
  CK(k_norm_fwd(L, T, h, S.x[L.n_local], nullptr, nullptr, L.gf, c.rms_eps, S.xf, S.rf, st));
  RET(gemm(ctx, T, V, h, S.xf, h, false, L.Wlm, h, false, L.logits, V, GEMM_STORE_F32, st));
  CK(ce_stats(T, V, L.logits, tgt, L.v0, L.stats, st));
  CK(ce_combine_max(T, L.stats, L.gmax, st));
  RET(tp_allreduce(ctx, L.gmax, (size_t)T, ncclMax, st));
  CK(ce_local_sum(T, L.stats, L.gmax, L.sumtgt, st));
  RET(tp_allreduce(ctx, L.sumtgt, (size_t)2 * T, ncclSum, st));
  duty_begin(ctx, 7, st);
  const double n_tok = (double)pp.n_micro * L.plan.b * c.seq_len;
  CK(ce_grad(T, V, L.logits, tgt, L.v0, L.gmax, L.sumtgt, L.sumtgt + T, (float)(1.0 / n_tok), dlogits,
             L.loss_rows, st, L.f32));
  if (L.member == 0)
    CK(reduce_loss(T, L.loss_rows, (float)(1.0 / ((double)L.plan.B * c.seq_len)), L.loss_acc, 1, st));
  RET(part_gemm(ctx, T, h, V, dlogits, V, false, L.Wlm, h, true, st));
  const int wm_lm = first ? GEMM_STORE_F32 : GEMM_ACCUM_F32;
  if (wg && tp_overlap(ctx)) {
    RET(tp_sum_begin(ctx, st));
    RET(gemm_co(ctx, V, h, Kw, w_dl, V, true, w_xf, h, true, L.dWlm, h, wm_lm, st));
    RET(tp_sum_end(ctx, st));
  } else {
    if (wg) {
      cudaStream_t ws;
      RET(wg_stream(ctx, pair, st, &ws));
      RET(gemm(ctx, V, h, Kw, w_dl, V, true, w_xf, h, true, L.dWlm, h, wm_lm, ws));
    }
    RET(tp_sum(ctx, st));
  }
  duty_begin(ctx, 8, st);
  CK(k_norm_bwd(L, T, h, S.x[L.n_local], L.gf, S.rf, L.part, nullptr, S.dlast, L.dgf, L.scratch, st, tp_sum_bf16(L)));
  duty_end(ctx, st);
  return MALLEUS_OK;
}

// ------------------------------------------------------------------ pipeline P2P
// forward: member r of stage j+1 receives from member (r mod TP_j) of stage j
static malleus_status pp_exchange(malleus_ctx* ctx, const uint16_t* send_fwd, uint16_t* recv_fwd,
                                  const uint16_t* send_bwd, uint16_t* recv_bwd, cudaStream_t st) {
  Layout& L = *ctx->L;
  const size_t n = (size_t)L.T * ctx->cfg.hidden;
  const ncclDataType_t adt = L.f32 ? ncclFloat : ncclBfloat16;
  if (!send_fwd && !recv_fwd && !send_bwd && !recv_bwd) return MALLEUS_OK;
  ev_begin(ctx, st, CAT_PP);
  NK(ncclGroupStart());
  if (send_fwd)
    for (size_t r = 0; r < L.next_ranks.size(); ++r)
      if ((int)(r % L.TP) == L.member) NK(ncclSend(send_fwd, n, adt, L.next_ranks[r], ctx->world_comm, st));
  if (recv_fwd)
    NK(ncclRecv(recv_fwd, n, adt, L.prev_ranks[L.member % L.prev_ranks.size()], ctx->world_comm, st));
  if (send_bwd)
    for (size_t q = 0; q < L.prev_ranks.size(); ++q)
      if ((int)(q % L.TP) == L.member) NK(ncclSend(send_bwd, n, adt, L.prev_ranks[q], ctx->world_comm, st));
  if (recv_bwd)
    NK(ncclRecv(recv_bwd, n, adt, L.next_ranks[L.member % L.next_ranks.size()], ctx->world_comm, st));
  NK(ncclGroupEnd());
  ev_end(ctx, st);
  return MALLEUS_OK;
}

// reduce + AdamW over the owned pieces: one fused pass, or with global-norm clipping two passes
// around a world all-reduce of the squared norm (collective either way when clipping)
static malleus_status reduce_and_update(malleus_ctx* ctx, const malleus_adam_cfg* a, cudaStream_t st) {
  Layout& L = *ctx->L;
  AdamHyper hp{a->lr, a->beta1, a->beta2, a->eps, a->weight_decay,
               (float)(1.0 - std::pow((double)a->beta1, a->step)), (float)(1.0 - std::pow((double)a->beta2, a->step)),
               a->apply_update};
  const int nc = (int)L.chunks.size();
  if (!(a->apply_update && a->max_grad_norm > 0.f)) {
    CK(reduce_adam(nc, L.d_chunks, L.d_pieces, hp, st));
    return MALLEUS_OK;
  }
  AdamHyper h1 = hp;  // pass 1: reduce into rgrad + per-chunk sum of G^2
  h1.apply = 0;
  h1.sq = L.d_sq;
  CK(reduce_adam(nc, L.d_chunks, L.d_pieces, h1, st));
  CK(sq_total(nc, L.d_sq, L.d_norm, st));  // nc == 0 -> 0
  NK(ncclAllReduce(L.d_norm, L.d_norm, 1, ncclDouble, ncclSum, ctx->world_comm, st));
  CK(clip_coef(L.d_norm, a->max_grad_norm, L.d_coef, L.d_coef + 1, st));
  AdamHyper h2 = hp;  // pass 2: AdamW on rgrad * coef, bf16 cast and push
  h2.apply = 3;
  h2.coef = L.d_coef;
  CK(reduce_adam(nc, L.d_chunks, L.d_pieces, h2, st));
  return MALLEUS_OK;
}

static malleus_status grad_sync_impl(malleus_ctx* ctx, const malleus_adam_cfg* a, cudaStream_t st) {
  Layout& L = *ctx->L;
  ev_begin(ctx, st, CAT_SYNC);
  if (L.p2p) {
    // peer-memory path: barrier (every rank's gradients final), fused reduce + AdamW reading the
    // other pipelines' gradient rows and storing the updated bf16 rows into every holder over
    // NVLink, barrier (all pushes landed; nobody still reads a gradient that the next step overwrites)
    float* bar = L.loss_acc + 2;
    NK(ncclAllReduce(bar, bar, 1, ncclFloat, ncclSum, ctx->world_comm, st));
    RET(reduce_and_update(ctx, a, st));
    NK(ncclAllReduce(bar, bar, 1, ncclFloat, ncclSum, ctx->world_comm, st));
    ev_end(ctx, st);
    return MALLEUS_OK;
  }
  if (!L.gops.empty()) {
    NK(ncclGroupStart());
    for (auto& o : L.gops) {
      if (o.send) NK(ncclSend(o.ptr, o.count, o.type, o.peer, ctx->world_comm, st));
      else NK(ncclRecv(o.ptr, o.count, o.type, o.peer, ctx->world_comm, st));
    }
    NK(ncclGroupEnd());
  }
  RET(reduce_and_update(ctx, a, st));
  if (a->apply_update && !L.pops.empty()) {
    NK(ncclGroupStart());
    for (auto& o : L.pops) {
      if (o.send) NK(ncclSend(o.ptr, o.count, o.type, o.peer, ctx->world_comm, st));
      else NK(ncclRecv(o.ptr, o.count, o.type, o.peer, ctx->world_comm, st));
    }
    NK(ncclGroupEnd());
  }
  ev_end(ctx, st);
  return MALLEUS_OK;
}

static malleus_status zero_grads(malleus_ctx* ctx, cudaStream_t st) {
  Layout& L = *ctx->L;
  for (TState& s : L.ts) {
    if (!s.held) continue;
    if (s.t.kind == SPLIT_REP) CK(cudaMemsetAsync(s.grad, 0, (s.rows.e - s.rows.b) * s.t.cols * 4, st));
  }
  return MALLEUS_OK;
}

static malleus_status train_step_impl(malleus_ctx* ctx, const int32_t* tokens, const int32_t* targets,
                                      float* loss_dev, const malleus_adam_cfg* adam, cudaStream_t st) {
  Layout& L = *ctx->L;
  const malleus_model_cfg& c = ctx->cfg;
  ctx->ev_used = 0;
  if (!ctx->step_beg) { cudaEventCreate(&ctx->step_beg); cudaEventCreate(&ctx->step_end); }
  cudaEventRecord(ctx->step_beg, st);
  CK(cudaMemsetAsync(L.loss_acc, 0, sizeof(float), st));
  if (!L.standby) {
    RET(zero_grads(ctx, st));
    const PipeInfo& pp = L.plan.pipes[L.pipe];
    const int m = pp.n_micro;
    int seq0 = 0;
    for (int i = 0; i < L.pipe; ++i) seq0 += L.plan.pipes[i].n_micro * L.plan.b;
    const long long s = c.seq_len;
    auto tok_mb = [&](int j) { return tokens + (seq0 + (long long)j * L.plan.b) * s; };
    auto tgt_mb = [&](int j) { return targets + (seq0 + (long long)j * L.plan.b) * s; };
    const int warm = std::min(L.PP - L.stage - 1, m);
    const int rem = m - warm;
    // pair mode (L.pair): micro-batches (2p, 2p + 1) share their weight-gradient GEMMs; an odd last one
    // runs alone.  pair_of(j) = -1 (alone), 0 (defer), 1 (flush the pair); first = the first GEMM that
    // writes the fp32 gradient (STORE), every later one accumulates.
    auto pair_of = [&](int j) { return !L.pair ? -1 : (j & 1) ? 1 : (j + 1 < m ? 0 : -1); };
    auto first_of = [&](int j) { return L.pair ? j <= 1 : j == 0; };
    auto fwd = [&](int j) -> malleus_status {
      const int si = j % L.slots;
      Slot& S = L.slot[si];
      RET(wg_join(ctx, st));  // the previous pair's side-stream wgrads read the slots this forward overwrites
      if (L.first) CK(k_embed_fwd(L, L.T, c.hidden, tok_mb(j), L.E, S.x[0], st));
      for (int li = 0; li < L.n_local; ++li) RET(layer_fwd_impl(ctx, li, si, st));
      if (L.last) RET(head_fwd_bwd(ctx, si, tgt_mb(j), first_of(j), st, pair_of(j)));
      return MALLEUS_OK;
    };
    // backward of micro-batch j; dy = grad of the stage output; returns grad of the stage input in *dx_out
    auto bwd = [&](int j, const uint16_t* dy, uint16_t** dx_out) -> malleus_status {
      const int si = j % L.slots;
      const uint16_t* cur = dy;
      uint16_t* bufs[2] = {L.dxa, L.dxb};
      int k = 0;
      for (int li = L.n_local - 1; li >= 0; --li) {
        // pair mode: layer li's input gradient is layer li-1's dy, kept in that layer's stash half
        uint16_t* out = (L.pair && li > 0) ? L.pdy[li - 1] + (size_t)si * L.T * c.hidden : bufs[k];
        k ^= 1;
        RET(layer_bwd_impl(ctx, li, si, cur, out, first_of(j), st, pair_of(j)));
        cur = out;
      }
      if (L.first) CK(k_embed_bwd(L, L.T, c.hidden, tok_mb(j), cur, L.dE, st));
      *dx_out = const_cast<uint16_t*>(cur);
      return MALLEUS_OK;
    };
    auto stage_dy = [&](int j) -> const uint16_t* { return L.last ? L.slot[j % L.slots].dlast : L.dyrecv; };
    for (int j = 0; j < warm; ++j) {
      if (!L.first) RET(pp_exchange(ctx, nullptr, L.slot[j % L.slots].x[0], nullptr, nullptr, st));
      RET(fwd(j));
      RET(pp_exchange(ctx, L.last ? nullptr : L.slot[j % L.slots].x[L.n_local], nullptr, nullptr, nullptr, st));
    }
    if (rem > 0 && !L.first) RET(pp_exchange(ctx, nullptr, L.slot[warm % L.slots].x[0], nullptr, nullptr, st));
    for (int i = 0; i < rem; ++i) {
      const int jf = warm + i;
      RET(fwd(jf));
      RET(pp_exchange(ctx, L.last ? nullptr : L.slot[jf % L.slots].x[L.n_local], nullptr, nullptr,
                      L.last ? nullptr : L.dyrecv, st));
      uint16_t* dx = nullptr;
      RET(bwd(i, stage_dy(i), &dx));
      if (i == rem - 1) {
        RET(pp_exchange(ctx, nullptr, nullptr, L.first ? nullptr : dx, nullptr, st));
      } else {
        RET(pp_exchange(ctx, nullptr, L.first ? nullptr : L.slot[(jf + 1) % L.slots].x[0], L.first ? nullptr : dx,
                        nullptr, st));
      }
    }
    for (int i = rem; i < m; ++i) {
      RET(pp_exchange(ctx, nullptr, nullptr, nullptr, L.last ? nullptr : L.dyrecv, st));
      uint16_t* dx = nullptr;
      RET(bwd(i, stage_dy(i), &dx));
      RET(pp_exchange(ctx, nullptr, nullptr, L.first ? nullptr : dx, nullptr, st));
    }
  }
  RET(wg_join(ctx, st));
  RET(grad_sync_impl(ctx, adam, st));
  // world loss: sum over pipelines of w_i * loss_i (only last-stage member 0 contributes)
  NK(ncclAllReduce(L.loss_acc, L.loss_acc, 1, ncclFloat, ncclSum, ctx->world_comm, st));
  if (loss_dev) CK(cudaMemcpyAsync(loss_dev, L.loss_acc, sizeof(float), cudaMemcpyDeviceToDevice, st));
  cudaEventRecord(ctx->step_end, st);
  ctx->have_timing = true;
  return MALLEUS_OK;
}

// ------------------------------------------------------------------ C-ABI
#define GUARD()                                                                \
  do {                                                                         \
    if (!ctx) return MALLEUS_E_ARG;                                            \
    if (ctx->sticky) return MALLEUS_E_STATE;                                   \
    cudaSetDevice(ctx->device);                                                \
  } while (0)
#define NEED_PLAN()                                                            \
  do {                                                                         \
    if (!ctx->L) return fail(ctx, MALLEUS_E_STATE, "no plan applied");         \
  } while (0)

extern "C" {

const char* malleus_version(void) { return "malleus-b200 0.2 (sm_100a)"; }

const char* malleus_last_error(const malleus_ctx* ctx) { return ctx ? ctx->err.c_str() : kNoCtx; }

malleus_status malleus_nccl_unique_id(uint8_t out[128]) {
  if (!out) return MALLEUS_E_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return MALLEUS_E_NCCL;
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  memcpy(out, &id, 128);
  return MALLEUS_OK;
}

malleus_status malleus_create(const malleus_model_cfg* cfg, int32_t rank, int32_t world, int32_t device,
                              const uint8_t nccl_uid[128], malleus_ctx** out) {
  if (!cfg || !out || !nccl_uid || rank < 0 || rank >= world) return MALLEUS_E_ARG;
  *out = nullptr;
  auto* ctx = new malleus_ctx();
  ctx->cfg = *cfg;
  ctx->rank = rank;
  ctx->world = world;
  ctx->device = device;
  if (cfg->hidden % 128 || cfg->head_dim % 32 || cfg->seq_len % 64 ||
      (cfg->dtype != MALLEUS_BF16 && cfg->dtype != MALLEUS_FP32)) {
    delete ctx;
    return MALLEUS_E_ARG;
  }
  if (cudaSetDevice(device) != cudaSuccess) { delete ctx; return MALLEUS_E_CUDA; }
  ncclUniqueId id;
  memcpy(&id, nccl_uid, 128);
  if (ncclCommInitRank(&ctx->world_comm, world, id, rank) != ncclSuccess) { delete ctx; return MALLEUS_E_NCCL; }
  *out = ctx;
  return MALLEUS_OK;
}

malleus_status malleus_set_slowdown(malleus_ctx* ctx, float x, int32_t mode);

// Failure detection and the failed state: see include/malleus.h.
malleus_status malleus_wait(malleus_ctx* ctx, void* stream, int32_t timeout_ms) {
  GUARD();
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaEvent_t ev;
  CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  CK(cudaEventRecord(ev, st));
  const auto t0 = std::chrono::steady_clock::now();
  auto elapsed_ms = [&] {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  };
  bool done = false;
  for (;;) {
    const cudaError_t q = cudaEventQuery(ev);
    if (q == cudaSuccess) { done = true; break; }
    if (q != cudaErrorNotReady) { cudaEventDestroy(ev); CK(q); }
    if (comm_status(false)) break;  // a device-side communication wait gave up
    if (timeout_ms > 0 && elapsed_ms() > timeout_ms) break;
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
  if (done && !comm_status(false)) {
    cudaEventDestroy(ev);
    return MALLEUS_OK;
  }
  // failure path: release our spin-waits (the abort word stays set: every later TP reduction of the
  // enqueued work gives up at once too).  NCCL communicators are not aborted here — ncclCommAbort
  // can block behind collectives that wait for the lost peer — and the failed context is not
  // reused: the process is expected to exit and the job to restart from the latest checkpoint
  // (PAPER.md:735), which process teardown makes safe for any kernel still waiting on the peer.
  const double waited = elapsed_ms();
  comm_abort(1u);
  cudaEventDestroy(ev);
  cudaGetLastError();
  ctx->sticky = true;
  ctx->failed = true;
  char msg[256];
  snprintf(msg, sizeof msg,
           "rank %d: communication did not complete within %.0f ms (PAPER.md:745 failure threshold); the context "
           "is failed: destroy it and resume the surviving GPUs from the latest checkpoint (PAPER.md:735)",
           ctx->rank, waited);
  ctx->err = msg;
  return MALLEUS_E_TIMEOUT;
}

malleus_status malleus_destroy(malleus_ctx* ctx) {
  if (!ctx) return MALLEUS_E_ARG;
  cudaSetDevice(ctx->device);
  if (ctx->failed) {  // host-side cleanup only: kernels may still wait on the lost peer (see malleus_wait)
    for (auto& e : ctx->ev_pool) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
    delete ctx;
    return MALLEUS_OK;
  }
  cudaDeviceSynchronize();
  cudaGetLastError();
  if (ctx->L) free_layout(ctx, ctx->L.get());
  if (ctx->world_comm) ncclCommDestroy(ctx->world_comm);
  for (auto& e : ctx->ev_pool) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
  if (ctx->step_beg) { cudaEventDestroy(ctx->step_beg); cudaEventDestroy(ctx->step_end); }
  if (ctx->tp_side) {
    cudaStreamSynchronize(ctx->tp_side);
    cudaStreamDestroy(ctx->tp_side);
    cudaEventDestroy(ctx->tp_ev_a);
    cudaEventDestroy(ctx->tp_ev_b);
  }
  if (ctx->wg_side) {
    cudaStreamSynchronize(ctx->wg_side);
    cudaStreamDestroy(ctx->wg_side);
    cudaEventDestroy(ctx->wg_fork_ev);
    cudaEventDestroy(ctx->wg_join_ev);
  }
  delete ctx;
  return MALLEUS_OK;
}

malleus_status malleus_plan_requirements(malleus_ctx* ctx, const malleus_plan* plan, malleus_requirements* out) {
  if (!ctx || !out) return MALLEUS_E_ARG;
  PlanInfo p;
  RET(check_plan(ctx, plan, &p));
  Layout L;
  build_shape(ctx->cfg, p, ctx->rank, L);
  assign(ctx->cfg, ctx->rank, L, 0, 0, 0);
  out->state = L.state_bytes;
  out->grads = L.grads_bytes;
  out->work = L.work_bytes;
  return MALLEUS_OK;
}

malleus_status malleus_plan_apply(malleus_ctx* ctx, const malleus_plan* plan, const malleus_arenas* arenas) {
  GUARD();
  PlanInfo p;
  RET(check_plan(ctx, plan, &p));
  auto L = std::make_unique<Layout>();
  build_shape(ctx->cfg, p, ctx->rank, *L);
  assign(ctx->cfg, ctx->rank, *L, 0, 0, 0);
  RET(bind_layout(ctx, *L, arenas));
  CK(cudaDeviceSynchronize());
  if (ctx->L) free_layout(ctx, ctx->L.get());
  ctx->L = std::move(L);
  duty_relearn(ctx);
  CK(cudaMemset(arenas->grads, 0, ctx->L->grads_bytes));
  return MALLEUS_OK;
}

static float bf16_to_f32(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

malleus_status malleus_write_tensor(malleus_ctx* ctx, int32_t tensor_id, int32_t kind, const void* host) {
  GUARD();
  NEED_PLAN();
  if (!host) return fail(ctx, MALLEUS_E_ARG, "host_full is NULL");
  Layout& L = *ctx->L;
  auto it = L.tix.find(tensor_id);
  if (it == L.tix.end()) return fail(ctx, MALLEUS_E_ARG, "unknown tensor id");
  TState& s = L.ts[it->second];
  const int64_t c = s.t.cols;
  if (kind == MALLEUS_KIND_PARAM) {  // bf16 bit patterns, or fp32 values in the parity mode
    const char* hb = static_cast<const char*>(host);
    if (s.held)
      CK(cudaMemcpy(s.param, hb + s.rows.b * c * L.aes, (s.rows.e - s.rows.b) * c * L.aes, cudaMemcpyHostToDevice));
    if (s.owned_elems) {
      std::vector<float> tmp(s.owned_elems);
      for (size_t i = 0; i < s.owned.size(); ++i)
        for (int64_t e = s.owned[i].e0; e < s.owned[i].e1; ++e)
          tmp[s.owned_off[i] + e - s.owned[i].e0] =
              L.f32 ? reinterpret_cast<const float*>(hb)[e] : bf16_to_f32(reinterpret_cast<const uint16_t*>(hb)[e]);
      CK(cudaMemcpy(s.master, tmp.data(), s.owned_elems * 4, cudaMemcpyHostToDevice));
      CK(cudaMemset(s.m, 0, s.owned_elems * 4));
      CK(cudaMemset(s.v, 0, s.owned_elems * 4));
    }
    return MALLEUS_OK;
  }
  if (kind != MALLEUS_KIND_MASTER && kind != MALLEUS_KIND_ADAM_M && kind != MALLEUS_KIND_ADAM_V)
    return fail(ctx, MALLEUS_E_ARG, "write_tensor: kind must be PARAM, MASTER, ADAM_M or ADAM_V");
  float* dst = kind == MALLEUS_KIND_MASTER ? s.master : kind == MALLEUS_KIND_ADAM_M ? s.m : s.v;
  if (s.owned.empty()) return MALLEUS_OK;  // this rank owns no piece of the tensor
  const float* h = static_cast<const float*>(host);
  for (size_t i = 0; i < s.owned.size(); ++i)
    CK(cudaMemcpy(dst + s.owned_off[i], h + s.owned[i].e0, (s.owned[i].e1 - s.owned[i].e0) * 4, cudaMemcpyHostToDevice));
  return MALLEUS_OK;
}

malleus_status malleus_read_local(malleus_ctx* ctx, int32_t tensor_id, int32_t kind, void* host_dst, int64_t* ranges,
                                  int32_t* n_ranges, int64_t* n_elems) {
  GUARD();
  NEED_PLAN();
  if (!n_ranges || !n_elems) return fail(ctx, MALLEUS_E_ARG, "n_ranges / n_elems NULL");
  Layout& L = *ctx->L;
  auto it = L.tix.find(tensor_id);
  if (it == L.tix.end()) return fail(ctx, MALLEUS_E_ARG, "unknown tensor id");
  TState& s = L.ts[it->second];
  const int64_t c = s.t.cols;
  std::vector<Range> rs;
  const void* src = nullptr;
  size_t esz = 4;
  if (kind == MALLEUS_KIND_PARAM || kind == MALLEUS_KIND_GRAD) {
    if (s.held) rs.push_back({s.rows.b * c, s.rows.e * c});
    src = kind == MALLEUS_KIND_PARAM ? (const void*)s.param : (const void*)s.grad;
    esz = kind == MALLEUS_KIND_PARAM ? (size_t)L.aes : 4;
  } else {
    for (auto& pc : s.owned) rs.push_back({pc.e0, pc.e1});
    src = kind == MALLEUS_KIND_MASTER ? s.master : kind == MALLEUS_KIND_ADAM_M ? s.m
        : kind == MALLEUS_KIND_ADAM_V ? s.v : kind == MALLEUS_KIND_RGRAD ? s.rgrad : nullptr;
    if (kind < MALLEUS_KIND_MASTER || kind > MALLEUS_KIND_RGRAD) return fail(ctx, MALLEUS_E_ARG, "bad kind");
  }
  int64_t tot = 0;
  for (auto& r : rs) tot += r.e - r.b;
  const int cap = *n_ranges;
  *n_ranges = (int32_t)rs.size();
  *n_elems = tot;
  if (!host_dst) return MALLEUS_OK;
  if ((int)rs.size() > cap || !ranges) return fail(ctx, MALLEUS_E_ARG, "ranges capacity too small");
  for (size_t i = 0; i < rs.size(); ++i) { ranges[2 * i] = rs[i].b; ranges[2 * i + 1] = rs[i].e; }
  if (tot) CK(cudaDeviceSynchronize());
  if (tot) CK(cudaMemcpy(host_dst, src, tot * esz, cudaMemcpyDeviceToHost));
  return MALLEUS_OK;
}

malleus_status malleus_layer_fwd(malleus_ctx* ctx, int32_t layer, int32_t slot, const void* x_in, void* x_out,
                                 void* stream) {
  GUARD();
  NEED_PLAN();
  Layout& L = *ctx->L;
  if (L.standby || layer < L.lb || layer >= L.le || slot < 0 || slot >= L.slots || !x_in || !x_out)
    return fail(ctx, MALLEUS_E_ARG, "layer not held by this rank or bad slot / pointers");
  cudaStream_t st = (cudaStream_t)stream;
  const int li = layer - L.lb;
  const size_t bytes = (size_t)L.T * ctx->cfg.hidden * L.aes;
  CK(cudaMemcpyAsync(L.slot[slot].x[li], x_in, bytes, cudaMemcpyDeviceToDevice, st));
  RET(layer_fwd_impl(ctx, li, slot, st));
  CK(cudaMemcpyAsync(x_out, L.slot[slot].x[li + 1], bytes, cudaMemcpyDeviceToDevice, st));
  return MALLEUS_OK;
}

malleus_status malleus_layer_bwd(malleus_ctx* ctx, int32_t layer, int32_t slot, const void* dy, void* dx,
                                 void* stream) {
  GUARD();
  NEED_PLAN();
  Layout& L = *ctx->L;
  if (L.standby || layer < L.lb || layer >= L.le || slot < 0 || slot >= L.slots || !dy || !dx)
    return fail(ctx, MALLEUS_E_ARG, "layer not held by this rank or bad slot / pointers");
  cudaStream_t st = (cudaStream_t)stream;
  RET(layer_bwd_impl(ctx, layer - L.lb, slot, (const uint16_t*)dy, L.dxb == dx ? L.dxa : L.dxb, false, st));
  CK(cudaMemcpyAsync(dx, L.dxb == dx ? L.dxa : L.dxb, (size_t)L.T * ctx->cfg.hidden * L.aes, cudaMemcpyDeviceToDevice, st));
  return MALLEUS_OK;
}

malleus_status malleus_train_step(malleus_ctx* ctx, const int32_t* tokens, const int32_t* targets, float* loss_dev,
                                  const malleus_adam_cfg* adam, void* stream) {
  GUARD();
  NEED_PLAN();
  if (!tokens || !targets || !adam || adam->step < 1) return fail(ctx, MALLEUS_E_ARG, "tokens/targets/adam");
  return train_step_impl(ctx, tokens, targets, loss_dev, adam, (cudaStream_t)stream);
}

malleus_status malleus_grad_sync(malleus_ctx* ctx, const malleus_adam_cfg* adam, void* stream) {
  GUARD();
  NEED_PLAN();
  if (!adam || adam->step < 1) return fail(ctx, MALLEUS_E_ARG, "adam cfg");
  ctx->ev_used = 0;
  return grad_sync_impl(ctx, adam, (cudaStream_t)stream);
}

malleus_status malleus_zero_grads(malleus_ctx* ctx, void* stream) {
  GUARD();
  NEED_PLAN();
  for (TState& s : ctx->L->ts)
    if (s.held) CK(cudaMemsetAsync(s.grad, 0, (s.rows.e - s.rows.b) * s.t.cols * 4, (cudaStream_t)stream));
  return MALLEUS_OK;
}

malleus_status malleus_last_step_timing(malleus_ctx* ctx, float out[5]) {
  GUARD();
  if (!out) return MALLEUS_E_ARG;
  for (int i = 0; i < 5; ++i) out[i] = 0.f;
  if (!ctx->have_timing) return fail(ctx, MALLEUS_E_STATE, "no step timed yet");
  CK(cudaEventSynchronize(ctx->step_end));
  float tot = 0.f;
  cudaEventElapsedTime(&tot, ctx->step_beg, ctx->step_end);
  for (size_t i = 0; i < ctx->ev_used; ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev_pool[i].first, ctx->ev_pool[i].second);
    out[ctx->ev_cat[i]] += ms;
  }
  out[4] = tot;
  out[0] = tot - out[1] - out[2] - out[3];
  return MALLEUS_OK;
}

malleus_status malleus_last_grad_norm(malleus_ctx* ctx, float* norm, float* coef) {
  GUARD();
  NEED_PLAN();
  if (!norm) return MALLEUS_E_ARG;
  float h[2] = {0.f, 1.f};
  if (ctx->L->d_coef) CK(cudaMemcpy(h, ctx->L->d_coef, sizeof(h), cudaMemcpyDeviceToHost));
  *norm = h[1];
  if (coef) *coef = h[0];
  return MALLEUS_OK;
}

// ------------------------------------------------------------------ migration
malleus_status malleus_migrate(malleus_ctx* ctx, const malleus_plan* new_plan, const malleus_arenas* new_arenas,
                               malleus_migrate_stats* stats) {
  GUARD();
  NEED_PLAN();
  PlanInfo np;
  RET(check_plan(ctx, new_plan, &np));
  auto NL = std::make_unique<Layout>();
  build_shape(ctx->cfg, np, ctx->rank, *NL);
  assign(ctx->cfg, ctx->rank, *NL, 0, 0, 0);
  RET(bind_layout(ctx, *NL, new_arenas));
  CK(cudaMemset(new_arenas->grads, 0, NL->grads_bytes));
  CK(cudaDeviceSynchronize());
  Layout& O = *ctx->L;
  const int me = ctx->rank;
  const auto t0 = std::chrono::steady_clock::now();
  // pointer of flat element e of tensor (kind) in a layout; nullptr if not resident
  auto locate_ptr = [](Layout& Lx, int32_t tid, int kind, int64_t e, size_t* esz) -> char* {
    TState& s = Lx.ts[Lx.tix[tid]];
    if (kind == MALLEUS_KIND_PARAM) {
      *esz = (size_t)Lx.aes;
      if (!s.held) return nullptr;
      return reinterpret_cast<char*>(param_at(Lx, s, e));
    }
    *esz = 4;
    for (size_t i = 0; i < s.owned.size(); ++i)
      if (s.owned[i].e0 <= e && e < s.owned[i].e1) {
        float* base = kind == MALLEUS_KIND_MASTER ? s.master : kind == MALLEUS_KIND_ADAM_M ? s.m : s.v;
        return reinterpret_cast<char*>(base + s.owned_off[i] + (e - s.owned[i].e0));
      }
    return nullptr;
  };
  cudaStream_t st = 0;
  uint64_t sent = 0, recvd = 0;
  constexpr long long CHUNK = COPY_CHUNK;
  auto add_copy = [&](std::vector<CopyDesc>& v, const char* s, char* d, long long bytes) {
    for (long long o = 0; o < bytes; o += CHUNK) v.push_back({s + o, d + o, std::min(CHUNK, bytes - o)});
  };
  auto pad16 = [](long long b) { return (b + 15) / 16 * 16; };
  // (1) keep-copies: everything this rank needs and already has (old arena -> new arena)
  std::vector<CopyDesc> keep;
  for (TState& ns : NL->ts) {
    const int64_t c = ns.t.cols;
    if (ns.held) {
      Range orow;
      if (held_rows(ctx->cfg, O.plan, ns.t, me, &orow)) {
        const int64_t lo = std::max(ns.rows.b, orow.b), hi = std::min(ns.rows.e, orow.e);
        if (hi > lo) {
          size_t es;
          char* src = locate_ptr(O, ns.t.id, MALLEUS_KIND_PARAM, lo * c, &es);
          char* dst = locate_ptr(*NL, ns.t.id, MALLEUS_KIND_PARAM, lo * c, &es);
          add_copy(keep, src, dst, (hi - lo) * c * NL->aes);
        }
      }
    }
    TState& os = O.ts[O.tix[ns.t.id]];
    for (size_t i = 0; i < ns.owned.size(); ++i)
      for (size_t j = 0; j < os.owned.size(); ++j) {
        const int64_t lo = std::max(ns.owned[i].e0, os.owned[j].e0), hi = std::min(ns.owned[i].e1, os.owned[j].e1);
        if (hi <= lo) continue;
        for (int kind : {MALLEUS_KIND_MASTER, MALLEUS_KIND_ADAM_M, MALLEUS_KIND_ADAM_V}) {
          size_t es;
          char* src = locate_ptr(O, ns.t.id, kind, lo, &es);
          char* dst = locate_ptr(*NL, ns.t.id, kind, lo, &es);
          add_copy(keep, src, dst, (hi - lo) * 4);
        }
      }
  }
  if (O.p2p) {
    // peer-memory path: every rank pulls its deltas straight from the sources' old arenas over
    // NVLink (no packing, no staging), in the same launch as its keep-copies, then a barrier so
    // no rank frees an old arena that a peer is still reading.
    const auto trp = migration_transfers(ctx->cfg, O.plan, np);
    std::vector<CopyDesc> descs = keep;
    // large remote ranges go to the copy engines (one cudaMemcpyAsync each, on a side stream, in
    // parallel with the SM kernel doing the keep-copies and the small pulls); MALLEUS_MIGRATE_CE=0
    // keeps every pull in the SM kernel
    static const long long ce_min = [] {
      const char* e = getenv("MALLEUS_MIGRATE_CE");
      return e && atoi(e) == 0 ? -1LL : (1LL << 20);
    }();
    struct CeCopy { const char* src; char* dst; long long bytes; };
    std::vector<CeCopy> ce;
    for (auto& t : trp) {
      if (t.dst != me) {
        if (t.src == me) sent += (t.e1 - t.e0) * (t.kind == MALLEUS_KIND_PARAM ? O.aes : 4);
        continue;
      }
      size_t es;
      const char* src = locate_ptr(*O.peer[t.src], t.tensor, t.kind, t.e0, &es);
      char* dst = locate_ptr(*NL, t.tensor, t.kind, t.e0, &es);
      const long long bytes = (t.e1 - t.e0) * (long long)es;
      if (ce_min > 0 && bytes >= ce_min) ce.push_back({src, dst, bytes});
      else add_copy(descs, src, dst, bytes);
      recvd += (t.e1 - t.e0) * es;
    }
    CopyDesc* d_desc = nullptr;
    if (!descs.empty()) {
      CK(cudaMalloc(&d_desc, descs.size() * sizeof(CopyDesc)));
      CK(cudaMemcpy(d_desc, descs.data(), descs.size() * sizeof(CopyDesc), cudaMemcpyHostToDevice));
    }
    float* bar = NL->loss_acc + 2;
    CK(cudaMemsetAsync(bar, 0, sizeof(float), st));
    NK(ncclAllReduce(bar, bar, 1, ncclFloat, ncclSum, ctx->world_comm, st));  // everyone ready
    CK(cudaStreamSynchronize(st));
    const auto t1 = std::chrono::steady_clock::now();
    if (!ce.empty()) {
      if (!ctx->tp_side) {
        CK(cudaStreamCreateWithFlags(&ctx->tp_side, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&ctx->tp_ev_a, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ctx->tp_ev_b, cudaEventDisableTiming));
      }
      CK(cudaEventRecord(ctx->tp_ev_a, st));
      CK(cudaStreamWaitEvent(ctx->tp_side, ctx->tp_ev_a, 0));
      for (const CeCopy& c : ce) CK(cudaMemcpyAsync(c.dst, c.src, (size_t)c.bytes, cudaMemcpyDeviceToDevice, ctx->tp_side));
      CK(cudaEventRecord(ctx->tp_ev_b, ctx->tp_side));
    }
    CK(copy_ranges((int)descs.size(), d_desc, st));
    if (!ce.empty()) CK(cudaStreamWaitEvent(st, ctx->tp_ev_b, 0));
    NK(ncclAllReduce(bar, bar, 1, ncclFloat, ncclSum, ctx->world_comm, st));  // everyone done reading
    CK(cudaStreamSynchronize(st));
    const double xfer = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
    if (d_desc) cudaFree(d_desc);
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    free_layout(ctx, ctx->L.get());
    ctx->L = std::move(NL);
    duty_relearn(ctx);
    if (stats) {
      stats->bytes_sent = sent;
      stats->bytes_recv = recvd;
      stats->seconds = xfer;
      stats->n_packs = 0;  // peer pull: nothing is packed
      stats->total_seconds = secs;
    }
    return MALLEUS_OK;
  }
  // (2) remote deltas in packs of 4 consecutive layers: per pack and peer, the
  // outgoing ranges are packed into one contiguous buffer (K11 pack), exchanged with one grouped
  // NCCL send / recv per peer, and unpacked into the new layout.  Every rank derives the same
  // transfer list (layout.cpp), so pack offsets agree on both sides.
  const auto tr = migration_transfers(ctx->cfg, O.plan, np);
  const int L_ = ctx->cfg.n_layers;
  const int n_packs = std::max(1, (L_ + 3) / 4);
  auto pack_of = [&](int32_t tid) {
    if (tid == MALLEUS_T_EMBED) return 0;
    if (tid >= MALLEUS_T_EMBED) return n_packs - 1;
    return (tid / 16) / 4;
  };
  struct PeerBuf {
    long long off = 0, bytes = 0;
  };
  struct Pack {
    std::map<int, PeerBuf> send, recv;
    long long send_bytes = 0, recv_bytes = 0;
    size_t pack_d0 = 0, pack_d1 = 0, unpack_d0 = 0, unpack_d1 = 0;
  };
  std::vector<Pack> packs(n_packs);
  std::vector<CopyDesc> descs = keep;
  // sizes per peer first (canonical order), then descriptors
  for (auto& t : tr) {
    size_t es = t.kind == MALLEUS_KIND_PARAM ? (size_t)O.aes : 4;
    const long long b = (t.e1 - t.e0) * (long long)es;
    Pack& P = packs[pack_of(t.tensor)];
    if (t.src == me) P.send[t.dst].bytes += pad16(b);
    if (t.dst == me) P.recv[t.src].bytes += pad16(b);
  }
  long long max_send = 0, max_recv = 0;
  for (Pack& P : packs) {
    for (auto& kv : P.send) { kv.second.off = P.send_bytes; P.send_bytes += kv.second.bytes; }
    for (auto& kv : P.recv) { kv.second.off = P.recv_bytes; P.recv_bytes += kv.second.bytes; }
    max_send = std::max(max_send, P.send_bytes);
    max_recv = std::max(max_recv, P.recv_bytes);
  }
  char *sbuf = nullptr, *rbuf = nullptr;
  if (max_send) CK(cudaMalloc(&sbuf, max_send));
  if (max_recv) CK(cudaMalloc(&rbuf, max_recv));
  for (int pk = 0; pk < n_packs; ++pk) {
    Pack& P = packs[pk];
    std::map<int, long long> scur, rcur;
    for (auto& kv : P.send) scur[kv.first] = kv.second.off;
    for (auto& kv : P.recv) rcur[kv.first] = kv.second.off;
    P.pack_d0 = descs.size();
    for (auto& t : tr) {
      if (pack_of(t.tensor) != pk || t.src != me) continue;
      size_t es;
      const char* p = locate_ptr(O, t.tensor, t.kind, t.e0, &es);
      const long long b = (t.e1 - t.e0) * (long long)es;
      add_copy(descs, p, sbuf + scur[t.dst], b);
      scur[t.dst] += pad16(b);
      sent += b;
    }
    P.pack_d1 = P.unpack_d0 = descs.size();
    for (auto& t : tr) {
      if (pack_of(t.tensor) != pk || t.dst != me) continue;
      size_t es;
      char* p = locate_ptr(*NL, t.tensor, t.kind, t.e0, &es);
      const long long b = (t.e1 - t.e0) * (long long)es;
      add_copy(descs, rbuf + rcur[t.src], p, b);
      rcur[t.src] += pad16(b);
      recvd += b;
    }
    P.unpack_d1 = descs.size();
  }
  CopyDesc* d_desc = nullptr;
  if (!descs.empty()) {
    CK(cudaMalloc(&d_desc, descs.size() * sizeof(CopyDesc)));
    CK(cudaMemcpy(d_desc, descs.data(), descs.size() * sizeof(CopyDesc), cudaMemcpyHostToDevice));
  }
  CK(cudaDeviceSynchronize());
  const auto t1 = std::chrono::steady_clock::now();
  CK(copy_ranges((int)keep.size(), d_desc, st));
  for (int pk = 0; pk < n_packs; ++pk) {
    Pack& P = packs[pk];
    CK(copy_ranges((int)(P.pack_d1 - P.pack_d0), d_desc + P.pack_d0, st));
    if (!P.send.empty() || !P.recv.empty()) {
      NK(ncclGroupStart());
      for (auto& kv : P.send) NK(ncclSend(sbuf + kv.second.off, kv.second.bytes, ncclUint8, kv.first, ctx->world_comm, st));
      for (auto& kv : P.recv) NK(ncclRecv(rbuf + kv.second.off, kv.second.bytes, ncclUint8, kv.first, ctx->world_comm, st));
      NK(ncclGroupEnd());
    }
    CK(copy_ranges((int)(P.unpack_d1 - P.unpack_d0), d_desc + P.unpack_d0, st));
  }
  CK(cudaStreamSynchronize(st));
  const double xfer_secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
  if (d_desc) cudaFree(d_desc);
  if (sbuf) cudaFree(sbuf);
  if (rbuf) cudaFree(rbuf);
  const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  free_layout(ctx, ctx->L.get());
  ctx->L = std::move(NL);
  duty_relearn(ctx);
  if (stats) {
    stats->bytes_sent = sent;
    stats->bytes_recv = recvd;
    stats->seconds = xfer_secs;
    stats->n_packs = n_packs;
    stats->total_seconds = secs;
  }
  return MALLEUS_OK;
}

// ------------------------------------------------------------------ probe / straggler emulation
malleus_status malleus_probe_speed(malleus_ctx* ctx, int32_t iters, float* ms_per_rank) {
  GUARD();
  if (!ms_per_rank || iters < 1) return MALLEUS_E_ARG;
  const int n = 4096;
  void *a = nullptr, *b = nullptr, *cbuf = nullptr;
  float* dev = nullptr;
  CK(cudaMalloc(&a, (size_t)n * n * 2));
  CK(cudaMalloc(&b, (size_t)n * n * 2));
  CK(cudaMalloc(&cbuf, (size_t)n * n * 2));
  CK(cudaMalloc(&dev, ctx->world * sizeof(float)));
  CK(cudaMemset(a, 0, (size_t)n * n * 2));
  CK(cudaMemset(b, 0, (size_t)n * n * 2));
  cudaStream_t st = 0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  GemmDesc g{n, n, n, a, n, false, b, n, false, cbuf, n, GEMM_STORE_BF16};
  // warm-up (also primes the DUTY timer of the probe segment so the emulated slowdown applies)
  for (int i = 0; i < 6; ++i) {
    duty_begin(ctx, 9, st);
    CK(gemm_bf16(g, st));
    CK(probe_copy((long long)n * n / 2, (const float*)a, (float*)cbuf, st));
    duty_end(ctx, st);
    if (i == 2) CK(cudaStreamSynchronize(st));
  }
  CK(cudaStreamSynchronize(st));
  // median of 5 rounds of `iters` iterations: robust against a clock excursion in one round (a
  // uniform cluster must read x = 1 +- 2%, SURVEY §8(c) probe pin)
  std::vector<float> rounds;
  for (int rd = 0; rd < 5; ++rd) {
    cudaEventRecord(e0, st);
    for (int i = 0; i < iters; ++i) {
      duty_begin(ctx, 9, st);
      CK(gemm_bf16(g, st));
      CK(probe_copy((long long)n * n / 2, (const float*)a, (float*)cbuf, st));
      duty_end(ctx, st);
    }
    cudaEventRecord(e1, st);
    CK(cudaEventSynchronize(e1));
    float t = 0.f;
    cudaEventElapsedTime(&t, e0, e1);
    rounds.push_back(t / iters);
  }
  std::sort(rounds.begin(), rounds.end());
  float ms = rounds[rounds.size() / 2];
  CK(cudaMemcpy(dev + ctx->rank, &ms, 4, cudaMemcpyHostToDevice));
  NK(ncclAllGather(dev + ctx->rank, dev, 1, ncclFloat, ctx->world_comm, st));
  CK(cudaStreamSynchronize(st));
  CK(cudaMemcpy(ms_per_rank, dev, ctx->world * sizeof(float), cudaMemcpyDeviceToHost));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(a);
  cudaFree(b);
  cudaFree(cbuf);
  cudaFree(dev);
  return MALLEUS_OK;
}

malleus_status malleus_set_slowdown(malleus_ctx* ctx, float x, int32_t mode) {
  if (!ctx) return MALLEUS_E_ARG;
  cudaSetDevice(ctx->device);
  if (x < 1.f || mode < 0 || mode > 2) return fail(ctx, MALLEUS_E_ARG, "x >= 1, mode in {0,1,2}");
  if (mode == 1)
    return fail(ctx, MALLEUS_E_ARG,
                "HOG mode is not available: a resident SM-occupying kernel deadlocks any device-wide "
                "synchronisation (cudaDeviceSynchronize / cudaFree) of the process; use DUTY (2)");
  ctx->slowdown = x;
  ctx->slow_mode = mode;
  for (auto& d : ctx->duty) { d.ms = -1.0; d.n = 0; }
  return MALLEUS_OK;
}

}  // extern "C"
