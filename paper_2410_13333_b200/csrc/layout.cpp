// Host-side plan validation and state placement (see layout.h).  Range arithmetic only; the
// per-element definitions it must agree with live in oracle/layout.py (tests compare them).
#include "layout.h"

#include <algorithm>
#include <set>
#include <sstream>

namespace mls {

PlanInfo plan_from_c(const malleus_plan* p) {
  PlanInfo out;
  out.plan_id = p->plan_id;
  out.b = p->micro_batch;
  out.B = p->global_batch;
  for (int i = 0; i < p->dp; ++i) {
    PipeInfo pi;
    pi.n_micro = p->pipes[i].n_micro;
    for (int j = 0; j < p->pipes[i].n_stages; ++j) {
      const malleus_stage& s = p->pipes[i].stages[j];
      StageInfo si;
      si.ranks.assign(s.ranks, s.ranks + s.n_members);
      si.heads.assign(s.heads, s.heads + s.n_members);
      si.ffn.assign(s.ffn_cols, s.ffn_cols + s.n_members);
      si.vocab.assign(s.vocab_rows, s.vocab_rows + s.n_members);
      si.lb = s.layer_begin;
      si.le = s.layer_end;
      pi.stages.push_back(std::move(si));
    }
    out.pipes.push_back(std::move(pi));
  }
  if (p->n_standby > 0) out.standby.assign(p->standby, p->standby + p->n_standby);
  return out;
}

std::string validate_plan(const malleus_model_cfg& cfg, const PlanInfo& p, int world) {
  std::ostringstream e;
  if (cfg.n_kv_heads < 1 || cfg.n_heads % cfg.n_kv_heads)
    return "n_kv_heads must divide n_heads (MHA: n_kv_heads == n_heads; GQA: whole query-head groups)";
  const int grp = cfg.n_heads / cfg.n_kv_heads;  // query heads per KV head
  if (cfg.hidden != cfg.n_heads * cfg.head_dim) return "hidden must equal n_heads * head_dim";
  if (p.b < 1 || p.B < 1 || p.pipes.empty()) return "b >= 1, B >= 1, DP >= 1";
  if (p.pipes.size() > 8) return "DP <= 8";
  if (world < 1 || world > 16) return "world <= 16 (peer tables hold at most 15 other holders)";
  long long tot = 0;
  for (auto& pp : p.pipes) {
    if (pp.n_micro < 0) return "m_i >= 0";
    tot += pp.n_micro;
  }
  if (tot * p.b != p.B) return "sum_i m_i * b == B violated (Eq.1, PAPER.md:523)";
  std::set<int> seen;
  for (size_t i = 0; i < p.pipes.size(); ++i) {
    auto& pp = p.pipes[i];
    if (pp.stages.empty()) return "pipeline with no stage";
    int nxt = 0;
    for (auto& st : pp.stages) {
      if (st.lb != nxt || st.le <= st.lb)
        return "stage layer ranges must partition [0, L) in stage order with l_ij >= 1 (PAPER.md:524, 556)";
      nxt = st.le;
      const size_t k = st.ranks.size();
      if (k < 1) return "empty stage";
      if (k > 16) return "TP degree <= 16 (MAX_TP)";
      if (st.heads.size() != k || st.ffn.size() != k || st.vocab.size() != k)
        return "split vectors need one entry per member";
      long long sh = 0, sf = 0, sv = 0;
      for (size_t m = 0; m < k; ++m) {
        if (st.heads[m] < 1) return "every member needs >= 1 head (zero-work GPUs are standby, PAPER.md:556)";
        if (st.heads[m] % grp) return "GQA: every member holds whole KV groups (heads split in multiples of n_heads / n_kv_heads)";
        if (st.ffn[m] < 16 || st.ffn[m] % 16) return "ffn split entries must be >= 16 and multiples of 16";
        if (st.vocab[m] < 16 || st.vocab[m] % 16) return "vocab split entries must be >= 16 and multiples of 16";
        sh += st.heads[m]; sf += st.ffn[m]; sv += st.vocab[m];
      }
      if (sh != cfg.n_heads) return "heads split must sum to n_heads";
      if (sf != cfg.ffn) return "ffn split must sum to ffn";
      if (sv != cfg.vocab) return "vocab split must sum to vocab";
      for (int r : st.ranks) {
        if (r < 0 || r >= world || seen.count(r)) {
          e << "rank " << r << " repeated or out of range";
          return e.str();
        }
        seen.insert(r);
      }
    }
    if (nxt != cfg.n_layers) return "stage layer ranges must cover [0, L) (PAPER.md:524)";
  }
  for (int r : p.standby) {
    if (r < 0 || r >= world || seen.count(r)) {
      e << "standby rank " << r << " also in a stage or out of range (PAPER.md:556)";
      return e.str();
    }
    seen.insert(r);
  }
  if ((int)seen.size() != world) return "every rank of [0, world) must be in exactly one stage or standby";
  return "";
}

std::string check_kernel_limits(const malleus_model_cfg& cfg, const PlanInfo& p) {
  // checked before any rank starts a plan the step cannot run (a kernel would fail mid-step on some
  // ranks while their peers block in a collective): embedding backward keeps the micro-batch's
  // token ids in shared memory (T = b*s <= 8192), RMSNorm and the TP reduction keep a row in
  // registers (h <= 8192, h % 128 for the GEMM tiles), attention has kernels for head_dim 32, 64
  // and 128 and sequence lengths in multiples of 64
  if ((long long)p.b * cfg.seq_len > 8192) return "b * seq_len must be <= 8192 (embedding backward)";
  if (cfg.hidden > 8192 || cfg.hidden % 128) return "hidden must be a multiple of 128 and <= 8192";
  if (cfg.head_dim != 32 && cfg.head_dim != 64 && cfg.head_dim != 128) return "head_dim must be 32, 64 or 128";
  if (cfg.seq_len % 64 || cfg.seq_len < 64) return "seq_len must be a multiple of 64";
  return "";
}

std::vector<TensorInfo> all_tensors(const malleus_model_cfg& c) {
  std::vector<TensorInfo> v;
  const int64_t h = c.hidden, nd = (int64_t)c.n_heads * c.head_dim, F = c.ffn, V = c.vocab;
  const int64_t kd = (int64_t)c.n_kv_heads * c.head_dim;  // W_k / W_v rows (GQA: n_kv heads)
  for (int l = 0; l < c.n_layers; ++l) {
    const int32_t b = l * 16;
    v.push_back({b + LT_G1, l, LT_G1, h, 1, SPLIT_REP, false});
    v.push_back({b + LT_WQ, l, LT_WQ, nd, h, SPLIT_HEADS, true});
    v.push_back({b + LT_WK, l, LT_WK, kd, h, SPLIT_HEADS, true});
    v.push_back({b + LT_WV, l, LT_WV, kd, h, SPLIT_HEADS, true});
    v.push_back({b + LT_WO, l, LT_WO, nd, h, SPLIT_HEADS, true});
    v.push_back({b + LT_G2, l, LT_G2, h, 1, SPLIT_REP, false});
    v.push_back({b + LT_WG, l, LT_WG, F, h, SPLIT_FFN, true});
    v.push_back({b + LT_WU, l, LT_WU, F, h, SPLIT_FFN, true});
    v.push_back({b + LT_WD, l, LT_WD, F, h, SPLIT_FFN, true});
  }
  v.push_back({MALLEUS_T_EMBED, -1, 0, V, h, SPLIT_REP, true});
  v.push_back({MALLEUS_T_FINAL_NORM, -1, 1, h, 1, SPLIT_REP, false});
  v.push_back({MALLEUS_T_LM_HEAD, -1, 2, V, h, SPLIT_VOCAB, true});
  return v;
}

bool tensor_info(const malleus_model_cfg& c, int32_t id, TensorInfo* out) {
  if (id >= MALLEUS_T_EMBED && id <= MALLEUS_T_LM_HEAD) {
    auto v = all_tensors(c);
    *out = v[v.size() - 3 + (id - MALLEUS_T_EMBED)];
    return true;
  }
  const int l = id / 16, k = id % 16;
  if (id < 0 || l >= c.n_layers || k >= LT_COUNT) return false;
  *out = all_tensors(c)[l * LT_COUNT + k];
  return true;
}

int stage_of(const malleus_model_cfg& cfg, const PipeInfo& pipe, const TensorInfo& t) {
  if (t.layer < 0) return t.idx == 0 ? 0 : (int)pipe.stages.size() - 1;
  for (size_t j = 0; j < pipe.stages.size(); ++j)
    if (pipe.stages[j].lb <= t.layer && t.layer < pipe.stages[j].le) return (int)j;
  return -1;
}

Range member_rows(const malleus_model_cfg& cfg, const StageInfo& st, const TensorInfo& t, int k) {
  if (t.kind == SPLIT_REP) return {0, t.rows};
  const std::vector<int>& v = t.kind == SPLIT_HEADS ? st.heads : (t.kind == SPLIT_FFN ? st.ffn : st.vocab);
  int64_t unit = t.kind == SPLIT_HEADS ? cfg.head_dim : 1;
  int64_t div = 1;
  if (t.kind == SPLIT_HEADS && (t.idx == LT_WK || t.idx == LT_WV)) div = cfg.n_heads / cfg.n_kv_heads;  // KV groups
  int64_t r0 = 0;
  for (int i = 0; i < k; ++i) r0 += v[i];
  return {r0 / div * unit, (r0 + v[k]) / div * unit};
}

void locate(const PlanInfo& p, int rank, int* pipe, int* stage, int* member) {
  *pipe = *stage = *member = -1;
  for (size_t i = 0; i < p.pipes.size(); ++i)
    for (size_t j = 0; j < p.pipes[i].stages.size(); ++j)
      for (size_t k = 0; k < p.pipes[i].stages[j].ranks.size(); ++k)
        if (p.pipes[i].stages[j].ranks[k] == rank) { *pipe = (int)i; *stage = (int)j; *member = (int)k; return; }
}

bool held_rows(const malleus_model_cfg& cfg, const PlanInfo& p, const TensorInfo& t, int rank, Range* rows) {
  int pi, sj, mk;
  locate(p, rank, &pi, &sj, &mk);
  if (pi < 0) return false;
  if (stage_of(cfg, p.pipes[pi], t) != sj) return false;
  *rows = member_rows(cfg, p.pipes[pi].stages[sj], t, mk);
  return true;
}

int sync_holder(const malleus_model_cfg& cfg, const PipeInfo& pipe, const TensorInfo& t, int64_t row) {
  const StageInfo& st = pipe.stages[stage_of(cfg, pipe, t)];
  if (t.kind == SPLIT_REP) return st.ranks[0];
  for (size_t k = 0; k < st.ranks.size(); ++k) {
    Range r = member_rows(cfg, st, t, (int)k);
    if (r.b <= row && row < r.e) return st.ranks[k];
  }
  return -1;
}

static std::vector<int64_t> refinement(const malleus_model_cfg& cfg, const PlanInfo& p, const TensorInfo& t) {
  std::set<int64_t> cuts{0, t.rows};
  if (t.kind != SPLIT_REP)
    for (auto& pp : p.pipes) {
      const StageInfo& st = pp.stages[stage_of(cfg, pp, t)];
      for (size_t k = 0; k < st.ranks.size(); ++k) {
        Range r = member_rows(cfg, st, t, (int)k);
        cuts.insert(r.b);
        cuts.insert(r.e);
      }
    }
  return std::vector<int64_t>(cuts.begin(), cuts.end());
}

std::vector<Piece> pieces(const malleus_model_cfg& cfg, const PlanInfo& p, const TensorInfo& t) {
  std::vector<Piece> out;
  const auto cuts = refinement(cfg, p, t);
  const int64_t c = t.cols, DP = (int64_t)p.pipes.size();
  for (size_t s = 0; s + 1 < cuts.size(); ++s) {
    const int64_t a = cuts[s], b = cuts[s + 1], nsig = (b - a) * c;
    for (int64_t q = 0; q < DP; ++q) {
      const int64_t lo = a * c + nsig * q / DP, hi = a * c + nsig * (q + 1) / DP;
      if (hi <= lo) continue;
      out.push_back({lo, hi, a, b, (int)q, sync_holder(cfg, p.pipes[q], t, a)});
    }
  }
  return out;
}

// Old holders of row segments: (row0, row1, lowest holder rank, set of holders)
struct HolderSeg {
  int64_t r0, r1;
  std::vector<int> holders;
};
static std::vector<HolderSeg> holder_segments(const malleus_model_cfg& cfg, const PlanInfo& p, const TensorInfo& t) {
  const auto cuts = refinement(cfg, p, t);
  std::vector<HolderSeg> out;
  for (size_t s = 0; s + 1 < cuts.size(); ++s) {
    HolderSeg hs{cuts[s], cuts[s + 1], {}};
    for (auto& pp : p.pipes) {
      const StageInfo& st = pp.stages[stage_of(cfg, pp, t)];
      for (size_t k = 0; k < st.ranks.size(); ++k) {
        Range r = member_rows(cfg, st, t, (int)k);
        if (r.b <= hs.r0 && hs.r0 < r.e) hs.holders.push_back(st.ranks[k]);
      }
    }
    std::sort(hs.holders.begin(), hs.holders.end());
    out.push_back(std::move(hs));
  }
  return out;
}

static std::vector<int> all_ranks(const PlanInfo& p) {
  std::vector<int> r;
  for (auto& pp : p.pipes)
    for (auto& st : pp.stages) r.insert(r.end(), st.ranks.begin(), st.ranks.end());
  std::sort(r.begin(), r.end());
  return r;
}

std::vector<Transfer> migration_transfers(const malleus_model_cfg& cfg, const PlanInfo& a, const PlanInfo& b) {
  std::vector<Transfer> out;
  const auto ranks_b = all_ranks(b);
  for (const TensorInfo& t : all_tensors(cfg)) {
    const int64_t c = t.cols;
    // bf16 params -> new holders from the lowest old holder (reading R11)
    const auto segs = holder_segments(cfg, a, t);
    for (int r : ranks_b) {
      Range need;
      if (!held_rows(cfg, b, t, r, &need)) continue;
      for (auto& s : segs) {
        const int64_t lo = std::max(need.b, s.r0), hi = std::min(need.e, s.r1);
        if (hi <= lo) continue;
        if (std::binary_search(s.holders.begin(), s.holders.end(), r)) continue;
        out.push_back({t.id, MALLEUS_KIND_PARAM, lo * c, hi * c, s.holders.front(), r});
      }
    }
    // fp32 master / m / v -> new owners from the unique old owner
    const auto po = pieces(cfg, a, t), pn = pieces(cfg, b, t);
    for (int kind : {MALLEUS_KIND_MASTER, MALLEUS_KIND_ADAM_M, MALLEUS_KIND_ADAM_V}) {
      size_t i = 0;
      for (const Piece& n : pn) {
        while (i < po.size() && po[i].e1 <= n.e0) ++i;
        for (size_t j = i; j < po.size() && po[j].e0 < n.e1; ++j) {
          const int64_t lo = std::max(n.e0, po[j].e0), hi = std::min(n.e1, po[j].e1);
          if (hi > lo && po[j].owner != n.owner) out.push_back({t.id, kind, lo, hi, po[j].owner, n.owner});
        }
      }
    }
  }
  return out;
}

}  // namespace mls

// ------------------------------------------------------------------ host-only C-ABI queries
using namespace mls;

extern "C" malleus_status malleus_layout_query(const malleus_model_cfg* cfg, const malleus_plan* plan,
                                               int32_t world, int32_t rank, int32_t tensor_id, int32_t kind,
                                               int64_t* ranges, int32_t* n_ranges) {
  if (!cfg || !plan || !n_ranges) return MALLEUS_E_ARG;
  PlanInfo p = plan_from_c(plan);
  if (!validate_plan(*cfg, p, world).empty()) return MALLEUS_E_PLAN;
  TensorInfo t;
  if (!tensor_info(*cfg, tensor_id, &t)) return MALLEUS_E_ARG;
  std::vector<Range> out;
  if (kind == MALLEUS_KIND_PARAM || kind == MALLEUS_KIND_GRAD) {
    Range r;
    if (held_rows(*cfg, p, t, rank, &r)) out.push_back({r.b * t.cols, r.e * t.cols});
  } else {
    for (const Piece& pc : pieces(*cfg, p, t))
      if (pc.owner == rank) out.push_back({pc.e0, pc.e1});
  }
  const int cap = *n_ranges;
  *n_ranges = (int32_t)out.size();
  if (ranges) {
    if ((int)out.size() > cap) return MALLEUS_E_ARG;
    for (size_t i = 0; i < out.size(); ++i) { ranges[2 * i] = out[i].b; ranges[2 * i + 1] = out[i].e; }
  }
  return MALLEUS_OK;
}

extern "C" malleus_status malleus_migration_query(const malleus_model_cfg* cfg, const malleus_plan* from,
                                                  const malleus_plan* to, int32_t world, int32_t dst_rank,
                                                  int32_t kind, int64_t* tbe, int32_t* src, int32_t* n) {
  if (!cfg || !from || !to || !n) return MALLEUS_E_ARG;
  PlanInfo a = plan_from_c(from), b = plan_from_c(to);
  if (!validate_plan(*cfg, a, world).empty() || !validate_plan(*cfg, b, world).empty()) return MALLEUS_E_PLAN;
  std::vector<Transfer> sel;
  for (auto& tr : migration_transfers(*cfg, a, b))
    if (tr.dst == dst_rank && tr.kind == kind) sel.push_back(tr);
  const int cap = *n;
  *n = (int32_t)sel.size();
  if (tbe && src) {
    if ((int)sel.size() > cap) return MALLEUS_E_ARG;
    for (size_t i = 0; i < sel.size(); ++i) {
      tbe[3 * i] = sel[i].tensor; tbe[3 * i + 1] = sel[i].e0; tbe[3 * i + 2] = sel[i].e1;
      src[i] = sel[i].src;
    }
  }
  return MALLEUS_OK;
}
