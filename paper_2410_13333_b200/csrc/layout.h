// Host-side plan model and state-placement arithmetic (no CUDA).
//
// Plan = grouping + orchestration + layer assignment + data assignment, with
// per-member split vectors (north-star extension).  Placement follows reading R9:
// every tensor is stored split-axis-outermost, so a member's shard is a contiguous row range;
// per tensor the common refinement of all pipelines' row partitions is cut into DP contiguous
// pieces per segment, piece p owned by pipeline p's holder of the segment.  For even
// power-of-two splits this is exactly PAPER.md:715 (DP x TP_max slices, TP_max/TP_i per GPU).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "malleus.h"

namespace mls {

struct StageInfo {
  std::vector<int> ranks, heads, ffn, vocab;
  int lb = 0, le = 0;
};
struct PipeInfo {
  std::vector<StageInfo> stages;
  int n_micro = 0;
};
struct PlanInfo {
  int plan_id = 0, b = 1, B = 1;
  std::vector<PipeInfo> pipes;
  std::vector<int> standby;
};

enum SplitKind { SPLIT_HEADS = 0, SPLIT_FFN = 1, SPLIT_VOCAB = 2, SPLIT_REP = 3 };
enum { LT_G1 = 0, LT_WQ, LT_WK, LT_WV, LT_WO, LT_G2, LT_WG, LT_WU, LT_WD, LT_COUNT };

struct TensorInfo {
  int32_t id;
  int layer;         // -1 for globals
  int idx;           // LT_* for layer tensors; 0 embed, 1 final norm, 2 lm head
  int64_t rows, cols;
  SplitKind kind;
  bool decay;        // AdamW weight decay (2-D tensors only, reading R5)
  int64_t numel() const { return rows * cols; }
};

struct Range {
  int64_t b, e;
};

// One DP piece of one refined segment of a tensor (flat element range, reading R9).
struct Piece {
  int64_t e0, e1;     // flat element range
  int64_t row0, row1; // segment rows
  int piece;          // DP piece index == owning pipeline index
  int owner;          // rank
};

// Where this rank finds / moves a piece's contributions in grad sync.
struct Contribution {
  int pipe;       // pipeline index (fixed summation order)
  int holder;     // rank holding the pipeline's gradient of the segment
};

PlanInfo plan_from_c(const malleus_plan* p);
std::string validate_plan(const malleus_model_cfg& cfg, const PlanInfo& p, int world);
// limits of the sm_100a kernels (checked by plan_requirements / plan_apply / migrate, not by the
// host-only layout queries)
std::string check_kernel_limits(const malleus_model_cfg& cfg, const PlanInfo& p);

std::vector<TensorInfo> all_tensors(const malleus_model_cfg& cfg);
bool tensor_info(const malleus_model_cfg& cfg, int32_t id, TensorInfo* out);

int stage_of(const malleus_model_cfg& cfg, const PipeInfo& pipe, const TensorInfo& t);
Range member_rows(const malleus_model_cfg& cfg, const StageInfo& st, const TensorInfo& t, int k);
// rank's (pipe, stage, member) or -1s if standby
void locate(const PlanInfo& p, int rank, int* pipe, int* stage, int* member);

// Rows of t held by `rank` (empty if none).  Replicated tensors: all rows.
bool held_rows(const malleus_model_cfg& cfg, const PlanInfo& p, const TensorInfo& t, int rank, Range* rows);
// Pipeline's holder-for-sync of `row` (first member for replicated tensors).
int sync_holder(const malleus_model_cfg& cfg, const PipeInfo& pipe, const TensorInfo& t, int64_t row);
// All pieces of t in canonical (segment, piece) order.
std::vector<Piece> pieces(const malleus_model_cfg& cfg, const PlanInfo& p, const TensorInfo& t);

// Every (tensor, kind) transfer needed to move from plan a to plan b (readings R10/R11).
struct Transfer {
  int32_t tensor;
  int kind;          // MALLEUS_KIND_PARAM or MASTER/ADAM_M/ADAM_V
  int64_t e0, e1;    // flat elements
  int src, dst;
};
std::vector<Transfer> migration_transfers(const malleus_model_cfg& cfg, const PlanInfo& a, const PlanInfo& b);

}  // namespace mls
