"""Oracle: plan validation, state placement (holders / owners) and migration deltas.

TEST INFRASTRUCTURE ONLY (see oracle/model.py header).

Definitions followed, element by element (deliberately brute force, no range
arithmetic, so that a reader can check it against the passages by eye):

* Plan = GPU grouping + pipeline orchestration + layer assignment + data
  assignment (§4.1), plus b and B (Table 1).
  Constraints of Eq.(1): sum_i m_i*b = B, sum_j l_ij = L.
  Zero-layer stages are omitted and their GPUs are standby.
* ZeRO-1 sharding with varying TP degrees (§5.1): a layer's
  states are cut into DP x TP_max slices and a GPU of pipeline i owns
  TP_max/TP_i of them.  Reading R9 generalises this to uneven and
  mismatched splits: per tensor, the common refinement of all pipelines' row
  partitions; every segment is cut into DP contiguous pieces, piece p owned by
  pipeline p's holder of the segment.  It reduces to PAPER.md:715 for even
  power-of-two splits (tests/test_oracle_layout.py pins that).
* Migration (§5.1; reading R10/R11): bf16 params move to new
  holders, fp32 master/m/v to new owners; delta = need_new(g) \\ have_old(g).
"""
from __future__ import annotations

from synth.gen import ModelCfg, tensor_shapes

KIND_PARAM, KIND_GRAD, KIND_MASTER, KIND_ADAM_M, KIND_ADAM_V = 0, 1, 2, 3, 4
KIND_BYTES = {KIND_PARAM: 2, KIND_MASTER: 4, KIND_ADAM_M: 4, KIND_ADAM_V: 4}


class PlanError(ValueError):
    pass


# ----------------------------------------------------------------------------- plan helpers
def split_kind(name: str) -> str:
    t = name.split(".")[-1]
    if t in ("wq", "wk", "wv", "wo"):
        return "heads"
    if t in ("wg", "wu", "wd"):
        return "ffn"
    if t == "Wlm":
        return "vocab"
    return "rep"  # g1, g2, gf, E (embedding replicated across the first stage's members)


def stage_of(pipe: dict, name: str, cfg: ModelCfg) -> int:
    """Index of the stage of `pipe` holding tensor `name` (embedding: first stage, LM head and
    final norm: last stage)."""
    if name == "E":
        return 0
    if name in ("gf", "Wlm"):
        return len(pipe["stages"]) - 1
    layer = int(name.split(".")[0])
    for j, st in enumerate(pipe["stages"]):
        if st["layers"][0] <= layer < st["layers"][1]:
            return j
    raise PlanError(f"layer {layer} not assigned")


def member_rows(cfg: ModelCfg, stage: dict, name: str, k: int):
    """Row range [r0, r1) of logical tensor `name` held by member k of `stage`."""
    kind = split_kind(name)
    n_rows = tensor_shapes(cfg)[name][0]
    if kind == "rep":
        return 0, n_rows
    unit = {"heads": cfg.head_dim, "ffn": 1, "vocab": 1}[kind]
    vec = {"heads": stage["heads"], "ffn": stage["ffn"], "vocab": stage["vocab"]}[kind]
    if name.endswith((".wk", ".wv")):  # GQA: a member holds the KV heads of its whole query-head groups
        g = cfg.n_heads // getattr(cfg, "kv_heads", cfg.n_heads)
        vec = [c // g for c in vec]
    r0 = unit * sum(vec[:k])
    return r0, r0 + unit * vec[k]


def validate(cfg: ModelCfg, plan: dict, world: int) -> None:
    """Raise PlanError naming the violated invariant (SURVEY §8(b) plan validation)."""
    b, B = plan["micro_batch"], plan["global_batch"]
    pipes = plan["pipes"]
    if b < 1 or B < 1 or len(pipes) < 1:
        raise PlanError("b >= 1, B >= 1, DP >= 1")
    if sum(p["n_micro"] for p in pipes) * b != B:
        raise PlanError("sum_i m_i * b == B (PAPER.md:523)")
    seen = set()
    for p in pipes:
        if p["n_micro"] < 0:
            raise PlanError("m_i >= 0")
        if not p["stages"]:
            raise PlanError("pipeline with no stage")
        nxt = 0
        for st in p["stages"]:
            lb, le = st["layers"]
            if lb != nxt or le <= lb:
                raise PlanError("stage layer ranges must partition [0, L) in order, l_ij >= 1 "
                                "(PAPER.md:524, 556)")
            nxt = le
            ks = len(st["ranks"])
            if ks < 1:
                raise PlanError("empty stage")
            for key, total, gran in (("heads", cfg.n_heads, 1), ("ffn", cfg.ffn, 16),
                                     ("vocab", cfg.vocab, 16)):
                vec = st[key]
                if len(vec) != ks or sum(vec) != total:
                    raise PlanError(f"{key} split must have one entry per member and sum to {total}")
                if key == "heads":  # whole KV groups per member (GQA; 1 for MHA)
                    gran = cfg.n_heads // getattr(cfg, "kv_heads", cfg.n_heads)
                if any(v < gran or v % gran for v in vec):
                    raise PlanError(f"{key} split entries must be >= {gran} and multiples of {gran}")
            for r in st["ranks"]:
                if r in seen or not (0 <= r < world):
                    raise PlanError(f"rank {r} repeated or out of range")
                seen.add(r)
        if nxt != cfg.n_layers:
            raise PlanError("stage layer ranges must cover [0, L) (PAPER.md:524)")
    for r in plan.get("standby", []):
        if r in seen or not (0 <= r < world):
            raise PlanError(f"standby rank {r} also in a stage or out of range (PAPER.md:556)")
        seen.add(r)
    if seen != set(range(world)):
        raise PlanError("every rank must be in exactly one stage or standby")


# ----------------------------------------------------------------------------- per element
def n_elems(cfg, name):
    sh = tensor_shapes(cfg)[name]
    return sh[0] * (sh[1] if len(sh) > 1 else 1)


def row_width(cfg, name):
    sh = tensor_shapes(cfg)[name]
    return sh[1] if len(sh) > 1 else 1


def holders_of_element(cfg, plan, name, e):
    """All ranks holding flat element e of `name` (bf16 param copies)."""
    row = e // row_width(cfg, name)
    out = []
    for p in plan["pipes"]:
        st = p["stages"][stage_of(p, name, cfg)]
        for k, r in enumerate(st["ranks"]):
            r0, r1 = member_rows(cfg, st, name, k)
            if r0 <= row < r1:
                out.append(r)
    return sorted(out)


def sync_holder(cfg, pipe, name, row):
    """Pipeline's holder of `row` for gradient sync: the member whose rows contain it;
    replicated tensors: the first member (its grad is bitwise equal to the others', R9)."""
    st = pipe["stages"][stage_of(pipe, name, cfg)]
    if split_kind(name) == "rep":
        return st["ranks"][0]
    for k, r in enumerate(st["ranks"]):
        r0, r1 = member_rows(cfg, st, name, k)
        if r0 <= row < r1:
            return r
    raise AssertionError("row not held")


def pipeline_cuts(cfg, pipe, name):
    st = pipe["stages"][stage_of(pipe, name, cfg)]
    n_rows = tensor_shapes(cfg)[name][0]
    cuts = {0, n_rows}
    if split_kind(name) != "rep":
        for k in range(len(st["ranks"])):
            cuts.update(member_rows(cfg, st, name, k))
    return cuts


def owner_of_element(cfg, plan, name, e):
    """Owner (rank) and DP piece index of flat element e (reading R9)."""
    c = row_width(cfg, name)
    row = e // c
    cuts = set()
    for p in plan["pipes"]:
        cuts |= pipeline_cuts(cfg, p, name)
    cuts = sorted(cuts)
    a = max(x for x in cuts if x <= row)
    b = min(x for x in cuts if x > row)
    DP = len(plan["pipes"])
    n_sig = (b - a) * c
    off = e - a * c
    piece = None
    for p in range(DP):
        lo, hi = (n_sig * p) // DP, (n_sig * (p + 1)) // DP
        if lo <= off < hi:
            piece = p
    return sync_holder(cfg, plan["pipes"][piece], name, row), piece


def owner_map(cfg, plan, name):
    return [owner_of_element(cfg, plan, name, e)[0] for e in range(n_elems(cfg, name))]


def holder_map(cfg, plan, name):
    return [holders_of_element(cfg, plan, name, e) for e in range(n_elems(cfg, name))]


def migration_deltas(cfg, old, new):
    """List of (name, kind, element, src, dst) moves (reading R10/R11).

    PARAM: every new holder that did not hold the element receives it from the lowest old
    holder.  MASTER/ADAM_M/ADAM_V: the new owner receives it from the unique old owner when
    they differ.  No self-transfers by construction."""
    moves = []
    for name in tensor_shapes(cfg):
        for e in range(n_elems(cfg, name)):
            oh = holders_of_element(cfg, old, name, e)
            for dst in holders_of_element(cfg, new, name, e):
                if dst not in oh:
                    moves.append((name, KIND_PARAM, e, oh[0], dst))
            oo = owner_of_element(cfg, old, name, e)[0]
            no = owner_of_element(cfg, new, name, e)[0]
            if oo != no:
                for kind in (KIND_MASTER, KIND_ADAM_M, KIND_ADAM_V):
                    moves.append((name, kind, e, oo, no))
    return moves


def delta_bytes(moves):
    return sum(KIND_BYTES[m[1]] for m in moves)
