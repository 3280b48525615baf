"""Malleable parallelization plans as plain dicts (host-side input, not the product).

A plan is the paper's four components (§4.1): GPU grouping (stage `ranks`),
pipeline orchestration (`pipes`, ordered `stages`), layer assignment (`layers` = [begin, end),
l_ij = end - begin), training-data assignment (`n_micro` = m_i), plus the micro-batch size b and
global batch B (Table 1) and the removed / standby GPUs.
North-star extension: per-member split vectors `heads`, `ffn`, `vocab` (uneven TP shards).

The split vectors below are the min-max apportionments of SURVEY §8(d) (reading R7); the tests
re-derive them with the oracle's split helper.
"""
from __future__ import annotations


def stage(ranks, heads, ffn, vocab, layers):
    return {"ranks": list(ranks), "heads": list(heads), "ffn": list(ffn), "vocab": list(vocab),
            "layers": list(layers)}


def even(total: int, k: int, gran: int = 1):
    """Even split of `total` units of granularity `gran` over k members (remainder to the front)."""
    units = total // gran
    base, rem = divmod(units, k)
    return [(base + (1 if i < rem else 0)) * gran for i in range(k)]


def plan(pipes, b, B, standby=(), plan_id=0):
    return {"plan_id": plan_id, "micro_batch": b, "global_batch": B, "pipes": pipes,
            "standby": list(standby)}


plan_fn = plan  # alias for helpers whose arguments shadow the name


def pipe(stages, n_micro):
    return {"stages": stages, "n_micro": n_micro}


def even_stage(cfg, ranks, layers):
    k = len(ranks)
    return stage(ranks, even(cfg.n_heads, k), even(cfg.ffn, k, 16), even(cfg.vocab, k, 16), layers)


def single_gpu(cfg, B, b=1, rank=0):
    return plan([pipe([even_stage(cfg, [rank], [0, cfg.n_layers])], B // b)], b, B)


def world_of(p) -> int:
    ranks = [r for pp in p["pipes"] for st in pp["stages"] for r in st["ranks"]] + p["standby"]
    return max(ranks) + 1


def plan_matrix_c1(cfg, B=8, b=2):
    """SURVEY §8(d) parity plan matrix P0-P8 on the tiny C1 model (4 heads, F 512, V 256, L 2), plus P9
    (TP 4, uneven FFN / vocab)."""
    L = cfg.n_layers
    m = B // b
    H, F, V = cfg.n_heads, cfg.ffn, cfg.vocab
    s31 = lambda ranks, layers: stage(ranks, [3 * H // 4, H // 4], [3 * F // 4, F // 4], [3 * V // 4, V // 4],
                                      layers)
    ev = lambda ranks, layers: even_stage(cfg, ranks, layers)
    P = {}
    P["P0"] = plan([pipe([ev([0], [0, L])], m)], b, B)
    P["P1"] = plan([pipe([ev([0, 1], [0, L])], m)], b, B)
    P["P2"] = plan([pipe([s31([0, 1], [0, L])], m)], b, B)
    P["P3"] = plan([pipe([ev([0], [0, L])], 3), pipe([ev([1], [0, L])], 1)], b, B)
    P["P4"] = plan([pipe([s31([0, 1], [0, L])], 1), pipe([ev([2, 3], [0, L])], 3)], b, B)
    P["P5"] = plan([pipe([s31([0, 1], [0, L])], 2), pipe([ev([2], [0, L])], 2)], b, B)
    P["P6"] = plan([pipe([ev([0], [0, 1]), s31([1, 2], [1, L])], m)], b, B)
    P["P7"] = plan([pipe([ev([0], [0, 1]), s31([1, 2], [1, L])], 1),
                    pipe([ev([3, 4, 5, 6], [0, L])], 3)], b, B, standby=[7])
    P["P8"] = plan([pipe([ev([0], [0, L])], 4), pipe([ev([1], [0, L])], 0)], b, B)
    # TP 4 with uneven FFN / vocab splits (3:2:2:1) on one pipeline: the stage shape of the 8-GPU
    # ladder (DP2 x TP4) on 4 GPUs
    f4 = [3 * F // 8, F // 4, F // 4, F // 8]
    v4 = [3 * V // 8, V // 4, V // 4, V // 8]
    P["P9"] = plan([pipe([stage([0, 1, 2, 3], [H // 4] * 4, f4, v4, [0, L])], m)], b, B)
    # standby ranks (a removed GPU) on 2 and 4 GPUs: P7's standby and PP-with-TP-change
    # features without its 8-GPU footprint
    P["P10"] = plan([pipe([ev([0], [0, L])], m)], b, B, standby=[1])
    P["P11"] = plan([pipe([ev([0], [0, 1]), s31([1, 2], [1, L])], m)], b, B, standby=[3])
    return P


def plan_matrix_gqa(cfg, B=8, b=2):
    """Parity plans for a GQA model (n_kv < n: every member holds whole KV groups, so the head splits
    are multiples of the group size): P0 1 GPU; P1 TP2 even; P3 DP2 m = (3, 1); P4 DP2 = {TP2, TP1}
    m = (1, 3) (cross-layout, different TP degrees); P6 PP2 = {TP1 layer 0, TP2 layer 1}."""
    L, m = cfg.n_layers, B // b
    ev = lambda ranks, layers: even_stage(cfg, ranks, layers)
    return {
        "P0": plan([pipe([ev([0], [0, L])], m)], b, B),
        "P1": plan([pipe([ev([0, 1], [0, L])], m)], b, B),
        "P3": plan([pipe([ev([0], [0, L])], 3 * m // 4), pipe([ev([1], [0, L])], m - 3 * m // 4)], b, B),
        "P4": plan([pipe([ev([0, 1], [0, L])], m // 4), pipe([ev([2], [0, L])], m - m // 4)], b, B),
        "P6": plan([pipe([ev([0], [0, 1]), ev([1, 2], [1, L])], m)], b, B),
    }


def ladder_plan(cfg, n_gpus: int, B: int, b: int = 1, straggle: bool = True):
    """1/2/4/8-GPU ladder on the C2 shape (SURVEY §8(d) 'Ladder 1/2/4/8').

    1: TP1.  2: TP2 with a 2x straggler on rank 1 (heads 22/10, min-max).  4: the C2 plan,
    DP2 x TP2, rank 1 at 1.5x (heads 19/13, FFN tiles 52/34, vocab 148/102 tiles, m = (7, 9)).
    8: DP2 x TP4, rank 3 at 2x (heads 10/10/10/2 ... min-max), m = (7, 9).
    straggle=False gives the uniform even plan (T0 / T_u runs)."""
    L, H, F, V = cfg.n_layers, cfg.n_heads, cfg.ffn, cfg.vocab
    m = B // b
    if n_gpus == 1:
        return plan([pipe([even_stage(cfg, [0], [0, L])], m)], b, B)
    if not straggle:
        if n_gpus == 2:
            return plan([pipe([even_stage(cfg, [0, 1], [0, L])], m)], b, B)
        if n_gpus == 4:
            return plan([pipe([even_stage(cfg, [0, 1], [0, L])], m // 2),
                         pipe([even_stage(cfg, [2, 3], [0, L])], m - m // 2)], b, B)
        if n_gpus == 8:
            return plan([pipe([even_stage(cfg, [0, 1, 2, 3], [0, L])], m // 2),
                         pipe([even_stage(cfg, [4, 5, 6, 7], [0, L])], m - m // 2)], b, B)
    tiles = lambda v: [t * 128 for t in v]
    if n_gpus == 2:
        # x = (1, 2): heads 22/10 (max(22, 20) = 22 vs 21/11 -> 22: both min-max), FFN/vocab by tiles
        st = stage([0, 1], [22, 10], _ffn_split(F, [1.0, 2.0]), _vocab_split(V, [1.0, 2.0]), [0, L])
        return plan([pipe([st], m)], b, B)
    if n_gpus == 4:
        st0 = stage([0, 1], [19, 13], _ffn_split(F, [1.0, 1.5]), _vocab_split(V, [1.0, 1.5]), [0, L])
        st1 = even_stage(cfg, [2, 3], [0, L])
        m0 = (7 * m) // 16
        return plan([pipe([st0], m0), pipe([st1], m - m0)], b, B)
    if n_gpus == 8:
        rates = [1.0, 1.0, 1.0, 2.0]
        st0 = stage([0, 1, 2, 3], _heads_split(H, rates), _ffn_split(F, rates),
                    _vocab_split(V, rates), [0, L])
        st1 = even_stage(cfg, [4, 5, 6, 7], [0, L])
        m0 = (7 * m) // 16
        return plan([pipe([st0], m0), pipe([st1], m - m0)], b, B)
    raise ValueError("ladder is defined for 1, 2, 4, 8 GPUs")


def _minmax(n_units, rates):
    """Min-max integer apportionment (reading R7); duplicated from the host planner side on purpose
    (the product never imports oracle/).  Fastest members are filled first on ties."""
    k = len(rates)
    cands = sorted({round(c * x, 9) for x in rates for c in range(1, n_units + 1)})
    for C in cands:
        caps = [int(C / x + 1e-9) for x in rates]
        if all(c >= 1 for c in caps) and sum(caps) >= n_units:
            break
    counts, left = [1] * k, n_units - k
    for i in sorted(range(k), key=lambda i: (rates[i], i)):
        add = min(left, caps[i] - counts[i])
        counts[i] += add
        left -= add
    return counts


def _apportion(n_units, weights, min_units=1):
    """Largest-remainder apportionment of n_units proportional to weights (each >= min_units)."""
    k = len(weights)
    tot = float(sum(weights))
    raw = [n_units * w / tot for w in weights]
    out = [max(min_units, int(r)) for r in raw]
    while sum(out) > n_units:  # min_units pushed us over: take from the largest
        j = max(range(k), key=lambda i: out[i])
        out[j] -= 1
    order = sorted(range(k), key=lambda i: -(raw[i] - int(raw[i])))
    i = 0
    while sum(out) < n_units:
        out[order[i % k]] += 1
        i += 1
    return out


def _damped(cur, target, damp):
    """(1 - damp) x the current shares + damp x the target weights, both normalised."""
    if damp >= 1.0:
        return target
    sc, st = float(sum(cur)), float(sum(target))
    return [(1.0 - damp) * c / sc + damp * w / st for c, w in zip(cur, target)]


def rebalance(cfg, plan, compute_ms: dict, min_micro: int = 0, damp: float = 1.0):
    """Re-plan from measured speeds (the profiler -> planner -> migration loop of PAPER.md:378-384).

    Reading R12 (work-normalised rates): member k of a TP group that processed share f_k of the
    columns in t_k ms of compute runs at speed f_k / t_k; new shares are proportional to the
    speeds (heads whole, FFN / vocab in 128-wide tiles).  Pipelines: a pipeline's time per
    micro-batch is the max over its members' compute; m_i is re-apportioned proportional to
    m_i / T_i (Eq.(3)'s min-max objective, with measured o_i).  Layers, groups
    and stage order are kept.

    damp in (0, 1]: the new shares are (1 - damp) x the current ones + damp x the speed-proportional
    ones.  A member's compute is not proportional to its share (per-kernel fixed costs, narrow
    GEMMs' wave quantisation on 148 SMs), so the full step (damp = 1) can overshoot; callers measure
    a damped candidate beside it and keep the faster (bench.py, tools/trace_run.py)."""
    import copy
    p = copy.deepcopy(plan)
    p["plan_id"] = plan.get("plan_id", 0) + 1
    pipe_speed = []
    for pp in p["pipes"]:
        t_pipe = 0.0
        for st in pp["stages"]:
            ranks = st["ranks"]
            t = [max(compute_ms[r], 1e-6) for r in ranks]
            t_pipe = max(t_pipe, max(t))
            if len(ranks) == 1:
                continue
            speed = _damped(st["heads"], [st["heads"][k] / t[k] for k in range(len(ranks))], damp)
            st["heads"] = _apportion(cfg.n_heads, speed)
            for key, total in (("ffn", cfg.ffn), ("vocab", cfg.vocab)):
                tile = 128 if total // 128 >= 4 * len(ranks) else 16  # GEMM-friendly tiles when possible
                n_t, rem = divmod(total, tile)
                spd = _damped(st[key], [st[key][k] / t[k] for k in range(len(ranks))], damp)
                tiles = _apportion(n_t, spd)
                st[key] = [x * tile for x in tiles]
                st[key][-1] += rem
        pipe_speed.append(pp["n_micro"] / t_pipe if pp["n_micro"] > 0 else 1.0 / t_pipe)
    total_m = sum(pp["n_micro"] for pp in p["pipes"])
    if len(p["pipes"]) > 1:
        ms = _apportion(total_m, _damped([pp["n_micro"] for pp in p["pipes"]], pipe_speed, damp),
                        min_units=min_micro)
        for pp, m in zip(p["pipes"], ms):
            pp["n_micro"] = m
    return p


def resplit_candidates(cfg, plan, compute_ms: dict, damps=(1.0, 2 / 3, 1 / 3)):
    """The measured re-split candidates of the straggler loop (DESIGN §3 "Measured re-split"):
    rebalance() with each damping, duplicates and the current plan's own split dropped, in damp order.
    The caller migrates to each, times it and keeps the fastest (the current plan included)."""
    import json
    seen, out = {json.dumps(plan["pipes"])}, []
    for a in damps:
        c = rebalance(cfg, plan, compute_ms, damp=a)
        key = json.dumps(c["pipes"])
        if key not in seen:
            seen.add(key)
            out.append(c)
    return out


def _heads_split(H, rates):
    return _minmax(H, rates)


def _ffn_split(F, rates, tile=128):
    """FFN columns in whole 128-column tiles (last member takes the ragged remainder)."""
    n_t, rem = divmod(F, tile)
    c = _minmax(n_t, rates)
    out = [x * tile for x in c]
    out[-1] += rem
    return out


def _vocab_split(V, rates, tile=128):
    return _ffn_split(V, rates, tile)


def stage_cost(cfg, st, xr, last: bool) -> float:
    """Per-micro-batch time of a stage in units of algorithmic FLOPs per token at rate 1:
    max over members of x_k * (layers * (8 h n_k d + 2 s n_k d + 6 h F_k) + [last] 2 h V_k), i.e. the
    member's QKV/O GEMMs, causal attention, gate/up/down GEMMs and LM-head share (forward; the
    backward is the same multiple for every term)."""
    h, d, s = cfg.hidden, cfg.head_dim, cfg.seq_len
    nl = st["layers"][1] - st["layers"][0]
    cost = 0.0
    for k, x in enumerate(xr):
        w = nl * (8 * h * st["heads"][k] * d + 2 * s * st["heads"][k] * d + 6 * h * st["ffn"][k])
        if last:
            w += 2 * h * st["vocab"][k]
        cost = max(cost, x * w)
    return cost


def plan_from_rates(cfg, plan, rates: dict, deadband: float = 0.05):
    """Re-plan from probed straggling rates x_g (PAPER.md:370-374 profiler -> §4 planner), keeping
    the grouping, stage order and layers: each TP group's heads / FFN tiles / vocab tiles by the
    min-max apportionment over its members' rates (reading R7), and the micro-batches over the
    pipelines by min-max on the pipelines' per-micro-batch cost y_i = max over members of
    (share x rate).  Rates within `deadband` of 1 count as 1 (the 5% trigger,
    PAPER.md:374), so a recovered cluster returns to the even plan exactly."""
    import copy
    x = {r: (1.0 if v < 1.0 + deadband else float(v)) for r, v in rates.items()}
    p = copy.deepcopy(plan)
    p["plan_id"] = plan.get("plan_id", 0) + 1
    H, F, V = cfg.n_heads, cfg.ffn, cfg.vocab
    y = []
    for pp in p["pipes"]:
        y_pipe = 0.0
        for j, st in enumerate(pp["stages"]):
            xr = [x[r] for r in st["ranks"]]
            if len(xr) > 1:
                st["heads"] = _heads_split(H, xr)
                tile = 128 if F // 128 >= 4 * len(xr) else 16
                st["ffn"] = _ffn_split(F, xr, tile)
                tile_v = 128 if V // 128 >= 4 * len(xr) else 16
                st["vocab"] = _vocab_split(V, xr, tile_v)
            # the pipeline's per-micro-batch cost is its slowest stage, o_i = max_j y_ij * l_ij
            # (lower problem 547-552); a stage's time is its slowest member's
            # rate x FLOPs of its shard (head / FFN columns per layer, vocab rows on the last stage)
            last = j == len(pp["stages"]) - 1
            y_pipe = max(y_pipe, stage_cost(cfg, st, xr, last))
        y.append(y_pipe)
    total_m = sum(pp["n_micro"] for pp in p["pipes"])
    if len(p["pipes"]) > 1:
        for pp, m in zip(p["pipes"], _minmax(total_m, y)):
            pp["n_micro"] = m
    return p


# TP efficiency per group size (the paper's rho_n: "the coefficient of efficiency
# degradation when the group consists of n GPUs ... profiled and computed beforehand"), as time per
# unit of work relative to one GPU: measured on B200 with the C2 shape (round-1 T0 runs):
# TP1 203.5 ms / step, TP2 120.3 ms (203.5 / (2 x 120.3) = 0.85), the TP-4 stage 92.4 ms (0.55).
TP_EFF = {1: 1.0, 2: 0.85, 3: 0.7, 4: 0.55}


def _group_cost(cfg, st, xr, last, eff):
    """Per-micro-batch time of a stage after a min-max re-split over its members (reading R8's
    group rate with the TP efficiency of its size), in FLOP units at rate 1."""
    k = len(xr)
    s2 = dict(st)
    if k > 1:
        s2["heads"] = _heads_split(cfg.n_heads, xr)
        s2["ffn"] = _ffn_split(cfg.ffn, xr, 128 if cfg.ffn // 128 >= 4 * k else 16)
        s2["vocab"] = _vocab_split(cfg.vocab, xr, 128 if cfg.vocab // 128 >= 4 * k else 16)
    else:
        s2["heads"], s2["ffn"], s2["vocab"] = [cfg.n_heads], [cfg.ffn], [cfg.vocab]
    return stage_cost(cfg, s2, xr, last) / eff.get(k, min(eff.values())), s2


def replan(cfg, base_plan, rates: dict, deadband: float = 0.05, eff=None, min_gain: float = 0.05):
    """The planner run by the asynchronous re-planning loop and the standby
    re-probe: always plans from the BASE grouping (all GPUs), so a GPU removed earlier
    is re-admitted as soon as its probed rate recovers.  Per TP group it chooses which members to
    keep — removing a heavy straggler when its group then runs faster by more than `min_gain`
    (zero layers for groups with high straggling rates; here per member, the group
    shrinks) — with the removed GPUs listed as standby; the kept members get min-max head / FFN /
    vocab splits (reading R7), and the micro-batches are apportioned min-max over the pipelines'
    per-micro-batch costs.  Layers and stage order are those of the base plan."""
    import copy
    import itertools
    eff = TP_EFF if eff is None else eff
    x = {r: (1.0 if v < 1.0 + deadband else float(v)) for r, v in rates.items()}
    p = copy.deepcopy(base_plan)
    p["plan_id"] = base_plan.get("plan_id", 0) + 1
    standby = set(base_plan.get("standby", []))
    y = []
    for pp in p["pipes"]:
        y_pipe = 0.0
        for j, st in enumerate(pp["stages"]):
            last = j == len(pp["stages"]) - 1
            ranks = list(st["ranks"])
            full_cost, best = _group_cost(cfg, st, [x[r] for r in ranks], last, eff)
            best_cost, best_ranks = full_cost, ranks
            for n_keep in range(len(ranks) - 1, 0, -1):
                for keep in itertools.combinations(ranks, n_keep):
                    c, s2 = _group_cost(cfg, st, [x[r] for r in keep], last, eff)
                    if c < best_cost * (1.0 - min_gain) and c < full_cost * (1.0 - min_gain):
                        best_cost, best, best_ranks = c, s2, list(keep)
            standby |= set(ranks) - set(best_ranks)
            st["ranks"] = best_ranks
            st["heads"], st["ffn"], st["vocab"] = best["heads"], best["ffn"], best["vocab"]
            y_pipe = max(y_pipe, best_cost)
        y.append(y_pipe)
    p["standby"] = sorted(standby)
    total_m = sum(pp["n_micro"] for pp in p["pipes"])
    if len(p["pipes"]) > 1:
        for pp, m in zip(p["pipes"], _minmax(total_m, y)):
            pp["n_micro"] = m
    return p


def survivor_plan(cfg, plan, failed, rates=None):
    """Recovery plan after a failure ("loading the latest model checkpoint onto the
    remaining GPUs and setting the straggling rates of unresponsive GPUs as infinite"): an infinite
    rate removes a GPU from its group, so the failed ranks leave their stages; a pipeline that lost a
    whole stage cannot run and is dropped (its micro-batches go to the others); the survivors are
    renumbered 0..N'-1 in rank order and re-split min-max by `rates` (default 1).  Returns
    (plan on the new ranks, {old rank: new rank})."""
    import copy
    failed = set(failed)
    rates = rates or {}
    pipes = []
    for pp in plan["pipes"]:
        stages = []
        for st in pp["stages"]:
            keep = [r for r in st["ranks"] if r not in failed]
            if not keep:
                break
            stages.append((keep, list(st["layers"])))
        else:
            pipes.append(stages)
    if not pipes:
        raise ValueError("no pipeline survives the failure")
    survivors = sorted({r for stages in pipes for keep, _ in stages for r in keep} |
                       (set(plan.get("standby", [])) - failed))
    remap = {r: i for i, r in enumerate(survivors)}
    out_pipes, y = [], []
    for stages in pipes:
        sts, y_pipe = [], 0.0
        for j, (keep, layers) in enumerate(stages):
            xr = [float(rates.get(r, 1.0)) for r in keep]
            last = j == len(stages) - 1
            c, s2 = _group_cost(cfg, {"layers": layers}, xr, last, TP_EFF)
            sts.append(stage([remap[r] for r in keep], s2["heads"], s2["ffn"], s2["vocab"], layers))
            y_pipe = max(y_pipe, c)
        out_pipes.append(sts)
        y.append(y_pipe)
    total_m = sum(pp["n_micro"] for pp in plan["pipes"])
    ms = _minmax(total_m, y) if len(out_pipes) > 1 else [total_m]
    new = plan_fn([pipe(sts, m) for sts, m in zip(out_pipes, ms)], plan["micro_batch"], plan["global_batch"],
                  standby=[remap[r] for r in plan.get("standby", []) if r not in failed],
                  plan_id=plan.get("plan_id", 0) + 1)
    return copy.deepcopy(new), remap


# ----------------------------------------------------------------------------- named workloads
# BASELINE.json configs C3 / C4 as concrete plans (SURVEY §8(d) "Concrete synthetic inputs"), so an
# 8-GPU run exercises non-uniform layers with PP and two-straggler cross-layout sync.  Each returns
# (plan, stragglers {rank: nominal x}, uniform plan for the T0 / T_u runs).

def c3_plan(cfg, B: int = 16):
    """C3 (32B-shaped 16-layer slice, 8 GPUs): TP4 x PP2, DP1.  Stage 0 = GPUs 0-3 with GPU 3 at 2x:
    heads 15/15/15/7 (min-max over rates (1, 1, 1, 2)), FFN 128-column tiles 40/40/40/20; stage 1 =
    GPUs 4-7 even (13 heads, 35 tiles).  Layers (7, 9): the slow stage takes fewer layers (PAPER.md:
    331-333 non-uniform layer assignment; even TP would need (5, 11)).  m = B (b = 1)."""
    rates = [1.0, 1.0, 1.0, 2.0]
    st0 = stage([0, 1, 2, 3], _heads_split(cfg.n_heads, rates), _ffn_split(cfg.ffn, rates),
                even(cfg.vocab, 4, 16), [0, 7])
    st1 = even_stage(cfg, [4, 5, 6, 7], [7, cfg.n_layers])
    uni = plan([pipe([even_stage(cfg, [0, 1, 2, 3], [0, cfg.n_layers // 2]),
                      even_stage(cfg, [4, 5, 6, 7], [cfg.n_layers // 2, cfg.n_layers])], B)], 1, B)
    return plan([pipe([st0, st1], B)], 1, B), {3: 2.0}, uni


def c4_plan(cfg, B: int = 32):
    """C4 (70B-shaped 4-layer slice, 8 GPUs): DP2 x TP4.  Pipeline A = GPUs 0-3 with GPU 1 at 1.3x,
    pipeline B = GPUs 4-7 with GPU 6 at 3x; heads / FFN tiles / vocab tiles by the min-max split of
    each group's rates (reading R7); micro-batches by min-max over the pipelines' per-micro-batch
    cost: the layouts of the two pipelines differ, so the gradient sync takes the
    cross-layout path."""
    ra, rb = [1.0, 1.3, 1.0, 1.0], [1.0, 1.0, 3.0, 1.0]
    L = cfg.n_layers
    sa = stage([0, 1, 2, 3], _heads_split(cfg.n_heads, ra), _ffn_split(cfg.ffn, ra), _vocab_split(cfg.vocab, ra),
               [0, L])
    sb = stage([4, 5, 6, 7], _heads_split(cfg.n_heads, rb), _ffn_split(cfg.ffn, rb), _vocab_split(cfg.vocab, rb),
               [0, L])
    y = [stage_cost(cfg, sa, ra, True), stage_cost(cfg, sb, rb, True)]
    ma, mb = _minmax(B, y)
    uni = plan([pipe([even_stage(cfg, [0, 1, 2, 3], [0, L])], B // 2),
                pipe([even_stage(cfg, [4, 5, 6, 7], [0, L])], B - B // 2)], 1, B)
    return plan([pipe([sa], ma), pipe([sb], mb)], 1, B), {1: 1.3, 6: 3.0}, uni


def member_flops(cfg, plan: dict, rank: int) -> float:
    """Algorithmic FLOPs of `rank` per step (reading R12's W_g): 3 x (forward per token of its shard:
    QKV/O 8 h n_k d, causal attention 2 (s + 1) n_k d ((s+1)/2 keys on average), gate/up/down 6 h F_k per
    layer, LM head 2 h V_k on the
    last stage) x the pipeline's m_i b s tokens.  0 for standby ranks."""
    for pp in plan["pipes"]:
        for j, st in enumerate(pp["stages"]):
            if rank in st["ranks"]:
                k = st["ranks"].index(rank)
                h, d, s = cfg.hidden, cfg.head_dim, cfg.seq_len
                nl = st["layers"][1] - st["layers"][0]
                w = nl * (8 * h * st["heads"][k] * d + 2 * (s + 1) * st["heads"][k] * d + 6 * h * st["ffn"][k])
                if j == len(pp["stages"]) - 1:
                    w += 2 * h * st["vocab"][k]
                return 3.0 * w * pp["n_micro"] * plan["micro_batch"] * s
    return 0.0
