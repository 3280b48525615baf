"""Pins for oracle/layout.py: paper-printed slice counts, SPEC examples, brute-force invariants,
and the paper's Table 4 plans as structural fixtures (tests/golden/table4_*.json)."""
import json
import os

import numpy as np
import pytest

from synth.gen import ModelCfg, C1_TINY, MICRO, tensor_shapes
from oracle import layout as Lo
from paper_2410_13333_b200 import plans as Pl
from tests.planutil import random_plan

GOLD = os.path.join(os.path.dirname(__file__), "golden")
# layout-only model: 8 heads of d=2 so that TP 8 has >= 1 head per member, tiny matrices
LAYOUT8 = ModelCfg(n_layers=4, hidden=16, n_heads=8, head_dim=2, ffn=128, vocab=128, seq_len=4)


def _slices_per_rank(cfg, plan, name):
    """Count distinct (segment, piece) pairs owned per rank = the paper's 'slices'."""
    c = Lo.row_width(cfg, name)
    cuts = sorted(set().union(*[Lo.pipeline_cuts(cfg, p, name) for p in plan["pipes"]]))
    seg_of = lambda e: max(i for i, x in enumerate(cuts) if x <= e // c)
    out = {}
    for e in range(Lo.n_elems(cfg, name)):
        r, pc = Lo.owner_of_element(cfg, plan, name, e)
        out.setdefault(r, set()).add((seg_of(e), pc))
    return {r: len(s) for r, s in out.items()}


def test_paper_rule_even_dp2_tp4_tp2():
    """PAPER.md:715 (§5.1) / SPEC S:537: DP=2, TP=(4,2) -> DP*TP_max = 8 slices; each GPU of
    pipeline i owns TP_max/TP_i slices: 1 per TP-4 GPU, 2 per TP-2 GPU."""
    cfg = LAYOUT8
    L = cfg.n_layers
    p = Pl.plan([Pl.pipe([Pl.even_stage(cfg, [0, 1, 2, 3], [0, L])], 2),
                 Pl.pipe([Pl.even_stage(cfg, [4, 5], [0, L])], 2)], 1, 4)
    Lo.validate(cfg, p, 6)
    for name in ("0.wq", "1.wd"):
        cnt = _slices_per_rank(cfg, p, name)
        assert sum(cnt.values()) == 8
        assert [cnt[r] for r in range(6)] == [1, 1, 1, 1, 2, 2]
        # owned elements: 1/(DP*TP_max) of the tensor per slice
        own = Lo.owner_map(cfg, p, name)
        n = Lo.n_elems(cfg, name)
        for r in range(6):
            assert own.count(r) == n // 8 * (1 if r < 4 else 2)


@pytest.mark.parametrize("dp_tp, expect", [((8,), 8), ((1, 1), 2)])
def test_spec_examples(dp_tp, expect):
    """DP=1, TP=8 -> 8 slices (classic ZeRO-1); DP=2, TP=(1,1) -> 2 slices."""
    cfg = LAYOUT8
    L = cfg.n_layers
    pipes, r = [], 0
    for tp in dp_tp:
        pipes.append(Pl.pipe([Pl.even_stage(cfg, list(range(r, r + tp)), [0, L])], 1))
        r += tp
    p = Pl.plan(pipes, 1, len(dp_tp))
    cnt = _slices_per_rank(cfg, p, "2.wk")
    assert sum(cnt.values()) == expect
    assert len(set(cnt.values())) == 1


def _check_invariants(cfg, plan):
    for name in tensor_shapes(cfg):
        n = Lo.n_elems(cfg, name)
        for e in range(0, n, max(1, n // 97)):
            hold = Lo.holders_of_element(cfg, plan, name, e)
            own, pc = Lo.owner_of_element(cfg, plan, name, e)
            assert own in hold, "owner must hold the element"
            assert not set(hold) & set(plan["standby"]), "standby ranks hold nothing"
            # one holder-for-sync per pipeline, all TP members for replicated tensors
            per_pipe = len(plan["pipes"])
            if Lo.split_kind(name) != "rep":
                assert len(hold) == per_pipe


def test_random_plan_invariants():
    rng = np.random.default_rng(7)
    for _ in range(60):
        p, world = random_plan(rng, MICRO, world_max=6, B=8, b=2)
        Lo.validate(MICRO, p, world)
        _check_invariants(MICRO, p)


def _table4_plan(d, cfg):
    pipes = []
    for pp in d["pipes"]:
        stages, l0 = [], 0
        for ranks, nl in pp["stages"]:
            stages.append(Pl.even_stage(cfg, ranks, [l0, l0 + nl]))
            l0 += nl
        pipes.append(Pl.pipe(stages, pp["n_micro"]))
    return Pl.plan(pipes, d["micro_batch"], d["global_batch"], standby=d["standby"])


@pytest.mark.parametrize("fname", ["table4_110b_s4.json", "table4_32b_s5.json"])
def test_paper_table4_plans(fname):
    """Table 4: per-pipeline layers sum to L, sum m = 64 = B, standby GPUs
    hold nothing, mixed TP degrees inside one pipeline and across pipelines validate, and every
    element of boundary layers has exactly one owner among its holders."""
    d = json.load(open(os.path.join(GOLD, fname)))
    cfg = ModelCfg(n_layers=d["n_layers"], hidden=16, n_heads=8, head_dim=2, ffn=128, vocab=128,
                   seq_len=4)
    p = _table4_plan(d, cfg)
    Lo.validate(cfg, p, d["world"])
    assert all(sum(st["layers"][1] - st["layers"][0] for st in pp["stages"]) == cfg.n_layers
               for pp in p["pipes"])
    assert sum(pp["n_micro"] for pp in p["pipes"]) * p["micro_batch"] == 64
    for name in ("0.wq", "1.g1", f"{cfg.n_layers - 1}.wd", "E", "Wlm"):
        own = Lo.owner_map(cfg, p, name)
        assert not set(own) & set(d["standby"])
        for e, r in enumerate(own):
            assert r in Lo.holders_of_element(cfg, p, name, e)


def _apply_moves(cfg, old, new, moves):
    """Simulate migration: start from old placement, apply moves, compare to new placement."""
    have = {}
    for name in tensor_shapes(cfg):
        for e in range(Lo.n_elems(cfg, name)):
            for r in Lo.holders_of_element(cfg, old, name, e):
                have[(name, Lo.KIND_PARAM, e, r)] = True
            r = Lo.owner_of_element(cfg, old, name, e)[0]
            for k in (Lo.KIND_MASTER, Lo.KIND_ADAM_M, Lo.KIND_ADAM_V):
                have[(name, k, e, r)] = True
    for name, kind, e, src, dst in moves:
        assert src != dst, "no self-transfer (SPEC S:553)"
        assert have.get((name, kind, e, src)), "source must hold the element in the old plan"
        have[(name, kind, e, dst)] = True
    for name in tensor_shapes(cfg):
        for e in range(Lo.n_elems(cfg, name)):
            for r in Lo.holders_of_element(cfg, new, name, e):
                assert have.get((name, Lo.KIND_PARAM, e, r))
            r = Lo.owner_of_element(cfg, new, name, e)[0]
            for k in (Lo.KIND_MASTER, Lo.KIND_ADAM_M, Lo.KIND_ADAM_V):
                assert have.get((name, k, e, r))


def test_migration_identity_and_roundtrip():
    cfg = MICRO
    P = Pl.plan_matrix_c1(C1_TINY)  # structure only; rebuild on MICRO dims
    rng = np.random.default_rng(11)
    for _ in range(12):
        a, wa = random_plan(rng, cfg, world_max=5, B=8, b=2)
        b, wb = random_plan(rng, cfg, world_max=5, B=8, b=2)
        if wa != wb:
            continue
        assert Lo.migration_deltas(cfg, a, a) == []  # identity -> empty
        mv = Lo.migration_deltas(cfg, a, b)
        _apply_moves(cfg, a, b, mv)
        back = Lo.migration_deltas(cfg, b, a)
        _apply_moves(cfg, b, a, back)


def test_data_only_replan_moves_nothing():
    """Holder / owner maps do not depend on m_i: a data-only re-plan moves 0 bytes."""
    cfg = MICRO
    L = cfg.n_layers
    mk = lambda m0: Pl.plan([Pl.pipe([Pl.even_stage(cfg, [0, 1], [0, L])], m0),
                             Pl.pipe([Pl.even_stage(cfg, [2], [0, L])], 4 - m0)], 2, 8)
    assert Lo.migration_deltas(cfg, mk(1), mk(3)) == []


def test_validation_errors():
    cfg = C1_TINY
    good = Pl.plan_matrix_c1(cfg)["P2"]
    Lo.validate(cfg, good, 2)
    import copy
    bad = copy.deepcopy(good); bad["pipes"][0]["n_micro"] = 3
    with pytest.raises(Lo.PlanError, match="PAPER.md:523"):
        Lo.validate(cfg, bad, 2)
    bad = copy.deepcopy(good); bad["pipes"][0]["stages"][0]["layers"] = [0, 1]
    with pytest.raises(Lo.PlanError):
        Lo.validate(cfg, bad, 2)
    bad = copy.deepcopy(good); bad["pipes"][0]["stages"][0]["heads"] = [4, 0]
    with pytest.raises(Lo.PlanError):
        Lo.validate(cfg, bad, 2)
    bad = copy.deepcopy(good); bad["pipes"][0]["stages"][0]["ffn"] = [500, 12]
    with pytest.raises(Lo.PlanError):
        Lo.validate(cfg, bad, 2)
    bad = copy.deepcopy(good); bad["standby"] = [1]
    with pytest.raises(Lo.PlanError):
        Lo.validate(cfg, bad, 2)


def test_plan_matrix_validates():
    cfg = C1_TINY
    for name, p in Pl.plan_matrix_c1(cfg).items():
        Lo.validate(cfg, p, Pl.world_of(p))


def test_gqa_rows_and_validation():
    """GQA: W_k / W_v rows follow the member's KV groups (query heads / g); a split that cuts a KV
    group is rejected."""
    from synth.gen import C1_GQA
    cfg = C1_GQA  # 4 query heads, 2 KV heads, d 32
    p = Pl.plan_matrix_gqa(cfg)["P1"]
    Lo.validate(cfg, p, 2)
    st = p["pipes"][0]["stages"][0]
    assert Lo.member_rows(cfg, st, "0.wq", 1) == (64, 128)
    assert Lo.member_rows(cfg, st, "0.wk", 0) == (0, 32) and Lo.member_rows(cfg, st, "0.wv", 1) == (32, 64)
    bad = Pl.plan([Pl.pipe([Pl.stage([0, 1], [3, 1], [256, 256], [128, 128], [0, cfg.n_layers])], 4)], 2, 8)
    with pytest.raises(Lo.PlanError):
        Lo.validate(cfg, bad, 2)
    # ownership still partitions every element exactly once (brute force)
    for name in ("0.wk", "1.wv", "0.wq"):
        own = Lo.owner_map(cfg, Pl.plan_matrix_gqa(cfg)["P4"], name)
        assert len(own) == Lo.n_elems(cfg, name) and all(o is not None for o in own)
