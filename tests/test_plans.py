"""Host-side plan builders: the ladder plans validate, and the measured-rate re-plan (profiler ->
planner loop, reading R12) keeps every invariant of Eq.(1)
while moving work away from slow ranks."""
import pytest

from synth.gen import C2_7B_SLICE, C1_TINY
from oracle.layout import validate
from paper_2410_13333_b200 import plans as Pl


@pytest.mark.parametrize("n", [1, 2, 4, 8])
@pytest.mark.parametrize("straggle", [True, False])
def test_ladder_plans_validate(n, straggle):
    p = Pl.ladder_plan(C2_7B_SLICE, n, 16, straggle=straggle)
    validate(C2_7B_SLICE, p, n)


def test_rebalance_moves_work_to_fast_ranks():
    cfg = C2_7B_SLICE
    p = Pl.ladder_plan(cfg, 2, 16)
    q = Pl.rebalance(cfg, p, {0: 137.0, 1: 189.0})
    validate(cfg, q, 2)
    a, b = p["pipes"][0]["stages"][0], q["pipes"][0]["stages"][0]
    assert b["heads"][0] > a["heads"][0] and b["ffn"][0] > a["ffn"][0] and b["vocab"][0] > a["vocab"][0]
    # balanced measurement (both members take equally long) -> unchanged
    r = Pl.rebalance(cfg, p, {0: 100.0, 1: 100.0})
    assert abs(r["pipes"][0]["stages"][0]["heads"][0] - 22) <= 1


def test_rebalance_micro_batches():
    cfg = C2_7B_SLICE
    p = Pl.ladder_plan(cfg, 4, 16)
    q = Pl.rebalance(cfg, p, {0: 60.0, 1: 60.0, 2: 40.0, 3: 40.0})
    validate(cfg, q, 4)
    assert sum(pp["n_micro"] for pp in q["pipes"]) == 16
    assert q["pipes"][1]["n_micro"] > p["pipes"][1]["n_micro"]


def test_rebalance_plan_matrix_c1():
    for name, p in Pl.plan_matrix_c1(C1_TINY).items():
        world = Pl.world_of(p)
        q = Pl.rebalance(C1_TINY, p, {r: 10.0 + r for r in range(world)})
        validate(C1_TINY, q, world)


def test_plan_from_rates_valid_and_recovers():
    """plans.plan_from_rates: every re-plan of the 4-GPU trace validates (layout ABI), stragglers get
    fewer heads / FFN tiles and their pipeline fewer micro-batches, rates inside the 5% dead band
    change nothing, and a recovered cluster returns to the even plan exactly."""
    cfg = C2_7B_SLICE
    even = Pl.ladder_plan(cfg, 4, 16, 1, straggle=False)
    p = even
    for xs in ({1: 1.62}, {1: 2.14}, {1: 2.14, 3: 1.62}, {3: 3.2}, {0: 1.03, 2: 1.049}, {}):
        q = Pl.plan_from_rates(cfg, p, {g: xs.get(g, 1.0) for g in range(4)})
        validate(cfg, q, 4)
        for pp in q["pipes"]:
            for st in pp["stages"]:
                assert sum(st["heads"]) == cfg.n_heads and sum(st["ffn"]) == cfg.ffn and sum(st["vocab"]) == cfg.vocab
                for k, r in enumerate(st["ranks"]):
                    if xs.get(r, 1.0) >= 1.05:
                        assert st["heads"][k] < cfg.n_heads // len(st["ranks"])
        assert sum(pp["n_micro"] for pp in q["pipes"]) == 16
        if any(v >= 1.05 for v in xs.values()):
            slow_pipes = [i for i, pp in enumerate(q["pipes"]) if any(xs.get(r, 1) >= 1.05 for st in pp["stages"] for r in st["ranks"])]
            if len(slow_pipes) == 1:
                assert q["pipes"][slow_pipes[0]]["n_micro"] < 8
        p = q
    assert [pp["stages"] for pp in p["pipes"]] == [pp["stages"] for pp in even["pipes"]]
    assert [pp["n_micro"] for pp in p["pipes"]] == [8, 8]
