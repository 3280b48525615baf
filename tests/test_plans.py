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


def test_rebalance_damped_between_current_and_full():
    """damp = 1: speed-proportional shares; damp -> 0: the current shares; in between, monotone
    (the measured 22/10 -> 25/7 overshoot of the C2 N = 2 straggler, bench_n2_r02z.json)."""
    cfg = C2_7B_SLICE
    p = Pl.ladder_plan(cfg, 2, 16)
    t = {0: 111.9, 1: 172.8}
    full = Pl.rebalance(cfg, p, t)["pipes"][0]["stages"][0]["heads"]
    assert full == [25, 7]  # 32 * (22/111.9) / (22/111.9 + 10/172.8) = 24.7
    h = [Pl.rebalance(cfg, p, t, damp=a)["pipes"][0]["stages"][0]["heads"][0] for a in (1e-6, 1 / 3, 2 / 3, 1.0)]
    assert h[0] == 22 and h == sorted(h) and h[2] == 24
    for a in (1 / 3, 2 / 3):
        validate(cfg, Pl.rebalance(cfg, p, t, damp=a), 2)
    q = Pl.ladder_plan(cfg, 4, 16)
    mm = [Pl.rebalance(cfg, q, {0: 60.0, 1: 60.0, 2: 40.0, 3: 40.0}, damp=a)["pipes"][1]["n_micro"] for a in (1e-6, 0.5, 1.0)]
    assert mm[0] == q["pipes"][1]["n_micro"] and mm == sorted(mm)


def test_resplit_candidates():
    """The straggler loop's measured candidates: distinct, valid, never the current split, full first."""
    cfg = C2_7B_SLICE
    p = Pl.ladder_plan(cfg, 2, 16)
    c = Pl.resplit_candidates(cfg, p, {0: 111.9, 1: 172.8})
    assert [x["pipes"][0]["stages"][0]["heads"] for x in c] == [[25, 7], [24, 8], [23, 9]]
    for x in c:
        validate(cfg, x, 2)
    # both members take equally long on their shares (the split is balanced): the heads stay (FFN /
    # vocab tiles may move by one tile of rounding)
    for x in Pl.resplit_candidates(cfg, p, {0: 100.0, 1: 100.0}):
        assert x["pipes"][0]["stages"][0]["heads"] == [22, 10]
    q = Pl.ladder_plan(cfg, 4, 16)
    cq = Pl.resplit_candidates(cfg, q, {0: 60.0, 1: 80.0, 2: 40.0, 3: 40.0})
    assert cq and len({str(x["pipes"]) for x in cq}) == len(cq)
    for x in cq:
        validate(cfg, x, 4)


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


def test_flops_per_token_matches_survey():
    """bench.py's algorithmic FLOPs per token (the tokens/s -> TF/s conversion) against SURVEY
    §8(d)'s per-config values (App. A.3: causal attention at (s+1)/2 keys, LM head included)."""
    import bench
    from synth.gen import C3_32B_SLICE, C4_70B_SLICE
    for cfg, ref in ((C2_7B_SLICE, 5.845e9), (C3_32B_SLICE, 5.526e10), (C4_70B_SLICE, 2.573e10)):
        assert abs(bench.flops_per_token(cfg) - ref) <= 5e-4 * ref, (cfg, bench.flops_per_token(cfg), ref)


@pytest.mark.parametrize("n,rates,want", [
    (32, [1.0, 1.5], [19, 13]),                  # C2 pipe 0
    (32, [1.0, 2.0], [22, 10]),                  # 2-GPU ladder rung
    (52, [1.0, 1.0, 1.0, 2.0], [15, 15, 15, 7]),  # C3 stage 0
    (64, [1.0, 1.3, 1.0, 1.0], [17, 13, 17, 17]),  # C4 pipe A
    (64, [1.0, 1.0, 3.0, 1.0], [20, 20, 4, 20]),   # C4 pipe B under reading R7's tie rule
])
def test_minmax_splits_match_survey(n, rates, want):
    got = Pl._minmax(n, rates)
    assert got == want
    # min-max optimality: no split has a smaller max cost (brute force over compositions for 2 members)
    if len(rates) == 2:
        best = min(max(a * rates[0], (n - a) * rates[1]) for a in range(1, n))
        assert max(c * x for c, x in zip(got, rates)) == best


@pytest.mark.parametrize("n", [2, 4, 8])
def test_plan_from_rates_random_rates_always_valid(n):
    """Property: for random probed rates (including extreme stragglers up to 20x), the re-plan keeps
    every plan invariant (oracle.layout.validate): whole heads >= 1 per member, FFN / vocab splits in
    multiples of 16 and >= 16, sums exact, sum of micro-batches = B / b."""
    import numpy as np
    rng = np.random.default_rng(11 + n)
    for cfg in (C2_7B_SLICE, C1_TINY):
        base = Pl.ladder_plan(cfg, n, 16, 1, straggle=False) if cfg is C2_7B_SLICE else None
        if base is None:
            if n == 8:
                continue
            base = Pl.plan_matrix_c1(cfg, B=8, b=2)["P9" if n == 4 else "P1"]
        p = base
        for _ in range(25):
            rates = {r: float(1.0 + (rng.pareto(1.5) if rng.random() < 0.5 else 0.0)) for r in range(n)}
            rates = {r: min(x, 20.0) for r, x in rates.items()}
            p = Pl.plan_from_rates(cfg, p, rates)
            validate(cfg, p, n)


@pytest.mark.parametrize("n", [2, 4, 8])
def test_rebalance_random_times_always_valid(n):
    """Property: plans.rebalance (re-plan from measured per-rank compute times) keeps every plan
    invariant for random, heavily skewed timings."""
    import numpy as np
    rng = np.random.default_rng(23 + n)
    p = Pl.ladder_plan(C2_7B_SLICE, n, 16, 1, straggle=True)
    for _ in range(25):
        t = {r: float(rng.uniform(10.0, 200.0)) for r in range(n)}
        p = Pl.rebalance(C2_7B_SLICE, p, t)
        validate(C2_7B_SLICE, p, n)


def test_plan_from_rates_mixed_pp_uses_slowest_stage():
    """a pipeline's per-micro-batch cost is its slowest stage (o_i = max_j y_ij l_ij,
    PAPER.md:503-506), not the sum of its stages.  A 2-stage 8 + 8-layer pipeline next to a
    16-layer single-stage pipeline runs a micro-batch in half the time, so at equal rates it must
    get twice the micro-batches (min-max, Eq.(3))."""
    from synth.gen import ModelCfg
    cfg = ModelCfg(n_layers=16, hidden=512, n_heads=4, head_dim=128, ffn=1536, vocab=2048, seq_len=256)
    ev = lambda ranks, layers: Pl.even_stage(cfg, ranks, layers)
    # the LM head sits on a last stage in both pipelines; embedding cost is not modelled
    p = Pl.plan([Pl.pipe([ev([0], [0, 8]), ev([1], [8, 16])], 6), Pl.pipe([ev([2], [0, 16])], 6)], 1, 12)
    q = Pl.plan_from_rates(cfg, p, {0: 1.0, 1: 1.0, 2: 1.0})
    validate(cfg, q, 3)
    assert [pp["n_micro"] for pp in q["pipes"]] == [8, 4]
    # the stage cost is FLOP-weighted: a 2x straggler that kept an even FFN share costs 2x
    st = ev([0, 1], [0, 16])
    c_even = Pl.stage_cost(cfg, st, [1.0, 1.0], False)
    assert Pl.stage_cost(cfg, st, [1.0, 2.0], False) == pytest.approx(2 * c_even)


@pytest.mark.parametrize("name", ["c3", "c4"])
def test_named_8gpu_workloads_validate(name):
    """BASELINE configs C3 / C4 as runnable plans: they validate under the
    oracle's Eq.(1) rules and the library's layout arithmetic, respect the
    kernel limits (b*s <= 8192, h <= 8192, h % 128), and carry SURVEY §8(d)'s shapes."""
    from synth.gen import C3_32B_SLICE, C4_70B_SLICE
    from tests.test_layout_abi import _query  # noqa: F401  (loads the library: host-only queries)
    cfg = C3_32B_SLICE if name == "c3" else C4_70B_SLICE
    plan, strag, uni = (Pl.c3_plan if name == "c3" else Pl.c4_plan)(cfg)
    validate(cfg, plan, 8)
    validate(cfg, uni, 8)
    assert plan["micro_batch"] * cfg.seq_len <= 8192 and cfg.hidden <= 8192 and cfg.hidden % 128 == 0
    if name == "c3":
        st0, st1 = plan["pipes"][0]["stages"]
        assert st0["heads"] == [15, 15, 15, 7] and [f // 128 for f in st0["ffn"]] == [40, 40, 40, 20]
        assert st0["layers"] == [0, 7] and st1["layers"] == [7, 16] and strag == {3: 2.0}
    else:
        assert [pp["n_micro"] for pp in plan["pipes"]] == [17, 15]  # m = (17, 15)
        assert plan["pipes"][0]["stages"][0]["heads"] != plan["pipes"][1]["stages"][0]["heads"]  # cross-layout
        assert strag == {1: 1.3, 6: 3.0}


def test_member_flops_sum_to_the_step():
    """reading R12's W_g: summed over the ranks of an even single-pipeline plan, the per-rank FLOPs
    equal the step's algorithmic FLOPs (bench.flops_per_token x tokens), embedding excluded."""
    import bench
    cfg = C2_7B_SLICE
    for n in (1, 2):
        p = Pl.ladder_plan(cfg, n, 16, straggle=False)
        tot = sum(Pl.member_flops(cfg, p, r) for r in range(n))
        assert tot == pytest.approx(bench.flops_per_token(cfg) * 16 * cfg.seq_len, rel=1e-12)


# ---- the asynchronous re-planner (plans.replan): standby removal and re-admission
def _rates(xs, n=4):
    return {r: xs.get(r, 1.0) for r in range(n)}


def test_replan_uniform_is_base():
    cfg = C2_7B_SLICE
    base = Pl.ladder_plan(cfg, 4, 16, straggle=False)
    p = Pl.replan(cfg, base, _rates({}))
    validate(cfg, p, 4)
    assert p["pipes"] == base["pipes"] and p["standby"] == []


@pytest.mark.parametrize("xs", [{1: 1.5}, {3: 3.0}, {1: 2.0, 3: 1.5}, {0: 1.3, 2: 2.5}])
def test_replan_moderate_stragglers_keep_every_gpu(xs):
    """Uneven splits absorb moderate stragglers: nobody is removed, the min-max splits follow x."""
    cfg = C2_7B_SLICE
    base = Pl.ladder_plan(cfg, 4, 16, straggle=False)
    p = Pl.replan(cfg, base, _rates(xs))
    validate(cfg, p, 4)
    assert p["standby"] == []
    for pp in p["pipes"]:
        st = pp["stages"][0]
        xr = [xs.get(r, 1.0) for r in st["ranks"]]
        slow = max(range(len(xr)), key=lambda k: xr[k])
        if xr[slow] > 1.05:
            assert st["heads"][slow] < cfg.n_heads // 2
    assert sum(pp["n_micro"] for pp in p["pipes"]) == 16


def test_replan_removes_heavy_straggler_and_readmits():
    """x = 12 (the paper's level-3 rate) in a TP-2 group: with the measured TP efficiency the
    group runs faster without it, so it goes to standby; when its (re-)probed rate recovers the
    next replan from the base grouping re-admits it."""
    cfg = C2_7B_SLICE
    base = Pl.ladder_plan(cfg, 4, 16, straggle=False)
    p = Pl.replan(cfg, base, _rates({3: 12.0}))
    validate(cfg, p, 4)
    assert p["standby"] == [3]
    assert [st["ranks"] for st in p["pipes"][1]["stages"]] == [[2]]
    assert p["pipes"][0]["n_micro"] > p["pipes"][1]["n_micro"]  # the shrunk pipeline takes fewer micro-batches
    q = Pl.replan(cfg, base, _rates({}))
    validate(cfg, q, 4)
    assert q["standby"] == [] and q["pipes"] == base["pipes"]


def test_replan_removal_only_when_it_pays():
    """Removal is chosen iff the group's cost (min-max split, TP efficiency of its size) drops by
    more than min_gain; with TP efficiency 1 (no TP overhead) keeping every GPU is never worse."""
    cfg = C2_7B_SLICE
    base = Pl.ladder_plan(cfg, 4, 16, straggle=False)
    p = Pl.replan(cfg, base, _rates({3: 12.0}), eff={1: 1.0, 2: 1.0})
    assert p["standby"] == []


# ---- recovery after a failure: survivors re-planned with x = infinity for the lost GPUs
@pytest.mark.parametrize("name,failed", [("P1", [1]), ("P2", [0]), ("P4", [1]), ("P4", [2, 3]), ("P6", [2]),
                                         ("P5", [2]), ("P9", [3])])
def test_survivor_plan_valid(name, failed):
    cfg = C1_TINY
    p = Pl.plan_matrix_c1(cfg)[name]
    world = Pl.world_of(p)
    q, remap = Pl.survivor_plan(cfg, p, failed)
    validate(cfg, q, len(remap))
    assert set(remap) == set(range(world)) - set(failed)
    assert sorted(remap.values()) == list(range(len(remap)))
    assert sum(pp["n_micro"] for pp in q["pipes"]) * q["micro_batch"] == q["global_batch"]
    used = {r for pp in q["pipes"] for st in pp["stages"] for r in st["ranks"]}
    assert used | set(q["standby"]) == set(range(len(remap)))


def test_survivor_plan_drops_broken_pipeline():
    """A pipeline that lost a whole stage cannot run: its micro-batches move to the others."""
    cfg = C1_TINY
    p = Pl.plan_matrix_c1(cfg)["P4"]  # pipe0 = TP2 {0, 1}, pipe1 = TP2 {2, 3}
    q, remap = Pl.survivor_plan(cfg, p, [0, 1])
    assert len(q["pipes"]) == 1 and q["pipes"][0]["n_micro"] * q["micro_batch"] == q["global_batch"]
    assert remap == {2: 0, 3: 1}
    with pytest.raises(ValueError):
        Pl.survivor_plan(cfg, Pl.plan_matrix_c1(cfg)["P1"], [0, 1])
