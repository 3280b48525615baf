"""Pins for oracle/costmodel.py against paper-printed values and brute force."""
import itertools

import numpy as np
import pytest

from oracle import costmodel as C
from paper_2410_13333_b200 import plans as Pl
from synth.gen import C2_7B_SLICE


def test_table2_theoretic_optimum_110b_s1():
    """Table 2 caption formula with the level-1 rate of Table 4 (2.62)
    and T_normal = 19.2 s (110B) gives the printed 19.4."""
    t = C.theoretic_optimum(19.2, 64, [2.62])
    assert round(t, 1) == 19.4


def test_spec_acceptance_9_ratio():
    """SPEC S:696 acceptance #9: N = 64, one x = 2.62 -> 1.0098 +- 1e-4."""
    assert abs(C.theoretic_optimum(1.0, 64, [2.62]) - 1.0098) <= 1e-4


def test_theoretic_optimum_edges():
    assert C.theoretic_optimum(1.0, 8, []) == 1.0
    assert abs(C.theoretic_optimum(1.0, 4, [float("inf")]) - 4 / 3) < 1e-15  # failed GPU
    # BJ target line: 1-of-8 at 2x -> surviving aggregate 7.5/8
    assert abs(1 / C.theoretic_optimum(1.0, 8, [2.0]) - 7.5 / 8) < 1e-15


def test_pipeline_time():
    """exact (m-1) max t + sum t >= approx m max t, equal for one stage."""
    y, l = [1.0, 2.0, 1.5], [4, 2, 3]
    ex = C.pipeline_time(y, l, 10, 0.1)
    ap = C.pipeline_time_approx(y, l, 10, 0.1)
    assert abs(ex - (9 * 0.45 + (0.4 + 0.4 + 0.45))) < 1e-12
    assert ex >= ap
    assert abs(C.pipeline_time([2.0], [3], 5, 1.0) - C.pipeline_time_approx([2.0], [3], 5, 1.0)) < 1e-12


def test_group_rates():
    """Reading R8 reduces to PAPER.md:491 (y = rho max x) for even splits."""
    rates = [1.0, 1.3, 1.0, 1.0]
    assert C.group_rate_uneven(rates, [16, 16, 16, 16]) == C.group_rate_even(rates)
    assert C.group_rate_uneven([1.0, 1.5], [19, 13]) == pytest.approx(2 * 19.5 / 32)


@pytest.mark.parametrize("seed", range(30))
def test_minmax_split_bruteforce(seed):
    rng = np.random.default_rng(seed)
    k = int(rng.integers(1, 5))
    n = int(rng.integers(k, 13))
    rates = [float(x) for x in rng.choice([1.0, 1.3, 1.5, 2.0, 3.0], size=k)]
    assert C.minmax_split(n, rates) == C.minmax_split_bruteforce(n, rates)


def test_survey_splits():
    """SURVEY App. A.5 examples (C2, C3; C4 pipeA) and the product-side duplicate agrees."""
    assert C.minmax_split(32, [1, 1.5]) == [19, 13]
    assert C.minmax_split(52, [1, 1, 1, 2]) == [15, 15, 15, 7]
    assert C.minmax_split(140, [1, 1, 1, 2]) == [40, 40, 40, 20]
    assert C.minmax_split(64, [1, 1.3, 1, 1]) == [17, 13, 17, 17]
    for n, r in ((32, [1, 2]), (64, [1, 1, 3, 1]), (86, [1, 1.5])):
        assert Pl._minmax(n, r) == C.minmax_split(n, r)
    p4 = Pl.ladder_plan(C2_7B_SLICE, 4, 16)
    assert p4["pipes"][0]["stages"][0]["heads"] == [19, 13]
    assert [pp["n_micro"] for pp in p4["pipes"]] == [7, 9]


def test_replan_threshold():
    """5% trigger, strict."""
    assert not C.replan_needed([1.0], [1.04])
    assert C.replan_needed([1.0], [1.06])
    assert not C.replan_needed([1.0], [1.05])
