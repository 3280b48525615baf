"""Oracle: the paper's closed forms used for measurement and plan construction.

TEST INFRASTRUCTURE ONLY (see oracle/model.py header).

* theoretic_optimum: T_normal * N / ((N - n) + sum_i 1/x_i)  (Table 2 caption).
* pipeline_time / approx: T_i = (m_i - 1) max_j t_ij + sum_j t_ij, t_ij = y_ij l_ij tau(b)
  and T_i ~ m_i max_j t_ij  (§4.2 "Cost Model").
* group_rate_even: y = rho_n * max x  (§4.2).
* group_rate_uneven: reading R8, y = rho_n * n * max_k f_k x_k for member fractions f_k.
* minmax_split: reading R7, integer apportionment argmin max_k c_k x_k s.t. sum c_k = n, the
  min-max form of Eq.(2) with heads / column tiles as the "layers";
  ties -> smallest sum c_k x_k (fastest members filled first), then lower index keeps more.
"""
from __future__ import annotations

import itertools
import math


def theoretic_optimum(t_normal: float, n_gpus: int, straggler_rates) -> float:
    n = len(straggler_rates)
    return t_normal * n_gpus / ((n_gpus - n) + sum(1.0 / x for x in straggler_rates))


def pipeline_time(y, l, m, tau):
    t = [yy * ll * tau for yy, ll in zip(y, l)]
    return (m - 1) * max(t) + sum(t)


def pipeline_time_approx(y, l, m, tau):
    return m * max(yy * ll for yy, ll in zip(y, l)) * tau


def group_rate_even(rates, rho=1.0):
    return rho * max(rates)


def group_rate_uneven(rates, counts, rho=1.0):
    n, tot = len(rates), sum(counts)
    return rho * n * max((c / tot) * x for c, x in zip(counts, rates))


def minmax_split(n_units: int, rates, min_units: int = 1):
    """Integer split of n_units over members with per-member rate x_k (reading R7).

    The optimal max-cost is the smallest candidate C = c*x_k with sum_k floor(C/x_k) >= n_units
    (every member >= min_units).  Ties at that C: smallest sum_k c_k x_k, i.e. fill the fastest
    members (smallest x, then lower index) up to their cap floor(C/x_k)."""
    k = len(rates)
    cands = sorted({round(c * x, 9) for x in rates for c in range(min_units, n_units + 1)})
    for C in cands:
        caps = [int(math.floor(C / x + 1e-9)) for x in rates]
        if all(cp >= min_units for cp in caps) and sum(caps) >= n_units:
            break
    counts = [min_units] * k
    left = n_units - min_units * k
    for i in sorted(range(k), key=lambda i: (rates[i], i)):
        add = min(left, caps[i] - counts[i])
        counts[i] += add
        left -= add
    assert left == 0
    return counts


def minmax_split_bruteforce(n_units: int, rates, min_units: int = 1):
    """Exhaustive reference for small n (tests only): key (max c x, sum c x, lower index more)."""
    best = None
    for c in itertools.product(range(min_units, n_units + 1), repeat=len(rates)):
        if sum(c) != n_units:
            continue
        key = (round(max(ci * x for ci, x in zip(c, rates)), 9),
               round(sum(ci * x for ci, x in zip(c, rates)), 9), tuple(-ci for ci in c))
        if best is None or key < best[0]:
            best = (key, list(c))
    return best[1]


def replan_needed(prev_rates, new_rates, threshold=0.05) -> bool:
    """5% trigger, strictly greater.  A change of exactly 5% in
    decimal (1.00 -> 1.05) is 0.05000000000000004 in binary, hence the 1e-12 guard."""
    return any(abs(n - p) / p > threshold + 1e-12 for p, n in zip(prev_rates, new_rates))
