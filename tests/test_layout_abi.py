"""Host logic of the C-ABI library (no GPU): the library loads, exports every function that
include/malleus.h declares, and its range arithmetic for holders / owners (reading R9) and
migration transfers (readings R10/R11) equals the oracle's per-element definitions."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from synth.gen import C1_TINY, MICRO, tensor_shapes, tensor_id
from oracle import layout as Lo
from paper_2410_13333_b200 import plans as Pl
from tests.planutil import random_plan

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2410_13333_b200 import _lib
    return _lib


def test_exports_every_header_function(L):
    src = open(os.path.join(ROOT, "include", "malleus.h")).read()
    names = set(re.findall(r"\b(malleus_[a-z0-9_]+)\s*\(", src))
    assert len(names) >= 20
    for n in sorted(names):
        assert hasattr(L.lib, n), f"libmalleus.so does not export {n}"
    assert set(L.EXPORTED) >= names


def _query(L, cfg, plan, world, rank, name, kind):
    ccfg = L.make_cfg(cfg)
    ps = L.PlanStruct(plan)
    n = C.c_int32(0)
    assert L.lib.malleus_layout_query(C.byref(ccfg), ps.ref, world, rank, tensor_id(name), kind, None,
                                      C.byref(n)) == 0
    buf = (C.c_int64 * max(1, 2 * n.value))()
    cap = C.c_int32(n.value)
    assert L.lib.malleus_layout_query(C.byref(ccfg), ps.ref, world, rank, tensor_id(name), kind, buf,
                                      C.byref(cap)) == 0
    out = set()
    for i in range(n.value):
        out.update(range(buf[2 * i], buf[2 * i + 1]))
    return out


def _check_plan(L, cfg, plan, world, names=None, max_samples=300, seed=0):
    """Every element's owner / holders (sampled on big tensors, always including row boundaries)."""
    rng = np.random.default_rng(seed)
    names = names or list(tensor_shapes(cfg))
    for name in names:
        n = Lo.n_elems(cfg, name)
        c = Lo.row_width(cfg, name)
        if n <= max_samples:
            sample = range(n)
        else:
            cuts = sorted(set().union(*[Lo.pipeline_cuts(cfg, pp, name) for pp in plan["pipes"]]))
            edge = {min(n - 1, max(0, r * c + d)) for r in cuts for d in (-1, 0)}
            sample = sorted(edge | set(rng.integers(0, n, size=max_samples).tolist()))
        own = {e: Lo.owner_of_element(cfg, plan, name, e)[0] for e in sample}
        hold = {e: Lo.holders_of_element(cfg, plan, name, e) for e in sample}
        for r in range(world):
            got_own = _query(L, cfg, plan, world, r, name, Lo.KIND_MASTER)
            got_hold = _query(L, cfg, plan, world, r, name, Lo.KIND_PARAM)
            for e in sample:
                assert (e in got_own) == (own[e] == r), (name, r, e)
                assert (e in got_hold) == (r in hold[e]), (name, r, e)
            if n <= max_samples:
                assert got_own <= set(range(n)) and got_hold <= set(range(n))


@pytest.mark.parametrize("pname", ["P0", "P1", "P2", "P3", "P4", "P5", "P6", "P7", "P8", "P9", "P10", "P11"])
def test_layout_plan_matrix(L, pname):
    cfg = C1_TINY
    p = Pl.plan_matrix_c1(cfg)[pname]
    _check_plan(L, cfg, p, Pl.world_of(p), names=["0.g1", "0.wq", "0.wo", "1.wd", "1.wu", "E", "gf", "Wlm"])


def test_layout_random_plans(L):
    rng = np.random.default_rng(99)
    for _ in range(25):
        p, world = random_plan(rng, MICRO, world_max=7, B=8, b=2)
        _check_plan(L, MICRO, p, world)


def test_plan_validation_errors(L):
    cfg = C1_TINY
    p = Pl.plan_matrix_c1(cfg)["P2"]
    p["pipes"][0]["n_micro"] = 3  # violates sum m_i b = B
    ccfg = L.make_cfg(cfg)
    n = C.c_int32(0)
    assert L.lib.malleus_layout_query(C.byref(ccfg), L.PlanStruct(p).ref, 2, 0, 1, 0, None, C.byref(n)) == 2


def _migration(L, cfg, a, b, world):
    ccfg = L.make_cfg(cfg)
    pa, pb = L.PlanStruct(a), L.PlanStruct(b)
    moves = set()
    for dst in range(world):
        for kind in (Lo.KIND_PARAM, Lo.KIND_MASTER, Lo.KIND_ADAM_M, Lo.KIND_ADAM_V):
            n = C.c_int32(0)
            assert L.lib.malleus_migration_query(C.byref(ccfg), pa.ref, pb.ref, world, dst, kind, None, None,
                                                 C.byref(n)) == 0
            tbe = (C.c_int64 * max(1, 3 * n.value))()
            src = (C.c_int32 * max(1, n.value))()
            cap = C.c_int32(n.value)
            assert L.lib.malleus_migration_query(C.byref(ccfg), pa.ref, pb.ref, world, dst, kind, tbe, src,
                                                 C.byref(cap)) == 0
            for i in range(n.value):
                for e in range(tbe[3 * i + 1], tbe[3 * i + 2]):
                    moves.add((tbe[3 * i], kind, e, src[i], dst))
    return moves


def test_migration_matches_oracle(L):
    cfg = MICRO
    rng = np.random.default_rng(5)
    done = 0
    while done < 12:
        a, wa = random_plan(rng, cfg, world_max=5, B=8, b=2)
        b, wb = random_plan(rng, cfg, world_max=5, B=8, b=2)
        if wa != wb:
            continue
        ref = {(tensor_id(n), k, e, s, d) for (n, k, e, s, d) in Lo.migration_deltas(cfg, a, b)}
        got = _migration(L, cfg, a, b, wa)
        assert got == ref
        done += 1
    assert _migration(L, cfg, a, a, wa) == set()


@pytest.mark.parametrize("pname", ["P0", "P1", "P3", "P4", "P6"])
def test_layout_gqa_plans(L, pname):
    """GQA: the library's W_k / W_v rows follow whole KV groups, as the oracle's member_rows."""
    from synth.gen import C1_GQA
    cfg = C1_GQA
    p = Pl.plan_matrix_gqa(cfg)[pname]
    _check_plan(L, cfg, p, Pl.world_of(p), names=["0.wq", "0.wk", "1.wv", "0.wo", "E", "Wlm"])


def test_layout_gqa_rejects_split_group(L):
    from synth.gen import C1_GQA
    cfg = C1_GQA
    p = Pl.plan([Pl.pipe([Pl.stage([0, 1], [3, 1], [256, 256], [128, 128], [0, cfg.n_layers])], 4)], 2, 8)
    ccfg = L.make_cfg(cfg)
    n = C.c_int32(0)
    assert L.lib.malleus_layout_query(C.byref(ccfg), L.PlanStruct(p).ref, 2, 0, 1, 0, None, C.byref(n)) == 2
