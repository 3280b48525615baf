"""Multi-process host logic on CPU (world_size 2 and 4, gloo): each rank computes only its own
layout through the C-ABI (malleus_layout_query / migration_query, no GPU), the ranks exchange them
with the process group exactly as the engine exchanges its NCCL bootstrap id, and the cross-rank
invariants of the placement (reading R9) and of a re-plan's migration (R10 / R11) are checked on
rank 0: every element owned by exactly one rank, which also holds it; after migration every rank
holds exactly its new rows, each either kept or received once from an old holder."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from synth.gen import C1_TINY, tensor_shapes, tensor_id

KIND_PARAM, KIND_MASTER = 0, 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ranges(L, fn, *args):
    n = C.c_int32(0)
    assert fn(*args, None, C.byref(n)) == 0
    buf = (C.c_int64 * max(1, 2 * n.value))()
    cap = C.c_int32(n.value)
    assert fn(*args, buf, C.byref(cap)) == 0
    return [(buf[2 * i], buf[2 * i + 1]) for i in range(n.value)]


def _own_view(L, cfg, plan, world, rank):
    ccfg, ps = L.make_cfg(cfg), L.PlanStruct(plan)
    out = {}
    for name in tensor_shapes(cfg):
        for kind in (KIND_PARAM, KIND_MASTER):
            out[(name, kind)] = _ranges(L, L.lib.malleus_layout_query, C.byref(ccfg), ps.ref, world, rank,
                                        tensor_id(name), kind)
    return out


def _recv_view(L, cfg, a, b, world, rank):
    ccfg, pa, pb = L.make_cfg(cfg), L.PlanStruct(a), L.PlanStruct(b)
    moves = []
    for kind in (KIND_PARAM, KIND_MASTER):
        n = C.c_int32(0)
        assert L.lib.malleus_migration_query(C.byref(ccfg), pa.ref, pb.ref, world, rank, kind, None, None,
                                             C.byref(n)) == 0
        tbe = (C.c_int64 * max(1, 3 * n.value))()
        src = (C.c_int32 * max(1, n.value))()
        cap = C.c_int32(n.value)
        assert L.lib.malleus_migration_query(C.byref(ccfg), pa.ref, pb.ref, world, rank, kind, tbe, src,
                                             C.byref(cap)) == 0
        moves += [(tbe[3 * i], kind, tbe[3 * i + 1], tbe[3 * i + 2], src[i]) for i in range(n.value)]
    return moves


def _worker(rank, world, port, plans, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2410_13333_b200 import _lib as L
        boot = [bytes(range(128)) if rank == 0 else None]  # the engine's NCCL-id bootstrap path
        dist.broadcast_object_list(boot, src=0)
        assert boot[0] == bytes(range(128))
        a, b = plans
        views = [None] * world
        dist.all_gather_object(views, (_own_view(L, C1_TINY, a, world, rank), _own_view(L, C1_TINY, b, world, rank),
                                       _recv_view(L, C1_TINY, a, b, world, rank)))
        if rank == 0:
            q.put(views)
    except Exception as e:  # surface the failure instead of letting rank 0's queue wait time out
        q.put(repr(e))
        raise
    finally:
        dist.destroy_process_group()


def _mask(rs, n):
    m = np.zeros(n, np.int32)
    for e0, e1 in rs:
        m[e0:e1] += 1
    return m


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_layout_and_migration_invariants(world):
    from paper_2410_13333_b200 import plans as Pl
    cfg = C1_TINY
    P = Pl.plan_matrix_c1(cfg, B=8, b=2)
    a, b = (P["P1"], P["P2"]) if world == 2 else (P["P4"], P["P9"])  # even -> 3:1; cross-layout DP2 -> TP4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, (a, b), q)) for r in range(world)]
    for p in procs:
        p.start()
    views = q.get(timeout=300)
    assert not isinstance(views, str), views
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    sizes = {n: int(np.prod(shp)) for n, shp in tensor_shapes(cfg).items()}
    for pi in (0, 1):
        for name, n in sizes.items():
            owned = sum(_mask(views[r][pi][(name, KIND_MASTER)], n) for r in range(world))
            assert np.all(owned == 1), (pi, name)  # every element owned exactly once
            for r in range(world):
                o = _mask(views[r][pi][(name, KIND_MASTER)], n) > 0
                h = _mask(views[r][pi][(name, KIND_PARAM)], n) > 0
                assert np.all(h[o]), (pi, name, r)  # the owner holds its rows
    # migration: each rank's new holdings = kept old holdings + rows received exactly once, each from
    # a rank that held (param) / owned (Adam state) them under the old plan
    by_tid = {tensor_id(nm): nm for nm in sizes}
    for r in range(world):
        for kind in (KIND_PARAM, KIND_MASTER):
            got = {nm: np.zeros(n, np.int32) for nm, n in sizes.items()}
            for (tid, k, e0, e1, src) in views[r][2]:
                if k != kind:
                    continue
                nm = by_tid[tid]
                got[nm][e0:e1] += 1
                assert src != r
                src_old = _mask(views[src][0][(nm, kind)], sizes[nm]) > 0
                assert np.all(src_old[e0:e1]), (r, nm, kind, e0, e1, src)
            for nm, n in sizes.items():
                new = _mask(views[r][1][(nm, kind)], n) > 0
                old = _mask(views[r][0][(nm, kind)], n) > 0
                assert np.all(got[nm] <= 1), (r, nm, kind)
                assert np.all(new[got[nm] > 0]), (r, nm, kind)          # received rows are needed
                assert np.all(old[new & (got[nm] == 0)]), (r, nm, kind)  # the rest was already here
