"""Migration worker: bit-exactness of malleus_migrate (readings R10/R11).

Every rank writes known logical params (bf16) and master / m / v (fp32, distinct random values)
under plan A, migrates to plan B, gathers the logical state and checks it is byte-identical to
what was written; then migrates back to A and checks again.  Also checks the bytes received
equal the oracle's delta bytes (oracle/layout.py, computed on rank 0).
Usage: python -m torch.distributed.run --nproc-per-node N tests/mp_migrate_worker.py <pair> <out.json>
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from synth.gen import C1_TINY, make_weights, tensor_shapes  # noqa: E402
from paper_2410_13333_b200 import plans as Pl  # noqa: E402
from paper_2410_13333_b200 import _lib as L  # noqa: E402
from paper_2410_13333_b200.engine import Engine, gather_logical  # noqa: E402

KINDS = (L.KIND_MASTER, L.KIND_ADAM_M, L.KIND_ADAM_V)


def plan_pair(name, cfg):
    M = Pl.plan_matrix_c1(cfg)
    if name == "P2-P1":
        return M["P2"], M["P1"]
    if name == "P4-swap":  # straggler moves from pipeline 0 to pipeline 1 (C5 analogue on 4 GPUs)
        s31 = lambda r: Pl.stage(r, [3, 1], [384, 128], [192, 64], [0, cfg.n_layers])
        ev = lambda r: Pl.even_stage(cfg, r, [0, cfg.n_layers])
        a = Pl.plan([Pl.pipe([s31([0, 1])], 1), Pl.pipe([ev([2, 3])], 3)], 2, 8)
        b = Pl.plan([Pl.pipe([ev([0, 1])], 3), Pl.pipe([s31([3, 2])], 1)], 2, 8, plan_id=1)
        return a, b
    if name == "P5-P6":  # different DP / PP structure on 3 GPUs
        return M["P5"], M["P6"]
    raise KeyError(name)


def run(pair, rank, world, local, group=None):
    cfg = C1_TINY
    a, b = plan_pair(pair, cfg)
    torch.cuda.set_device(local)
    eng = Engine(cfg, rank, world, local, group=group)
    eng.apply(a)
    W = make_weights(cfg)
    eng.write_weights(W)
    rng = np.random.default_rng(77)
    state = {n: {k: rng.standard_normal(int(np.prod(s))).astype(np.float32) for k in KINDS}
             for n, s in tensor_shapes(cfg).items()}
    for n in state:
        for k in KINDS:
            eng.write_state(n, k, state[n][k])

    def snapshot():
        return {n: {k: eng.read(n, k) for k in (L.KIND_PARAM,) + KINDS} for n in state}

    snaps = [snapshot()]
    st1 = eng.migrate(b)
    snaps.append(snapshot())
    st2 = eng.migrate(a)
    snaps.append(snapshot())
    eng.close()
    import torch.distributed as dist
    allr = [None] * world
    dist.all_gather_object(allr, {"snaps": snaps, "stats": [st1, st2]}, group=group)
    if rank != 0:
        return None
    from oracle import layout as Lo
    out = {"ok": True, "errors": [], "bytes_recv": [sum(r["stats"][i]["bytes_recv"] for r in allr) for i in (0, 1)]}
    out["oracle_bytes"] = [Lo.delta_bytes(Lo.migration_deltas(cfg, a, b)), Lo.delta_bytes(Lo.migration_deltas(cfg, b, a))]
    for si in range(3):
        for n, shp in tensor_shapes(cfg).items():
            for k in (L.KIND_PARAM,) + KINDS:
                dt = np.uint16 if k == L.KIND_PARAM else np.float32
                full, seen = gather_logical([r["snaps"][si][n][k] for r in allr], shp, dtype=dt)
                want = W[n].reshape(shp) if k == L.KIND_PARAM else state[n][k].reshape(shp)
                if not seen.all() or not np.array_equal(full.view(np.uint8), np.ascontiguousarray(want).view(np.uint8)):
                    out["ok"] = False
                    out["errors"].append((si, n, k))
                # every holder of a param must carry the same bytes
                if k == L.KIND_PARAM:
                    flat = want.reshape(-1)
                    for r in allr:
                        ranges, vals = r["snaps"][si][n][k]
                        off = 0
                        for e0, e1 in ranges:
                            if not np.array_equal(vals[off:off + e1 - e0], flat[e0:e1]):
                                out["ok"] = False
                                out["errors"].append((si, n, "holder"))
                            off += e1 - e0
    out["errors"] = out["errors"][:20]
    return out


if __name__ == "__main__":
    import torch.distributed as dist
    pair, out_path = sys.argv[1], sys.argv[2]
    dist.init_process_group("gloo")
    r = run(pair, dist.get_rank(), dist.get_world_size(), int(os.environ.get("LOCAL_RANK", 0)))
    if dist.get_rank() == 0:
        json.dump(r, open(out_path, "w"), indent=1)
    dist.barrier()
    dist.destroy_process_group()
