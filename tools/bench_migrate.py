"""Migration GB/s (BASELINE.json metric, second half): re-plan when the straggler moves.

C5 (BASELINE.json configs[4]): LLaMA-110B-shaped 4-layer slice (h 8192, 64 heads, ffn 49152,
V 32000, seq 4096, B 16), DP2 x TP4 on 8 GPUs; plan A has the 2x straggler on GPU 3 (pipeline 0,
heads 19/19/19/7), plan B on GPU 6 (pipeline 1).  With --gpus 4 the same shapes run DP2 x TP2 and
the straggler moves GPU 1 -> GPU 3.  Timed: malleus_migrate(A -> B) (peer pulls over NVLink by
default; 4-layer packs with grouped NCCL P2P, under MALLEUS_NO_P2P=1) between barriers; GB/s = bytes moved over all ranks / max seconds over ranks.
Parameter values are not initialised (the copy moves bytes regardless of content); bit-exactness is
tests/test_gpu_migrate.py's job.
  python -m torch.distributed.run --nproc-per-node N tools/bench_migrate.py --gpus N
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def plans(cfg, n):
    from paper_2410_13333_b200 import plans as Pl
    L = cfg.n_layers
    if n == 8:
        rates_a = [1.0, 1.0, 1.0, 2.0]
        rates_b = [1.0, 1.0, 2.0, 1.0]
        tp = 4
    elif n == 4:
        rates_a = [1.0, 2.0]
        rates_b = [1.0, 2.0]
        tp = 2
    else:
        raise SystemExit("--gpus 4 or 8")
    st = lambda ranks, rates: Pl.stage(ranks, Pl._heads_split(cfg.n_heads, rates), Pl._ffn_split(cfg.ffn, rates),
                                       Pl._vocab_split(cfg.vocab, rates), [0, L])
    ev = lambda ranks: Pl.even_stage(cfg, ranks, [0, L])
    r0, r1 = list(range(tp)), list(range(tp, 2 * tp))
    a = Pl.plan([Pl.pipe([st(r0, rates_a)], 7), Pl.pipe([ev(r1)], 9)], 1, 16)
    b = Pl.plan([Pl.pipe([ev(r0)], 9), Pl.pipe([st(r1, rates_b)], 7)], 1, 16, plan_id=1)
    return a, b


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=8)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist
    from synth.gen import C5_110B_SLICE
    from paper_2410_13333_b200.engine import Engine
    cfg = C5_110B_SLICE
    world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    a, b = plans(cfg, world)
    eng = Engine(cfg, rank, world, local)
    eng.apply(a)
    torch.cuda.synchronize()
    dist.barrier()
    # warm-up round trip: NCCL establishes peer connections lazily on first use; in a training job
    # they exist from previous re-plans / grad syncs
    eng.migrate(b)
    dist.barrier()
    eng.migrate(a)
    dist.barrier()
    st = eng.migrate(b)
    dist.barrier()
    # and back (A -> B -> A)
    st2 = eng.migrate(a)
    dist.barrier()
    allst = [None] * world
    dist.all_gather_object(allst, (st, st2))
    if rank == 0:
        out = {}
        for i, name in enumerate(("A->B", "B->A")):
            tot = sum(s[i]["bytes_recv"] for s in allst)
            secs = max(s[i]["seconds"] for s in allst)
            mx = max(s[i]["bytes_recv"] for s in allst)
            out[name] = {"bytes_total": tot, "seconds_max": secs, "GBps_total": tot / secs / 1e9,
                         "max_recv_bytes_per_gpu": mx, "GBps_per_gpu_max": mx / secs / 1e9,
                         "n_packs": allst[0][i]["n_packs"]}
        line = {"metric": "migration GB/s", "value": out["A->B"]["GBps_total"], "unit": "GB/s", "n_gpus": world,
                "config": {"workload": f"C5 LLaMA-110B-shaped {cfg.n_layers}-layer slice",
                           "plan": "DP2 x TP%d, straggler moves pipeline 0 -> 1" % (world // 2)},
                "nvlink_peak_GBps_per_dir": 900, "nvlink_measured_peer_copy_GBps": 770, "detail": out}
        print(json.dumps(line), flush=True)
    eng.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
