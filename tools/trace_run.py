"""Dynamic straggler trace, end to end on 4 B200 (the PAPER.md:822-825
S1-S6 experiment at 4-GPU scale): a sequence of straggler situations is injected (DUTY mode) while
training continues; at every transition the Malleus loop runs — probe the per-rank speed
(malleus_probe_speed), re-plan from the probed rates (plans.plan_from_rates:
min-max splits and micro-batches, 5% dead band), migrate the model states (malleus_migrate,
PAPER.md:731-733) — and the step time before (stale plan) and after (re-planned) is measured.

  python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 tools/trace_run.py

Reports per situation: injected and probed x, the plan, T_stale, T_replanned, migration time, and
R_actual = T_replanned / T0 against R_opt = N / sum(1/x) (the paper's theoretic optimum)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

from synth.gen import C2_7B_SLICE, make_weights, make_tokens
from paper_2410_13333_b200 import plans as Pl
from paper_2410_13333_b200.engine import Engine

SITUATIONS = [  # rank -> x
    ("S0 none", {}),
    ("S1 rank1 1.5x", {1: 1.5}),
    ("S2 rank1 2x", {1: 2.0}),
    ("S3 rank1 2x + rank3 1.5x", {1: 2.0, 3: 1.5}),
    ("S4 rank3 3x", {3: 3.0}),
    ("S5 recovered", {}),
]


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    assert world == 4, "the trace is defined for 4 GPUs (DP2 x TP2)"
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    cfg, B = C2_7B_SLICE, 16
    plan = Pl.ladder_plan(cfg, world, B, b=1, straggle=False)
    eng = Engine(cfg, rank, world, local)
    eng.apply(plan)
    eng.write_weights(make_weights(cfg, parity=False))
    tok, tgt = make_tokens(cfg, B)
    dtok, dtgt = torch.tensor(tok, device="cuda"), torch.tensor(tgt, device="cuda")
    stream = torch.cuda.current_stream()
    step = [1]

    def steps(n):
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(n):
            eng.train_step(dtok, dtgt, step=step[0], apply_update=2)
            step[0] += 1
        b.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        t = torch.tensor([a.elapsed_time(b) / n], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    steps(3)  # warm-up
    t0 = steps(5)
    rows = []
    for name, xs in SITUATIONS:
        x = xs.get(rank, 1.0)
        eng.set_slowdown(x, 2 if x > 1.0 else 0)
        steps(2)  # the DUTY timers learn the segment durations
        t_stale = steps(4)
        probe = eng.probe(10)
        ref = sorted(probe)[0]
        x_probe = [p / ref for p in probe]
        obj = [Pl.plan_from_rates(cfg, plan, {r: x_probe[r] for r in range(world)}) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        new_plan = obj[0]
        mig = eng.migrate(new_plan)
        allm = [None] * world
        dist.all_gather_object(allm, mig)
        steps(2)
        t_new = steps(4)
        plan = new_plan
        xs_all = [xs.get(r, 1.0) for r in range(world)]
        r_opt = world / sum(1.0 / v for v in xs_all)
        rows.append({
            "situation": name, "x_injected": xs_all, "x_probed": [round(v, 3) for v in x_probe],
            "plan": [{"m": p["n_micro"], "heads": [s["heads"] for s in p["stages"]]} for p in plan["pipes"]],
            "ms_stale_plan": round(t_stale, 2), "ms_replanned": round(t_new, 2),
            "migration_s": round(max(m["total_seconds"] for m in allm), 4),
            "migration_GB": round(sum(m["bytes_recv"] for m in allm) / 1e9, 3),
            "R_actual": round(t_new / t0, 4), "R_opt": round(r_opt, 4),
            "R_opt_over_R_actual": round(r_opt / (t_new / t0), 4),
            "tokens_s": round(B * cfg.seq_len / (t_new / 1e3)),
        })
        if rank == 0:
            print(json.dumps(rows[-1]), flush=True)
    if rank == 0:
        print(json.dumps({"T0_ms": round(t0, 2), "T0_tokens_s": round(B * cfg.seq_len / (t0 / 1e3)),
                          "situations": len(rows)}), flush=True)
    eng.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
