"""Dynamic straggler trace, end to end on 4 B200 (the PAPER.md:822-825
S1-S6 experiment at 4-GPU scale): a sequence of straggler situations is injected (DUTY mode) while
training continues, and the Malleus loop reacts:

  * profiler: every situation is probed with malleus_probe_speed; the probe is
    world-collective, so GPUs on standby are re-probed too and are re-admitted when
    their rate recovers; rates are x_g = t_g / t_ref with t_ref the median probe of a start-up
    calibration without injection (reading R12); a change beyond 5% triggers re-planning;
  * planner, asynchronous: rank 0 runs plans.replan (min-max splits per group,
    removal of a heavy straggler when its group runs faster without it, micro-batches min-max over
    the pipelines) on a background thread while all ranks keep training on the stale plan; after
    every step the ranks agree (one broadcast) whether the new plan is ready, and migrate at that
    step boundary (malleus_migrate);
  * the profiler's in-run view refines the new plan once (plans.rebalance from the measured compute
    times, reading R12, full and damped re-split; the fastest is kept);
  * the step time with the stale plan and with the (refined) new plan is measured.

  python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 tools/trace_run.py [--sync]

--sync: the round-1 loop (plan_from_rates between steps, no overlap, no removal).
Reports per situation: injected and probed x, the plan and standby set, planner wall time and the
number of steps trained while it ran, T_stale, T_replanned, migration time / bytes, and
R_actual = T_replanned / T0 against R_opt = N / sum(1/x) (the paper's theoretic optimum)."""
import argparse
import concurrent.futures as cf
import json
import os
import statistics
import sys
import time

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
    ("S5 rank3 12x (removed)", {3: 12.0}),
    ("S6 recovered (re-admitted)", {}),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sync", action="store_true")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    assert world == 4, "the trace is defined for 4 GPUs (DP2 x TP2)"
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    cfg, B = C2_7B_SLICE, 16
    base = Pl.ladder_plan(cfg, world, B, b=1, straggle=False)
    plan = base
    eng = Engine(cfg, rank, world, local)
    eng.apply(plan)
    eng.write_weights(make_weights(cfg, parity=False))
    tok, tgt = make_tokens(cfg, B)
    dtok, dtgt = torch.tensor(tok, device="cuda"), torch.tensor(tgt, device="cuda")
    stream = torch.cuda.current_stream()
    step = [1]
    pool = cf.ThreadPoolExecutor(max_workers=1) if rank == 0 else None

    def one_step():
        eng.train_step(dtok, dtgt, step=step[0], apply_update=2)
        step[0] += 1

    def steps(n):
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(n):
            one_step()
        b.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        t = torch.tensor([a.elapsed_time(b) / n], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    steps(3)  # warm-up
    t0 = steps(5)
    t_ref = statistics.median(eng.probe(10))  # start-up calibration, no injection (reading R12)
    x_prev = [1.0] * world
    rows = []
    for name, xs in SITUATIONS:
        x = xs.get(rank, 1.0)
        eng.set_slowdown(x, 2 if x > 1.0 else 0)
        steps(2)  # the DUTY timers learn the segment durations
        t_stale = steps(3)
        probe = eng.probe(10)  # every rank, standby included
        x_probe = [p / t_ref for p in probe]
        trig = any(abs(a - b) / b > 0.05 + 1e-12 for a, b in zip(x_probe, x_prev))
        x_prev = x_probe
        plan_s, stale_steps = 0.0, 0
        if args.sync:
            obj = [Pl.plan_from_rates(cfg, plan, {r: x_probe[r] for r in range(world)}) if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            new_plan = obj[0]
        else:
            fut = None
            if rank == 0:
                def planner(rates):
                    t = time.perf_counter()
                    p = Pl.replan(cfg, base, rates)
                    return p, time.perf_counter() - t
                fut = pool.submit(planner, {r: x_probe[r] for r in range(world)})
            while True:  # keep training on the stale plan until the planner is done
                one_step()
                stale_steps += 1
                flag = torch.tensor([1 if (rank == 0 and fut.done()) else 0])
                dist.broadcast(flag, src=0)
                if flag.item():
                    break
            obj = [fut.result() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            new_plan, plan_s = obj[0]
        changed = json.dumps(new_plan["pipes"]) != json.dumps(plan["pipes"]) or new_plan["standby"] != plan["standby"]
        mig = {"total_seconds": 0.0, "bytes_recv": 0}
        if changed:
            mig = eng.migrate(new_plan)
            plan = new_plan
        allm = [None] * world
        dist.all_gather_object(allm, mig)
        steps(2)
        t_new = steps(4)
        # the profiler keeps measuring: one refinement from the measured compute
        # times of the new plan (reading R12, plans.rebalance re-splits within the groups), kept only
        # if it is faster — the planner's FLOP-proportional costs miss the narrow shards' lower
        # GEMM efficiency (wave quantisation on 148 SMs)
        refined = False
        if not args.sync and changed:
            comp = [None] * world
            dist.all_gather_object(comp, eng.timing()["compute"])
            obj = [Pl.resplit_candidates(cfg, plan, {r: comp[r] for r in range(world)}, damps=(1.0, 2 / 3))
                   if rank == 0 else None]  # full and damped re-split (plans.rebalance docstring)
            dist.broadcast_object_list(obj, src=0)
            at = best = plan
            for cand in obj[0]:
                eng.migrate(cand)
                at = cand
                steps(2)
                t_cand = steps(4)
                if t_cand < t_new:
                    best, t_new, refined = cand, t_cand, True
            if at is not best:
                eng.migrate(best)
                steps(2)
            plan = best
        xs_all = [xs.get(r, 1.0) for r in range(world)]
        r_opt = world / sum(1.0 / v for v in xs_all)
        rows.append({
            "situation": name, "x_injected": xs_all, "x_probed": [round(v, 3) for v in x_probe], "triggered": trig,
            "plan": [{"m": p["n_micro"], "ranks": [s["ranks"] for s in p["stages"]],
                      "heads": [s["heads"] for s in p["stages"]]} for p in plan["pipes"]],
            "standby": plan["standby"], "planner_s": round(plan_s, 4), "steps_during_planning": stale_steps,
            "refined_from_measured_compute": refined,
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
        summary = {"T0_ms": round(t0, 2), "T0_tokens_s": round(B * cfg.seq_len / (t0 / 1e3)),
                   "situations": len(rows), "mode": "sync" if args.sync else "async planner + standby re-probe"}
        print(json.dumps(summary), flush=True)
        if args.out:
            json.dump({"summary": summary, "rows": rows}, open(args.out, "w"), indent=1)
    eng.set_slowdown(1.0, 0)
    eng.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
