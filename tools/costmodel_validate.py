"""Cost-model validation on B200 (the analogue of PAPER.md:1417-1434, App. A.1,
Fig. hetero_layer_batch): enumerate the layers and the micro-batches given to a straggler and compare
the measured step time with the paper's cost model:

    t_ij = y_ij * l_ij * tau(b)               (stage time for one micro-batch)
    T_i  = (m_i - 1) * max_j t_ij + sum_j t_ij (1F1B phase + warm-up / cool-down)
    T    = max_i T_i                           (the slowest pipeline bounds the step)
and its simplification T_i ~ m_i * max_j t_ij (the form the planner optimises, Eq. lower problem).

Two parameter sets are evaluated.  "advance": tau(b) profiled in advance as in the paper — one layer's
forward + backward for one micro-batch through the C-ABI (malleus_layer_fwd / malleus_layer_bwd) on a
non-straggling GPU — and y = the probe-measured rate.  "in-run": tau and x from the profiler's view of
a training step (reading R12 work-normalised): the uniform plan with the injection on.  The LM head and
embedding, which the paper's model folds into "identical layers", enter as layer equivalents by their
algorithmic FLOP ratio (h_eq = 2 h V / per-layer forward FLOPs per token); the straggler's y is the
probe-measured rate (reading R13).  Grad sync + AdamW are not in the paper's model; they
are measured separately and reported beside it.

Two enumerations on 2 GPUs, GPU 0 slowed by DUTY emulation:
  layers: one pipeline PP2 = {GPU 0: layers [0, l) + embedding, GPU 1: [l, L) + LM head}, m = B / b;
  data:   DP2 of TP1 pipelines (GPU 0, GPU 1) with all L layers each, m_0 = 0..B/b, m_1 = B/b - m_0.
For each point: measured step ms (max over ranks), per-rank compute ms, model T and the simplified model.
The paper's claim checked here: the argmin of the model coincides with the measured argmin.

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/costmodel_validate.py
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from synth.gen import C2_7B_SLICE, make_weights, make_tokens  # noqa: E402
from paper_2410_13333_b200 import plans as Pl  # noqa: E402
from paper_2410_13333_b200 import _lib as L  # noqa: E402
from paper_2410_13333_b200.engine import Engine  # noqa: E402


def layer_flops_per_token(cfg):
    h, F, s, d, n = cfg.hidden, cfg.ffn, cfg.seq_len, cfg.head_dim, cfg.n_heads
    return 8 * h * n * d + 2 * (s + 1) * n * d + 6 * h * F


def model_T(m, stages_t):
    """T_i = (m - 1) max_j t_ij + sum_j t_ij, and the simplification m max_j t_ij."""
    if m == 0:
        return 0.0, 0.0
    return (m - 1) * max(stages_t) + sum(stages_t), m * max(stages_t)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--x", type=float, default=1.5, help="straggling rate injected on GPU 0")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", 1))
    rank = int(os.environ.get("RANK", 0))
    assert world == 2, "run with 2 processes (one per GPU)"
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    dist.init_process_group("gloo")
    cfg = dataclasses.replace(C2_7B_SLICE, n_layers=args.layers)
    Lyr, B, b = cfg.n_layers, args.batch, 1
    m_all = B // b
    h_eq = 2 * cfg.hidden * cfg.vocab / layer_flops_per_token(cfg)
    eng = Engine(cfg, rank, world)
    tok, tgt = make_tokens(cfg, B)
    dtok, dtgt = torch.tensor(tok, device="cuda"), torch.tensor(tgt, device="cuda")
    W = make_weights(cfg, parity=False)
    stream = torch.cuda.current_stream()
    step = [1]

    def timed(n):
        for _ in range(2):
            eng.train_step(dtok, dtgt, step=step[0], apply_update=2)
            step[0] += 1
        torch.cuda.synchronize()
        dist.barrier()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(n):
            eng.train_step(dtok, dtgt, step=step[0], apply_update=2)
            step[0] += 1
        e.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        t = torch.tensor([a.elapsed_time(e) / n], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        comp = [None] * world
        dist.all_gather_object(comp, eng.timing())
        return float(t.item()), comp

    # ---- tau(b): one layer fwd + bwd for one micro-batch via the C-ABI, on a plan with no straggler
    dp = Pl.plan([Pl.pipe([Pl.even_stage(cfg, [r], [0, Lyr])], m_all // 2) for r in range(2)], b, B)
    eng.apply(dp)
    eng.write_weights(W)
    T, h = b * cfg.seq_len, cfg.hidden
    x = (torch.randn(T, h, device="cuda") * 0.5).to(torch.bfloat16)
    y = torch.empty_like(x)
    dy = (torch.randn(T, h, device="cuda") * 1e-3).to(torch.bfloat16)
    dx = torch.empty_like(x)
    st = stream.cuda_stream

    def layer_once():
        L.check(L.lib.malleus_layer_fwd(eng.ctx, 0, 0, x.data_ptr(), y.data_ptr(), st), eng.ctx, "layer_fwd")
        L.check(L.lib.malleus_layer_bwd(eng.ctx, 0, 0, dy.data_ptr(), dx.data_ptr(), st), eng.ctx, "layer_bwd")

    for _ in range(5):
        layer_once()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(20):
        layer_once()
    e.record(stream)
    torch.cuda.synchronize()
    tau_ms = a.elapsed_time(e) / 20
    taus = [None] * world
    dist.all_gather_object(taus, tau_ms)
    tau = taus[1]  # the non-straggling GPU's profile (GPU 0 is slowed below)
    # grad sync + AdamW time of the uniform DP plan (not modelled by the paper)
    base_ms, base_comp = timed(args.steps)

    # ---- straggler on GPU 0, rate measured by the probe (reading R13)
    nominal, x_meas = eng.calibrate_slowdown(0, args.x, mode=2)
    # in-run profile (the paper's profiler, reading R12): the uniform DP plan with the
    # injection on; both ranks do the same work, so x = t_comp(GPU 0) / t_comp(GPU 1), and the
    # in-step per-layer time tau_run = t_comp(GPU 1) / (m_1 (L + h_eq))
    eng.migrate(dp)
    _, comp_u = timed(args.steps)
    x_run = comp_u[0]["compute"] / comp_u[1]["compute"]
    tau_run = comp_u[1]["compute"] / ((m_all - m_all // 2) * (Lyr + h_eq))
    y0 = x_meas

    rows_l = []
    for l in range(1, Lyr):
        p = Pl.plan([Pl.pipe([Pl.even_stage(cfg, [0], [0, l]), Pl.even_stage(cfg, [1], [l, Lyr])], m_all)], b, B)
        eng.migrate(p)
        ms, comp = timed(args.steps)
        t0 = y0 * l * tau                       # embedding: negligible (a gather)
        t1 = (Lyr - l + h_eq) * tau
        Tm, Ts = model_T(m_all, [t0, t1])
        Tr, _ = model_T(m_all, [x_run * l * tau_run, (Lyr - l + h_eq) * tau_run])
        rows_l.append({"l_straggler": l, "l_other": Lyr - l, "measured_ms": ms,
                       "compute_ms": [c["compute"] for c in comp], "grad_sync_ms": [c["grad_sync"] for c in comp],
                       "model_ms": Tm, "model_simplified_ms": Ts, "model_inrun_ms": Tr})
    rows_m = []
    for m0 in range(0, m_all + 1):
        p = Pl.plan([Pl.pipe([Pl.even_stage(cfg, [0], [0, Lyr])], m0),
                     Pl.pipe([Pl.even_stage(cfg, [1], [0, Lyr])], m_all - m0)], b, B)
        eng.migrate(p)
        ms, comp = timed(args.steps)
        T0, S0 = model_T(m0, [y0 * (Lyr + h_eq) * tau])
        T1, S1 = model_T(m_all - m0, [(Lyr + h_eq) * tau])
        R0, _ = model_T(m0, [x_run * (Lyr + h_eq) * tau_run])
        R1, _ = model_T(m_all - m0, [(Lyr + h_eq) * tau_run])
        rows_m.append({"m_straggler": m0, "m_other": m_all - m0, "measured_ms": ms,
                       "compute_ms": [c["compute"] for c in comp], "grad_sync_ms": [c["grad_sync"] for c in comp],
                       "model_ms": max(T0, T1), "model_simplified_ms": max(S0, S1), "model_inrun_ms": max(R0, R1)})
    eng.set_slowdown(1.0, 0)
    eng.close()
    if rank == 0:
        def summary(rows, key):
            best_meas = min(rows, key=lambda r: r["measured_ms"])[key]
            best_model = min(rows, key=lambda r: r["model_ms"])[key]
            best_simpl = min(rows, key=lambda r: r["model_simplified_ms"])[key]
            best_run = min(rows, key=lambda r: r["model_inrun_ms"])[key]
            gs = min(min(r["grad_sync_ms"]) for r in rows)  # the exchange + AdamW floor (not modelled)
            err = [abs(r["measured_ms"] - gs - r["model_ms"]) / r["measured_ms"] for r in rows if r["model_ms"] > 0]
            err_r = [abs(r["measured_ms"] - gs - r["model_inrun_ms"]) / r["measured_ms"] for r in rows
                     if r["model_inrun_ms"] > 0]
            return {"argmin_measured": best_meas,
                    "advance_profile": {"argmin": best_model, "argmin_simplified": best_simpl,
                                        "coincide": best_meas == best_model,
                                        "mean_abs_rel_err_model_plus_sync": sum(err) / len(err),
                                        "max_abs_rel_err": max(err)},
                    "inrun_profile": {"argmin": best_run, "coincide": best_meas == best_run,
                                      "mean_abs_rel_err_model_plus_sync": sum(err_r) / len(err_r),
                                      "max_abs_rel_err": max(err_r)}}
        out = {"config": {"model": f"C2 shape, {Lyr} layers (h {cfg.hidden}, 32 heads, ffn {cfg.ffn}, V {cfg.vocab}, "
                                   f"s {cfg.seq_len})", "B": B, "b": b, "x_nominal": args.x,
                          "duty_nominal_used": nominal, "x_measured_probe": x_meas},
               "tau_ms": tau, "tau_ms_per_rank": taus, "h_eq": h_eq,
               "inrun": {"x_work_normalised": x_run, "tau_ms": tau_run,
                         "how": "uniform DP plan, injection on: x = t_comp(GPU0) / t_comp(GPU1) (equal work, "
                                "reading R12), tau = t_comp(GPU1) / (m_1 (L + h_eq))"},
               "uniform_dp_step_ms": base_ms, "uniform_dp_grad_sync_ms": [c["grad_sync"] for c in base_comp],
               "layers": {"rows": rows_l, "summary": summary(rows_l, "l_straggler")},
               "data": {"rows": rows_m, "summary": summary(rows_m, "m_straggler")}}
        s = json.dumps(out, indent=1)
        print(s, flush=True)
        if args.out:
            open(args.out, "w").write(s)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
