"""Step-parity worker: runs one malleable plan through libmalleus.so on N GPUs (one process per
GPU; launched by torchrun for N > 1) and compares against the oracle on rank 0.

Checks (readings R15, R16):
  * loss: |l - l_ref| / |l_ref| <= 1e-3 (bf16 path);
  * reduced gradients (sum_i w_i g_i on the owners, gathered over ranks into logical tensors):
    ||g - g_ref||_inf / ||g_ref||_inf <= 2e-2 per tensor, every element owned exactly once;
  * AdamW on owned pieces vs the oracle's AdamW applied to the GPU's own reduced gradient
    (fp32 vs fp64): <= 1e-6 relative on master;
  * param push: every holder's bf16 copy == RNE(owner's fp32 master), bit for bit.
Usage: python -m torch.distributed.run --nproc-per-node N tests/mp_worker.py <plan> <out.json>
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

from synth.gen import C1_TINY, C1_MED, C1_MED_GQA, C1_GQA, make_weights, make_tokens, bf16_rne, tensor_shapes  # noqa: E402
from paper_2410_13333_b200 import plans as Pl  # noqa: E402
from paper_2410_13333_b200 import _lib as L  # noqa: E402
from paper_2410_13333_b200.engine import Engine, gather_logical  # noqa: E402

import dataclasses  # noqa: E402
from synth.gen import C2_7B_SLICE  # noqa: E402

# c2l1: the bench's C2 shapes (h 4096, 32 heads of 128, ffn 11008, V 32000, s 2048) with one layer:
# full-size parity in the launch configuration bench.py times (CTA-pair GEMMs with the fused
# epilogues, tcgen05 attention at s = 2048, the TP-2 peer reduction with the scatter epilogue)
C2_1L = dataclasses.replace(C2_7B_SLICE, n_layers=1)
CONFIGS = {"c1": C1_TINY, "c1m": C1_MED, "c1mg": C1_MED_GQA, "c1g": C1_GQA, "c2l1": C2_1L}


def _plans(cfg_name, cfg, B, b):
    if cfg_name == "c2l1":  # B = 2 sequences, b = 1: two micro-batches (STORE then ACCUM weight gradients)
        L = cfg.n_layers
        tp2 = Pl.stage([0, 1], [22, 10], Pl._ffn_split(cfg.ffn, [1.0, 2.0]), Pl._vocab_split(cfg.vocab, [1.0, 2.0]),
                       [0, L])
        return {"P0": Pl.plan([Pl.pipe([Pl.even_stage(cfg, [0], [0, L])], B // b)], b, B),
                "P2": Pl.plan([Pl.pipe([tp2], B // b)], b, B)}
    if cfg.kv_heads != cfg.n_heads:
        return Pl.plan_matrix_gqa(cfg, B=B, b=b)
    return Pl.plan_matrix_c1(cfg, B=B, b=b)


def run(plan_name: str, rank: int = 0, world: int = 1, local_rank: int = 0, group=None, steps: int = 1,
        cfg_name: str = "c1", dtype: str = "bf16"):
    cfg = CONFIGS[cfg_name]
    B, b = (2, 1) if cfg_name == "c2l1" else (8, 2)
    plan = _plans(cfg_name, cfg, B, b)[plan_name]
    assert Pl.world_of(plan) == world, (plan_name, world)
    torch.cuda.set_device(local_rank)
    eng = Engine(cfg, rank, world, local_rank, group=group, dtype=dtype)
    eng.apply(plan)
    W = make_weights(cfg)
    eng.write_weights(W)
    tok, tgt = make_tokens(cfg, B)
    dtok = torch.tensor(tok, device="cuda")
    dtgt = torch.tensor(tgt, device="cuda")
    names = list(tensor_shapes(cfg))
    results = {"losses": []}
    reads_step1 = None
    clip = float(os.environ.get("MALLEUS_TEST_CLIP", "0"))  # global-norm clipping (max_grad_norm)
    for step in range(1, steps + 1):
        loss = eng.train_step(dtok, dtgt, step=step, apply_update=True, max_grad_norm=clip)
        torch.cuda.synchronize()
        results["losses"].append(float(loss.item()))
        if clip > 0:
            results.setdefault("grad_norms", []).append(eng.grad_norm()[0])
        if step == 1:
            reads_step1 = {n: (eng.read(n, L.KIND_RGRAD), eng.read(n, L.KIND_MASTER), eng.read(n, L.KIND_PARAM))
                           for n in names}
    eng.close()
    if world > 1:
        import torch.distributed as dist
        allr = [None] * world
        dist.all_gather_object(allr, reads_step1, group=group)
    else:
        allr = [reads_step1]
    if rank != 0:
        return None
    return check(cfg, W, tok, tgt, names, allr, results, plan, dtype)


def check(cfg, W, tok, tgt, names, allr, results, plan, dtype="bf16"):
    from oracle import model as M
    P = M.params_f64(W)
    loss_ref, g_ref = M.forward_backward(cfg, P, tok, tgt)
    out = {"loss": results["losses"][0], "loss_ref": loss_ref,
           "loss_rel": abs(results["losses"][0] - loss_ref) / abs(loss_ref), "grad_rel": {}, "adam_rel": {},
           "push_ok": True, "owned_once": True}
    hp = dict(M.ADAM_DEFAULT)
    clip = float(os.environ.get("MALLEUS_TEST_CLIP", "0"))
    coef = 1.0
    if clip > 0:  # the GPU clips its own reduced gradient: reproduce that from the gathered rgrads
        gs = {n: gather_logical([r[n][0] for r in allr], tensor_shapes(cfg)[n])[0].astype(np.float64) for n in names}
        _, gpu_norm = M.clip_grad_norm(gs, clip)
        coef = min(1.0, clip / (gpu_norm + 1e-6))
        out["grad_norm"] = results["grad_norms"][0]
        out["grad_norm_rgrad"] = gpu_norm
        out["clip_coef"] = coef
        hp["max_grad_norm"] = clip
    for n in names:
        shp = tensor_shapes(cfg)[n]
        g, seen = gather_logical([r[n][0] for r in allr], shp)
        cnt = np.zeros(int(np.prod(shp)), np.int64)
        for r in allr:
            for e0, e1 in r[n][0][0]:
                cnt[e0:e1] += 1
        out["owned_once"] &= bool(np.all(cnt == 1))
        out["grad_rel"][n] = float(np.abs(g - g_ref[n]).max() / max(np.abs(g_ref[n]).max(), 1e-30))
        master, _ = gather_logical([r[n][1] for r in allr], shp)
        wd = hp["weight_decay"] if M.decays(n) else 0.0
        th, _, _ = M.adamw(P[n], np.zeros(shp), np.zeros(shp), g.astype(np.float64) * coef, 1, hp["lr"], hp["beta1"],
                           hp["beta2"], hp["eps"], wd)
        out["adam_rel"][n] = float(np.abs(master - th).max() / max(np.abs(th).max(), 1e-30))
        # param push: each holder's bf16 == RNE(master) (fp32 mode: == master)
        want = bf16_rne(master.reshape(-1).astype(np.float32)) if dtype == "bf16" else \
            master.reshape(-1).astype(np.float32)
        for r in allr:
            (ranges, vals) = r[n][2]
            off = 0
            for e0, e1 in ranges:
                if not np.array_equal(vals[off:off + e1 - e0], want[e0:e1]):
                    out["push_ok"] = False
                off += e1 - e0
    # multi-step loss curve vs the oracle fed with bf16(master) each step (the GPU's param definition)
    if len(results["losses"]) > 1:
        Pm = {k: v.copy() for k, v in P.items()}
        Mm = {k: np.zeros_like(v) for k, v in P.items()}
        Vm = {k: np.zeros_like(v) for k, v in P.items()}
        ref_losses = []
        from synth.gen import bf16_to_f64
        for step in range(1, len(results["losses"]) + 1):
            Pb = {k: bf16_to_f64(bf16_rne(v.astype(np.float32))) if dtype == "bf16" else
                  v.astype(np.float32).astype(np.float64) for k, v in Pm.items()}
            l, g = M.forward_backward(cfg, Pb, tok, tgt)
            ref_losses.append(l)
            if clip > 0:
                g, _ = M.clip_grad_norm(g, clip)
            for k in Pm:
                wd = hp["weight_decay"] if M.decays(k) else 0.0
                Pm[k], Mm[k], Vm[k] = M.adamw(Pm[k], Mm[k], Vm[k], g[k], step, hp["lr"], hp["beta1"], hp["beta2"],
                                              hp["eps"], wd)
        out["losses"] = results["losses"]
        out["ref_losses"] = ref_losses
    return out


if __name__ == "__main__":
    import torch.distributed as dist
    plan_name, out_path = sys.argv[1], sys.argv[2]
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    dist.init_process_group("gloo")
    cfg_name = sys.argv[4] if len(sys.argv) > 4 else "c1"
    dtype = sys.argv[5] if len(sys.argv) > 5 else "bf16"
    r = run(plan_name, dist.get_rank(), dist.get_world_size(), int(os.environ.get("LOCAL_RANK", 0)), steps=steps,
            cfg_name=cfg_name, dtype=dtype)
    if dist.get_rank() == 0:
        json.dump(r, open(out_path, "w"), indent=1)
    dist.barrier()
    dist.destroy_process_group()
