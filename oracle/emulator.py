"""Oracle: fp64 partition emulator — executes a malleable plan's arithmetic member by member.

TEST INFRASTRUCTURE ONLY (see oracle/model.py header).  Shares code with oracle/model.py
(allowed, SURVEY §8(c) "Partition emulator") and never with the CUDA path.

For each pipeline i with m_i > 0 it takes its contiguous sequences (reading R14), runs every
micro-batch through its stages, splitting every layer over the stage's TP members exactly as
Megatron TP does (column-parallel QKV / gate-up, row-parallel O / down with member partial sums
added in member order, §2.1) and the LM head vocab-parallel (per-member max and
sum-exp combined).  Member-local gradients accumulate over the pipeline's micro-batches; each
pipeline's gradient is the mean over its own m_i*b*s tokens and pipelines are combined with
w_i = m_i*b/B (reading R4, Eq.(1)) piece by piece through the owner map of
oracle/layout.py (reading R9).  AdamW then runs on owned pieces only.  The
result must equal the unpartitioned oracle step to <= 1e-12 relative (the lossless property,
PAPER.md:303).
"""
from __future__ import annotations

import numpy as np

from synth.gen import ModelCfg, tensor_shapes
from oracle import model as M
from oracle.layout import (member_rows, stage_of, split_kind, pipeline_cuts, row_width,
                           sync_holder)


def _layer_fwd(cfg, P, l, st, x, phi, Bn, s):
    d = cfg.head_dim
    g = lambda t: P[f"{l}.{t}"]
    a, r1 = M.rmsnorm_fwd(x, g("g1"), cfg.rms_eps)
    part = np.zeros_like(x)
    mem = []
    for k in range(len(st["ranks"])):
        r0, r1_ = member_rows(cfg, st, f"{l}.wq", k)
        c0, c1 = member_rows(cfg, st, f"{l}.wk", k)  # the member's KV heads (GQA groups)
        nk, nkv = (r1_ - r0) // d, (c1 - c0) // d
        hd = lambda t, n_: t.reshape(Bn, s, n_, d).transpose(0, 2, 1, 3)
        q = M.rope_fwd(hd(a @ g("wq")[r0:r1_].T, nk), phi)
        kk = M.rope_fwd(hd(a @ g("wk")[c0:c1].T, nkv), phi)
        v = hd(a @ g("wv")[c0:c1].T, nkv)
        o4, Pm = M.attention_fwd(q, kk, v)
        o = o4.transpose(0, 2, 1, 3).reshape(Bn, s, nk * d)
        part = part + o @ g("wo")[r0:r1_]
        mem.append((r0, r1_, nk, q, kk, v, o4, Pm, o, c0, c1))
    x1 = x + part
    a2, r2 = M.rmsnorm_fwd(x1, g("g2"), cfg.rms_eps)
    part = np.zeros_like(x)
    mlp = []
    for k in range(len(st["ranks"])):
        f0, f1 = member_rows(cfg, st, f"{l}.wg", k)
        G = a2 @ g("wg")[f0:f1].T
        U = a2 @ g("wu")[f0:f1].T
        u = M.swiglu_fwd(G, U)
        part = part + u @ g("wd")[f0:f1]
        mlp.append((f0, f1, G, U, u))
    return x1 + part, (x, a, r1, mem, x1, a2, r2, mlp)


def _layer_bwd(cfg, P, l, st, saved, dx, phi, Bn, s, acc):
    """acc: dict (member k, name) -> local grad rows; returns dx of the layer input."""
    d, h = cfg.head_dim, cfg.hidden
    g = lambda t: P[f"{l}.{t}"]
    x0, a, r1, mem, x1, a2, r2, mlp = saved
    da2 = np.zeros_like(dx)
    for k, (f0, f1, G, U, u) in enumerate(mlp):
        du = dx @ g("wd")[f0:f1].T
        acc[(k, f"{l}.wd")] += u.reshape(-1, f1 - f0).T @ dx.reshape(-1, h)
        dG, dU = M.swiglu_bwd(G, U, du)
        acc[(k, f"{l}.wg")] += dG.reshape(-1, f1 - f0).T @ a2.reshape(-1, h)
        acc[(k, f"{l}.wu")] += dU.reshape(-1, f1 - f0).T @ a2.reshape(-1, h)
        da2 = da2 + dG @ g("wg")[f0:f1] + dU @ g("wu")[f0:f1]
    dxn, dg2 = M.rmsnorm_bwd(x1, g("g2"), r2, da2)
    for k in range(len(st["ranks"])):
        acc[(k, f"{l}.g2")] += dg2
    dx1 = dx + dxn
    da = np.zeros_like(dx)
    for k, (r0, r1_, nk, q, kk, v, o4, Pm, o, c0, c1) in enumerate(mem):
        hd = lambda t: t.reshape(Bn, s, nk, d).transpose(0, 2, 1, 3)
        uh = lambda t: t.transpose(0, 2, 1, 3).reshape(Bn, s, t.shape[1] * d)
        do = dx1 @ g("wo")[r0:r1_].T
        acc[(k, f"{l}.wo")] += o.reshape(-1, nk * d).T @ dx1.reshape(-1, h)
        dq4, dk4, dv4 = M.attention_bwd(q, kk, v, o4, Pm, hd(do))
        dq, dk, dv = uh(M.rope_bwd(dq4, phi)), uh(M.rope_bwd(dk4, phi)), uh(dv4)
        af = a.reshape(-1, h)
        acc[(k, f"{l}.wq")] += dq.reshape(-1, nk * d).T @ af
        acc[(k, f"{l}.wk")] += dk.reshape(-1, c1 - c0).T @ af
        acc[(k, f"{l}.wv")] += dv.reshape(-1, c1 - c0).T @ af
        da = da + dq @ g("wq")[r0:r1_] + dk @ g("wk")[c0:c1] + dv @ g("wv")[c0:c1]
    dxn, dg1 = M.rmsnorm_bwd(x0, g("g1"), r1, da)
    for k in range(len(st["ranks"])):
        acc[(k, f"{l}.g1")] += dg1
    return dx1 + dxn


def _pipeline_grads(cfg, P, pipe, tokens, targets, b):
    """Member-local gradients of one pipeline (mean over its m_i*b*s tokens) and its loss."""
    s, h = cfg.seq_len, cfg.hidden
    m = pipe["n_micro"]
    n_tok = m * b * s
    phi = M.rope_angles(cfg, s)
    shapes = tensor_shapes(cfg)
    accs = []  # per stage: (k, name) -> array
    for j, st in enumerate(pipe["stages"]):
        acc = {}
        for name in shapes:
            if stage_of(pipe, name, cfg) == j:
                for k in range(len(st["ranks"])):
                    r0, r1 = member_rows(cfg, st, name, k)
                    shp = (r1 - r0,) + shapes[name][1:]
                    acc[(k, name)] = np.zeros(shp)
        accs.append(acc)
    loss = 0.0
    for mb in range(m):
        tok, tgt = tokens[mb * b:(mb + 1) * b], targets[mb * b:(mb + 1) * b]
        x = P["E"][tok]
        saved = []
        for j, st in enumerate(pipe["stages"]):
            for l in range(*st["layers"]):
                x, sv = _layer_fwd(cfg, P, l, st, x, phi, b, s)
                saved.append((j, l, sv))
        last = pipe["stages"][-1]
        xf, rf = M.rmsnorm_fwd(x, P["gf"], cfg.rms_eps)
        # vocab-parallel CE: per-member max / sum-exp / target logit, combined
        zs = []
        for k in range(len(last["ranks"])):
            v0, v1 = member_rows(cfg, last, "Wlm", k)
            zs.append((v0, v1, xf @ P["Wlm"][v0:v1].T))
        gmax = np.max(np.stack([z.max(axis=-1) for _, _, z in zs]), axis=0)
        se = sum(np.exp(z - gmax[..., None]).sum(axis=-1) for _, _, z in zs)
        lse = gmax + np.log(se)
        zt = np.zeros_like(lse)
        for v0, v1, z in zs:
            inr = (tgt >= v0) & (tgt < v1)
            idx = np.clip(tgt - v0, 0, v1 - v0 - 1)
            zt = zt + np.where(inr, np.take_along_axis(z, idx[..., None], -1)[..., 0], 0.0)
        loss += float((lse - zt).sum()) / n_tok
        dxf = np.zeros_like(xf)
        accL = accs[-1]
        for k, (v0, v1, z) in enumerate(zs):
            dz = np.exp(z - lse[..., None])
            inr = (tgt >= v0) & (tgt < v1)
            bi, si = np.nonzero(inr)
            dz[bi, si, tgt[bi, si] - v0] -= 1.0
            dz /= n_tok
            accL[(k, "Wlm")] += dz.reshape(-1, v1 - v0).T @ xf.reshape(-1, h)
            dxf = dxf + dz @ P["Wlm"][v0:v1]
        dx, dgf = M.rmsnorm_bwd(x, P["gf"], rf, dxf)
        for k in range(len(last["ranks"])):
            accL[(k, "gf")] += dgf
        for j, l, sv in reversed(saved):
            dx = _layer_bwd(cfg, P, l, pipe["stages"][j], sv, dx, phi, b, s, accs[j])
        gE = np.zeros_like(P["E"])
        np.add.at(gE, tok.reshape(-1), dx.reshape(-1, h))
        for k in range(len(pipe["stages"][0]["ranks"])):
            accs[0][(k, "E")] += gE
    local = {}
    for j, st in enumerate(pipe["stages"]):
        for (k, name), arr in accs[j].items():
            local[(st["ranks"][k], name)] = arr
    return loss, local


def emulate_step(cfg: ModelCfg, P: dict, Mo: dict, Vo: dict, plan: dict, tokens, targets,
                 step: int, hp=None):
    """Returns (loss, reduced_grads_full, newP, newM, newV, local_grads).  Full logical tensors
    are assembled from owned pieces only, so a wrong owner map shows up as a mismatch."""
    hp = dict(M.ADAM_DEFAULT if hp is None else hp)
    b, B = plan["micro_batch"], plan["global_batch"]
    pipes = plan["pipes"]
    DP = len(pipes)
    w = [p["n_micro"] * b / B for p in pipes]
    local, loss = [], 0.0
    start = 0
    for i, p in enumerate(pipes):
        n = p["n_micro"] * b
        if n > 0:
            li, gi = _pipeline_grads(cfg, P, p, tokens[start:start + n], targets[start:start + n], b)
            loss += w[i] * li
        else:
            gi = None
        local.append(gi)
        start += n
    G, nP, nM, nV = {}, {}, {}, {}
    for name, (full, newp, newm, newv) in _reduce_and_adam(cfg, plan, local, P, Mo, Vo, step, hp).items():
        G[name] = full
        nP[name], nM[name], nV[name] = newp, newm, newv
    return loss, G, nP, nM, nV, local


def weighted_reduce(cfg: ModelCfg, plan: dict, local: list) -> dict:
    """The grad-sync reduction alone (reading R4 / R9): local[i] maps (holder rank,
    name) -> pipeline i's member-local gradient rows (None for m_i = 0).  Returns the full logical
    G[name] = sum_i w_i g_i assembled from owned pieces (each element owned exactly once)."""
    return {n: v[0] for n, v in _reduce_and_adam(cfg, plan, local, None, None, None, 1, None).items()}


def _reduce_and_adam(cfg, plan, local, P, Mo, Vo, step, hp):
    hp = dict(M.ADAM_DEFAULT if hp is None else hp)
    b, B = plan["micro_batch"], plan["global_batch"]
    pipes = plan["pipes"]
    DP = len(pipes)
    w = [p["n_micro"] * b / B for p in pipes]
    shapes = tensor_shapes(cfg)
    out = {}
    for name, shp in shapes.items():
        c = row_width(cfg, name)
        full = np.zeros(int(np.prod(shp)))
        newp, newm, newv = (np.zeros_like(full) for _ in range(3))
        covered = np.zeros(full.shape, dtype=np.int64)
        cuts = sorted(set().union(*[pipeline_cuts(cfg, p, name) for p in pipes]))
        for a, bb in zip(cuts[:-1], cuts[1:]):
            nsig = (bb - a) * c
            for pc in range(DP):
                lo, hi = a * c + (nsig * pc) // DP, a * c + (nsig * (pc + 1)) // DP
                if hi <= lo:
                    continue
                acc = np.zeros(hi - lo)
                for i, p in enumerate(pipes):  # fixed pipeline order (determinism)
                    if local[i] is None:
                        continue
                    hr = sync_holder(cfg, p, name, a)
                    st = p["stages"][stage_of(p, name, cfg)]
                    k = st["ranks"].index(hr)
                    r0 = member_rows(cfg, st, name, k)[0] if split_kind(name) != "rep" else 0
                    loc = local[i][(hr, name)].reshape(-1)
                    acc = acc + w[i] * loc[lo - r0 * c:hi - r0 * c]
                full[lo:hi] = acc
                covered[lo:hi] += 1
                if P is None:
                    continue
                wd = hp["weight_decay"] if M.decays(name) else 0.0
                th = P[name].reshape(-1)[lo:hi]
                mm = Mo[name].reshape(-1)[lo:hi]
                vv = Vo[name].reshape(-1)[lo:hi]
                newp[lo:hi], newm[lo:hi], newv[lo:hi] = M.adamw(
                    th, mm, vv, acc, step, hp["lr"], hp["beta1"], hp["beta2"], hp["eps"], wd)
        assert np.all(covered == 1), f"{name}: every element must be owned exactly once"
        out[name] = tuple(t.reshape(shp) for t in (full, newp, newm, newv))
    return out
