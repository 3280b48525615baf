"""Pins for oracle/model.py against things other than itself (SURVEY §8(c) "What pins each part").

* finite differences (fp64, central) on a micro model;
* an independent library implementation: torch CPU fp64 autograd with F.rms_norm-equivalent,
  F.scaled_dot_product_attention(is_causal=True), F.silu, F.cross_entropy;
* closed-form special cases;
* torch.optim.AdamW on CPU fp64.
"""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from synth.gen import MICRO, MICRO_GQA, C1_TINY, C1_GQA, ModelCfg, make_weights, make_tokens
from oracle import model as M


def _setup(cfg, B=2, seed=1234):
    P = M.params_f64(make_weights(cfg, seed=seed))
    tok, tgt = make_tokens(cfg, B)
    return P, tok, tgt


@pytest.mark.parametrize("cfg", [MICRO, MICRO_GQA], ids=["mha", "gqa"])
def test_finite_differences_micro(cfg):
    P, tok, tgt = _setup(cfg)
    # larger weights so that every term matters at fp64 FD resolution
    rng = np.random.default_rng(0)
    P = {k: v + (0.3 * rng.standard_normal(v.shape) if v.ndim == 2 else 0.0) for k, v in P.items()}
    loss, g = M.forward_backward(cfg, P, tok, tgt)
    eps = 1e-6
    for name, arr in P.items():
        flat = arr.reshape(-1)
        idx = rng.choice(flat.size, size=min(6, flat.size), replace=False)
        for i in idx:
            Pp = dict(P)
            Pm = dict(P)
            a = flat.copy(); a[i] += eps; Pp[name] = a.reshape(arr.shape)
            b = flat.copy(); b[i] -= eps; Pm[name] = b.reshape(arr.shape)
            fd = (M.loss_only(cfg, Pp, tok, tgt) - M.loss_only(cfg, Pm, tok, tgt)) / (2 * eps)
            an = g[name].reshape(-1)[i]
            scale = max(np.abs(g[name]).max(), 1e-12)
            assert abs(fd - an) <= 1e-6 * scale + 1e-10, (name, i, fd, an)


def _torch_loss(cfg: ModelCfg, P: dict, tok, tgt):
    """Independent implementation with torch library routines (fp64)."""
    T = {k: torch.tensor(v, dtype=torch.float64, requires_grad=True) for k, v in P.items()}
    Bn, s = tok.shape
    n, d, h = cfg.n_heads, cfg.head_dim, cfg.hidden
    nkv = cfg.kv_heads
    tok_t = torch.tensor(tok, dtype=torch.long)
    x = T["E"][tok_t]
    pos = torch.arange(s, dtype=torch.float64)
    inv = cfg.rope_theta ** (-torch.arange(0, d, 2, dtype=torch.float64) / d)
    ang = pos[:, None] * inv[None, :]
    cos, sin = torch.cos(ang), torch.sin(ang)

    def rms(x, g):
        return F.rms_norm(x, (h,), weight=g, eps=cfg.rms_eps)

    def rope(t):  # [B, n, s, d], rotate_half convention
        t1, t2 = t[..., : d // 2], t[..., d // 2:]
        return torch.cat([t1 * cos - t2 * sin, t2 * cos + t1 * sin], dim=-1)

    for l in range(cfg.n_layers):
        p = lambda t: T[f"{l}.{t}"]
        a = rms(x, p("g1"))
        q = (a @ p("wq").T).view(Bn, s, n, d).transpose(1, 2)
        k = (a @ p("wk").T).view(Bn, s, nkv, d).transpose(1, 2)
        v = (a @ p("wv").T).view(Bn, s, nkv, d).transpose(1, 2)
        o = F.scaled_dot_product_attention(rope(q), rope(k), v, is_causal=True, enable_gqa=nkv != n)
        x = x + o.transpose(1, 2).reshape(Bn, s, n * d) @ p("wo")
        a2 = rms(x, p("g2"))
        x = x + (F.silu(a2 @ p("wg").T) * (a2 @ p("wu").T)) @ p("wd")
    z = rms(x, T["gf"]) @ T["Wlm"].T
    loss = F.cross_entropy(z.reshape(-1, cfg.vocab), torch.tensor(tgt, dtype=torch.long).reshape(-1))
    loss.backward()
    return loss.item(), {k: t.grad.numpy() for k, t in T.items()}


@pytest.mark.parametrize("cfg", [MICRO, C1_TINY, MICRO_GQA, C1_GQA])
def test_torch_autograd_fp64(cfg):
    P, tok, tgt = _setup(cfg, B=2)
    loss, g = M.forward_backward(cfg, P, tok, tgt)
    tl, tg = _torch_loss(cfg, P, tok, tgt)
    assert abs(loss - tl) <= 1e-12 * abs(tl)
    for k in P:
        err = np.abs(g[k] - tg[k]).max() / max(np.abs(tg[k]).max(), 1e-300)
        assert err <= 1e-10, (k, err)


def test_special_case_zero_lm_head():
    """(i) W_lm = 0 => loss = ln V exactly and dz = (1/V - onehot)/(B s) => dW_lm closed form."""
    cfg = C1_TINY
    P, tok, tgt = _setup(cfg)
    P["Wlm"] = np.zeros_like(P["Wlm"])
    loss, g = M.forward_backward(cfg, P, tok, tgt)
    assert abs(loss - math.log(cfg.vocab)) < 1e-12
    # z = 0 -> every non-LM-head grad is zero (dxf = dz @ Wlm = 0)
    assert np.abs(g["0.wq"]).max() == 0.0 and np.abs(g["E"]).max() == 0.0
    # dWlm = dz^T xf with dz = (1/V - onehot)/N: its rows are exact closed forms of xf, and the
    # sum over vocab rows vanishes because sum_v dz_v = 0 for every token.
    colsum = g["Wlm"].sum(axis=0)  # sum over vocab rows of dz^T xf = (sum_v dz_v) xf = 0
    assert np.abs(colsum).max() < 1e-12


def test_special_case_identity_blocks():
    """(ii) W_o = W_d = 0 => every block is the identity: z = RMSNorm(E[tok]) W_lm^T."""
    cfg = C1_TINY
    P, tok, tgt = _setup(cfg)
    for l in range(cfg.n_layers):
        P[f"{l}.wo"] = np.zeros_like(P[f"{l}.wo"])
        P[f"{l}.wd"] = np.zeros_like(P[f"{l}.wd"])
    loss, _ = M.forward_backward(cfg, P, tok, tgt)
    x = P["E"][tok]
    r = 1.0 / np.sqrt((x * x).mean(-1, keepdims=True) + cfg.rms_eps)
    z = (x * r * P["gf"]) @ P["Wlm"].T
    zt = np.take_along_axis(z, tgt[..., None], -1)[..., 0]
    ref = np.mean(np.log(np.exp(z).sum(-1)) - zt)
    assert abs(loss - ref) < 1e-12


def test_special_case_attention_position0_and_rope_identity():
    """(iii) position 0 attends only to itself => o_0 = v_0; (iv) RoPE at pos 0 = identity and
    rotations preserve pair norms."""
    rng = np.random.default_rng(1)
    q, k, v = (rng.standard_normal((2, 3, 7, 8)) for _ in range(3))
    o, _ = M.attention_fwd(q, k, v)
    assert np.abs(o[:, :, 0] - v[:, :, 0]).max() == 0.0
    phi = M.rope_angles(C1_TINY, 7)
    qr = M.rope_fwd(rng.standard_normal((7, 32)), phi)
    q0 = rng.standard_normal((7, 32))
    qr = M.rope_fwd(q0, phi)
    assert np.abs(qr[0] - q0[0]).max() == 0.0
    n0 = q0[:, :16] ** 2 + q0[:, 16:] ** 2
    n1 = qr[:, :16] ** 2 + qr[:, 16:] ** 2
    assert np.abs(n0 - n1).max() < 1e-12
    assert np.abs(M.rope_bwd(qr, phi) - q0).max() < 1e-12


def test_special_case_rmsnorm_constant_row():
    """(v) RMSNorm(c * 1) = sign(c) * g  (up to eps)."""
    g = np.linspace(0.5, 1.5, 16)
    for c in (3.0, -2.0):
        y, _ = M.rmsnorm_fwd(np.full((1, 16), c), g, 0.0)
        assert np.abs(y[0] - np.sign(c) * g).max() < 1e-14


def test_init_loss_near_ln_v():
    """(vi) at init the loss is close to ln V (sanity of the generator recipe)."""
    cfg = C1_TINY
    P, tok, tgt = _setup(cfg, B=4)
    loss, _ = M.forward_backward(cfg, P, tok, tgt)
    assert abs(loss - math.log(cfg.vocab)) < 0.05


def test_adamw_vs_torch():
    rng = np.random.default_rng(3)
    theta = rng.standard_normal(50)
    hp = M.ADAM_DEFAULT
    p = torch.tensor(theta.copy(), dtype=torch.float64, requires_grad=True)
    opt = torch.optim.AdamW([p], lr=hp["lr"], betas=(hp["beta1"], hp["beta2"]), eps=hp["eps"],
                            weight_decay=hp["weight_decay"])
    m = np.zeros(50)
    v = np.zeros(50)
    th = theta.copy()
    for step in range(1, 6):
        g = rng.standard_normal(50)
        p.grad = torch.tensor(g, dtype=torch.float64)
        opt.step()
        th, m, v = M.adamw(th, m, v, g, step, hp["lr"], hp["beta1"], hp["beta2"], hp["eps"],
                           hp["weight_decay"])
    assert np.abs(th - p.detach().numpy()).max() <= 1e-15 * 10


@pytest.mark.parametrize("max_norm", [0.05, 1.0, 1e6])
def test_clip_grad_norm_vs_torch(max_norm):
    """Pin of oracle.model.clip_grad_norm: torch.nn.utils.clip_grad_norm_ (an independent
    implementation) in float64 on random multi-tensor gradients, active (0.05, 1.0) and inactive
    (1e6) clipping; the clipped global norm equals max_norm when clipping is active."""
    rng = np.random.default_rng(3)
    g = {f"t{i}": rng.normal(size=shp) * s for i, (shp, s) in enumerate([((7, 5), 0.3), ((11,), 2.0), ((3, 4, 2), 0.05)])}
    ts = [torch.tensor(v, dtype=torch.float64, requires_grad=True) for v in g.values()]
    for t, v in zip(ts, g.values()):
        t.grad = torch.tensor(v, dtype=torch.float64)
    tot_ref = float(torch.nn.utils.clip_grad_norm_(ts, max_norm))
    out, tot = M.clip_grad_norm(g, max_norm)
    assert abs(tot - tot_ref) <= 1e-12 * tot_ref
    for t, k in zip(ts, g):
        np.testing.assert_allclose(out[k], t.grad.numpy(), rtol=1e-13, atol=0)
    new_norm = math.sqrt(sum(float(np.sum(v ** 2)) for v in out.values()))
    if max_norm < tot_ref:
        assert abs(new_norm - max_norm) <= 1e-5 * max_norm
    else:
        assert abs(new_norm - tot_ref) <= 1e-12 * tot_ref


def test_gqa_equals_mha_with_repeated_kv_weights():
    """GQA with n_kv KV heads is exactly MHA whose W_k / W_v repeat each KV head's rows for the g
    query heads of its group (query head j <- KV head j // g); the GQA weight gradient of a KV head
    is the sum of the MHA gradients of its g copies."""
    import dataclasses
    cfg = C1_GQA
    mha = dataclasses.replace(cfg, n_kv_heads=0)
    P, tok, tgt = _setup(cfg, B=2)
    g_sz, d = cfg.n_heads // cfg.kv_heads, cfg.head_dim
    Q = dict(P)
    for l in range(cfg.n_layers):
        for t in ("wk", "wv"):
            w = P[f"{l}.{t}"].reshape(cfg.kv_heads, d, -1)
            Q[f"{l}.{t}"] = np.repeat(w, g_sz, axis=0).reshape(cfg.n_heads * d, -1)
    la, ga = M.forward_backward(cfg, P, tok, tgt)
    lb, gb = M.forward_backward(mha, Q, tok, tgt)
    assert abs(la - lb) <= 1e-13 * abs(lb)
    for k in P:
        if k.endswith((".wk", ".wv")):
            red = gb[k].reshape(cfg.kv_heads, g_sz, d, -1).sum(axis=1).reshape(ga[k].shape)
            assert np.abs(ga[k] - red).max() <= 1e-12 * max(np.abs(red).max(), 1e-300), k
        else:
            assert np.abs(ga[k] - gb[k]).max() <= 1e-12 * max(np.abs(gb[k]).max(), 1e-300), k
