"""Oracle: the plain, single-device, unpartitioned training step in NumPy float64.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module.  The product path
(paper_2410_13333_b200) never imports, links or executes anything under oracle/.

What it computes (readings R1-R6):
  Malleus is lossless: "does not adjust the global batch size and the
  synchronization protocol across pipelines" (§2.3), data parallel
  means every replica gets the same update from synchronised gradients
  (§2.1).  So every valid malleable plan must reproduce exactly this
  step: a LLaMA-2-architecture decoder (§7.1 "Workloads") forward,
  mean cross-entropy over all B*s target tokens, textbook backward, AdamW.

  x = E[tok]
  per layer:  a = rmsnorm(x; g1); q,k,v = a Wq^T, a Wk^T, a Wv^T; rope(q,k)
              o = softmax(q k^T / sqrt(d) + causal) v;  x += o @ WoT
              a2 = rmsnorm(x; g2); x += (silu(a2 Wg^T) * (a2 Wu^T)) @ WdT
  xf = rmsnorm(x; gf); z = xf Wlm^T; loss = mean(logsumexp(z) - z[target])

Backward equations are the ones written in SURVEY §8(c) ("Backward equations"),
implemented literally; AdamW follows torch.optim.AdamW semantics (reading R5).
"""
from __future__ import annotations

import numpy as np

from synth.gen import ModelCfg, bf16_to_f64


def params_f64(weights_bf16: dict) -> dict:
    """bf16 bit patterns -> float64 values (exact)."""
    return {k: bf16_to_f64(v) for k, v in weights_bf16.items()}


# ----------------------------------------------------------------------------- pieces
def rmsnorm_fwd(x, g, eps):
    """y = g * x * r,  r = (mean(x^2) + eps)^-1/2 (per row).  Returns y, r."""
    r = 1.0 / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps)
    return x * r * g, r


def rmsnorm_bwd(x, g, r, dy):
    """u = g*dy;  dx = r*u - x*r^3*mean(x*u);  dg = sum_rows dy*x*r."""
    u = g * dy
    dx = r * u - x * (r ** 3) * np.mean(x * u, axis=-1, keepdims=True)
    dg = np.sum((dy * x * r).reshape(-1, x.shape[-1]), axis=0)
    return dx, dg


def rope_angles(cfg: ModelCfg, s: int):
    """phi[p, i] = p * theta^(-2i/d), i < d/2 (reading R2/R3: theta=1e4, half-split)."""
    d = cfg.head_dim
    i = np.arange(d // 2, dtype=np.float64)
    inv = cfg.rope_theta ** (-2.0 * i / d)
    return np.arange(s, dtype=np.float64)[:, None] * inv[None, :]


def rope_fwd(q, phi):
    """q [..., s, d] rotated per half-split pairs (i, i+d/2)."""
    d2 = q.shape[-1] // 2
    c, s_ = np.cos(phi), np.sin(phi)
    q1, q2 = q[..., :d2], q[..., d2:]
    return np.concatenate([q1 * c - q2 * s_, q2 * c + q1 * s_], axis=-1)


def rope_bwd(dq, phi):
    """Backward of a rotation is the rotation by -phi."""
    return rope_fwd(dq, -phi)


def _expand_kv(t, n):
    """GQA: [B, n_kv, s, d] -> [B, n, s, d], query head j reads KV head j // (n / n_kv) (LLaMA-2-70B
    grouping: each KV head serves a block of consecutive query heads).  n_kv == n: unchanged."""
    return np.repeat(t, n // t.shape[1], axis=1)


def _reduce_kv(t, n_kv):
    """Backward of _expand_kv: sum the gradients of each KV head's group of query heads."""
    B, n, s, d = t.shape
    return t.reshape(B, n_kv, n // n_kv, s, d).sum(axis=2)


def attention_fwd(q, k, v):
    """q [B, n, s, d]; k, v [B, n_kv, s, d] (n_kv = n: MHA).  S = q k^T/sqrt(d) + causal;
    P = softmax(S); o = P v."""
    k, v = _expand_kv(k, q.shape[1]), _expand_kv(v, q.shape[1])
    d = q.shape[-1]
    s = q.shape[-2]
    S = (q @ np.swapaxes(k, -1, -2)) / np.sqrt(d)          # [B, n, s, s]
    mask = np.triu(np.ones((s, s), dtype=bool), k=1)
    S = np.where(mask, -np.inf, S)
    S = S - S.max(axis=-1, keepdims=True)
    P = np.exp(S)
    P = P / P.sum(axis=-1, keepdims=True)
    o = P @ v
    return o, P


def attention_bwd(q, k, v, o, P, do):
    """dV = P^T dO; dP = dO V^T; dS = P*(dP - rowsum(dO*O)); dQ = dS K/sqrt(d); dK = dS^T Q/sqrt(d).
    GQA: K / V expanded to the query heads as in the forward, dK / dV summed over each group."""
    n_kv = k.shape[1]
    k, v = _expand_kv(k, q.shape[1]), _expand_kv(v, q.shape[1])
    d = q.shape[-1]
    dv = np.swapaxes(P, -1, -2) @ do
    dP = do @ np.swapaxes(v, -1, -2)
    D = np.sum(do * o, axis=-1, keepdims=True)
    dS = P * (dP - D)
    dq = (dS @ k) / np.sqrt(d)
    dk = (np.swapaxes(dS, -1, -2) @ q) / np.sqrt(d)
    return dq, _reduce_kv(dk, n_kv), _reduce_kv(dv, n_kv)


def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def swiglu_fwd(G, U):
    return G * sigmoid(G) * U


def swiglu_bwd(G, U, du):
    """dU = du*silu(G);  dG = du*U*sig(G)*(1 + G*(1-sig(G)))."""
    sg = sigmoid(G)
    return du * U * sg * (1.0 + G * (1.0 - sg)), du * G * sg


def cross_entropy(z, y):
    """Per-token CE and dz/dlogit-per-token (softmax - onehot); caller scales by 1/N_tok."""
    zmax = z.max(axis=-1, keepdims=True)
    ez = np.exp(z - zmax)
    se = ez.sum(axis=-1, keepdims=True)
    lse = zmax[..., 0] + np.log(se[..., 0])
    zt = np.take_along_axis(z, y[..., None], axis=-1)[..., 0]
    p = ez / se
    onehot = np.zeros_like(z)
    np.put_along_axis(onehot, y[..., None], 1.0, axis=-1)
    return lse - zt, p - onehot


# ----------------------------------------------------------------------------- one layer
def _heads(t, n, d):  # [Bn, s, n*d] -> [Bn, n, s, d]
    Bn, s = t.shape[0], t.shape[1]
    return t.reshape(Bn, s, n, d).transpose(0, 2, 1, 3)


def _unheads(t):  # [Bn, n, s, d] -> [Bn, s, n*d]
    Bn, n, s, d = t.shape
    return t.transpose(0, 2, 1, 3).reshape(Bn, s, n * d)


def layer_fwd(cfg: ModelCfg, p, x0, phi):
    """One decoder layer (SURVEY §8(c) algorithm): p(name) -> that layer's tensor; x0 [Bn, s, h].
    Returns (x_out, saved activations for layer_bwd)."""
    n, d, eps = cfg.n_heads, cfg.head_dim, cfg.rms_eps
    nkv = getattr(cfg, "kv_heads", n)
    a, r1 = rmsnorm_fwd(x0, p("g1"), eps)
    q = rope_fwd(_heads(a @ p("wq").T, n, d), phi)
    k = rope_fwd(_heads(a @ p("wk").T, nkv, d), phi)
    v = _heads(a @ p("wv").T, nkv, d)
    o4, Pm = attention_fwd(q, k, v)
    o = _unheads(o4)
    x1 = x0 + o @ p("wo")
    a2, r2 = rmsnorm_fwd(x1, p("g2"), eps)
    G = a2 @ p("wg").T
    U = a2 @ p("wu").T
    u = swiglu_fwd(G, U)
    return x1 + u @ p("wd"), (x0, a, r1, q, k, v, o4, Pm, o, x1, a2, r2, G, U, u)


def layer_bwd(cfg: ModelCfg, p, saved, dx, phi):
    """Backward of layer_fwd: dx = gradient of the layer output.  Returns (gradient of the layer
    input, {tensor: weight gradient}) with the SURVEY §8(c) backward equations."""
    n, d, h = cfg.n_heads, cfg.head_dim, cfg.hidden
    x0, a, r1, q, k, v, o4, Pm, o, x1, a2, r2, G, U, u = saved
    g = {}
    # MLP
    du = dx @ p("wd").T
    g["wd"] = u.reshape(-1, cfg.ffn).T @ dx.reshape(-1, h)
    dG, dU = swiglu_bwd(G, U, du)
    g["wg"] = dG.reshape(-1, cfg.ffn).T @ a2.reshape(-1, h)
    g["wu"] = dU.reshape(-1, cfg.ffn).T @ a2.reshape(-1, h)
    da2 = dG @ p("wg") + dU @ p("wu")
    dxn, g["g2"] = rmsnorm_bwd(x1, p("g2"), r2, da2)
    dx1 = dx + dxn
    # attention
    do = dx1 @ p("wo").T
    g["wo"] = o.reshape(-1, n * d).T @ dx1.reshape(-1, h)
    dq4, dk4, dv4 = attention_bwd(q, k, v, o4, Pm, _heads(do, n, d))
    dq = _unheads(rope_bwd(dq4, phi))
    dk = _unheads(rope_bwd(dk4, phi))
    dv = _unheads(dv4)
    a_f = a.reshape(-1, h)
    kd = getattr(cfg, "kv_heads", n) * d
    g["wq"] = dq.reshape(-1, n * d).T @ a_f
    g["wk"] = dk.reshape(-1, kd).T @ a_f
    g["wv"] = dv.reshape(-1, kd).T @ a_f
    da = dq @ p("wq") + dk @ p("wk") + dv @ p("wv")
    dxn, g["g1"] = rmsnorm_bwd(x0, p("g1"), r1, da)
    return dx1 + dxn, g


# ----------------------------------------------------------------------------- step
def forward_backward(cfg: ModelCfg, P: dict, tokens: np.ndarray, targets: np.ndarray,
                     n_norm: int | None = None):
    """Loss (mean CE over the given tokens unless n_norm overrides the divisor) and grads.

    tokens/targets: int [Bn, s].  Returns (loss, grads: name -> float64 array)."""
    Bn, s = tokens.shape
    h, n, d = cfg.hidden, cfg.n_heads, cfg.head_dim
    eps = cfg.rms_eps
    N = Bn * s if n_norm is None else n_norm
    phi = rope_angles(cfg, s)

    x = P["E"][tokens]                                      # [Bn, s, h]
    saved = []
    for l in range(cfg.n_layers):
        x, sv = layer_fwd(cfg, lambda t, l=l: P[f"{l}.{t}"], x, phi)
        saved.append(sv)

    xf, rf = rmsnorm_fwd(x, P["gf"], eps)
    z = xf @ P["Wlm"].T                                      # [Bn, s, V]
    ce, dz1 = cross_entropy(z, targets)
    loss = ce.sum() / N
    dz = dz1 / N

    g = {}
    g["Wlm"] = dz.reshape(-1, cfg.vocab).T @ xf.reshape(-1, h)
    dxf = dz @ P["Wlm"]
    dx, g["gf"] = rmsnorm_bwd(x, P["gf"], rf, dxf)
    for l in reversed(range(cfg.n_layers)):
        dx, gl = layer_bwd(cfg, lambda t, l=l: P[f"{l}.{t}"], saved[l], dx, phi)
        g.update({f"{l}.{t}": v for t, v in gl.items()})
    gE = np.zeros_like(P["E"])
    np.add.at(gE, tokens.reshape(-1), dx.reshape(-1, h))
    g["E"] = gE
    return loss, g


def loss_only(cfg: ModelCfg, P: dict, tokens, targets) -> float:
    return forward_backward(cfg, P, tokens, targets)[0]


# ----------------------------------------------------------------------------- AdamW
ADAM_DEFAULT = dict(lr=3e-4, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1)


def decays(name: str) -> bool:
    """Reading R5: weight decay on 2-D tensors only (not on norm gains)."""
    return not (name.endswith("g1") or name.endswith("g2") or name == "gf")


def adamw(theta, m, v, g, step: int, lr, beta1, beta2, eps, weight_decay):
    """torch.optim.AdamW semantics (reading R5), one tensor, float64.  Returns new (theta, m, v)."""
    theta = theta * (1.0 - lr * weight_decay)
    m = beta1 * m + (1.0 - beta1) * g
    v = beta2 * v + (1.0 - beta2) * g * g
    mhat = m / (1.0 - beta1 ** step)
    vhat = v / (1.0 - beta2 ** step)
    theta = theta - lr * mhat / (np.sqrt(vhat) + eps)
    return theta, m, v


def clip_grad_norm(g: dict, max_norm: float):
    """Global-norm gradient clipping, torch.nn.utils.clip_grad_norm_ semantics:
    total = sqrt(sum over all tensors of sum g^2); coef = max_norm / (total + 1e-6); every gradient
    is scaled by coef when coef < 1.  float64.  Returns (clipped grads, total)."""
    total = float(np.sqrt(sum(float(np.sum(np.asarray(v, np.float64) ** 2)) for v in g.values())))
    coef = max_norm / (total + 1e-6)
    if coef < 1.0:
        return {k: np.asarray(v, np.float64) * coef for k, v in g.items()}, total
    return {k: np.asarray(v, np.float64) for k, v in g.items()}, total


def train_step(cfg: ModelCfg, P: dict, M: dict, Vs: dict, tokens, targets, step: int, hp=None):
    """Full step: fwd, bwd, AdamW on all tensors.  Returns (loss, grads, newP, newM, newV)."""
    hp = dict(ADAM_DEFAULT if hp is None else hp)
    loss, g = forward_backward(cfg, P, tokens, targets)
    gu = g
    if hp.get("max_grad_norm", 0.0) > 0.0:  # optional global-norm clipping before AdamW
        gu, _ = clip_grad_norm(g, hp["max_grad_norm"])
    nP, nM, nV = {}, {}, {}
    for k in P:
        wd = hp["weight_decay"] if decays(k) else 0.0
        nP[k], nM[k], nV[k] = adamw(P[k], M[k], Vs[k], gu[k], step, hp["lr"], hp["beta1"],
                                    hp["beta2"], hp["eps"], wd)
    return loss, g, nP, nM, nV
