"""The per-layer boundary calls: malleus_layer_fwd / malleus_layer_bwd /
malleus_zero_grads / malleus_grad_sync on one GPU (plan P0), layer by layer against the oracle's
layer_fwd / layer_bwd (oracle/model.py, SURVEY §8(c) equations) fed with the GPU's own bf16 layer
input, and grad_sync's reduce + AdamW + bf16 cast against oracle.model.adamw (reading R16).
Tolerances (reading R15): ||gpu - ref||_inf / ||ref||_inf <= tol per tensor on the bf16 path;
AdamW fp32 vs fp64 <= 1e-6; bf16 param == RNE(master) bit for bit; P0 has w = 1, so the reduced
gradient equals the accumulated gradient bit for bit."""
import numpy as np
import pytest
import torch

from synth.gen import C1_TINY, C1_MED, C2_7B_SLICE, make_weights, make_tokens, tensor_shapes, bf16_rne, normal_matrix
from oracle import model as M
from paper_2410_13333_b200 import plans as Pl

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def _f64(t):
    return t.float().cpu().numpy().astype(np.float64)


@pytest.fixture(scope="module")
def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
@pytest.mark.parametrize("cfg", [C1_TINY, C1_MED], ids=["c1", "c1m"])
def test_layer_fwd_bwd_grad_sync_p0(need_gpu, cfg, dtype):
    from paper_2410_13333_b200 import _lib as L
    from paper_2410_13333_b200.engine import Engine
    b, B = 2, 8
    plan = Pl.plan_matrix_c1(cfg, B=B, b=b)["P0"]
    tol = 2e-2 if dtype == "bf16" else 1e-4  # reading R15; fp32 parity mode (north star)
    act = torch.bfloat16 if dtype == "bf16" else torch.float32
    eng = Engine(cfg, 0, 1, 0, dtype=dtype)
    eng.apply(plan)
    W = make_weights(cfg)
    eng.write_weights(W)
    P = M.params_f64(W)
    tok, _ = make_tokens(cfg, b)
    s, h = cfg.seq_len, cfg.hidden
    phi = M.rope_angles(cfg, s)
    st = torch.cuda.current_stream().cuda_stream
    x = torch.tensor(W["E"][tok.reshape(-1)].view(np.int16)).cuda().view(torch.bfloat16).to(act)  # E[tok], exact
    saved = []
    for l in range(cfg.n_layers):
        y = torch.empty_like(x)
        assert L.lib.malleus_layer_fwd(eng.ctx, l, 0, x.data_ptr(), y.data_ptr(), st) == 0
        torch.cuda.synchronize()
        xin = _f64(x).reshape(b, s, h)
        ref, sv = M.layer_fwd(cfg, lambda t, l=l: P[f"{l}.{t}"], xin, phi)
        assert _rel(_f64(y).reshape(b, s, h), ref) <= tol, l
        saved.append(sv)
        x = y
    # backward from a random output gradient, weight grads accumulated from zero
    assert L.lib.malleus_zero_grads(eng.ctx, st) == 0
    dy = torch.tensor(normal_matrix((b * s, h), 77, 1e-2)).to(act).cuda()
    for l in reversed(range(cfg.n_layers)):
        dx = torch.empty_like(dy)
        assert L.lib.malleus_layer_bwd(eng.ctx, l, 0, dy.data_ptr(), dx.data_ptr(), st) == 0
        torch.cuda.synchronize()
        ref_dx, ref_g = M.layer_bwd(cfg, lambda t, l=l: P[f"{l}.{t}"], saved[l], _f64(dy).reshape(b, s, h), phi)
        assert _rel(_f64(dx).reshape(b, s, h), ref_dx) <= tol, l
        for t, gref in ref_g.items():
            (rng,), vals = eng.read(f"{l}.{t}", L.KIND_GRAD)
            assert rng == (0, gref.size)
            assert _rel(vals.astype(np.float64).reshape(gref.shape), gref) <= tol, (l, t)
        dy = dx
    # accumulation: a second layer_bwd of the top layer with the same dy doubles its weight grads
    top = cfg.n_layers - 1
    before = eng.read(f"{top}.wd", L.KIND_GRAD)[1].copy()
    dy2 = torch.tensor(normal_matrix((b * s, h), 78, 1e-2)).to(act).cuda()
    dx2 = torch.empty_like(dy2)
    assert L.lib.malleus_layer_bwd(eng.ctx, top, 0, dy2.data_ptr(), dx2.data_ptr(), st) == 0
    torch.cuda.synchronize()
    _, g2 = M.layer_bwd(cfg, lambda t: P[f"{top}.{t}"], saved[top], _f64(dy2).reshape(b, s, h), phi)
    after = eng.read(f"{top}.wd", L.KIND_GRAD)[1].astype(np.float64)
    assert _rel(after - before, g2["wd"].reshape(-1)) <= tol
    # grad_sync: reduce (w = 1) + AdamW + bf16 push on the accumulated gradients
    a = eng.adam(1, True)
    assert L.lib.malleus_grad_sync(eng.ctx, a, st) == 0
    torch.cuda.synchronize()
    hp = M.ADAM_DEFAULT
    for name in tensor_shapes(cfg):
        _, g = eng.read(name, L.KIND_GRAD)
        _, rg = eng.read(name, L.KIND_RGRAD)
        assert np.array_equal(rg, g), name
        _, master = eng.read(name, L.KIND_MASTER)
        wd = hp["weight_decay"] if M.decays(name) else 0.0
        th, _, _ = M.adamw(P[name].reshape(-1), 0.0, 0.0, g.astype(np.float64), 1, hp["lr"], hp["beta1"],
                           hp["beta2"], hp["eps"], wd)
        assert _rel(master.astype(np.float64), th) <= 1e-6, name
        _, par = eng.read(name, L.KIND_PARAM)
        assert np.array_equal(par, bf16_rne(master) if dtype == "bf16" else master), name
    # argument checks: a layer this rank does not hold / a bad slot
    assert L.lib.malleus_layer_fwd(eng.ctx, cfg.n_layers, 0, x.data_ptr(), x.data_ptr(), st) == 1
    assert L.lib.malleus_layer_bwd(eng.ctx, 0, 5, x.data_ptr(), x.data_ptr(), st) == 1
    eng.close()


def test_plan_rejected_at_kernel_limits(need_gpu):
    """a plan the kernels cannot run (C2 with b = 8: b*s = 16384 tokens > the embedding
    backward's 8192) is rejected by plan_requirements / plan_apply with E_PLAN, before any step."""
    from paper_2410_13333_b200._lib import MalleusError
    from paper_2410_13333_b200.engine import Engine
    cfg = C2_7B_SLICE
    eng = Engine(cfg, 0, 1, 0)
    with pytest.raises(MalleusError, match="E_PLAN.*8192"):
        eng.requirements(Pl.single_gpu(cfg, 16, b=8))
    s, g, w = eng.requirements(Pl.single_gpu(cfg, 16, b=4))
    assert s > 0 and g > 0 and w > 0
    eng.close()
