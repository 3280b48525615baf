"""Single-GPU parity of the multi-GPU rows: the kernels that run the
cross-layout batch-weighted reduce + AdamW + param push (S15-S17, K14/K9), the migration copies
(S20, K11) and the vocab-parallel cross entropy (S11), driven through the C-ABI with every "rank's"
buffers on ONE device and the piece / transfer tables taken from the library's own layout
arithmetic (malleus_layout_query / malleus_migration_query), compared against the oracle.

* K14: small-integer gradients and dyadic weights w_i = m_i b / B (e.g. m = (1, 3), b = 2, B = 8 ->
  1/4, 3/4) make every fp32 partial sum exact, so the reduced gradient is compared BIT FOR BIT
  with the oracle's reduction (oracle.emulator.weighted_reduce, readings R4/R9;
  SURVEY §8(c) "Reshard-reduce kernel" pin); AdamW on the owned pieces vs oracle.model.adamw
  (fp32 vs fp64, <= 1e-6 relative, reading R16); every holder's bf16 copy == RNE(master) bit for bit.
* Migration: per-rank compact state buffers laid out like the runtime's (held rows, owned pieces
  concatenated in canonical order); the keep-copies plus the transfers of migration_query, moved by
  malleus_k_copy_ranges, must leave every rank's new buffers byte-identical to the logical state
  under the new plan (readings R10/R11), with the byte count equal to the
  oracle's delta bytes.
* Vocab-parallel CE: k member slices with v0 != 0 against oracle.model.cross_entropy (R15).
"""
import ctypes as C

import numpy as np
import pytest
import torch

from synth.gen import C1_TINY, ModelCfg, make_weights, tensor_shapes, tensor_id, small_int_matrix, bf16_rne
from oracle import model as M
from oracle import layout as Lo
from oracle.emulator import weighted_reduce
from paper_2410_13333_b200 import plans as Pl

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2410_13333_b200 import _lib
    return _lib


def _ranges(L, cfg, plan, world, rank, name, kind):
    """Flat element ranges of (name, kind) that `rank` holds / owns, in the library's canonical order."""
    ccfg = L.make_cfg(cfg)
    ps = L.PlanStruct(plan)
    n = C.c_int32(0)
    assert L.lib.malleus_layout_query(C.byref(ccfg), ps.ref, world, rank, tensor_id(name), kind, None, C.byref(n)) == 0
    buf = (C.c_int64 * max(1, 2 * n.value))()
    cap = C.c_int32(n.value)
    assert L.lib.malleus_layout_query(C.byref(ccfg), ps.ref, world, rank, tensor_id(name), kind, buf, C.byref(cap)) == 0
    return [(buf[2 * i], buf[2 * i + 1]) for i in range(n.value)]


def _stream():
    return torch.cuda.current_stream().cuda_stream


# ----------------------------------------------------------------------------------------- K14
def _local_from_logical(cfg, plan, g_pipe):
    """oracle input: local[i][(holder rank, name)] = pipeline i's gradient rows held by that member."""
    local = []
    for i, pp in enumerate(plan["pipes"]):
        if g_pipe[i] is None:
            local.append(None)
            continue
        d = {}
        for name in tensor_shapes(cfg):
            st = pp["stages"][Lo.stage_of(pp, name, cfg)]
            for k, r in enumerate(st["ranks"]):
                if Lo.split_kind(name) == "rep":
                    d[(r, name)] = g_pipe[i][name]
                else:
                    r0, r1 = Lo.member_rows(cfg, st, name, k)
                    d[(r, name)] = g_pipe[i][name][r0:r1]
        local.append(d)
    return local


def _run_reduce_adam(L, cfg, plan, world, seed, clip=0.0, misalign=False):
    shapes = tensor_shapes(cfg)
    names = list(shapes)
    b, B = plan["micro_batch"], plan["global_batch"]
    w = [pp["n_micro"] * b / B for pp in plan["pipes"]]
    # small integers |g| <= 45: every fp32 sum of <= 8 terms with dyadic weights is exact
    g_pipe = [None if pp["n_micro"] == 0 else
              {n: small_int_matrix(shapes[n], 45, seed + 97 * i + j).astype(np.float64)
               for j, n in enumerate(names)} for i, pp in enumerate(plan["pipes"])]
    G_ref = weighted_reduce(cfg, plan, _local_from_logical(cfg, plan, g_pipe))
    W = make_weights(cfg)
    P = M.params_f64(W)
    pad = 1 if misalign else 0  # misaligned sources force the kernel's scalar path
    dev_g = [None if g is None else {n: torch.tensor(np.concatenate([np.zeros(pad), g[n].reshape(-1)]),
                                                     dtype=torch.float32, device="cuda") for n in names}
             for g in g_pipe]
    # every rank: a full-size bf16 param buffer per tensor (zero outside its held rows)
    params = {(r, n): torch.zeros(int(np.prod(shapes[n])), dtype=torch.int16, device="cuda")
              for r in range(world) for n in names}
    held = {(r, n): _ranges(L, cfg, plan, world, r, n, Lo.KIND_PARAM) for r in range(world) for n in names}
    states, pieces = {}, []
    for r in range(world):
        for n in names:
            own = _ranges(L, cfg, plan, world, r, n, Lo.KIND_MASTER)
            tot = sum(e1 - e0 for e0, e1 in own)
            if tot == 0:
                continue
            master = torch.tensor(np.concatenate([P[n].reshape(-1)[e0:e1] for e0, e1 in own]), dtype=torch.float32,
                                  device="cuda")
            st = dict(own=own, master=master, m=torch.zeros_like(master), v=torch.zeros_like(master),
                      rgrad=torch.full_like(master, float("nan")))
            states[(r, n)] = st
            off = 0
            for e0, e1 in own:
                pc = L.Piece()
                pc.len = e1 - e0
                srcs = [(i, dg) for i, dg in enumerate(dev_g) if dg is not None]
                pc.n_src = len(srcs)
                for q, (i, dg) in enumerate(srcs):
                    pc.src[q] = dg[n].data_ptr() + 4 * (e0 + pad)
                    pc.w[q] = w[i]
                pc.decay = 1 if M.decays(n) else 0
                for key in ("master", "m", "v", "rgrad"):
                    setattr(pc, key, st[key].data_ptr() + 4 * off)
                pc.param = params[(r, n)].data_ptr() + 2 * e0
                others = [q for q in range(world) if q != r and any(a <= e0 < z for a, z in held[(q, n)])]
                pc.n_push = len(others)
                for q, hr in enumerate(others):
                    pc.push[q] = params[(hr, n)].data_ptr() + 2 * e0
                pieces.append(pc)
                off += e1 - e0
    arr = (L.Piece * len(pieces))(*pieces)
    hp = dict(M.ADAM_DEFAULT)
    adam = L.AdamCfg(hp["lr"], hp["beta1"], hp["beta2"], hp["eps"], hp["weight_decay"], 1, 1, clip)
    nc = torch.zeros(2, device="cuda")
    assert L.lib.malleus_k_reduce_adam(len(pieces), C.cast(arr, C.c_void_p), C.byref(adam), nc.data_ptr(),
                                       _stream()) == 0
    torch.cuda.synchronize()
    return G_ref, P, states, params, held, nc.cpu().numpy(), hp


@pytest.mark.parametrize("pname", ["P3", "P4", "P5", "P7", "P8"])
def test_reduce_adam_cross_layout_bitwise(L, pname):
    """P3 DP2 m = (3, 1); P4 cross-layout {TP2 3:1, TP2 even} m = (1, 3); P5 different TP degrees;
    P7 PP + TP4 + standby (8 'ranks' on one device); P8 a pipeline with m_i = 0 (w = 0)."""
    cfg = C1_TINY
    plan = Pl.plan_matrix_c1(cfg)[pname]
    world = Pl.world_of(plan)
    G_ref, P, states, params, held, _, hp = _run_reduce_adam(L, cfg, plan, world, seed=31)
    seen = {n: np.zeros(int(np.prod(v.shape)), np.int64) for n, v in G_ref.items()}
    master_full = {n: np.zeros(int(np.prod(v.shape))) for n, v in G_ref.items()}
    for (r, n), st in states.items():
        rg = st["rgrad"].cpu().numpy()
        ms = st["master"].cpu().numpy().astype(np.float64)
        mm = st["m"].cpu().numpy().astype(np.float64)
        vv = st["v"].cpu().numpy().astype(np.float64)
        off = 0
        for e0, e1 in st["own"]:
            ref = G_ref[n].reshape(-1)[e0:e1]
            got = rg[off:off + e1 - e0]
            assert np.array_equal(got.astype(np.float64), ref), (pname, r, n, e0)  # exact: bitwise
            wd = hp["weight_decay"] if M.decays(n) else 0.0
            th, m1, v1 = M.adamw(P[n].reshape(-1)[e0:e1], 0.0, 0.0, ref, 1, hp["lr"], hp["beta1"], hp["beta2"],
                                 hp["eps"], wd)
            for got_x, want in ((ms, th), (mm, m1), (vv, v1)):
                g_ = got_x[off:off + e1 - e0]
                assert np.abs(g_ - want).max() <= 1e-6 * max(np.abs(want).max(), 1e-30), (pname, r, n)
            master_full[n][e0:e1] = ms[off:off + e1 - e0]
            seen[n][e0:e1] += 1
            off += e1 - e0
    for n in seen:
        assert np.all(seen[n] == 1), (pname, n, "every element owned exactly once")
    # param push (S17): every holder's bf16 copy == RNE(fp32 master), nothing written elsewhere
    for (r, n), buf in params.items():
        got = buf.cpu().numpy().view(np.uint16)
        want = bf16_rne(master_full[n].astype(np.float32))
        mask = np.zeros(got.shape, bool)
        for e0, e1 in held[(r, n)]:
            mask[e0:e1] = True
        assert np.array_equal(got[mask], want[mask]), (pname, r, n)
        assert not got[~mask].any(), (pname, r, n, "stray write")


def test_reduce_adam_scalar_path_and_clipping(L):
    """Misaligned sources (scalar path) give the same bits; global-norm clipping
    (torch clip_grad_norm_ semantics) on the same pieces: norm and coefficient vs the oracle."""
    cfg = C1_TINY
    plan = Pl.plan_matrix_c1(cfg)["P4"]
    G_ref, P, states, _, _, nc, hp = _run_reduce_adam(L, cfg, plan, 4, seed=5, clip=100.0, misalign=True)
    gc, total = M.clip_grad_norm(G_ref, 100.0)
    coef = min(1.0, 100.0 / (total + 1e-6))
    assert coef < 1.0
    assert abs(nc[1] - total) <= 1e-6 * total and abs(nc[0] - coef) <= 1e-6 * coef, (nc, total, coef)
    for (r, n), st in states.items():
        rg = st["rgrad"].cpu().numpy()
        ms = st["master"].cpu().numpy().astype(np.float64)
        off = 0
        for e0, e1 in st["own"]:
            assert np.array_equal(rg[off:off + e1 - e0].astype(np.float64), G_ref[n].reshape(-1)[e0:e1])
            wd = hp["weight_decay"] if M.decays(n) else 0.0
            th, _, _ = M.adamw(P[n].reshape(-1)[e0:e1], 0.0, 0.0, gc[n].reshape(-1)[e0:e1], 1, hp["lr"],
                               hp["beta1"], hp["beta2"], hp["eps"], wd)
            assert np.abs(ms[off:off + e1 - e0] - th).max() <= 2e-6 * max(np.abs(th).max(), 1e-30), (r, n)
            off += e1 - e0


# ------------------------------------------------------------------------------------ migration
def _transfers(L, cfg, a, b, world, dst, kind):
    ccfg = L.make_cfg(cfg)
    pa, pb = L.PlanStruct(a), L.PlanStruct(b)
    n = C.c_int32(0)
    assert L.lib.malleus_migration_query(C.byref(ccfg), pa.ref, pb.ref, world, dst, kind, None, None, C.byref(n)) == 0
    tbe = (C.c_int64 * max(1, 3 * n.value))()
    src = (C.c_int32 * max(1, n.value))()
    cap = C.c_int32(n.value)
    assert L.lib.malleus_migration_query(C.byref(ccfg), pa.ref, pb.ref, world, dst, kind, tbe, src, C.byref(cap)) == 0
    return [(tbe[3 * i], tbe[3 * i + 1], tbe[3 * i + 2], src[i]) for i in range(cap.value)]


KINDS = (Lo.KIND_PARAM, Lo.KIND_MASTER, Lo.KIND_ADAM_M, Lo.KIND_ADAM_V)


def _compact(L, cfg, plan, world, logical):
    """rank -> (name, kind) -> (ranges, device buffer of those elements concatenated): the runtime's
    storage order (held rows; owned pieces in canonical order)."""
    out = {}
    for r in range(world):
        for n in tensor_shapes(cfg):
            for kind in KINDS:
                rk = Lo.KIND_PARAM if kind == Lo.KIND_PARAM else Lo.KIND_MASTER
                rs = _ranges(L, cfg, plan, world, r, n, rk)
                data = logical[(n, kind)]
                vals = np.concatenate([data[e0:e1] for e0, e1 in rs]) if rs else data[:0]
                out[(r, n, kind)] = (rs, torch.tensor(vals.view(np.int16 if kind == Lo.KIND_PARAM else np.int32),
                                                      device="cuda"))
    return out


def _addr(entry, e, es):
    rs, buf = entry
    off = 0
    for e0, e1 in rs:
        if e0 <= e < e1:
            return buf.data_ptr() + es * (off + e - e0)
        off += e1 - e0
    raise AssertionError(f"element {e} not resident")


def _migrate_one_device(L, cfg, a, b, world, seed):
    rng = np.random.default_rng(seed)
    shapes = tensor_shapes(cfg)
    logical = {}
    for n, shp in shapes.items():
        ne = int(np.prod(shp))
        logical[(n, Lo.KIND_PARAM)] = rng.integers(0, 1 << 16, ne, dtype=np.uint64).astype(np.uint16)
        for kind in KINDS[1:]:
            logical[(n, kind)] = rng.integers(0, 1 << 32, ne, dtype=np.uint64).astype(np.uint32)
    old = _compact(L, cfg, a, world, logical)
    new = {k: (rs, torch.zeros_like(buf)) for k, (rs, buf) in _compact(L, cfg, b, world, logical).items()}
    copies, moved = [], 0
    for r in range(world):
        for n in shapes:
            for kind in KINDS:
                es = 2 if kind == Lo.KIND_PARAM else 4
                ors, nrs = old[(r, n, kind)][0], new[(r, n, kind)][0]
                for (o0, o1) in ors:  # keep-copies: what r needs and already has
                    for (n0, n1) in nrs:
                        lo, hi = max(o0, n0), min(o1, n1)
                        if hi > lo:
                            copies.append(L.Copy(_addr(old[(r, n, kind)], lo, es), _addr(new[(r, n, kind)], lo, es),
                                                 (hi - lo) * es))
        for kind in KINDS:
            es = 2 if kind == Lo.KIND_PARAM else 4
            for tid, e0, e1, src in _transfers(L, cfg, a, b, world, r, kind):
                n = next(x for x in shapes if tensor_id(x) == tid)
                assert src != r
                copies.append(L.Copy(_addr(old[(src, n, kind)], e0, es), _addr(new[(r, n, kind)], e0, es),
                                     (e1 - e0) * es))
                moved += (e1 - e0) * es
    arr = (L.Copy * max(1, len(copies)))(*copies)
    assert L.lib.malleus_k_copy_ranges(len(copies), C.cast(arr, C.c_void_p), _stream()) == 0
    torch.cuda.synchronize()
    for (r, n, kind), (rs, buf) in new.items():
        got = buf.cpu().numpy()
        want = np.concatenate([logical[(n, kind)][e0:e1] for e0, e1 in rs]) if rs else logical[(n, kind)][:0]
        assert np.array_equal(got.view(want.dtype), want), (r, n, kind)
    return moved


# the C1 plan matrix's shapes on a model small enough for the oracle's per-element delta loop
LAYOUT_TINY = ModelCfg(n_layers=2, hidden=32, n_heads=4, head_dim=8, ffn=128, vocab=128, seq_len=8)


@pytest.mark.parametrize("pair", [("P2", "P1"), ("P1", "P2"), ("P3", "P10"), ("P4", "P9"), ("P9", "P4")])
def test_migration_copies_one_device_tiny(L, pair):
    """Byte-identical new state and moved bytes == the oracle's per-element delta bytes."""
    cfg = LAYOUT_TINY
    pm = Pl.plan_matrix_c1(cfg)
    a, b = pm[pair[0]], pm[pair[1]]
    world = Pl.world_of(a)
    assert Pl.world_of(b) == world
    moved = _migrate_one_device(L, cfg, a, b, world, seed=3)
    assert moved == Lo.delta_bytes(Lo.migration_deltas(cfg, a, b))


def test_migration_copies_one_device_random_c1(L):
    """C1 (16-byte vector path), random plan pairs with the same world (the dynamic re-plan case),
    including an A -> B -> A-shaped pair: the state is rebuilt exactly every time."""
    from tests.planutil import random_plan
    rng = np.random.default_rng(17)
    done = 0
    while done < 6:
        a, wa = random_plan(rng, C1_TINY, world_max=6)
        b, wb = random_plan(rng, C1_TINY, world_max=6)
        if wa != wb:
            continue
        _migrate_one_device(L, C1_TINY, a, b, wa, seed=done)
        _migrate_one_device(L, C1_TINY, b, a, wa, seed=100 + done)
        done += 1


# --------------------------------------------------------------------------- vocab-parallel CE
@pytest.mark.parametrize("splits", [[256], [192, 64], [64, 64, 64, 64], [96, 80, 80], [16, 224, 16]])
def test_vocab_parallel_ce_one_device(L, splits):
    V, T = sum(splits), 128
    rng = np.random.default_rng(len(splits))
    z = (3 * rng.standard_normal((T, V))).astype(np.float32)
    tgt = rng.integers(0, V, T).astype(np.int32)
    scale = 1.0 / (4 * T)
    zs, dzs, v0 = [], [], 0
    for Vj in splits:
        zs.append(torch.tensor(z[:, v0:v0 + Vj].copy(), device="cuda"))
        dzs.append(torch.empty(T, Vj, dtype=torch.bfloat16, device="cuda"))
        v0 += Vj
    loss = torch.empty(T, device="cuda")
    dt = torch.tensor(tgt, device="cuda")
    Va = (C.c_int32 * len(splits))(*splits)
    zp = (C.c_void_p * len(splits))(*[t.data_ptr() for t in zs])
    dp = (C.c_void_p * len(splits))(*[t.data_ptr() for t in dzs])
    assert L.lib.malleus_k_vocab_ce(len(splits), T, C.cast(Va, C.c_void_p), C.cast(zp, C.c_void_p), dt.data_ptr(),
                                    scale, C.cast(dp, C.c_void_p), loss.data_ptr(), _stream()) == 0
    torch.cuda.synchronize()
    ce, dz1 = M.cross_entropy(z.astype(np.float64), tgt.astype(np.int64))
    assert np.abs(loss.cpu().numpy() - ce).max() <= 1e-5 * np.abs(ce).max()
    got = torch.cat([d.float() for d in dzs], dim=1).cpu().numpy().astype(np.float64)
    ref = dz1 * scale
    # one bf16 rounding of an fp32 value (2^-8 relative) plus fp32 softmax error
    assert (np.abs(got - ref) <= np.abs(ref) * 2.0 ** -8 + 1e-6 * scale).all()
