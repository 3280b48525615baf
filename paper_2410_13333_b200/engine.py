"""Python front end of libmalleus.so: argument marshalling only.

PyTorch provides device memory (the arenas), streams and the process group used to broadcast
the NCCL unique id; every step of the hot path runs inside the library.
"""
from __future__ import annotations

import ctypes as C
import glob
import json
import os

import numpy as np
import torch

from . import _lib as L
from ._lib import check

_ADAM_DEFAULT = dict(lr=3e-4, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1)


def name_to_id(name: str) -> int:
    if name == "E":
        return L.T_EMBED
    if name == "gf":
        return L.T_FINAL_NORM
    if name == "Wlm":
        return L.T_LM_HEAD
    layer, t = name.split(".")
    return int(layer) * 16 + ("g1", "wq", "wk", "wv", "wo", "g2", "wg", "wu", "wd").index(t)


def _numel(cfg, name: str) -> int:
    h, nd, F, V = cfg.hidden, cfg.n_heads * cfg.head_dim, cfg.ffn, cfg.vocab
    kd = getattr(cfg, "kv_heads", cfg.n_heads) * cfg.head_dim
    if name in ("E", "Wlm"):
        return V * h
    if name == "gf":
        return h
    t = name.split(".")[1]
    return {"g1": h, "g2": h, "wq": nd * h, "wk": kd * h, "wv": kd * h, "wo": nd * h,
            "wg": F * h, "wu": F * h, "wd": F * h}[t]


def tensor_names(cfg):
    names = []
    for l in range(cfg.n_layers):
        names += [f"{l}.{t}" for t in ("g1", "wq", "wk", "wv", "wo", "g2", "wg", "wu", "wd")]
    return names + ["E", "gf", "Wlm"]


class Engine:
    """One malleus context (one process == one GPU)."""

    def __init__(self, cfg, rank: int = 0, world: int = 1, device: int | None = None, group=None,
                 dtype: str = "bf16"):
        self.cfg = cfg
        self.dtype = dtype  # "bf16", or "fp32" (parity mode: fp32 params / activations, SIMT kernels)
        self.rank, self.world = rank, world
        self.device = torch.cuda.current_device() if device is None else device
        torch.cuda.set_device(self.device)
        uid = C.create_string_buffer(128)
        if rank == 0:
            check(L.lib.malleus_nccl_unique_id(uid), None, "nccl_unique_id")
        if world > 1:
            import torch.distributed as dist
            obj = [bytes(uid.raw) if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0, group=group)
            uid = C.create_string_buffer(obj[0], 128)
        self._ccfg = L.make_cfg(cfg, dtype)
        ctx = C.c_void_p()
        check(L.lib.malleus_create(C.byref(self._ccfg), rank, world, self.device, uid, C.byref(ctx)), None, "create")
        self.ctx = ctx
        self.plan = None
        self._arenas = None
        self._plan_struct = None

    # ------------------------------------------------------------------ plans
    def requirements(self, plan: dict):
        ps = L.PlanStruct(plan)
        req = L.Requirements()
        check(L.lib.malleus_plan_requirements(self.ctx, ps.ref, C.byref(req)), self.ctx, "plan_requirements")
        return req.state, req.grads, req.work

    def _alloc(self, plan):
        s, g, w = self.requirements(plan)
        bufs = [torch.empty(n, dtype=torch.uint8, device=f"cuda:{self.device}") for n in (s, g, w)]
        ar = L.Arenas(bufs[0].data_ptr(), s, bufs[1].data_ptr(), g, bufs[2].data_ptr(), w)
        return bufs, ar

    def apply(self, plan: dict):
        bufs, ar = self._alloc(plan)
        ps = L.PlanStruct(plan)
        check(L.lib.malleus_plan_apply(self.ctx, ps.ref, C.byref(ar)), self.ctx, "plan_apply")
        self.plan, self._arenas, self._plan_struct = plan, bufs, ps

    def migrate(self, plan: dict) -> dict:
        bufs, ar = self._alloc(plan)
        ps = L.PlanStruct(plan)
        st = L.MigrateStats()
        check(L.lib.malleus_migrate(self.ctx, ps.ref, C.byref(ar), C.byref(st)), self.ctx, "migrate")
        self.plan, self._arenas, self._plan_struct = plan, bufs, ps
        return dict(bytes_sent=st.bytes_sent, bytes_recv=st.bytes_recv, seconds=st.seconds, n_packs=st.n_packs,
                    total_seconds=st.total_seconds)

    # ------------------------------------------------------------------ state I/O
    def write_weights(self, weights_bf16: dict):
        """bf16 bit patterns per tensor (synth.gen); in fp32 mode their exact fp32 values are written."""
        for name, arr in weights_bf16.items():
            a = np.ascontiguousarray(arr, dtype=np.uint16)
            if self.dtype == "fp32":
                a = np.ascontiguousarray((a.astype(np.uint32) << 16).view(np.float32))
            check(L.lib.malleus_write_tensor(self.ctx, name_to_id(name), L.KIND_PARAM, a.ctypes.data), self.ctx,
                  f"write_tensor {name}")

    def write_state(self, name: str, kind: int, values: np.ndarray):
        a = np.ascontiguousarray(values, dtype=np.float32)
        check(L.lib.malleus_write_tensor(self.ctx, name_to_id(name), kind, a.ctypes.data), self.ctx, "write_tensor")

    def read(self, name: str, kind: int):
        """(list of (e0, e1) flat ranges, values concatenated as np array)."""
        nr, ne = C.c_int32(0), C.c_int64(0)
        tid = name_to_id(name)
        check(L.lib.malleus_read_local(self.ctx, tid, kind, None, None, C.byref(nr), C.byref(ne)), self.ctx, "read")
        ranges = (C.c_int64 * max(1, 2 * nr.value))()
        dtype = np.uint16 if kind == L.KIND_PARAM and self.dtype == "bf16" else np.float32
        out = np.empty(max(ne.value, 1), dtype=dtype)
        check(L.lib.malleus_read_local(self.ctx, tid, kind, out.ctypes.data, ranges, C.byref(nr), C.byref(ne)),
              self.ctx, "read")
        return [(ranges[2 * i], ranges[2 * i + 1]) for i in range(nr.value)], out[:ne.value]

    # ------------------------------------------------------------------ checkpoint
    _KINDS = (("param", L.KIND_PARAM), ("master", L.KIND_MASTER), ("m", L.KIND_ADAM_M), ("v", L.KIND_ADAM_V))

    def save_checkpoint(self, path: str, step: int):
        """Collective over the caller's ranks (each writes its own file): every rank stores its OWNED
        pieces (ZeRO-1, reading R9) of fp32 master / m / v and the bf16 (fp32 in parity mode) params
        of the same element ranges, so the files partition the model state exactly once and can be
        loaded onto any other plan or world size (the surviving GPUs).
        Format: <path>/rank<r>.npz with '<tensor>|<kind>|ranges' (int64 [n, 2] flat element ranges)
        and '<tensor>|<kind>|vals'; <path>/meta.json (step, world, dtype, model shape) from rank 0."""
        os.makedirs(path, exist_ok=True)
        torch.cuda.synchronize(self.device)
        arrs = {}
        for name in tensor_names(self.cfg):
            owned, master = self.read(name, L.KIND_MASTER)
            if not owned:
                continue
            held, param = self.read(name, L.KIND_PARAM)
            pv = []
            for e0, e1 in owned:  # params of the owned ranges (owned pieces lie inside held rows)
                off = 0
                for h0, h1 in held:
                    if h0 <= e0 and e1 <= h1:
                        pv.append(param[off + e0 - h0: off + e1 - h0])
                        break
                    off += h1 - h0
                else:
                    raise RuntimeError(f"owned range {e0, e1} of {name} not held")
            rg = np.asarray(owned, dtype=np.int64).reshape(-1, 2)
            arrs[f"{name}|param|vals"] = np.concatenate(pv)
            arrs[f"{name}|master|vals"] = master
            for tag, kind in self._KINDS[2:]:
                _, vals = self.read(name, kind)
                arrs[f"{name}|{tag}|vals"] = vals
            arrs[f"{name}|ranges"] = rg
        np.savez(os.path.join(path, f"rank{self.rank}.npz"), **arrs)
        if self.rank == 0:
            c = self.cfg
            meta = {"step": int(step), "world": self.world, "dtype": self.dtype,
                    "model": [c.n_layers, c.hidden, c.n_heads, c.head_dim, c.ffn, c.vocab, c.seq_len]}
            with open(os.path.join(path, "meta.json"), "w") as f:
                json.dump(meta, f)

    def load_checkpoint(self, path: str) -> int:
        """Load a checkpoint written by save_checkpoint (on any plan / world) into this rank's current
        plan: the logical tensors are assembled from every rank file (each element exactly once) and
        written with write_tensor, PARAM first (it resets master / m / v), then MASTER, ADAM_M, ADAM_V.
        Returns the step stored in meta.json."""
        meta = json.load(open(os.path.join(path, "meta.json")))
        c = self.cfg
        if meta["model"] != [c.n_layers, c.hidden, c.n_heads, c.head_dim, c.ffn, c.vocab, c.seq_len] or \
                meta["dtype"] != self.dtype:
            raise ValueError("checkpoint model shape / dtype does not match this engine")
        files = [np.load(f) for f in sorted(glob.glob(os.path.join(path, "rank*.npz")))]
        for name in tensor_names(c):
            n = _numel(c, name)
            full = {tag: np.zeros(n, dtype=np.float32) for tag, _ in self._KINDS}
            pbits = self.dtype == "bf16"
            full["param"] = np.zeros(n, dtype=np.uint16 if pbits else np.float32)
            seen = np.zeros(n, dtype=np.int32)
            for f in files:
                key = f"{name}|ranges"
                if key not in f:
                    continue
                off = 0
                vals = {tag: f[f"{name}|{tag}|vals"] for tag, _ in self._KINDS}
                for e0, e1 in f[key]:
                    for tag in vals:
                        full[tag][e0:e1] = vals[tag][off: off + e1 - e0]
                    seen[e0:e1] += 1
                    off += e1 - e0
            if not np.all(seen == 1):
                raise ValueError(f"checkpoint does not cover {name} exactly once")
            for tag, kind in self._KINDS:
                a = np.ascontiguousarray(full[tag])
                check(L.lib.malleus_write_tensor(self.ctx, name_to_id(name), kind, a.ctypes.data), self.ctx,
                      f"write_tensor {name} {tag}")
        return int(meta["step"])

    def wait(self, timeout_ms: int, stream=None):
        """Failure detector: raises _lib.CommTimeout when the enqueued work does not
        finish within timeout_ms; the context is then failed (destroy it, resume from a checkpoint)."""
        st = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        check(L.lib.malleus_wait(self.ctx, st, int(timeout_ms)), self.ctx, "wait")

    # ------------------------------------------------------------------ step
    def adam(self, step: int, apply_update: bool = True, **kw):
        hp = dict(_ADAM_DEFAULT, **kw)
        return L.AdamCfg(hp["lr"], hp["beta1"], hp["beta2"], hp["eps"], hp["weight_decay"], step, int(apply_update),
                         float(hp.get("max_grad_norm", 0.0)))

    def grad_norm(self):
        """(global gradient norm, clipping coefficient) of the last clipped step."""
        n, c = C.c_float(0), C.c_float(1)
        check(L.lib.malleus_last_grad_norm(self.ctx, C.byref(n), C.byref(c)), self.ctx, "grad_norm")
        return n.value, c.value

    def train_step(self, tokens: torch.Tensor, targets: torch.Tensor, step: int, apply_update: bool = True,
                   loss_out: torch.Tensor | None = None, stream=None, **adam_kw) -> torch.Tensor:
        """tokens/targets: device int32 [B, s] (whole global batch).  Returns the device loss."""
        assert tokens.dtype == torch.int32 and tokens.is_cuda and tokens.is_contiguous()
        if loss_out is None:
            loss_out = torch.zeros(1, dtype=torch.float32, device=tokens.device)
        st = (stream or torch.cuda.current_stream()).cuda_stream
        a = self.adam(step, apply_update, **adam_kw)
        check(L.lib.malleus_train_step(self.ctx, tokens.data_ptr(), targets.data_ptr(), loss_out.data_ptr(),
                                       C.byref(a), st), self.ctx, "train_step")
        return loss_out

    def timing(self):
        out = (C.c_float * 5)()
        check(L.lib.malleus_last_step_timing(self.ctx, out), self.ctx, "timing")
        return dict(compute=out[0], tp_comm=out[1], pp_comm=out[2], grad_sync=out[3], total=out[4])

    def probe(self, iters: int = 10):
        out = (C.c_float * self.world)()
        check(L.lib.malleus_probe_speed(self.ctx, iters, out), self.ctx, "probe")
        return list(out)

    def set_slowdown(self, x: float, mode: int = 1):
        check(L.lib.malleus_set_slowdown(self.ctx, float(x), int(mode)), self.ctx, "set_slowdown")

    def calibrate_slowdown(self, slow_rank: int, x_target: float, mode: int = 2, iters: int = 10, tol: float = 0.05,
                           max_rounds: int = 8):
        """Collective.  Reading R13: inject on `slow_rank` until the probe measures
        x = t_slow / t_ref within `tol` of x_target; t_ref = median probe of the other ranks (or the
        rank's own uninjected probe on one GPU).  Returns (nominal x used, measured x)."""
        if self.rank == slow_rank:
            self.set_slowdown(1.0, 0)
        base = self.probe(iters)
        t_ref_self = base[slow_rank]
        lo, hi, nominal = 1.0, max(2.0, 4.0 * x_target), x_target
        measured = 1.0
        for _ in range(max_rounds):
            if self.rank == slow_rank:
                self.set_slowdown(nominal, mode)
            t = self.probe(iters)
            others = [v for i, v in enumerate(t) if i != slow_rank]
            t_ref = sorted(others)[len(others) // 2] if others else t_ref_self
            measured = t[slow_rank] / t_ref
            if abs(measured / x_target - 1.0) <= tol:
                break
            if measured < x_target:
                lo = nominal
            else:
                hi = nominal
            nominal = 0.5 * (lo + hi)
        return nominal, measured

    def close(self):
        if self.ctx:
            L.lib.malleus_destroy(self.ctx)
            self.ctx = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def gather_logical(engines_reads, shape, dtype=np.float32):
    """Assemble a logical tensor from (ranges, values) pieces of several ranks."""
    full = np.zeros(int(np.prod(shape)), dtype=dtype)
    seen = np.zeros(full.shape, dtype=bool)
    for ranges, vals in engines_reads:
        off = 0
        for e0, e1 in ranges:
            full[e0:e1] = vals[off:off + e1 - e0]
            seen[e0:e1] = True
            off += e1 - e0
    return full.reshape(shape), seen.reshape(shape)
