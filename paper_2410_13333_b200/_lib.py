"""ctypes binding of include/malleus.h (argument marshalling only).

Every step of the hot path runs inside libmalleus.so (hand-written sm_100a kernels + NCCL).
There is no fallback: importing this module raises if the library is missing.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmalleus.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2410_13333_b200.build` "
                      "(there is no CPU fallback)")

# torch must load its bundled NCCL first when present so that both use the same libnccl.so.2
try:  # pragma: no cover - plumbing
    import torch  # noqa: F401
except Exception:  # noqa: BLE001
    pass

lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)

i32, i64, f32, vp = C.c_int32, C.c_int64, C.c_float, C.c_void_p
P_i32, P_i64, P_f32 = C.POINTER(i32), C.POINTER(i64), C.POINTER(f32)

T_EMBED, T_FINAL_NORM, T_LM_HEAD = 0x7FFF0000, 0x7FFF0001, 0x7FFF0002
KIND_PARAM, KIND_GRAD, KIND_MASTER, KIND_ADAM_M, KIND_ADAM_V, KIND_RGRAD = range(6)
STATUS = {0: "OK", 1: "E_ARG", 2: "E_PLAN", 3: "E_CUDA", 4: "E_NCCL", 5: "E_NOMEM", 6: "E_STATE",
          7: "E_TIMEOUT"}


class ModelCfg(C.Structure):
    _fields_ = [("n_layers", i32), ("hidden", i32), ("n_heads", i32), ("n_kv_heads", i32),
                ("head_dim", i32), ("ffn", i32), ("vocab", i32), ("seq_len", i32),
                ("rms_eps", f32), ("rope_theta", f32), ("dtype", i32)]


class Stage(C.Structure):
    _fields_ = [("n_members", i32), ("ranks", P_i32), ("heads", P_i32), ("ffn_cols", P_i32),
                ("vocab_rows", P_i32), ("layer_begin", i32), ("layer_end", i32)]


class Pipeline(C.Structure):
    _fields_ = [("n_stages", i32), ("stages", C.POINTER(Stage)), ("n_micro", i32)]


class Plan(C.Structure):
    _fields_ = [("plan_id", i32), ("dp", i32), ("pipes", C.POINTER(Pipeline)),
                ("micro_batch", i32), ("global_batch", i32), ("n_standby", i32),
                ("standby", P_i32)]


class Arenas(C.Structure):
    _fields_ = [("state", vp), ("state_bytes", C.c_size_t), ("grads", vp), ("grads_bytes", C.c_size_t),
                ("work", vp), ("work_bytes", C.c_size_t)]


class Requirements(C.Structure):
    _fields_ = [("state", C.c_size_t), ("grads", C.c_size_t), ("work", C.c_size_t)]


class AdamCfg(C.Structure):
    _fields_ = [("lr", f32), ("beta1", f32), ("beta2", f32), ("eps", f32), ("weight_decay", f32),
                ("step", i32), ("apply_update", i32), ("max_grad_norm", f32)]


class Piece(C.Structure):
    _fields_ = [("len", i64), ("n_src", i32), ("decay", i32), ("src", vp * 8), ("w", f32 * 8),
                ("master", vp), ("m", vp), ("v", vp), ("rgrad", vp), ("param", vp), ("n_push", i32),
                ("push", vp * 15)]


class Copy(C.Structure):
    _fields_ = [("src", vp), ("dst", vp), ("bytes", i64)]


class MigrateStats(C.Structure):
    _fields_ = [("bytes_sent", C.c_uint64), ("bytes_recv", C.c_uint64), ("seconds", C.c_double),
                ("n_packs", i32), ("total_seconds", C.c_double)]


_SIGS = {
    "malleus_version": ([], C.c_char_p),
    "malleus_last_error": ([vp], C.c_char_p),
    "malleus_nccl_unique_id": ([C.c_char_p], i32),
    "malleus_create": ([C.POINTER(ModelCfg), i32, i32, i32, C.c_char_p, C.POINTER(vp)], i32),
    "malleus_destroy": ([vp], i32),
    "malleus_plan_requirements": ([vp, C.POINTER(Plan), C.POINTER(Requirements)], i32),
    "malleus_plan_apply": ([vp, C.POINTER(Plan), C.POINTER(Arenas)], i32),
    "malleus_write_tensor": ([vp, i32, i32, vp], i32),
    "malleus_read_local": ([vp, i32, i32, vp, P_i64, P_i32, P_i64], i32),
    "malleus_layout_query": ([C.POINTER(ModelCfg), C.POINTER(Plan), i32, i32, i32, i32, P_i64, P_i32], i32),
    "malleus_migration_query": ([C.POINTER(ModelCfg), C.POINTER(Plan), C.POINTER(Plan), i32, i32, i32,
                                 P_i64, P_i32, P_i32], i32),
    "malleus_layer_fwd": ([vp, i32, i32, vp, vp, vp], i32),
    "malleus_layer_bwd": ([vp, i32, i32, vp, vp, vp], i32),
    "malleus_train_step": ([vp, vp, vp, vp, C.POINTER(AdamCfg), vp], i32),
    "malleus_grad_sync": ([vp, C.POINTER(AdamCfg), vp], i32),
    "malleus_migrate": ([vp, C.POINTER(Plan), C.POINTER(Arenas), C.POINTER(MigrateStats)], i32),
    "malleus_probe_speed": ([vp, i32, P_f32], i32),
    "malleus_set_slowdown": ([vp, f32, i32], i32),
    "malleus_last_step_timing": ([vp, P_f32], i32),
    "malleus_last_grad_norm": ([vp, P_f32, P_f32], i32),
    "malleus_kernel_launches": ([], i64),
    "malleus_gemm_profile": ([i32, P_i64, C.POINTER(C.c_double), C.POINTER(C.c_double)], i32),
    "malleus_k_gemm": ([i32, i32, i32, vp, i64, i32, vp, i64, i32, vp, i64, i32, vp], i32),
    "malleus_k_gemm_variant": ([i32], i32),
    "malleus_k_comm_abort": ([i32], i32),
    "malleus_k_rmsnorm_bwd16": ([i32, i32, vp, vp, vp, vp, vp, vp, vp, vp], i32),
    "malleus_k_comm_status": ([i32], i32),
    "malleus_wait": ([vp, vp, i32], i32),
    "malleus_k_gemm_fused": ([i32, i32, i32, vp, i64, vp, i64, vp, i64, vp, i64, i32, vp, vp, vp, vp], i32),
    "malleus_k_attention_variant": ([i32], i32),
    "malleus_k_rmsnorm_fwd": ([i32, i32, vp, vp, vp, vp, f32, vp, vp, vp], i32),
    "malleus_k_rmsnorm_bwd": ([i32, i32, vp, vp, vp, vp, vp, vp, vp, vp], i32),
    "malleus_k_attention_fwd": ([i32, i32, i32, i32, vp, vp, vp, f32, vp], i32),
    "malleus_k_attention_bwd": ([i32, i32, i32, i32, vp, vp, vp, vp, vp, f32, vp], i32),
    "malleus_k_tp_reduce": ([i32, i32, i32, i32, i32, i32, f32, C.c_uint64, vp, vp, vp, vp, vp, vp, vp, vp, vp],
                            i32),
    "malleus_k_reduce_adam": ([i32, vp, C.POINTER(AdamCfg), vp, vp], i32),
    "malleus_k_copy_ranges": ([i32, vp, vp], i32),
    "malleus_k_vocab_ce": ([i32, i32, vp, vp, vp, f32, vp, vp, vp], i32),
    "malleus_zero_grads": ([vp, vp], i32),
}

EXPORTED = tuple(_SIGS)

for _name, (_args, _res) in _SIGS.items():
    _f = getattr(lib, _name)  # AttributeError if the library does not export it
    _f.argtypes = _args
    _f.restype = _res


class MalleusError(RuntimeError):
    pass


class CommTimeout(MalleusError):
    """MALLEUS_E_TIMEOUT: a communication call exceeded the failure threshold."""


def check(status: int, ctx=None, what: str = ""):
    if status != 0:
        msg = lib.malleus_last_error(ctx).decode() if ctx is not None else ""
        cls = CommTimeout if status == 7 else MalleusError
        raise cls(f"{what}: {STATUS.get(status, status)}: {msg}")


DTYPES = {"bf16": 0, "fp32": 1}


def make_cfg(cfg, dtype: str = "bf16") -> ModelCfg:
    return ModelCfg(cfg.n_layers, cfg.hidden, cfg.n_heads, getattr(cfg, "kv_heads", cfg.n_heads), cfg.head_dim, cfg.ffn,
                    cfg.vocab, cfg.seq_len, cfg.rms_eps, cfg.rope_theta, DTYPES[dtype])


class PlanStruct:
    """Owns the ctypes arrays behind a malleus_plan built from a plan dict (plans.py format)."""

    def __init__(self, plan: dict):
        self._keep = []
        arr = lambda xs: self._hold((i32 * max(1, len(xs)))(*xs))
        pipes = []
        for p in plan["pipes"]:
            stages = []
            for st in p["stages"]:
                stages.append(Stage(len(st["ranks"]), arr(st["ranks"]), arr(st["heads"]), arr(st["ffn"]),
                                    arr(st["vocab"]), st["layers"][0], st["layers"][1]))
            sarr = self._hold((Stage * len(stages))(*stages))
            pipes.append(Pipeline(len(stages), sarr, p["n_micro"]))
        parr = self._hold((Pipeline * len(pipes))(*pipes))
        sb = plan.get("standby", [])
        self.c = Plan(plan.get("plan_id", 0), len(pipes), parr, plan["micro_batch"], plan["global_batch"],
                      len(sb), arr(sb))

    def _hold(self, x):
        self._keep.append(x)
        return x

    @property
    def ref(self):
        return C.byref(self.c)
