"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no layer math, no sharding rule,
no optimiser): it only draws random numbers and rounds them to bf16, so that both
sides load the same bytes (SURVEY §8(c) "Synthetic inputs, shared bytes with no
shared code").  Recipe:

* weights, seed 1234 (PCG64): every matrix ~ N(0, 0.02^2) drawn in float32;
  W_o^T and W_d^T additionally scaled by 1/sqrt(2L); RMSNorm gains
  1 + 0.1*N(0,1) in parity mode, exactly 1 in perf mode.  Everything is rounded
  to bf16 with round-to-nearest-even.
* tokens, seed 5678 (PCG64): uniform integers in [0, V), shape [B, s+1];
  inputs = [:, :s], targets = [:, 1:]  (the paper names no dataset).

Logical tensor storage (reading R9): every matrix is stored
split-axis-outermost with the hidden dim innermost, i.e. shape [rows, h]:
  Wq         : [n*d, h]     (out, in)
  Wk, Wv     : [n_kv*d, h]  (GQA: n_kv KV heads, each shared by n/n_kv query heads)
  WoT        : [n*d, h]     (= W_o transposed: x += o @ WoT)
  Wg, Wu     : [F, h]
  WdT        : [F, h]       (= W_d transposed: x += u @ WdT)
  E, Wlm     : [V, h]
  g1, g2, gf : [h]
"""
from __future__ import annotations

import dataclasses
import numpy as np

LAYER_TENSORS = ("g1", "wq", "wk", "wv", "wo", "g2", "wg", "wu", "wd")
# tensor id = layer*16 + index in LAYER_TENSORS; globals below (include/malleus.h)
T_EMBED = 0x7FFF0000 + 0
T_FINAL_NORM = 0x7FFF0000 + 1
T_LM_HEAD = 0x7FFF0000 + 2


@dataclasses.dataclass(frozen=True)
class ModelCfg:
    n_layers: int
    hidden: int
    n_heads: int
    head_dim: int
    ffn: int
    vocab: int
    seq_len: int
    rms_eps: float = 1e-5
    rope_theta: float = 10000.0
    n_kv_heads: int = 0  # GQA: 0 = MHA (n_kv = n_heads, reading R1)

    def __post_init__(self):
        assert self.hidden == self.n_heads * self.head_dim, "h = n*d (reading R1)"
        assert self.kv_heads >= 1 and self.n_heads % self.kv_heads == 0, "query heads in whole KV groups"

    @property
    def kv_heads(self) -> int:
        return self.n_kv_heads or self.n_heads


# Named configurations (BASELINE.json configs)
C1_TINY = ModelCfg(n_layers=2, hidden=128, n_heads=4, head_dim=32, ffn=512, vocab=256, seq_len=64)
C2_7B_SLICE = ModelCfg(n_layers=4, hidden=4096, n_heads=32, head_dim=128, ffn=11008, vocab=32000,
                       seq_len=2048)
C3_32B_SLICE = ModelCfg(n_layers=16, hidden=6656, n_heads=52, head_dim=128, ffn=17920, vocab=32000,
                        seq_len=4096)
C4_70B_SLICE = ModelCfg(n_layers=4, hidden=8192, n_heads=64, head_dim=128, ffn=28672, vocab=32000,
                        seq_len=4096)
C5_110B_SLICE = ModelCfg(n_layers=4, hidden=8192, n_heads=64, head_dim=128, ffn=49152, vocab=32000,
                         seq_len=4096)
# C1 with d = 128 and 256-token sequences: exercises the tcgen05 attention and CTA-pair GEMM paths
C1_MED = ModelCfg(n_layers=2, hidden=512, n_heads=4, head_dim=128, ffn=1536, vocab=2048, seq_len=256)
MICRO = ModelCfg(n_layers=2, hidden=16, n_heads=2, head_dim=8, ffn=32, vocab=16, seq_len=8)
# GQA variants (LLaMA-2-70B groups 8 query heads per KV head; here 2 per KV head): the tiny model on the
# mma.sync attention and the d = 128 model on the tcgen05 kernels
C1_GQA = ModelCfg(n_layers=2, hidden=128, n_heads=4, head_dim=32, ffn=512, vocab=256, seq_len=64, n_kv_heads=2)
C1_MED_GQA = ModelCfg(n_layers=2, hidden=512, n_heads=4, head_dim=128, ffn=1536, vocab=2048, seq_len=256,
                      n_kv_heads=2)
MICRO_GQA = ModelCfg(n_layers=2, hidden=32, n_heads=4, head_dim=8, ffn=32, vocab=16, seq_len=8, n_kv_heads=2)


def tensor_shapes(cfg: ModelCfg) -> dict:
    """name -> shape of every logical tensor (storage layout above)."""
    h, nd, F, V = cfg.hidden, cfg.n_heads * cfg.head_dim, cfg.ffn, cfg.vocab
    kd = cfg.kv_heads * cfg.head_dim
    shapes = {"E": (V, h), "gf": (h,), "Wlm": (V, h)}
    for l in range(cfg.n_layers):
        shapes.update({f"{l}.g1": (h,), f"{l}.wq": (nd, h), f"{l}.wk": (kd, h), f"{l}.wv": (kd, h),
                       f"{l}.wo": (nd, h), f"{l}.g2": (h,), f"{l}.wg": (F, h), f"{l}.wu": (F, h),
                       f"{l}.wd": (F, h)})
    return shapes


def tensor_id(name: str) -> int:
    if name == "E":
        return T_EMBED
    if name == "gf":
        return T_FINAL_NORM
    if name == "Wlm":
        return T_LM_HEAD
    l, t = name.split(".")
    return int(l) * 16 + LAYER_TENSORS.index(t)


def bf16_rne(x32: np.ndarray) -> np.ndarray:
    """Round float32 values to bf16 (round-to-nearest-even); returns uint16 bit patterns."""
    u = np.ascontiguousarray(x32, dtype=np.float32).view(np.uint32).astype(np.uint64)
    bias = 0x7FFF + ((u >> 16) & 1)
    return ((u + bias) >> 16).astype(np.uint16)


def bf16_to_f64(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def make_weights(cfg: ModelCfg, seed: int = 1234, parity: bool = True) -> dict:
    """name -> uint16 bf16 bit patterns, shaped per tensor_shapes()."""
    rng = np.random.Generator(np.random.PCG64(seed))
    out = {}
    for name, shape in tensor_shapes(cfg).items():
        short = name.split(".")[-1]
        if len(shape) == 1:
            if parity:
                w = 1.0 + 0.1 * rng.standard_normal(shape, dtype=np.float32)
            else:
                w = np.ones(shape, np.float32)
        else:
            w = 0.02 * rng.standard_normal(shape, dtype=np.float32)
            if short in ("wo", "wd"):
                w = w * np.float32(1.0 / np.sqrt(2.0 * cfg.n_layers))
        out[name] = bf16_rne(w.astype(np.float32))
    return out


def make_tokens(cfg: ModelCfg, batch: int, seed: int = 5678):
    """(inputs [B,s] int32, targets [B,s] int32), uniform over the vocabulary."""
    rng = np.random.Generator(np.random.PCG64(seed))
    t = rng.integers(0, cfg.vocab, size=(batch, cfg.seq_len + 1), dtype=np.int64).astype(np.int32)
    return np.ascontiguousarray(t[:, :-1]), np.ascontiguousarray(t[:, 1:])


def small_int_matrix(shape, vmax: int, seed: int) -> np.ndarray:
    """Integers in [-vmax, vmax] as float32 (exact in bf16 when vmax <= 256): kernel bitwise pins."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.integers(-vmax, vmax + 1, size=shape).astype(np.float32)


def normal_matrix(shape, seed: int, scale: float = 1.0) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    return (scale * rng.standard_normal(shape, dtype=np.float32)).astype(np.float32)
