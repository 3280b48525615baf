"""Fused-epilogue GEMMs vs the plain GEMM of the same shape (C2 TP1 shapes, CUDA events, 20 reps):
gate/up + SwiGLU (glu 1), down-projection dgrad + SwiGLU backward (glu 2), O-proj / down + residual.
The unfused path adds the standalone SwiGLU / residual kernels (times from the ncu launch list).
  python tools/gemm_fused_bench.py"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_13333_b200 import _lib as L

st = torch.cuda.current_stream().cuda_stream


def bench(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters * 1e3


T, h, F = 2048, 4096, 11008
bf = torch.bfloat16
fused = (ctypes.c_int32 * 1)()


def plain(M, N, K, A, B, C):
    return lambda: L.lib.malleus_k_gemm(M, N, K, A.data_ptr(), K, 0, B.data_ptr(), K, 0, C.data_ptr(), N, 0, st)


def fz(M, N, K, A, B, C, ldc, res=None, glu=0, aux=None, aux_in=None):
    return lambda: L.lib.malleus_k_gemm_fused(M, N, K, A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), ldc,
                                              res.data_ptr() if res is not None else None, N if res is not None else 0,
                                              glu, aux.data_ptr() if aux is not None else None,
                                              aux_in.data_ptr() if aux_in is not None else None, fused, st)


a2 = torch.randn(T, h, device="cuda").to(bf)
wgu = (torch.randn(2 * F, h, device="cuda") * 0.02).to(bf)
gu = torch.empty(T, 2 * F, device="cuda", dtype=bf)
u = torch.empty(T, F, device="cuda", dtype=bf)
dy = torch.randn(T, h, device="cuda").to(bf)
wd = (torch.randn(F, h, device="cuda") * 0.02).to(bf)
du = torch.empty(T, F, device="cuda", dtype=bf)
dgu = torch.empty(T, 2 * F, device="cuda", dtype=bf)
o = torch.randn(T, h, device="cuda").to(bf)
wo = (torch.randn(h, h, device="cuda") * 0.02).to(bf)
x = torch.randn(T, h, device="cuda").to(bf)
x1 = torch.empty(T, h, device="cuda", dtype=bf)
ud = torch.randn(T, F, device="cuda").to(bf)
wdT = (torch.randn(h, F, device="cuda") * 0.02).to(bf)
rows = [
    ("gate/up      plain", plain(T, 2 * F, h, a2, wgu, gu), 2 * T * 2 * F * h),
    ("gate/up      +SwiGLU (glu 1)", fz(T, 2 * F, h, a2, wgu, gu, 2 * F, glu=1, aux=u), 2 * T * 2 * F * h),
    ("du           plain", plain(T, F, h, dy, wd, du), 2 * T * F * h),
    ("du           +SwiGLU bwd (glu 2)", fz(T, F, h, dy, wd, du, F, glu=2, aux=dgu, aux_in=gu), 2 * T * F * h),
    ("O-proj       plain", plain(T, h, h, o, wo, x1), 2 * T * h * h),
    ("O-proj       +residual", fz(T, h, h, o, wo, x1, h, res=x), 2 * T * h * h),
    ("down         plain", plain(T, h, F, ud, wdT, x1), 2 * T * h * F),
    ("down         +residual", fz(T, h, F, ud, wdT, x1, h, res=x), 2 * T * h * F),
]
for name, fn, fl in rows:
    us = bench(fn)
    print(f"{name:34s} {us:8.1f} us  {fl / us / 1e6:7.1f} TF/s  fused={fused[0]}", flush=True)
