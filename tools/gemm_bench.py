"""Quick GEMM throughput check: malleus_k_gemm vs torch.matmul (cuBLAS) on hot-path shapes."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_13333_b200 import _lib as L

def bench(fn, iters=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters

st = torch.cuda.current_stream().cuda_stream
shapes = [("sq8192", 8192, 8192, 8192, 0, 0), ("qkv", 2048, 12288, 4096, 0, 0), ("gu", 2048, 22016, 4096, 0, 0),
          ("down_KMN", 2048, 4096, 11008, 0, 1), ("wgrad_gu", 22016, 4096, 2048, 1, 1), ("lmhead", 2048, 32000, 4096, 0, 0)]
for name, M, N, K, amn, bmn in shapes:
    A = torch.randn(K, M, device="cuda").to(torch.bfloat16) if amn else torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(K, N, device="cuda").to(torch.bfloat16) if bmn else torch.randn(N, K, device="cuda").to(torch.bfloat16)
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    f = lambda: L.lib.malleus_k_gemm(M, N, K, A.data_ptr(), A.shape[1], amn, B.data_ptr(), B.shape[1], bmn, C.data_ptr(), N, 0, st)
    ms = bench(f)
    At = A.t() if amn else A
    Bt = B if bmn else B.t()
    ref = bench(lambda: torch.matmul(At, Bt))
    err = (C.float() - torch.matmul(At, Bt).float()).abs().max().item()
    print(f"{name:10s} M={M} N={N} K={K}: malleus {ms*1e3:8.1f} us {2*M*N*K/ms/1e9:7.1f} TF | cublas {ref*1e3:8.1f} us {2*M*N*K/ref/1e9:7.1f} TF | maxdiff {err:.3g}", flush=True)

# CTA-pair vs single-CTA on the same shapes
for var in (1, 3, 2):
    L.lib.malleus_k_gemm_variant(var)
    for name, M, N, K, amn, bmn in shapes:
        A = torch.randn(K, M, device="cuda").to(torch.bfloat16) if amn else torch.randn(M, K, device="cuda").to(torch.bfloat16)
        B = torch.randn(K, N, device="cuda").to(torch.bfloat16) if bmn else torch.randn(N, K, device="cuda").to(torch.bfloat16)
        C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        f = lambda: L.lib.malleus_k_gemm(M, N, K, A.data_ptr(), A.shape[1], amn, B.data_ptr(), B.shape[1], bmn, C.data_ptr(), N, 0, st)
        ms = bench(f)
        print(f"variant {var} {name:10s}: {ms*1e3:8.1f} us {2*M*N*K/ms/1e9:7.1f} TF", flush=True)
L.lib.malleus_k_gemm_variant(0)
