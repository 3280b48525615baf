"""Launch one hot-path GEMM shape a few times (for `ncu --set full` captures).
  python tools/gemm_one.py M N K a_mn b_mn mode variant"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_13333_b200 import _lib as L

M, N, K, amn, bmn, mode, var = (int(x) for x in sys.argv[1:8])
L.lib.malleus_k_gemm_variant(var)
A = (torch.randn(K, M, device="cuda") if amn else torch.randn(M, K, device="cuda")).to(torch.bfloat16)
B = (torch.randn(K, N, device="cuda") if bmn else torch.randn(N, K, device="cuda")).to(torch.bfloat16)
C = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16 if mode == 0 else torch.float32)
st = torch.cuda.current_stream().cuda_stream
for _ in range(4):
    assert L.lib.malleus_k_gemm(M, N, K, A.data_ptr(), A.shape[1], amn, B.data_ptr(), B.shape[1], bmn,
                                C.data_ptr(), N, mode, st) == 0
torch.cuda.synchronize()
print("ok", M, N, K, amn, bmn, mode, var)
