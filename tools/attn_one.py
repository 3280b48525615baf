"""Launch attention fwd + bwd on the C2 shape a few times (for `ncu --set full` captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_13333_b200 import _lib as L

nb, s, n, d = 1, 2048, 32, 128
T = nb * s
st = torch.cuda.current_stream().cuda_stream
qkv = (torch.randn(T, 3 * n * d, device="cuda") * 0.5).to(torch.bfloat16)
o = torch.empty(T, n * d, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(nb, n, s, device="cuda")
do = torch.randn(T, n * d, device="cuda").to(torch.bfloat16)
dqkv = torch.empty_like(qkv)
for _ in range(3):
    assert L.lib.malleus_k_attention_fwd(nb, s, n, d, qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), 1e4, st) == 0
    assert L.lib.malleus_k_attention_bwd(nb, s, n, d, qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), do.data_ptr(),
                                         dqkv.data_ptr(), 1e4, st) == 0
torch.cuda.synchronize()
print("ok")
