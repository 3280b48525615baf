"""Pipeline timeline of the tcgen05 attention forward (MALLEUS_ATTN_TRACE=1): per key tile of the
heaviest CTA, when the producer issued K / V, the MMA warp issued QK / PV, and softmax warp 2 started,
passed the max exchange and finished.  Times in microseconds from the CTA's start."""
import ctypes as C
import os
import sys

os.environ["MALLEUS_ATTN_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2410_13333_b200 import _lib as L

L.lib.malleus_k_attn_trace_buffer.restype = C.c_void_p
nb, s, n, d = 1, 2048, 32, 128
T = nb * s
qkv = (torch.randn(T, 3 * n * d, device="cuda") * 0.5).to(torch.bfloat16)
o = torch.empty(T, n * d, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(nb, n, s, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    L.lib.malleus_k_attention_fwd(nb, s, n, d, qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), 1e4, st)
torch.cuda.synchronize()
addr = L.lib.malleus_k_attn_trace_buffer()
buf = np.ctypeslib.as_array((C.c_uint64 * (2 * 8 * 64)).from_address(addr)).reshape(2, 8, 64).astype(np.int64)
names = ["K_issue", "V_issue", "QK_issue", "PV_issue", "sm_start", "sm_xchg", "sm_end"]
for cta in range(2):
    b = buf[cta]
    t0 = b[7, 0]
    print(f"CTA (0,{cta}): epilogue start {(b[7,1]-t0)/1e3:.2f} us, end {(b[7,2]-t0)/1e3:.2f} us")
    print("tile " + " ".join(f"{x:>9s}" for x in names))
    for i in range(s // 128):
        print(f"{i:4d} " + " ".join(f"{(b[e, i]-t0)/1e3:9.2f}" for e in range(7)))

# ---- backward dK / dV kernel: per 64-query sub-tile
do = torch.randn(T, n * d, device="cuda").to(torch.bfloat16)
dqkv = torch.empty_like(qkv)
L.lib.malleus_k_attn_bwd_trace_buffer.restype = C.c_void_p
for _ in range(3):
    L.lib.malleus_k_attention_bwd(nb, s, n, d, qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), do.data_ptr(),
                                  dqkv.data_ptr(), 1e4, st)
torch.cuda.synchronize()
addr = L.lib.malleus_k_attn_bwd_trace_buffer()
buf = np.ctypeslib.as_array((C.c_uint64 * (2 * 16 * 64)).from_address(addr)).reshape(2, 16, 64).astype(np.int64)
names = ["QdO_issue", "c_tmem", "S_issue", "dVdK_iss", "c_start", "c_math", "c_end"] + [f"end_w{w}" for w in range(2, 10)]
for cta in range(1):
    b = buf[cta]
    t0 = b[7, 0]
    print(f"dKV CTA (0,{cta}): epilogue start {(b[7,1]-t0)/1e3:.2f} us, end {(b[7,2]-t0)/1e3:.2f} us")
    print("iter " + " ".join(f"{x:>8s}" for x in names))
    for i in range(s // 64):
        print(f"{i:4d} " + " ".join(f"{(b[e, i]-t0)/1e3:8.2f}" for e in list(range(7)) + list(range(8, 16))))

# ---- backward dQ kernel: per 128-key tile of CTA (0, 0, 0)
L.lib.malleus_k_attn_dq_trace_buffer.restype = C.c_void_p
addr = L.lib.malleus_k_attn_dq_trace_buffer()
b = np.ctypeslib.as_array((C.c_uint64 * (8 * 64)).from_address(addr)).reshape(8, 64).astype(np.int64)
t0 = b[7, 0]
names = ["KV_issue", "c_s_ok", "S_issue", "dQ_issue", "c_dp_ok", "c_math", "c_end"]
print("dQ CTA (0,0,0)")
print("tile " + " ".join(f"{x:>8s}" for x in names))
for i in range(s // 128):
    print(f"{i:4d} " + " ".join(f"{(b[e, i]-t0)/1e3:8.2f}" for e in range(7)))
