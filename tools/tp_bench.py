"""Peer-memory TP reduction (malleus_k_tp_reduce) timing at the C2 shape (T = 2048, h = 4096):
k members on k GPUs in one process; per-mode microseconds per reduction (max over members) and
the NVLink bytes each member moves ((k-1)/k of its rows in, and out to k-1 peers)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from tests.tputil import Group, enable_peer_access

T, h = int(os.environ.get("TP_T", 2048)), int(os.environ.get("TP_H", 4096))
for k in (2, 4, 8):
    if torch.cuda.device_count() < k:
        break
    enable_peer_access(k)
    G = Group(k, T, h, part_dtype=torch.bfloat16 if os.environ.get("TP_BF16") else torch.float32)
    xs = [torch.randn(T, h, device=f"cuda:{j}").to(torch.bfloat16) for j in range(k)]
    gs = [torch.ones(h, device=f"cuda:{j}").to(torch.bfloat16) for j in range(k)]
    for mode, name, out_b in ((0, "SUM", 4), (1, "RESID_NORM", 4), (2, "RESID", 2)):
        for _ in range(5):
            G.launch(mode, xs, gs)
        G.sync()
        n = 50
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
        # hold every device in a sleep kernel while the host enqueues all launches, so the timed
        # region is GPU-bound (no host launch gaps, no member waiting for the host to reach it)
        for j in range(k):
            with torch.cuda.device(j):
                torch.cuda._sleep(int(60e6))  # ~30 ms
                ev[j][0].record()
        for _ in range(n):
            G.launch(mode, xs, gs)
        for j in range(k):
            with torch.cuda.device(j):
                ev[j][1].record()
        G.sync()
        us = max(ev[j][0].elapsed_time(ev[j][1]) for j in range(k)) / n * 1e3
        rows = T / k
        nv_in = (k - 1) * rows * h * (2 if os.environ.get("TP_BF16") else 4)
        nv_out = (k - 1) * rows * h * out_b
        print(f"k={k} T={T} h={h} {name:10s}: {us:7.1f} us/reduce | per member NVLink in {nv_in/us/1e3:6.0f} GB/s, "
              f"out {nv_out/us/1e3:6.0f} GB/s", flush=True)
    # context: one peer copy of the full fp32 partial
    a = torch.empty(T, h, device="cuda:0")
    b = torch.empty(T, h, device="cuda:1")
    for _ in range(3):
        b.copy_(a)
    torch.cuda.synchronize(0); torch.cuda.synchronize(1)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.device(0):
        s.record()
        for _ in range(20):
            b.copy_(a)
        e.record()
    torch.cuda.synchronize(0); torch.cuda.synchronize(1)
    us = s.elapsed_time(e) / 20 * 1e3
    print(f"  context: cuda:0 -> cuda:1 copy of {T*h*4/1e6:.0f} MB: {us:.1f} us ({T*h*4/us/1e3:.0f} GB/s)", flush=True)

# ---- optional stage trace (MALLEUS_TP_TRACE=1): where one k=2 reduction spends its time
if os.environ.get("MALLEUS_TP_TRACE") and torch.cuda.device_count() >= 2:
    import ctypes as C
    import numpy as np
    from paper_2410_13333_b200 import _lib as L
    L.lib.malleus_k_tp_trace_buffer.restype = C.c_void_p
    k = 2
    G = Group(k, T, h)
    xs = [torch.randn(T, h, device=f"cuda:{j}").to(torch.bfloat16) for j in range(k)]
    gs = [torch.ones(h, device=f"cuda:{j}").to(torch.bfloat16) for j in range(k)]
    for mode in (0, 1, 2):
        for _ in range(3):
            G.launch(mode, xs, gs)
        G.sync()
        for j in range(k):
            with torch.cuda.device(j):
                torch.cuda._sleep(int(60e6))
        G.launch(mode, xs, gs)
        G.sync()
        addr = L.lib.malleus_k_tp_trace_buffer()
        buf = np.ctypeslib.as_array((C.c_uint64 * (4 * 592 * k)).from_address(addr)).reshape(k, 592, 4).astype(np.int64)
        t0 = buf[:, :, 0].min()
        for j in range(k):
            b = buf[j] - t0
            print(f"mode {mode} member {j}: start {np.median(b[:,0])/1e3:.1f}..{b[:,0].max()/1e3:.1f} us, "
                  f"ready med {np.median(b[:,1])/1e3:.1f} max {b[:,1].max()/1e3:.1f}, rows med {np.median(b[:,2])/1e3:.1f} "
                  f"max {b[:,2].max()/1e3:.1f}, end med {np.median(b[:,3])/1e3:.1f} max {b[:,3].max()/1e3:.1f} us", flush=True)
