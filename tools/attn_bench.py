"""Attention kernel throughput (malleus_k_attention_fwd / bwd incl. RoPE) on the C2 shape.
Algorithmic causal FLOPs: fwd 2 * 2 * s^2/2 * d * n * nb, bwd 2.5x fwd."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_13333_b200 import _lib as L


def bench(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


st = torch.cuda.current_stream().cuda_stream
for nb, s, n, d in [(1, 2048, 32, 128), (1, 4096, 16, 128), (2, 2048, 16, 128)]:
    T = nb * s
    qkv = (torch.randn(T, 3 * n * d, device="cuda") * 0.5).to(torch.bfloat16)
    o = torch.empty(T, n * d, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(nb, n, s, device="cuda")
    do = torch.randn(T, n * d, device="cuda").to(torch.bfloat16)
    dqkv = torch.empty_like(qkv)
    f = lambda: L.lib.malleus_k_attention_fwd(nb, s, n, d, qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), 1e4, st)
    b = lambda: L.lib.malleus_k_attention_bwd(nb, s, n, d, qkv.data_ptr(), o.data_ptr(), lse.data_ptr(),
                                              do.data_ptr(), dqkv.data_ptr(), 1e4, st)
    flops = 2 * 2 * s * s / 2 * d * n * nb
    tf, tb = bench(f), bench(b)
    # reference: torch SDPA (flash) for context
    q = torch.randn(nb, n, s, d, device="cuda", dtype=torch.bfloat16)
    ref = bench(lambda: torch.nn.functional.scaled_dot_product_attention(q, q, q, is_causal=True))
    qg = q.clone().requires_grad_(True)
    out = torch.nn.functional.scaled_dot_product_attention(qg, qg, qg, is_causal=True)
    g = torch.randn_like(out)
    refb = bench(lambda: torch.autograd.grad(out, qg, g, retain_graph=True))
    tb2 = bench(b)  # re-time ours after the others (first-call effects)
    print(f"nb={nb} s={s} n={n} d={d}: fwd {tf*1e3:.0f} us {flops/tf/1e9:.0f} TF | bwd {tb*1e3:.0f} us "
          f"{2.5*flops/tb/1e9:.0f} TF (again {tb2*1e3:.0f} us) | torch sdpa fwd {ref*1e3:.0f} us "
          f"{flops/ref/1e9:.0f} TF bwd {refb*1e3:.0f} us {2.5*flops/refb/1e9:.0f} TF", flush=True)
