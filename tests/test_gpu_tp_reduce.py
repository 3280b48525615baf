"""Parity of the peer-memory TP reduction (malleus_k_tp_reduce, tp_reduce.cu) against plain
torch-CPU arithmetic: one process drives k members on k GPUs.  The sum is taken in member order
on the GPU, and the CPU reference adds in the same order, so the fp32 sum and the bf16 residual are
compared bit for bit; the RMSNorm output (different summation order inside the row) to 1 bf16 ulp
and rstd to 1e-6 relative."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def _need(k):
    if not torch.cuda.is_available() or torch.cuda.device_count() < k:
        pytest.skip(f"needs {k} GPUs")


def _ref_sum(parts):
    s = parts[0].cpu().clone()
    for p in parts[1:]:
        s = s + p.cpu()
    return s


@pytest.mark.parametrize("k,T,h,pdt", [(2, 300, 512, "f32"), (2, 2048, 4096, "f32"), (4, 257, 1024, "f32"),
                                      (2, 300, 512, "bf16"), (4, 2048, 8192, "bf16"), (3, 301, 2048, "bf16"),
                                      (2, 2048, 4096, "bf16sum"), (4, 515, 1024, "bf16sum")])
def test_tp_reduce_modes(k, T, h, pdt):
    _need(k)
    from tests.tputil import Group, enable_peer_access
    enable_peer_access(k)
    dt = torch.bfloat16 if pdt.startswith("bf16") else torch.float32
    G = Group(k, T, h, part_dtype=dt, sum_bf16=pdt == "bf16sum")
    gen = torch.Generator().manual_seed(7)
    x_cpu = (torch.randn(T, h, generator=gen) * 2).to(torch.bfloat16)
    g_cpu = (1 + 0.1 * torch.randn(h, generator=gen)).to(torch.bfloat16)
    xs = [x_cpu.to(f"cuda:{j}") for j in range(k)]
    gs = [g_cpu.to(f"cuda:{j}") for j in range(k)]
    for rep, mode in enumerate([0, 1, 2, 0, 1]):  # epochs 1..5: both partial buffers, every mode
        buf = (G.epoch + 1) & 1
        parts = [torch.randn(T, h, generator=gen).to(dt) for _ in range(k)]
        for j in range(k):
            G.part[buf][j].copy_(parts[j])
        parts = [q.float() for q in parts]
        G.sync()
        G.launch(mode, xs, gs)
        G.sync()
        s = _ref_sum(parts)
        if mode == 0:
            ref = s.to(torch.bfloat16) if pdt == "bf16sum" else s
            for j in range(k):
                assert torch.equal(G.out32[j].cpu(), ref), (rep, j)
            continue
        x1 = (x_cpu.float() + s).to(torch.bfloat16)
        for j in range(k):
            assert torch.equal(G.x1[j].cpu(), x1), (rep, mode, j)
        if mode == 1:
            xf = x1.double()
            rstd = torch.rsqrt((xf * xf).mean(1) + 1e-5)
            a = (xf * rstd[:, None] * g_cpu.double())
            for j in range(k):
                assert torch.allclose(G.rstd[j].cpu().double(), rstd, rtol=1e-6, atol=0), (rep, j)
                diff = (G.a[j].cpu().double() - a).abs()
                assert (diff <= a.abs() * 2.0 ** -7 + 1e-30).all(), (rep, j, diff.max())
