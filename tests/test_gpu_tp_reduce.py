"""Parity of the peer-memory TP reduction (malleus_k_tp_reduce, tp_reduce.cu) against plain
torch-CPU arithmetic: one process drives k members on k GPUs.  The sum is taken in member order
on the GPU, and the CPU reference adds in the same order, so the fp32 sum and the bf16 residual are
compared bit for bit; the RMSNorm output (different summation order inside the row) to 1 bf16 ulp
and rstd to 1e-6 relative.  The same kernel also runs with all k members on ONE GPU (co-resident
grids, one stream per member), which is how the driver's single-GPU box checks K15."""
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


def _run(G, k, T, h, pdt, seed=7, modes=(0, 1, 2, 0, 1)):
    """Epochs 1..len(modes): both partial buffers, every mode; member-order fp32 sums bitwise,
    residual bitwise, RMSNorm to 1 bf16 ulp, rstd 1e-6."""
    dt = torch.bfloat16 if pdt.startswith("bf16") else torch.float32
    gen = torch.Generator().manual_seed(seed)
    x_cpu = (torch.randn(T, h, generator=gen) * 2).to(torch.bfloat16)
    g_cpu = (1 + 0.1 * torch.randn(h, generator=gen)).to(torch.bfloat16)
    xs = [x_cpu.to(f"cuda:{d}") for d in G.devices]
    gs = [g_cpu.to(f"cuda:{d}") for d in G.devices]
    for rep, mode in enumerate(modes):
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


@pytest.mark.parametrize("k,T,h,pdt", [(2, 300, 512, "f32"), (2, 2048, 4096, "f32"), (4, 257, 1024, "f32"),
                                      (2, 300, 512, "bf16"), (4, 2048, 8192, "bf16"), (3, 301, 2048, "bf16"),
                                      (2, 2048, 4096, "bf16sum"), (4, 515, 1024, "bf16sum")])
def test_tp_reduce_modes(k, T, h, pdt):
    _need(k)
    from tests.tputil import Group, enable_peer_access
    enable_peer_access(k)
    dt = torch.bfloat16 if pdt.startswith("bf16") else torch.float32
    _run(Group(k, T, h, part_dtype=dt, sum_bf16=pdt == "bf16sum"), k, T, h, pdt)


# Single-GPU driver of the same kernel: k members co-resident on cuda:0,
# each on its own stream, peer pointers = local buffers.  Grids stay small (rows per member <= 148 or
# so) so every member's CTAs can be resident at once; even and uneven (speed-proportional) row
# splits, including a member with no rows.
@pytest.mark.parametrize("k,T,h,pdt,rows", [
    (2, 128, 512, "f32", None), (2, 128, 4096, "bf16", None), (3, 97, 2048, "bf16sum", None),
    (4, 200, 1024, "f32", None), (4, 64, 8192, "bf16", None),
    (2, 128, 512, "bf16", [0, 96, 128]), (3, 150, 1024, "f32", [0, 20, 20, 150]),
    (4, 160, 4096, "bf16sum", [0, 64, 96, 128, 160])])
def test_tp_reduce_one_device(k, T, h, pdt, rows):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from tests.tputil import Group
    dt = torch.bfloat16 if pdt.startswith("bf16") else torch.float32
    G = Group(k, T, h, part_dtype=dt, sum_bf16=pdt == "bf16sum", devices=[0] * k, rows=rows)
    _run(G, k, T, h, pdt, seed=11 + k)


def test_tp_reduce_rejects_bad_row_split():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import ctypes as C
    from paper_2410_13333_b200 import _lib as L
    from tests.tputil import Group
    G = Group(2, 64, 512, devices=[0, 0], rows=[0, 40, 63])  # does not end at T
    with pytest.raises(AssertionError):
        G.launch(0)
    G.rows = (C.c_int32 * 3)(0, 50, 40)  # decreasing
    G.epoch = 0
    with pytest.raises(AssertionError):
        G.launch(0)
    assert L.lib.malleus_kernel_launches() >= 0
