"""GPU parity of the GEMM's fused epilogues (malleus_k_gemm_fused) against the oracle.

* residual (TP-1 row-parallel O-proj / down projection, SURVEY §8(a) S7/S10 + the residual of S8):
  small-integer operands make the fp32 product exact, so C must equal RNE_bf16(A B^T + res) bit for
  bit (§8(c) small-integer pin);
* SwiGLU forward in the gate/up GEMM (S9) and SwiGLU backward in the down-projection dgrad (S12):
  the GEMM part is exact on small integers (gu / du bitwise); u, dG, dU are compared with
  oracle.model.swiglu_fwd / swiglu_bwd evaluated in fp64 on the same bf16 inputs, within one bf16
  rounding plus the fp32 __expf error (reading R15's elementwise floor).
Ragged F (not a multiple of the 128-column half tile) and M tails are included."""
import ctypes

import numpy as np
import pytest
import torch

from oracle import model as OM
from synth.gen import small_int_matrix, normal_matrix

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2410_13333_b200 import _lib
    return _lib


def _bf(x):
    return torch.tensor(np.asarray(x, dtype=np.float32)).to(torch.bfloat16)


def _rne(x64):
    """RNE to bf16 of exactly-representable-in-fp32 values (fp64 -> fp32 exact here)."""
    return torch.tensor(x64.astype(np.float32)).to(torch.bfloat16).float().numpy().astype(np.float64)


def _call(L, M, N, K, A, B, C, ldc, res=None, ldr=0, glu=0, aux=None, aux_in=None):
    fused = (ctypes.c_int32 * 1)(-1)
    st = torch.cuda.current_stream().cuda_stream
    rc = L.lib.malleus_k_gemm_fused(M, N, K, A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), ldc,
                                    res.data_ptr() if res is not None else None, ldr, glu,
                                    aux.data_ptr() if aux is not None else None,
                                    aux_in.data_ptr() if aux_in is not None else None, fused, st)
    assert rc == 0
    torch.cuda.synchronize()
    return fused[0]


@pytest.mark.parametrize("variant", [0, 1, 3], ids=["auto", "cta1", "cta2_direct_epi"])
@pytest.mark.parametrize("shape", [(2048, 4096, 512), (1000, 776, 520), (200, 304, 136), (512, 128, 4096)])
def test_residual_epilogue_bitwise(L, variant, shape):
    M, N, K = shape
    assert L.lib.malleus_k_gemm_variant(variant) == 0
    try:
        A = small_int_matrix((M, K), 6, seed=M + K)
        B = small_int_matrix((N, K), 6, seed=N + 3 * K)      # stored [N][K]: C = A B^T
        R = small_int_matrix((M, N), 200, seed=11)           # bf16-exact residual
        exact = A.astype(np.float64) @ B.astype(np.float64).T + R
        assert np.abs(exact).max() < 2 ** 24
        dA, dB, dR = _bf(A).cuda(), _bf(B).cuda(), _bf(R).cuda()
        dC = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
        _call(L, M, N, K, dA, dB, dC, N, res=dR, ldr=N)
        assert np.array_equal(dC.float().cpu().numpy().astype(np.float64), _rne(exact))
    finally:
        L.lib.malleus_k_gemm_variant(0)


@pytest.mark.parametrize("M,F,K", [(2048, 5504, 4096), (512, 1376, 512), (768, 272, 256), (300, 1536, 512)])
def test_swiglu_fwd_epilogue(L, M, F, K):
    A = small_int_matrix((M, K), 4, seed=5 + M)
    W = small_int_matrix((2 * F, K), 4, seed=7 + F)          # [W_g; W_u] stored [2F][K]
    scale = 2.0 ** -6                                         # exact power-of-two scaling keeps sums exact
    Af, Wf = A * scale, W * scale
    dA, dW = _bf(Af).cuda(), _bf(Wf).cuda()
    gu = torch.zeros(M, 2 * F, dtype=torch.bfloat16, device="cuda")
    u = torch.full((M, F), float("nan"), dtype=torch.bfloat16, device="cuda")
    fused = _call(L, M, 2 * F, K, dA, dW, gu, 2 * F, glu=1, aux=u)
    exact = Af.astype(np.float64) @ Wf.astype(np.float64).T
    gu_h = gu.float().cpu().numpy().astype(np.float64)
    assert np.array_equal(gu_h, _rne(exact))                 # pre-activations: exact, then RNE
    if M < 256:
        assert fused == 0                                     # single-CTA kernel: no fused epilogue
        return
    assert fused == 1
    G, U = gu_h[:, :F], gu_h[:, F:]
    ref = OM.swiglu_fwd(G, U)                                 # oracle, fp64 on the bf16 values
    got = u.float().cpu().numpy().astype(np.float64)
    tol = 2.0 ** -8 * np.abs(ref) + 1e-3 * np.abs(ref).max()
    assert np.all(np.abs(got - ref) <= tol), np.abs(got - ref).max()


@pytest.mark.parametrize("M,F,K", [(2048, 5504, 4096), (512, 1376, 512), (768, 272, 256)])
def test_swiglu_bwd_epilogue(L, M, F, K):
    dy = small_int_matrix((M, K), 4, seed=21 + M)
    Wd = small_int_matrix((F, K), 4, seed=23 + F)            # W_d^T stored [F][K]: du = dy W_d
    scale = 2.0 ** -6
    dyf, Wdf = dy * scale, Wd * scale
    gu = torch.tensor(normal_matrix((M, 2 * F), 31)).to(torch.bfloat16)
    d_dy, d_W, d_gu = _bf(dyf).cuda(), _bf(Wdf).cuda(), gu.cuda()
    du = torch.zeros(M, F, dtype=torch.bfloat16, device="cuda")
    dgu = torch.full((M, 2 * F), float("nan"), dtype=torch.bfloat16, device="cuda")
    fused = _call(L, M, F, K, d_dy, d_W, du, F, glu=2, aux=dgu, aux_in=d_gu)
    assert fused == 1
    D = _rne(dyf.astype(np.float64) @ Wdf.astype(np.float64).T)  # du rounded to bf16 (reading R6)
    g = gu.float().numpy().astype(np.float64)
    dG_ref, dU_ref = OM.swiglu_bwd(g[:, :F], g[:, F:], D)
    got = dgu.float().cpu().numpy().astype(np.float64)
    for ref, out in ((dG_ref, got[:, :F]), (dU_ref, got[:, F:])):
        tol = 2.0 ** -8 * np.abs(ref) + 1e-3 * np.abs(ref).max()
        assert np.all(np.abs(out - ref) <= tol), np.abs(out - ref).max()


def test_fused_rejects_bad_layouts(L):
    st = torch.cuda.current_stream().cuda_stream
    A = torch.zeros(256, 64, dtype=torch.bfloat16, device="cuda")
    B = torch.zeros(96, 64, dtype=torch.bfloat16, device="cuda")
    C = torch.zeros(256, 96, dtype=torch.bfloat16, device="cuda")
    u = torch.zeros(256, 48, dtype=torch.bfloat16, device="cuda")
    # glu 1 needs F = N / 2 a multiple of 16: N = 96 -> F = 48 is fine, N = 80 -> F = 40 is not
    assert L.lib.malleus_k_gemm_fused(256, 80, 64, A.data_ptr(), 64, B.data_ptr(), 64, C.data_ptr(), 96, None, 0,
                                      1, u.data_ptr(), None, None, st) == 1
    # glu and a residual together are not a fused mode
    assert L.lib.malleus_k_gemm_fused(256, 96, 64, A.data_ptr(), 64, B.data_ptr(), 64, C.data_ptr(), 96,
                                      C.data_ptr(), 96, 1, u.data_ptr(), None, None, st) == 1
