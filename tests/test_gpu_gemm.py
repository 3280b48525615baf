"""GPU parity of the tcgen05 GEMM (malleus_k_gemm) — every layout and epilogue the layer uses.

Small-integer operands make every fp32 partial sum exact regardless of summation order
(K * vmax^2 < 2^24, SURVEY §8(c) pins), so fp32 outputs must equal the exact integer product
bit for bit and bf16 outputs must equal RNE(exact).  Random bf16 operands are checked against
the fp64 product of the same bf16 values with an fp32-accumulation tolerance."""
import numpy as np
import pytest
import torch

from synth.gen import small_int_matrix, normal_matrix

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2410_13333_b200 import _lib
    return _lib


def _run(L, A, B, a_mn, b_mn, mode, C0=None):
    """A: logical [M,K] float32, B: logical [K,N] float32 (values bf16-exact)."""
    M, K = A.shape
    N = B.shape[1]
    Ast = A.T.copy() if a_mn else A          # a_mn: stored [K][M]
    Bst = B.copy() if b_mn else B.T.copy()   # b_mn: stored [K][N]; else [N][K]
    dA = torch.tensor(Ast).to(torch.bfloat16).cuda()
    dB = torch.tensor(Bst).to(torch.bfloat16).cuda()
    if mode == 0:
        dC = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
    else:
        dC = (torch.tensor(C0) if C0 is not None else torch.zeros(M, N)).float().cuda()
    st = torch.cuda.current_stream().cuda_stream
    rc = L.lib.malleus_k_gemm(M, N, K, dA.data_ptr(), dA.shape[1], a_mn, dB.data_ptr(), dB.shape[1],
                              b_mn, dC.data_ptr(), N, mode, st)
    assert rc == 0
    torch.cuda.synchronize()
    return dC.float().cpu().numpy()


SHAPES = [(128, 256, 64), (256, 512, 1024), (200, 304, 136), (96, 48, 2048), (1000, 776, 520),
          (2048, 2304, 4096)]


@pytest.fixture(params=[1, 2, 3], ids=["cta1", "cta2_tma_epi", "cta2_direct_epi"])
def variant(request, L):
    """1: single-CTA 128x256 tiles; 2: CTA pair (tcgen05.mma.cta_group::2) 256x256 tiles with TMA
    store / reduce-add epilogue; 3: CTA pair with direct stores."""
    assert L.lib.malleus_k_gemm_variant(request.param) == 0
    yield request.param
    L.lib.malleus_k_gemm_variant(0)


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 1), (1, 0)])
@pytest.mark.parametrize("shape", SHAPES)
def test_gemm_small_int_bitwise(L, variant, a_mn, b_mn, shape):
    M, N, K = shape
    A = small_int_matrix((M, K), 8, seed=M + K)
    B = small_int_matrix((K, N), 8, seed=N + 7 * K)
    exact = A.astype(np.float64) @ B.astype(np.float64)  # exact: |products| < 2^53
    assert np.abs(exact).max() < 2 ** 24
    C = _run(L, A, B, a_mn, b_mn, 1)
    assert np.array_equal(C, exact.astype(np.float32))
    C0 = small_int_matrix((M, N), 100, seed=3)
    C = _run(L, A, B, a_mn, b_mn, 2, C0=C0)
    assert np.array_equal(C, (exact + C0).astype(np.float32))
    Cb = _run(L, A, B, a_mn, b_mn, 0)
    ref = torch.tensor(exact.astype(np.float32)).to(torch.bfloat16).float().numpy()
    assert np.array_equal(Cb, ref)


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 1)])
def test_gemm_random_tolerance(L, variant, a_mn, b_mn):
    M, N, K = 1536, 1000, 4096
    A = torch.tensor(normal_matrix((M, K), 1)).to(torch.bfloat16).float().numpy()
    B = torch.tensor(normal_matrix((K, N), 2)).to(torch.bfloat16).float().numpy()
    ref = A.astype(np.float64) @ B.astype(np.float64)
    C = _run(L, A, B, a_mn, b_mn, 1)
    err = np.abs(C - ref).max() / np.abs(ref).max()
    assert err < 1e-5, err


def test_gemm_rejects_unaligned_strides(L):
    """TMA needs 16-byte row strides: ld not a multiple of 8 bf16 elements is E_ARG, not a fault."""
    A = torch.zeros(64, 100, dtype=torch.bfloat16, device="cuda")
    B = torch.zeros(64, 100, dtype=torch.bfloat16, device="cuda")
    C = torch.zeros(64, 64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    assert L.lib.malleus_k_gemm(64, 64, 100, A.data_ptr(), 100, 0, B.data_ptr(), 100, 0, C.data_ptr(), 64, 1,
                                st) == 1
