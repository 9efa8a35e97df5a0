"""tcgen05 GEMM (C = alpha A B^T + beta C, bf16/fp16, fp32 accumulation in TMEM) against a
plain fp32 product of the same 16-bit operands (-m gpu)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    import paper_2510_02126_b200 as G
    G.lib()
    return G


@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (256, 384, 256), (200, 130, 32), (1024, 96, 1024),
                                   (300, 1000, 40), (1, 1, 16),
                                   # >= one tile per SM: the persistent warp-specialised kernel
                                   (2048, 2048, 256), (2000, 2100, 96), (1536, 1536, 640), (4096, 1280, 64)])
@pytest.mark.parametrize("beta", [0.0, 1.0])
def test_tc_gemm_matches_fp32_reference(gpu, dt, M, N, K, beta):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N * 3 + K)
    A = torch.randn(M, K, device="cuda", generator=g).to(dt)
    B = torch.randn(N, K, device="cuda", generator=g).to(dt)
    C0 = torch.randn(M, N, device="cuda", generator=g).to(dt)
    C = C0.clone()
    gpu.tc_gemm(A, B, C, alpha=-1.0, beta=beta)
    ref = -(A.float() @ B.float().T) + beta * C0.float()
    u = 2.0 ** -8 if dt == torch.bfloat16 else 2.0 ** -11
    err = (C.float() - ref).abs()
    # output rounding (u |ref|) + fp32 accumulation of K products
    bound = u * ref.abs() + 1e-5 * K * (A.float().abs() @ B.float().abs().T + 1)
    assert torch.all(err <= bound), (err - bound).max().item()
