"""tcgen05 GEMM (and the ordered fp32 GEMM) against a plain PyTorch fp32
reference of the same op, through the C-ABI (hzp_gemm_bf16 / hzp_gemm_f32)."""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SHAPES = [
    # (M, N, K)
    (128, 256, 64),
    (256, 512, 512),
    (384, 640, 1024),
    (200, 136, 72),     # M/N/K tails (TMA zero-fill, masked stores)
    (8, 64, 128),       # tiny M
    (1024, 1024, 2048),
]


def _mk(M, N, K, a_mn, b_mn, dev):
    g = torch.Generator(device="cpu").manual_seed(M * 7 + N * 3 + K)
    A = torch.randn(M, K, generator=g).to(dev, torch.bfloat16)
    B = torch.randn(N, K, generator=g).to(dev, torch.bfloat16)
    As = A.t().contiguous() if a_mn else A  # MN-major storage: [K, M]
    Bs = B.t().contiguous() if b_mn else B
    lda = M if a_mn else K
    ldb = N if b_mn else K
    return A, B, As, Bs, lda, ldb


@pytest.mark.parametrize("a_mn", [0, 1])
@pytest.mark.parametrize("b_mn", [0, 1])
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_tcgen05_gemm_matches_torch(gpu, shape, a_mn, b_mn):
    from paper_2510_20111_b200.engine import gemm_bf16
    M, N, K = shape
    if (a_mn and M % 8) or (b_mn and N % 8):
        pytest.skip("MN-major leading dim must be a multiple of 8 for TMA")
    A, B, As, Bs, lda, ldb = _mk(M, N, K, a_mn, b_mn, gpu)
    ref = A.float() @ B.float().t()
    C32 = torch.full((M, N), float("nan"), device=gpu, dtype=torch.float32)
    gemm_bf16(As.data_ptr(), Bs.data_ptr(), C32.data_ptr(), M, N, K, lda, ldb, N, a_mn, b_mn, 1)
    torch.cuda.synchronize()
    err = (C32 - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-5, err  # fp32 accumulation of exact bf16 products
    C16 = torch.zeros((M, N), device=gpu, dtype=torch.bfloat16)
    gemm_bf16(As.data_ptr(), Bs.data_ptr(), C16.data_ptr(), M, N, K, lda, ldb, N, a_mn, b_mn, 0)
    torch.cuda.synchronize()
    err16 = (C16.float() - ref).abs().max().item() / ref.abs().max().item()
    assert err16 < 1e-2, err16


def test_tcgen05_gemm_accumulate(gpu):
    from paper_2510_20111_b200.engine import gemm_bf16
    M, N, K = 256, 384, 256
    A, B, As, Bs, lda, ldb = _mk(M, N, K, 1, 1, gpu)
    C = torch.randn(M, N, device=gpu)
    ref = C + A.float() @ B.float().t()
    gemm_bf16(As.data_ptr(), Bs.data_ptr(), C.data_ptr(), M, N, K, lda, ldb, N, 1, 1, 2)
    torch.cuda.synchronize()
    assert (C - ref).abs().max().item() < 1e-3


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 1)])
def test_ordered_f32_gemm_is_sequential_fp32(gpu, a_mn, b_mn):
    from paper_2510_20111_b200.engine import gemm_f32
    M, N, K = 40, 24, 70
    g = torch.Generator().manual_seed(3)
    A = torch.randn(M, K, generator=g)
    B = torch.randn(N, K, generator=g)
    # CPU reference with the same left-fold order, separate rounding per op
    ref = torch.zeros(M, N)
    acc = torch.zeros(M, N, dtype=torch.float32)
    for k in range(K):
        acc = acc + (A[:, k:k + 1] * B[:, k].view(1, -1))
    ref = acc
    As = (A.t().contiguous() if a_mn else A).to(gpu)
    Bs = (B.t().contiguous() if b_mn else B).to(gpu)
    C = torch.empty(M, N, device=gpu)
    gemm_f32(As.data_ptr(), Bs.data_ptr(), C.data_ptr(), M, N, K, M if a_mn else K,
             N if b_mn else K, N, a_mn, b_mn, 1)
    torch.cuda.synchronize()
    assert torch.equal(C.cpu(), ref)
