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
    (8192, 2048, 128),  # CTA pairs with the tail wave split into half-width units
    (6144, 2048, 192),
    # MN-major through the 5-D maps with a chunk past the end (MN % 128 == 64:
    # the second 64-wide chunk of the last tile is out of bounds -> zero fill)
    (320, 192, 256),
    (704, 320, 128),
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
    if a_mn and not b_mn:
        pytest.skip("A MN-major x B K-major is not used by any layer product (not instantiated)")
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


def test_gemm_profile_busy_union(gpu):
    """hzp_gemm_profile_read_busy: GEMMs on two streams overlap, so the union
    of the launch intervals is <= the summed launch time (and > 0)."""
    from paper_2510_20111_b200.engine import gemm_bf16, gemm_profile, gemm_profile_read_busy
    M = N = K = 2048
    A, B, As, Bs, lda, ldb = _mk(M, N, K, 0, 0, gpu)
    C1 = torch.empty(M, N, device=gpu, dtype=torch.bfloat16)
    C2 = torch.empty(M, N, device=gpu, dtype=torch.bfloat16)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    gemm_profile(True)
    for _ in range(4):
        gemm_bf16(As.data_ptr(), Bs.data_ptr(), C1.data_ptr(), M, N, K, lda, ldb, N, 0, 0, 0, s1.cuda_stream)
        gemm_bf16(As.data_ptr(), Bs.data_ptr(), C2.data_ptr(), M, N, K, lda, ldb, N, 0, 0, 0, s2.cuda_stream)
    torch.cuda.synchronize()
    gemm_profile(False)
    flops, ms, busy, n = gemm_profile_read_busy()
    assert n == 8 and flops == 8 * 2.0 * M * N * K
    assert 0 < busy <= ms * (1 + 1e-6)


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


def _ex(A, B, C, M, N, K, lda, ldb, ldc, a_mn, b_mn, mode=0, out_bf16=1, act=0, bias=None, aux=None,
        ldaux=0, resid=None, ldres=0, rowvec=None, alpha=1.0):
    import ctypes as C_
    from paper_2510_20111_b200 import _native as Nn
    p = lambda t: C_.c_void_p(t.data_ptr() if t is not None else 0)  # noqa: E731
    Nn.check(Nn.lib.hzp_gemm_bf16_ex(p(A), p(B), p(C), M, N, K, lda, ldb, ldc, a_mn, b_mn, mode,
                                     out_bf16, act, p(bias), p(aux), ldaux, p(resid), ldres, p(rowvec),
                                     alpha, None))


@pytest.mark.parametrize("M,N,K", [(256, 512, 256), (200, 328, 136), (96, 96, 64)])
def test_epilogues_match_torch(gpu, M, N, K):
    A, B, As, Bs, lda, ldb = _mk(M, N, K, 0, 0, gpu)
    acc = A.float() @ B.float().t()
    bias = torch.randn(N, device=gpu).to(torch.bfloat16)
    resid = torch.randn(M, N, device=gpu).to(torch.bfloat16)
    aux_in = (torch.rand(M, N, device=gpu) * 2 - 1).to(torch.bfloat16)
    rowvec = torch.randn(M, device=gpu)
    k = 0.7978845608028654
    gelu = lambda u: 0.5 * u * (1 + torch.tanh(k * (u + 0.044715 * u ** 3)))  # noqa: E731

    def dgelu(x):
        t = torch.tanh(k * (x + 0.044715 * x ** 3))
        return 0.5 * (1 + t) + 0.5 * x * (1 - t * t) * k * (1 + 3 * 0.044715 * x * x)
    cases = [
        (dict(act=0, bias=bias, resid=resid, ldres=N, alpha=0.5), 0.5 * acc + bias.float() + resid.float(), None),
        (dict(act=1, bias=bias), torch.tanh(acc + bias.float()), None),
        (dict(act=2, bias=bias), gelu(acc + bias.float()), acc + bias.float()),
        (dict(act=3, aux=aux_in, ldaux=N), acc * (1 - aux_in.float() ** 2), None),
        (dict(act=4, aux=aux_in, ldaux=N), acc * dgelu(aux_in.float()), None),
        (dict(act=5, aux=aux_in, ldaux=N, rowvec=rowvec, alpha=0.25),
         aux_in.float() * (0.25 * acc - 0.25 * rowvec[:, None]), None),
    ]
    for kw, want, want_aux in cases:
        C = torch.zeros(M, N, device=gpu, dtype=torch.bfloat16)
        aux_out = None
        if kw["act"] == 2:
            aux_out = torch.zeros(M, N, device=gpu, dtype=torch.bfloat16)
            kw = dict(kw, aux=aux_out, ldaux=N)
        _ex(As, Bs, C, M, N, K, lda, ldb, N, 0, 0, **kw)
        torch.cuda.synchronize()
        err = (C.float() - want).abs().max().item() / max(want.abs().max().item(), 1e-6)
        assert err < 2e-2, (kw["act"], err)
        if want_aux is not None:
            e2 = (aux_out.float() - want_aux).abs().max().item() / want_aux.abs().max().item()
            assert e2 < 1e-2, e2
    # fp32 assign / accumulate through the TMA reduce-add path
    C = torch.randn(M, N, device=gpu)
    base = C.clone()
    _ex(As, Bs, C, M, N, K, lda, ldb, N, 0, 0, mode=1, out_bf16=0)
    torch.cuda.synchronize()
    assert (C - (base + acc)).abs().max().item() < 1e-3
    _ex(As, Bs, C, M, N, K, lda, ldb, N, 0, 0, mode=2, out_bf16=0)
    torch.cuda.synchronize()
    assert (C - acc).abs().max().item() < 1e-3


def test_f32_tanh_epilogue_is_libm_tanhf(gpu, oracle):
    """The fp32 tier's tanh epilogue (libm_f32.cuh) against the host libm's
    tanhf — what the reference's std::tanh on float calls — bit for bit, on
    every 61st float of [-12, 12] plus the branch edges of the fdlibm
    algorithm (2^-55, 2^-25, ln2/2, 1.5 ln2, 1, 27 ln2, 22).  Through the
    GEMM itself: K = 1, A = 1, so acc = x exactly."""
    import numpy as np
    from paper_2510_20111_b200.engine import gemm_f32
    lo = np.float32(-12.0).view(np.uint32)
    hi = np.float32(12.0).view(np.uint32)
    pos = np.arange(61, int(hi), 61, dtype=np.uint32)  # (x = -0 would reach the epilogue as 0 + -0 = +0)
    edges = np.array([2.0 ** -55, 2.0 ** -25, 0.34657359, 0.5, 1.0, 1.03972077, 18.714973, 22.0, 11.0],
                     dtype=np.float32)
    nb = np.concatenate([edges, np.nextafter(edges, np.float32(0)), np.nextafter(edges, np.float32(30))])
    x = np.concatenate([pos.view(np.float32), nb]).astype(np.float32)
    x = np.concatenate([x, -x, np.zeros(1, np.float32)])
    assert int(lo) & 0x80000000
    want = oracle.tanhf(x)
    n = x.size  # C [1, n] = 1 x B^T, B = x as [n, 1] (the grid spans n along x)
    X = torch.from_numpy(x).to(gpu).view(n, 1)
    one = torch.ones(1, 1, device=gpu)
    Y = torch.empty(1, n, device=gpu)
    gemm_f32(one.data_ptr(), X.data_ptr(), Y.data_ptr(), 1, n, 1, 1, 1, n, 0, 0, 3)
    torch.cuda.synchronize()
    got = Y.view(-1).cpu().numpy()
    bad = np.flatnonzero(got.view(np.uint32) != want.view(np.uint32))
    assert bad.size == 0, (bad.size, x[bad[:4]], got[bad[:4]], want[bad[:4]])
