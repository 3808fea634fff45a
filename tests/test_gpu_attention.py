"""Fused tcgen05 causal attention (head dim 128) vs a PyTorch fp32 reference:
forward O and lse, backward dQ / dK / dV, through the C-ABI."""
import ctypes as C
import math

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _ref(q, k, v, do):
    S = q.shape[2]
    q, k, v = (t.float().requires_grad_(True) for t in (q, k, v))
    att = (q @ k.transpose(-1, -2)) / math.sqrt(q.shape[-1])
    mask = torch.triu(torch.ones(S, S, dtype=torch.bool, device=q.device), 1)
    att = att.masked_fill(mask, float("-inf"))
    lse = torch.logsumexp(att, -1)
    o = att.softmax(-1) @ v
    o.backward(do.float())
    return o.detach(), lse.detach(), q.grad, k.grad, v.grad


# (4, 16, 2048) is the bench shape (1.3B config: b = 4 sequences per microbatch,
# 16 heads, S = 2048): the LPT-ordered two-tile forward and the full backward grid
@pytest.mark.parametrize("legacy", [False, True], ids=["dq-tmem", "dq-gemm"])
@pytest.mark.parametrize("b,nh,S", [(1, 1, 128), (2, 2, 256), (1, 4, 512), (2, 1, 1024), (4, 16, 2048)])
def test_fused_attention_fwd_bwd(gpu, b, nh, S, legacy):
    from paper_2510_20111_b200 import _native as N
    hd, h = 128, 128 * nh
    g = torch.Generator(device="cpu").manual_seed(b * 100 + nh * 10 + S)
    qkv = (torch.randn(b, S, 3 * h, generator=g) * 0.5).to(gpu, torch.bfloat16)
    do = (torch.randn(b, S, h, generator=g) * 0.1).to(gpu, torch.bfloat16)
    O = torch.zeros(b, S, h, device=gpu, dtype=torch.bfloat16)
    lse = torch.zeros(b * nh, S, device=gpu)
    p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    N.check(N.lib.hzp_attention_fwd(p(qkv), p(O), p(lse), b, nh, S, h, None))
    D = torch.zeros(2, b * nh, S, device=gpu)  # backward workspace (per-query vectors)
    dqkv = torch.zeros(b, S, 3 * h, device=gpu, dtype=torch.bfloat16)
    # dQ recomputed in TMEM (production, dsT = NULL) and the legacy dS^T + GEMM path
    dsT = torch.zeros(b * nh, S, S, device=gpu, dtype=torch.bfloat16) if legacy else None
    N.check(N.lib.hzp_attention_bwd(p(qkv), p(O), p(do), p(lse), p(D), p(dqkv),
                                    p(dsT) if legacy else None, b, nh, S, h, None))
    torch.cuda.synchronize()
    split = lambda t: t.view(b, S, nh, hd).transpose(1, 2)  # noqa: E731
    q, k, v = (split(t) for t in qkv.split(h, dim=-1))
    o_ref, lse_ref, dq, dk, dv = _ref(q, k, v, split(do))
    rel = lambda a, r: ((a.float() - r).norm() / r.norm()).item()  # noqa: E731
    assert rel(split(O), o_ref) < 1e-2
    assert (lse.view(b, nh, S) - lse_ref).abs().max().item() < 2e-2
    gq, gk, gv = (split(t) for t in dqkv.split(h, dim=-1))
    assert rel(gv, dv) < 2e-2
    assert rel(gk, dk) < 2e-2
    assert rel(gq, dq) < 2e-2
