"""Mixture-of-experts GPT block (BASELINE configs[3] family) on the engine vs
a plain PyTorch fp32 reference of the same network: top-k router with
renormalised gates, GELU experts, capacity large enough that no token is
dropped.  One dp=1 step leaves the full fp32 gradient in the grad shard; it
must match autograd (through the gates) on the same bf16 working copy."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CFG = dict(layers=1, hidden=256, heads=2, ffn=512, vocab=512, seq=256, batch=2, experts=8, topk=2)
# SwiGLU experts (BASELINE configs[3]: 16 x SwiGLU): fc1 [2f, h] = gate | up, no biases
CFG_SWIGLU = dict(CFG, ffn=320, swiglu=1)


def layout(c):
    h, f, V, S, L, E = c["hidden"], c["ffn"], c["vocab"], c["seq"], c["layers"], c["experts"]
    blk = [("ln1_g", (h,)), ("ln1_b", (h,)), ("w_qkv", (3 * h, h)), ("b_qkv", (3 * h,)),
           ("w_o", (h, h)), ("b_o", (h,)), ("ln2_g", (h,)), ("ln2_b", (h,)), ("w_router", (E, h))]
    for e in range(E):
        if c.get("swiglu"):
            blk += [(f"e{e}.w_fc1", (2 * f, h)), (f"e{e}.w_fc2", (h, f))]
        else:
            blk += [(f"e{e}.w_fc1", (f, h)), (f"e{e}.b_fc1", (f,)), (f"e{e}.w_fc2", (h, f)), (f"e{e}.b_fc2", (h,))]
    names, off = [], 0
    for n, shp in [("wte", (V, h)), ("wpe", (S, h))]:
        names.append((n, shp, off))
        off += int(np.prod(shp))
    for l in range(L):
        for n, shp in blk:
            names.append((f"{l}.{n}", shp, off))
            off += int(np.prod(shp))
    for n, shp in [("lnf_g", (h,)), ("lnf_b", (h,)), ("w_head", (V, h))]:
        names.append((n, shp, off))
        off += int(np.prod(shp))
    return names, off


def init_params(c, seed=0):
    names, P = layout(c)
    rng = np.random.default_rng(seed)
    p = np.zeros(P, np.float32)
    for n, shp, off in names:
        k = int(np.prod(shp))
        if n.endswith("_g"):
            p[off:off + k] = 1.0
        elif n.endswith("w_router"):
            p[off:off + k] = rng.normal(0, 0.3, k)  # well-separated routing probabilities
        else:
            p[off:off + k] = rng.normal(0, 0.02, k)
    return p


def torch_loss(c, flat, tokens):
    names, _ = layout(c)
    P = {n: flat[off:off + int(np.prod(shp))].view(*shp) for n, shp, off in names}
    h, nh, S, E, K = c["hidden"], c["heads"], c["seq"], c["experts"], c["topk"]
    hd = h // nh
    inp, tgt = tokens[:, :S], tokens[:, 1:]
    x = P["wte"][inp] + P["wpe"][torch.arange(S, device=flat.device)]
    gelu = lambda u: 0.5 * u * (1 + torch.tanh(0.7978845608028654 * (u + 0.044715 * u ** 3)))  # noqa: E731
    for l in range(c["layers"]):
        g = lambda n: P[f"{l}.{n}"]  # noqa: E731
        a = torch.nn.functional.layer_norm(x, (h,), g("ln1_g"), g("ln1_b"), 1e-5)
        qkv = a @ g("w_qkv").t() + g("b_qkv")
        q, k, v = qkv.split(h, dim=-1)
        q, k, v = (t.view(t.shape[0], S, nh, hd).transpose(1, 2) for t in (q, k, v))
        att = (q @ k.transpose(-1, -2)) / math.sqrt(hd)
        mask = torch.triu(torch.ones(S, S, dtype=torch.bool, device=flat.device), 1)
        att = att.masked_fill(mask, float("-inf")).softmax(-1)
        o = (att @ v).transpose(1, 2).reshape(x.shape[0], S, h)
        x = x + o @ g("w_o").t() + g("b_o")
        a = torch.nn.functional.layer_norm(x, (h,), g("ln2_g"), g("ln2_b"), 1e-5)
        a2 = a.reshape(-1, h)
        p = (a2 @ g("w_router").t()).softmax(-1)
        topv, topi = p.topk(K, dim=-1)
        gates = topv / topv.sum(-1, keepdim=True)
        out = torch.zeros_like(a2)
        for e in range(E):
            ti, ki = (topi == e).nonzero(as_tuple=True)
            if ti.numel() == 0:
                continue
            if c.get("swiglu"):
                gate, up = (a2[ti] @ g(f"e{e}.w_fc1").t()).split(c["ffn"], dim=-1)
                y = (torch.nn.functional.silu(gate) * up) @ g(f"e{e}.w_fc2").t()
            else:
                hh = gelu(a2[ti] @ g(f"e{e}.w_fc1").t() + g(f"e{e}.b_fc1"))
                y = hh @ g(f"e{e}.w_fc2").t() + g(f"e{e}.b_fc2")
            out = out.index_add(0, ti, gates[ti, ki, None] * y)
        x = x + out.view_as(x)
    a = torch.nn.functional.layer_norm(x, (h,), P["lnf_g"], P["lnf_b"], 1e-5)
    logits = a @ P["w_head"].t()
    return torch.nn.functional.cross_entropy(logits.reshape(-1, logits.shape[-1]), tgt.reshape(-1))


def _bf16_bits(x):
    u = np.ascontiguousarray(x, np.float32).view(np.uint32)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


@pytest.mark.parametrize("c", [CFG, CFG_SWIGLU], ids=["gelu", "swiglu"])
def test_moe_gradient_matches_torch(gpu, c):
    from paper_2510_20111_b200 import EngineConfig, HzpEngine, ParallelConfig
    T = c["batch"] * c["seq"]
    eng = HzpEngine(EngineConfig(model=1, precision=1, gpt_layers=c["layers"], gpt_hidden=c["hidden"],
                                 gpt_heads=c["heads"], gpt_ffn=c["ffn"], gpt_vocab=c["vocab"],
                                 gpt_seq=c["seq"], batch=c["batch"], num_microbatches=1,
                                 gpt_experts=c["experts"], gpt_topk=c["topk"], gpt_capacity=T,
                                 gpt_swiglu=c.get("swiglu", 0),
                                 par=ParallelConfig()))
    master = init_params(c)
    work = _bf16_bits(master)
    assert eng.P == master.size
    eng.upload(0, 0, work)
    eng.upload(0, 2, master)
    eng.upload(0, 3, np.zeros_like(master))
    eng.upload(0, 4, np.zeros_like(master))
    rng = np.random.default_rng(1)
    tokens = rng.integers(0, c["vocab"], size=(1, 1, c["batch"], c["seq"] + 1), dtype=np.int32)
    loss = eng.step(tokens)[0]
    g_eng = eng.download(0, 1)
    flat = torch.tensor((work.astype(np.uint32) << 16).view(np.float32), device=gpu, requires_grad=True)
    tok = torch.tensor(tokens[0, 0], device=gpu, dtype=torch.long)
    ref = torch_loss(c, flat, tok)
    ref.backward()
    g_ref = flat.grad.cpu().numpy()
    assert abs(loss - ref.item()) / ref.item() < 1e-2, (loss, ref.item())
    names, _ = layout(c)
    errs = {}
    for n, shp, off in names:
        k = int(np.prod(shp))
        a, b = g_eng[off:off + k], g_ref[off:off + k]
        nb = np.linalg.norm(b)
        if nb < 1e-6:  # an expert no token chose: both must be ~0
            assert np.linalg.norm(a) < 1e-4, n
            continue
        errs[n] = float(np.linalg.norm(a - b) / nb)
    print({n: round(e, 4) for n, e in errs.items()})
    # The router gradient goes through the renormalised top-k softmax Jacobian
    # (differences of nearly equal terms) fed by dgate = <dout, y> of bf16
    # expert outputs, and reaches everything upstream through the large router
    # weights (std 0.3 here): bf16 rounding shows up there at the 5-10 % level
    # (measured: GELU f = 320 6.3 %, SwiGLU f = 320 10.6 % on the router, the
    # expert weights 1-4 %), so those get the looser bound.
    tol = 6e-2 if not c.get("swiglu") and c["ffn"] == 512 else 1.2e-1
    bad = {n: e for n, e in errs.items() if e >= tol}
    assert not bad, bad
    eng.close()
