"""GPT decoder on the engine vs a plain PyTorch fp32 reference of the same
network (the reference repo has no transformer, so this is the numerics
oracle for the GPU-scale model).  One engine step at dp=1 leaves the full
fp32 gradient in the grad shard; it must match autograd through the
fp32 torch model evaluated on the same bf16 working copy."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CFG = dict(layers=2, hidden=256, heads=2, ffn=1024, vocab=512, seq=256, batch=2)
# the 1.3B block width: CTA-pair GEMMs (incl. split tail waves), the h = 2048
# register-resident LayerNorm kernels, two-tile attention, bias column sums
CFG_WIDE = dict(layers=1, hidden=2048, heads=16, ffn=8192, vocab=1024, seq=512, batch=2)
# the bench's exact shapes (BASELINE configs[1]): S = 2048, 16 heads, b = 4
# sequences per microbatch, the 50304-way head / cross-entropy
CFG_BENCH = dict(layers=1, hidden=2048, heads=16, ffn=8192, vocab=50304, seq=2048, batch=4)


# SwiGLU FFN (BASELINE configs[2] / [3]): fc1 [2f, h] = gate | up, no FFN biases
# the 7B width (h = 4096: the fused LayerNorm backward's two-vector path, the
# two-warp LayerNorm rows), GELU FFN so the b_fc2 hand-over is exercised
CFG_H4096 = dict(layers=2, hidden=4096, heads=32, ffn=1024, vocab=512, seq=256, batch=1)
CFG_SWIGLU = dict(layers=2, hidden=256, heads=2, ffn=704, vocab=512, seq=256, batch=2, swiglu=1)


def layout(c):
    h, f, V, S, L = c["hidden"], c["ffn"], c["vocab"], c["seq"], c["layers"]
    blk = [("ln1_g", (h,)), ("ln1_b", (h,)), ("w_qkv", (3 * h, h)), ("b_qkv", (3 * h,)),
           ("w_o", (h, h)), ("b_o", (h,)), ("ln2_g", (h,)), ("ln2_b", (h,))]
    if c.get("swiglu"):
        blk += [("w_fc1", (2 * f, h)), ("w_fc2", (h, f))]
    else:
        blk += [("w_fc1", (f, h)), ("b_fc1", (f,)), ("w_fc2", (h, f)), ("b_fc2", (h,))]
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
        elif n.split(".")[-1].startswith("b_") or n.endswith("_b"):
            p[off:off + k] = rng.normal(0, 0.02, k)
        else:
            p[off:off + k] = rng.normal(0, 0.02, k)
    return p


def torch_loss(c, flat, tokens):
    names, _ = layout(c)
    P = {n: flat[off:off + int(np.prod(shp))].view(*shp) for n, shp, off in names}
    h, nh, S = c["hidden"], c["heads"], c["seq"]
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
        if c.get("swiglu"):
            gate, up = (a @ g("w_fc1").t()).split(c["ffn"], dim=-1)
            x = x + (torch.nn.functional.silu(gate) * up) @ g("w_fc2").t()
        else:
            x = x + gelu(a @ g("w_fc1").t() + g("b_fc1")) @ g("w_fc2").t() + g("b_fc2")
    a = torch.nn.functional.layer_norm(x, (h,), P["lnf_g"], P["lnf_b"], 1e-5)
    logits = a @ P["w_head"].t()
    return torch.nn.functional.cross_entropy(logits.reshape(-1, logits.shape[-1]), tgt.reshape(-1))


def _engine(c, dp=1, z=(1, 1, 1), mbs=1, **kw):
    from paper_2510_20111_b200 import EngineConfig, HzpEngine, ParallelConfig
    return HzpEngine(EngineConfig(model=1, precision=1, gpt_layers=c["layers"], gpt_hidden=c["hidden"],
                                  gpt_heads=c["heads"], gpt_ffn=c["ffn"], gpt_vocab=c["vocab"],
                                  gpt_seq=c["seq"], batch=c["batch"], num_microbatches=mbs,
                                  gpt_swiglu=c.get("swiglu", 0),
                                  par=ParallelConfig(dp=dp, z1=z[0], z2=z[1], z3=z[2]), **kw))


def _bf16_bits(x):
    return (np.ascontiguousarray(x, np.float32).view(np.uint32) + 0x7FFF +
            ((np.ascontiguousarray(x, np.float32).view(np.uint32) >> 16) & 1) >> 16).astype(np.uint16)


@pytest.mark.parametrize("c", [CFG, CFG_WIDE, CFG_BENCH, CFG_SWIGLU, CFG_H4096],
                         ids=["small", "wide", "bench", "swiglu", "h4096"])
def test_gpt_gradient_matches_torch(gpu, c):
    eng = _engine(c)
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
    for n, shp, off in names:
        k = int(np.prod(shp))
        a, b = g_eng[off:off + k], g_ref[off:off + k]
        err = np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-12)
        assert err < 5e-2, (n, err)
    eng.close()


def test_gpt_emulated_dp_matches_single_rank(gpu):
    """dp=2 hierarchical (z1=2, z2=2, z3=2) emulated on one GPU, each rank its
    own batch, vs dp=1 with 2 microbatches on the same two batches: both sum
    the same gradients, so the Adam step must agree (bf16 tolerance)."""
    c = dict(CFG, layers=1)
    master = init_params(c, 3)
    work = _bf16_bits(master)
    rng = np.random.default_rng(2)
    tok = rng.integers(0, c["vocab"], size=(2, c["batch"], c["seq"] + 1), dtype=np.int32)
    e1 = _engine(c, mbs=2)
    e1.upload(0, 0, work)
    e1.upload(0, 2, master)
    for f in (3, 4):
        e1.upload(0, f, np.zeros_like(master))
    e1.step(tok[None])  # [local=1][mb=2][b][S+1]
    p1 = e1.param_f32(0)
    e2 = _engine(c, dp=2, z=(2, 2, 2))
    s1, s3 = e2.s1, e2.s3
    for r in range(2):
        w = np.zeros(s3 * 2, np.uint16)
        w[:work.size] = work
        e2.upload(r, 0, w[r * s3:(r + 1) * s3])
        m = np.zeros(s1 * 2, np.float32)
        m[:master.size] = master
        e2.upload(r, 2, m[r * s1:(r + 1) * s1])
        for f in (3, 4):
            e2.upload(r, f, np.zeros(s1, np.float32))
    e2.step(tok[:, None])  # [local=2][mb=1][b][S+1]
    p2 = np.concatenate([e2.param_f32(0), e2.param_f32(1)])[:master.size]
    d = np.abs(p1 - p2)
    # Adam moves every element by ~lr; only near-zero gradients (sign decided
    # by bf16-wire rounding) may land on the other side
    assert np.max(d) <= 2.5e-3 and np.mean(d > 1e-3) < 1e-2, (np.max(d), np.mean(d > 1e-3))
    e1.close()
    e2.close()


@pytest.mark.parametrize("experts", [0, 8], ids=["dense", "moe"])
def test_gpt_reuse_and_recompute_are_bitwise_neutral(gpu, experts):
    """§8(f)-3 on the GPT engine: the CLI's reuse (R3: microbatch 1's forward
    reads microbatch 0's gathered blocks from the side cache) and activation
    recomputation (recompute_rule: one shared activation set, rebuilt by a
    FWD-recompute before each BWD) change where data lives and what is
    recomputed, never the arithmetic — losses and updated parameters are
    bitwise those of the plain schedule.  dp=2 emulated (z3 = 2: real AGs)."""
    c = dict(CFG, layers=3)
    rng = np.random.default_rng(5)
    tok = rng.integers(0, c["vocab"], size=(2, 2, c["batch"], c["seq"] + 1), dtype=np.int32)
    out = {}
    for reuse, rc in ((0, 0), (1, 0), (0, 1), (1, 1)):
        e = _engine(c, dp=2, z=(2, 2, 2), mbs=2, reuse=reuse, recompute=rc, gpt_experts=experts)
        e.init_random(seed=11, scale=0.04)
        losses = [np.asarray(e.step(tok)) for _ in range(2)]
        out[(reuse, rc)] = (losses, [e.param_f32(r) for r in range(2)])
        if rc:
            assert sum(1 for r in e.launch_log() if r[1] == 2) > 0  # FWD-recompute tasks ran
        e.close()
    base_l, base_p = out[(0, 0)]
    for k, (l, p) in out.items():
        for a, b in zip(l, base_l):
            assert np.array_equal(a, b), k
        for a, b in zip(p, base_p):
            assert np.array_equal(a, b), k
