"""AG / RS / fused Z1 on the REAL 1.3B layer table (BASELINE configs[1]
dims: h 2048, ffn 8192, vocab 50304, seq 2048), truncated to 3 decoder
blocks so four emulated dp ranks fit one GPU: the embedding layer
(wte + wpe, 107.2 M elements), 50.4 M-element blocks, the 103 M-element
head, layers that straddle Z3 shard boundaries, single-owner spans.

  AG : every rank's slot == the oracle all_gather of the Z3 group, bitwise
       (collective.cpp:44-67);
  RS : bf16 wire, every rank's grad shard == the ordered fp32 sum of the
       members' bf16 gradients, rounded to bf16 (the switch's result), bitwise;
  Z1 : master / m / v / param shards after the fused replica reduce + Adam +
       bf16 push == oracle adam_update (train.cpp:171-189) on the ordered
       replica sum (collective.cpp:99-115), bitwise.
"""
import numpy as np
import pytest

from test_gpu_comm import bf16_rne, rs_bf16_model

pytestmark = pytest.mark.gpu

C3 = dict(layers=3, hidden=2048, heads=16, ffn=8192, vocab=50304, seq=2048, batch=1)


def _engine(dp, z):
    from paper_2510_20111_b200 import EngineConfig, HzpEngine, ParallelConfig
    c = C3
    return HzpEngine(EngineConfig(model=1, precision=1, gpt_layers=c["layers"], gpt_hidden=c["hidden"],
                                  gpt_heads=c["heads"], gpt_ffn=c["ffn"], gpt_vocab=c["vocab"],
                                  gpt_seq=c["seq"], batch=c["batch"], num_microbatches=1,
                                  par=ParallelConfig(dp=dp, z1=z[0], z2=z[1], z3=z[2])))


# (dp, (z1, z2, z3)): flat ZeRO-3 (1.3B), hierarchical with 2 DZP replicas
# (7B-shaped), and dp = 3 (shard boundaries not 16-byte aligned)
LAYOUTS = [(4, (4, 4, 4)), (4, (4, 2, 2)), (3, (3, 3, 3))]


@pytest.mark.parametrize("dp,z", LAYOUTS, ids=lambda v: str(v))
def test_ag_rs_z1_on_13b_layer_table(gpu, oracle, dp, z):
    z1, z2, z3 = z
    eng = _engine(dp, z)
    P, s1, s2, s3 = eng.P, eng.s1, eng.s2, eng.s3
    sizes = [n for _, n in eng.layers]
    assert max(sizes) > 100_000_000 and min(sizes[1:-1]) > 50_000_000
    rng = np.random.default_rng(7)
    master = np.zeros(s1 * z1, np.float32)
    master[:P] = (rng.random(P, dtype=np.float32) - 0.5) * 0.04
    work = bf16_rne(oracle, master)  # bf16-valued working copy
    wbits = (work.view(np.uint32) >> 16).astype(np.uint16)
    wpad = np.zeros(s3 * z3, np.uint16)
    wpad[:P] = wbits[:P]
    for r in range(dp):
        eng.upload(r, 0, wpad[(r % z3) * s3:(r % z3 + 1) * s3])
        eng.upload(r, 2, master[(r % z1) * s1:(r % z1 + 1) * s1])
        eng.upload(r, 3, np.zeros(s1, np.float32))
        eng.upload(r, 4, np.zeros(s1, np.float32))
        eng.set_step(r, 0)
    # ---- AG: every layer, every rank's slot ----
    for l, (off, n) in enumerate(eng.layers):
        slot = l % 2
        eng.ag_layer(l, slot)
        for r in range(dp):
            assert np.array_equal(eng.ag_slot(r, slot, n), wpad[off:off + n]), (l, r)
    # ---- RS: blocks 0, 1 and the head (bf16 wire) ----
    eng.zero_grads()
    want = np.zeros((dp, s2), np.float32)
    for l in (1, 2, len(sizes) - 1):
        off, n = eng.layers[l]
        g = rng.standard_normal((dp, n), dtype=np.float32)
        for r in range(dp):
            eng.wgrad_upload(r, l, 0, g[r])
        eng.rs_layer(l, 0)
        for g0 in range(0, dp, z2):
            red = rs_bf16_model(oracle, g[g0:g0 + z2])
            for r in range(g0, g0 + z2):
                lo, hi = max(off, (r % z2) * s2), min(off + n, (r % z2 + 1) * s2)
                if lo < hi:
                    want[r, lo - (r % z2) * s2:hi - (r % z2) * s2] = red[lo - off:hi - off]
        del g
    for r in range(dp):
        assert np.array_equal(eng.download(r, 1).view(np.uint32), want[r].view(np.uint32)), r
    # ---- Z1: replica reduce + Adam + bf16 push, from random Z2 grad shards ----
    grads = rng.standard_normal((dp, s2), dtype=np.float32) * 1e-3
    for r in range(dp):
        eng.upload(r, 1, grads[r])
    eng.z1_adam_step()
    newp = np.zeros(s1 * z1, np.float32)
    # the flat gradient summed over the DZP replicas in ascending order: element
    # e of replica b lives on rank b * z2 + e // s2
    full = np.stack([np.concatenate([grads[b * z2 + j] for j in range(z2)]) for b in range(dp // z2)])
    gall = oracle.all_reduce(full)
    del full
    for r in range(dp):
        e0 = (r % z1) * s1
        gsum = np.ascontiguousarray(gall[e0:e0 + s1])
        m = master[e0:e0 + s1].copy()
        mo = np.zeros(s1, np.float32)
        va = np.zeros(s1, np.float32)
        oracle.adam_update(m, mo, va, gsum, 1)
        m[max(0, P - e0):] = 0.0  # padding stays 0 (kernels skip [P, s*z))
        assert np.array_equal(eng.download(r, 2).view(np.uint32), m.view(np.uint32)), (r, "master")
        assert np.array_equal(eng.download(r, 3)[:max(0, min(s1, P - e0))].view(np.uint32),
                              mo[:max(0, min(s1, P - e0))].view(np.uint32)), (r, "m")
        newp[e0:e0 + s1] = m
    pbits = (bf16_rne(oracle, newp).view(np.uint32) >> 16).astype(np.uint16)
    ppad = np.zeros(s3 * z3, np.uint16)
    ppad[:P] = pbits[:P]
    for r in range(dp):
        got = eng.download(r, 0)
        assert np.array_equal(got, ppad[(r % z3) * s3:(r % z3 + 1) * s3]), (r, "param")
    eng.close()
