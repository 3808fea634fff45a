"""Parity of the collective kernels against the oracle (tier A, bitwise).

All dp ranks are emulated on one GPU: the AG / RS / Z1 kernels of the
multi-GPU path run over the same tile tables, with the NVLS primitive
replaced by its unicast model (owner stores to every member's slot; the
reducer sums the members' slots in ascending order, bf16 wire rounded to
bf16 like the switch).  The multi-process path (multimem over NVSwitch) is
covered by tests/test_gpu_multi.py on >= 2 GPUs.

  AG  : slot contents == oracle all_gather of the Z3 group (collective.cpp:44-67)
  RS  : grad shards == 0 + ascending-rank sum (collective.cpp:69-97, train.cpp:313-322);
        bf16 wire: the same sum of the bf16-rounded gradients, rounded to bf16
  Z1  : master/m/v/param shards after the fused replica-reduce + Adam + bf16
        push == oracle train_step_hzp (train.cpp:326-379)
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CONFIGS = [
    # dims, dp, z1, z2, z3
    ([12, 20, 8], 4, 4, 2, 2),      # CPU reference config
    ([12, 20, 8], 4, 2, 2, 2),
    ([12, 20, 8], 8, 8, 4, 4),
    ([12, 20, 8], 8, 2, 4, 8),
    ([12, 20, 8], 8, 4, 8, 2),
    ([64, 128, 64], 8, 8, 4, 4),    # 7B-shaped hierarchy (z3=z2=4, z1=8), aligned
    ([64, 128, 64], 8, 8, 2, 2),    # MoE-shaped (z3=z2=2, z1=8)
    ([64, 128, 64], 8, 8, 8, 8),    # 1.3B-shaped flat ZeRO-3
    ([96, 200, 40], 6, 3, 2, 6),
]


def _ids(c):
    return "{}-dp{}-z{}{}{}".format("x".join(map(str, c[0])), *c[1:])


def _engine(dims, dp, z1, z2, z3, prec, mbs=1, batch=4, **kw):
    from paper_2510_20111_b200 import EngineConfig, HzpEngine, ParallelConfig
    cfg = EngineConfig(model=0, precision=prec, dims=dims, batch=batch, num_microbatches=mbs,
                       par=ParallelConfig(dp=dp, z1=z1, z2=z2, z3=z3), **kw)
    return HzpEngine(cfg)


@pytest.mark.parametrize("prec", [0, 1], ids=["fp32", "bf16"])
@pytest.mark.parametrize("cfg", CONFIGS, ids=_ids)
def test_ag_pull_bitwise(gpu, oracle, cfg, prec):
    dims, dp, z1, z2, z3 = cfg
    st = oracle.shard_init(dims, dp, z1, z2, z3, 2024, bool(prec))
    eng = _engine(dims, dp, z1, z2, z3, prec)
    eng.load_state(st)
    for l, (off, n) in enumerate(eng.layers):
        slot = l % 2
        eng.ag_layer(l, slot)
        for r in range(dp):
            g0 = r - r % z3
            want = oracle.all_gather(st.param[g0:g0 + z3])[off:off + n]
            got = eng.ag_slot(r, slot, n)
            if prec:
                got = (got.astype(np.uint32) << 16).view(np.float32)
            assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (l, r)
    eng.close()


@pytest.mark.parametrize("cfg", [c for c in CONFIGS if c[3] > 1], ids=_ids)
def test_rs_pull_bitwise(gpu, oracle, cfg):
    dims, dp, z1, z2, z3 = cfg
    st = oracle.shard_init(dims, dp, z1, z2, z3, 7, False)
    x = oracle.make_inputs(dims, dp, 2, 4, 7, 0)
    ref = st.copy()
    _, rank_grads = oracle.train_step_hzp(ref, x, 4, False, want_rank_grads=True)
    eng = _engine(dims, dp, z1, z2, z3, 0, mbs=2)
    eng.load_state(st)
    eng.zero_grads()
    want = np.zeros((dp, st.s2), np.float32)
    for mb in range(2):
        for l, (off, n) in enumerate(eng.layers):
            for r in range(dp):
                eng.wgrad_upload(r, l, mb % 2, rank_grads[mb, r, off:off + n])
            eng.rs_layer(l, mb % 2)
        for g0 in range(0, dp, z2):
            seg = oracle.reduce_scatter(rank_grads[mb, g0:g0 + z2])
            for i in range(z2):
                want[g0 + i] = want[g0 + i] + seg[i]
    for r in range(dp):
        got = eng.download(r, 2 - 1)  # F_GRAD
        assert np.array_equal(got.view(np.uint32), want[r].view(np.uint32)), r
    eng.close()


def bf16_rne(o, x):
    return o.bf16_round(np.ascontiguousarray(x, np.float32)).astype(np.float32)


def rs_bf16_model(o, grads):
    """The bf16-wire reduce: each member's gradient rounded to bf16 (the wgrad
    GEMM's bf16 store), summed in fp32 in ascending rank order; in groups of
    >= 3 (in-switch multimem.ld_reduce .acc::f32, which returns bf16) the sum
    is rounded to bf16, in groups of 2 (ordered unicast pull) it stays fp32."""
    w = [bf16_rne(o, g) for g in grads]
    s = w[0].copy()
    for x in w[1:]:
        s = (s + x).astype(np.float32)
    return bf16_rne(o, s) if len(grads) >= 3 else s


@pytest.mark.parametrize("cfg", [c for c in CONFIGS if c[3] > 1], ids=_ids)
def test_rs_bf16_wire_bitwise(gpu, oracle, cfg):
    dims, dp, z1, z2, z3 = cfg
    st = oracle.shard_init(dims, dp, z1, z2, z3, 7, True)
    rng = np.random.default_rng(3)
    eng = _engine(dims, dp, z1, z2, z3, 1, mbs=2)
    eng.load_state(st)
    eng.zero_grads()
    want = np.zeros((dp, st.s2), np.float32)
    for mb in range(2):
        full = rng.standard_normal((dp, st.s2 * z2)).astype(np.float32)
        for l, (off, n) in enumerate(eng.layers):
            for r in range(dp):
                eng.wgrad_upload(r, l, mb % 2, full[r, off:off + n])
            eng.rs_layer(l, mb % 2)
        for g0 in range(0, dp, z2):
            red = rs_bf16_model(oracle, full[g0:g0 + z2])
            for i in range(z2):
                seg = red[i * st.s2:(i + 1) * st.s2]
                want[g0 + i] = (want[g0 + i] + seg).astype(np.float32)
    for r in range(dp):
        got = eng.download(r, 1)
        P = eng.P
        lo = (r % z2) * st.s2
        n_valid = max(0, min(st.s2, P - lo))
        assert np.array_equal(got[:n_valid].view(np.uint32), want[r][:n_valid].view(np.uint32)), r
    eng.close()


@pytest.mark.parametrize("prec", [0, 1], ids=["fp32", "bf16"])
@pytest.mark.parametrize("cfg", CONFIGS, ids=_ids)
def test_z1_adam_push_bitwise(gpu, oracle, cfg, prec):
    """Tier A: feed the oracle's pre-all-reduce Z2 grad shards, run the fused
    Z1 kernel, compare every optimizer state and working-copy shard bitwise."""
    dims, dp, z1, z2, z3 = cfg
    bf16 = bool(prec)
    st = oracle.shard_init(dims, dp, z1, z2, z3, 11, bf16)
    eng = _engine(dims, dp, z1, z2, z3, prec, mbs=2)
    for step in range(3):
        x = oracle.make_inputs(dims, dp, 2, 4, 11, step)
        pre = st.copy()
        _, rank_grads = oracle.train_step_hzp(st, x, 4, bf16, want_rank_grads=True)
        # the Z2 shards as they stand before the DZP all-reduce (train.cpp:306-323)
        shards = np.zeros((dp, st.s2), np.float32)
        for mb in range(2):
            for g0 in range(0, dp, z2):
                seg = oracle.reduce_scatter(rank_grads[mb, g0:g0 + z2])
                for i in range(z2):
                    shards[g0 + i] = shards[g0 + i] + seg[i]
        pre.grad = shards
        eng.load_state(pre)
        eng.z1_adam_step()
        for r in range(dp):
            for f, name in ((2, "master"), (3, "mom"), (4, "var")):
                got = eng.download(r, f)
                assert np.array_equal(got.view(np.uint32), getattr(st, name)[r].view(np.uint32)), (step, r, name)
            got = eng.param_f32(r)
            assert np.array_equal(got.view(np.uint32), st.param[r].view(np.uint32)), (step, r, "param")
    eng.close()
