"""Full train_step_hzp on the device vs the oracle (SURVEY §7.4 tiers B/C),
plus launch-order / slot parity of the executor against the LaunchPlan.

fp32 engine: ordered fp32 GEMMs (the reference's summation order) and the
  host libm's tanhf restated on the device — params, optimizer state and
  losses bitwise equal to the oracle after N steps.
bf16 engine: tcgen05 bf16 GEMMs with fp32 accumulation vs the reference's
  mixed mode — within 1e-2 relative.
"""
import numpy as np
import pytest

from paper_2510_20111_b200 import hzp as H

pytestmark = pytest.mark.gpu

STEP_CONFIGS = [
    # dims, dp, z1, z2, z3, mbs, batch, steps
    ([12, 20, 8], 4, 4, 2, 2, 1, 4, 10),   # the CPU reference config
    ([12, 20, 8], 4, 4, 2, 2, 2, 4, 10),
    ([12, 20, 8], 8, 8, 4, 4, 2, 4, 5),
    ([12, 20, 8], 8, 2, 4, 8, 1, 4, 5),
    ([12, 20, 8], 1, 1, 1, 1, 2, 4, 5),
    ([64, 128, 128, 64], 8, 8, 2, 2, 2, 16, 5),
    ([64, 128, 64], 8, 8, 8, 8, 1, 32, 5),
    # ragged / degenerate shards: P = 8 over 8 ranks (1-element Z1 chunks),
    # P = 23 (padding in the last Z3 / Z1 shards), a layer smaller than a shard
    ([3, 2], 8, 8, 4, 4, 1, 2, 3),
    ([5, 3, 2], 4, 4, 2, 2, 2, 3, 3),
    ([1, 1], 2, 2, 2, 2, 1, 1, 3),
    # SURVEY §8(d)-2 parity size: {256, 1024, 256}, B = 8 rows per microbatch,
    # dp = 4 with the CPU config's hierarchy and flat; multi-tile tcgen05 GEMMs
    ([256, 1024, 256], 4, 4, 2, 2, 2, 8, 3),
    ([256, 1024, 256], 4, 4, 4, 4, 2, 8, 3),
]


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


def _run(oracle, cfg, prec, mode=1, timeline=0, reuse=0):
    from paper_2510_20111_b200 import EngineConfig, HzpEngine, ParallelConfig
    dims, dp, z1, z2, z3, mbs, batch, steps = cfg
    bf16 = bool(prec)
    st = oracle.shard_init(dims, dp, z1, z2, z3, 2024, bf16)
    eng = HzpEngine(EngineConfig(model=0, precision=prec, dims=dims, batch=batch,
                                 num_microbatches=mbs, par=ParallelConfig(dp=dp, z1=z1, z2=z2, z3=z3),
                                 mode=mode, timeline=timeline, reuse=reuse))
    eng.load_state(st)
    for step in range(steps):
        x = oracle.make_inputs(dims, dp, mbs, batch, 2024, step)
        ref_losses, _ = oracle.train_step_hzp(st, x, batch, bf16)
        losses = eng.step(x)
    return eng, st, losses, ref_losses


@pytest.mark.parametrize("cfg", STEP_CONFIGS, ids=lambda c: "{}-dp{}-z{}{}{}-mb{}".format("x".join(map(str, c[0])), *c[1:6]))
def test_fp32_step_matches_oracle(gpu, oracle, cfg):
    """Bitwise: ordered fp32 GEMMs, the libm tanhf restatement, ordered
    reductions and the reference's Adam expression order leave no rounding
    difference (the reference's own fp32 check allows 1e-6 absolute,
    train.cpp:519-531)."""
    eng, st, losses, ref_losses = _run(oracle, cfg, 0)
    dp = cfg[1]
    for r in range(dp):
        for got, want in ((eng.param_f32(r), st.param[r]), (eng.download(r, 2), st.master[r]),
                          (eng.download(r, 3), st.mom[r]), (eng.download(r, 4), st.var[r])):
            assert np.array_equal(np.asarray(got, np.float32), np.asarray(want, np.float32)), (r, rel(got, want))
    assert np.array_equal(np.asarray(losses, np.float32), np.asarray(ref_losses, np.float32)), rel(losses, ref_losses)
    eng.close()


@pytest.mark.parametrize("cfg", STEP_CONFIGS, ids=lambda c: "{}-dp{}-z{}{}{}-mb{}".format("x".join(map(str, c[0])), *c[1:6]))
def test_bf16_step_matches_oracle_mixed(gpu, oracle, cfg):
    eng, st, losses, ref_losses = _run(oracle, cfg, 1)
    for r in range(cfg[1]):
        assert rel(eng.param_f32(r), st.param[r]) <= 1e-2, r
        assert rel(eng.download(r, 2), st.master[r]) <= 1e-2, r
    assert rel(losses, ref_losses) <= 1e-2
    eng.close()


@pytest.mark.parametrize("mode", [1, 0], ids=["async", "vanilla"])
def test_launch_log_follows_plan(gpu, oracle, mode):
    cfg = ([64, 128, 64], 8, 8, 4, 4, 2, 16, 1)
    eng, st, _, _ = _run(oracle, cfg, 1, mode=mode, timeline=1)
    log = eng.launch_log()
    g = H.build_task_graph(H.ModelSpec(num_layers=2, params_per_layer=1, num_microbatches=2),
                           H.ParallelConfig(dp=8, z1=8, z2=4, z3=4), H.CostModel(ranks_per_node=8))
    plan = H.launch_plan(g, 2, 1)
    assert [r[0] for r in log] == [p.id for p in plan]           # issue order == task-id order
    assert [r[1] for r in log] == [p.kind for p in plan]
    assert [r[5] for r in log] == [p.slot for p in plan]          # ring slots bit-exact
    fused = [r for r in log if r[1] == H.OPT_STEP][0]
    # async: each layer's Z1 (covering AR-dzp(l)) ran on the RS stream right
    # after the layer's last RS; the OPT record covers OPT + AG-post-step.
    # vanilla: one Z1 at the tail covers AR-dzp, OPT and AG-post-step.
    kinds = (H.AG_POST_STEP,) if mode == 1 else (H.AR_DZP, H.AG_POST_STEP)
    ids = [p.id for p in plan if p.kind in kinds]
    assert (fused[6], fused[7]) == (min(ids + [fused[0]]), max(ids + [fused[0]]))
    for r in log:
        if r[1] == H.AR_DZP:
            assert (r[4], r[6], r[7]) == ((2, r[0], r[0]) if mode == 1 else (-1, fused[0], fused[0]))
    tl = eng.timeline()
    assert tl["makespan_ms"] > 0 and tl["compute_busy_ms"] > 0
    # every task starts after each of its waits ended (device clock)
    for p in plan:
        for w in p.waits:
            assert tl["start_ms"][p.id] >= tl["end_ms"][w] - 1e-3
    eng.close()


REUSE_CONFIGS = [c for c in STEP_CONFIGS if c[5] >= 2] + [([12, 20, 8], 4, 4, 2, 2, 3, 4, 5)]


@pytest.mark.parametrize("cfg", REUSE_CONFIGS, ids=lambda c: "{}-dp{}-z{}{}{}-mb{}".format("x".join(map(str, c[0])), *c[1:6]))
def test_reuse_step_matches_oracle_and_no_reuse(gpu, oracle, cfg):
    """The CLI's apply_reuse (pipeline.cpp:167-279) on the executor: at pp=1 R3
    drops every later forward's AGs and those forwards read microbatch 0's
    gathered layers from the side cache.  Same numbers as the oracle (which
    runs the un-reused step) and bitwise the same as the engine without reuse."""
    eng, st, losses, ref_losses = _run(oracle, cfg, 0, reuse=1)
    base, _, base_losses, _ = _run(oracle, cfg, 0, reuse=0)
    for r in range(cfg[1]):
        assert np.array_equal(eng.param_f32(r), np.asarray(st.param[r], np.float32)), (r, rel(eng.param_f32(r), st.param[r]))
        assert np.array_equal(eng.download(r, 2), np.asarray(st.master[r], np.float32)), r
        assert np.array_equal(eng.param_f32(r), base.param_f32(r)), r
    assert np.array_equal(np.asarray(losses, np.float32), np.asarray(ref_losses, np.float32))
    assert np.array_equal(np.asarray(losses), np.asarray(base_losses))
    eng.close()
    base.close()


def test_reuse_launch_log_follows_reused_plan(gpu, oracle):
    cfg = ([64, 128, 64], 8, 8, 4, 4, 3, 16, 1)
    eng, st, _, _ = _run(oracle, cfg, 1, timeline=1, reuse=1)
    log = eng.launch_log()
    g = H.build_task_graph(H.ModelSpec(num_layers=2, params_per_layer=1, num_microbatches=3),
                           H.ParallelConfig(dp=8, z1=8, z2=4, z3=4), H.CostModel(ranks_per_node=8), reuse=True)
    assert g.reuse_report["r3_eliminated_ag"] == 4
    plan = H.launch_plan(g, 2, 1)
    assert [r[0] for r in log] == [p.id for p in plan]
    assert [r[1] for r in log] == [p.kind for p in plan]
    assert [r[5] for r in log] == [p.slot for p in plan]
    assert sum(1 for r in log if r[1] == H.AG_PARAM) == 2 * 3 * 2 - 4
    tl = eng.timeline()
    for p in plan:
        for w in p.waits:
            assert tl["start_ms"][p.id] >= tl["end_ms"][w] - 1e-3
    eng.close()


@pytest.mark.parametrize("prec", [0, 1], ids=["fp32", "bf16"])
def test_device_seeded_init_is_reference_shard_init(gpu, oracle, prec):
    """hzp_state_init_seeded (scale 1) == the reference's shard_init
    (train.cpp:224-253) bit for bit, every rank and field."""
    from paper_2510_20111_b200 import EngineConfig, HzpEngine, ParallelConfig
    dims, dp, z1, z2, z3 = [64, 128, 72], 8, 8, 4, 2
    st = oracle.shard_init(dims, dp, z1, z2, z3, 2024, bool(prec))
    eng = HzpEngine(EngineConfig(model=0, precision=prec, dims=dims, batch=4,
                                 par=ParallelConfig(dp=dp, z1=z1, z2=z2, z3=z3)))
    eng.init_seeded(2024, 1.0)
    for r in range(dp):
        assert np.array_equal(eng.param_f32(r).view(np.uint32), st.param[r].view(np.uint32)), r
        assert np.array_equal(eng.download(r, 2).view(np.uint32), st.master[r].view(np.uint32)), r
        assert not eng.download(r, 3).any() and not eng.download(r, 1).any()
    eng.close()
