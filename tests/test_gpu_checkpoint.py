"""ShardedState checkpoint round trip and measured Chrome trace (SURVEY
§8(f)-4).  Saving after k steps, restoring into a fresh ctx and stepping
must reproduce the uninterrupted run bit for bit (fp32 tier: every kernel
on that path is deterministic)."""
import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DIMS, DP, Z, MBS, BATCH = [12, 20, 8], 4, (4, 2, 2), 2, 4


def _engine(timeline=0, precision=0):
    from paper_2510_20111_b200 import EngineConfig, HzpEngine, ParallelConfig
    return HzpEngine(EngineConfig(model=0, precision=precision, dims=DIMS, batch=BATCH, num_microbatches=MBS,
                                  par=ParallelConfig(dp=DP, z1=Z[0], z2=Z[1], z3=Z[2]), timeline=timeline))


def test_checkpoint_round_trip_is_bitwise(gpu, oracle, tmp_path):
    st = oracle.shard_init(DIMS, DP, *Z, 2024, False)
    a = _engine()
    a.load_state(st)
    for step in range(3):
        a.step(oracle.make_inputs(DIMS, DP, MBS, BATCH, 2024, step))
    a.save_checkpoint(str(tmp_path))
    x = oracle.make_inputs(DIMS, DP, MBS, BATCH, 2024, 3)
    la = a.step(x)
    b = _engine()
    b.load_checkpoint(str(tmp_path))
    assert [b.get_step(r) for r in range(DP)] == [3] * DP
    lb = b.step(x)
    assert np.array_equal(np.asarray(la), np.asarray(lb))
    for r in range(DP):
        for f in range(5):
            assert np.array_equal(a.download(r, f), b.download(r, f)), (r, f)
    a.close()
    b.close()


def test_checkpoint_rejects_other_precision(gpu, oracle, tmp_path):
    """A bf16 checkpoint (param = uint16 bit patterns) must not load into an
    fp32 ctx (same element count) and vice versa."""
    st = oracle.shard_init(DIMS, DP, *Z, 2024, True)
    a = _engine(precision=1)
    a.load_state(st)
    a.save_checkpoint(str(tmp_path))
    b = _engine(precision=0)
    with pytest.raises(ValueError, match="precision"):
        b.load_checkpoint(str(tmp_path))
    a.close()
    b.close()


def test_measured_chrome_trace(gpu, oracle, tmp_path):
    from paper_2510_20111_b200 import hzp as H
    from paper_2510_20111_b200.trace import measured_trace
    st = oracle.shard_init(DIMS, DP, *Z, 2024, False)
    e = _engine(timeline=1)
    e.load_state(st)
    e.step(oracle.make_inputs(DIMS, DP, MBS, BATCH, 2024, 0))
    g = H.build_task_graph(H.ModelSpec(num_layers=len(DIMS) - 1, params_per_layer=1, num_microbatches=MBS),
                           H.ParallelConfig(dp=DP, z1=Z[0], z2=Z[1], z3=Z[2]), H.CostModel())
    tr = measured_trace(e, g)
    xs = [v for v in tr["traceEvents"] if v["ph"] == "X"]
    assert len(xs) == len(g.tasks)
    assert all(v["dur"] >= 0 and v["ts"] >= 0 for v in xs)
    (tmp_path / "t.json").write_text(json.dumps(tr))
    e.close()
