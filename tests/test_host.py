"""Host side of the product (no GPU): the C-ABI library loads, exports every
declared symbol, and its C++ partition/scheduler drop-in reproduces the
reference bit-exactly (tests/golden/{layout,sched}.json were produced by the
reference itself).  Mirrors tests/test_config.cpp, test_memory.cpp and
test_sched.cpp of the reference."""
import ctypes
import os
import re

import pytest

from conftest import ROOT, golden
from oracle import sched_oracle as so

import paper_2510_20111_b200 as hzp
from paper_2510_20111_b200 import _native as N

LAYOUT = golden("layout")
SCHED = golden("sched")


def declared_symbols():
    with open(os.path.join(ROOT, "include", "hzp_b200.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(hzp_[a-z0-9_]+)\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    names = declared_symbols()
    assert len(names) >= 35
    lib = ctypes.CDLL(N.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    bound = {s[0] for s in N.SIGNATURES}
    assert set(names) == bound


def test_version():
    assert b"sm_100a" in N.lib.hzp_version()


def test_groups_match_reference():
    for c in LAYOUT["groups"]:
        g = hzp.build_process_groups(hzp.ParallelConfig(dp=c["dp"], z1=c["z1"], z2=c["z2"], z3=c["z3"]))
        for k in ("Z1", "Z2", "Z3", "DZP"):
            assert g[k] == c[k], (c, k)


def test_shard_elems_match_reference():
    for c in LAYOUT["shard_elems"]:
        assert hzp.shard_elems(c["n"], c["parts"]) == c["s"]


def test_validation_codes_match_reference():
    for c in LAYOUT["validate"]:
        spec = hzp.ModelSpec(num_layers=c["layers"], params_per_layer=c["ppl"])
        topo = hzp.CostModel(num_nodes=1, ranks_per_node=c["dp"])
        cfg = hzp.ParallelConfig(dp=c["dp"], z1=c["z1"], z2=c["z2"], z3=c["z3"])
        if c["code"] == 0:
            hzp.validate_config(spec, cfg, topo)
        else:
            with pytest.raises(hzp.ValidationError) as ei:
                hzp.validate_config(spec, cfg, topo)
            assert ei.value.code == c["code"]


def _graph(case):
    spec = hzp.ModelSpec(num_layers=case["layers"], params_per_layer=case["ppl"],
                         seq_len=case["seq"], num_microbatches=case["num_mb"],
                         flops_per_token_per_layer=case["flops"])
    cfg = hzp.ParallelConfig(dp=case["dp"], z1=case["z1"], z2=case["z2"], z3=case["z3"])
    cost = hzp.CostModel(num_nodes=1, ranks_per_node=case["dp"], intra_bw=case["intra_bw"],
                         inter_bw=case["intra_bw"], intra_latency=case["intra_lat"],
                         device_flops=case["device_flops"])
    return hzp.build_task_graph(spec, cfg, cost, defer_rs=case["defer_rs"])


@pytest.mark.parametrize("case", SCHED["graphs"], ids=lambda c: "L{layers}-M{num_mb}-z{z2}-d{depth}-r{rs_slots}-{defer_rs}-{vanilla}".format(**c))
def test_task_graph_and_simulation_bit_exact(case):
    g = _graph(case)
    assert len(g.tasks) == len(case["tasks"])
    for a, b in zip(g.tasks, case["tasks"]):
        assert (a.kind, a.layer, a.microbatch, a.pass_, a.bytes, a.deps) == \
               (b["kind"], b["layer"], b["mb"], b["pass"], b["bytes"], b["deps"])
    assert [t.duration for t in g.tasks] == case["dur"]
    tl = hzp.simulate(g, case["depth"], case["rs_slots"], hzp.VANILLA if case["vanilla"] else hzp.ASYNC)
    assert tl.start == case["start"] and tl.end == case["end"]
    assert tl.compute_idle == case["summary"]["compute_idle"]
    assert tl.makespan == case["summary"]["makespan"]
    assert tl.compute_busy == case["summary"]["compute_busy"]
    ag, rs = hzp.make_pools(g, case["depth"], case["rs_slots"])
    assert (ag["slot_count"], ag["slot_bytes"]) == (case["summary"]["ag_slot_count"], case["summary"]["ag_slot_bytes"])
    assert (rs["slot_count"], rs["slot_bytes"]) == (case["summary"]["rs_slot_count"], case["summary"]["rs_slot_bytes"])


@pytest.mark.parametrize("case", SCHED["graphs"][::2], ids=lambda c: "L{layers}-M{num_mb}-z{z2}-d{depth}".format(**c))
def test_launch_plan_slots_and_waits(case):
    g = _graph(case)
    plan = hzp.launch_plan(g, case["depth"], case["rs_slots"])
    ref = so.launch_plan(case["tasks"] and [dict(id=i, **t) for i, t in enumerate(case["tasks"])],
                         case["depth"], case["rs_slots"])
    assert [(p.stream, p.slot, p.ring_wait, p.waits) for p in plan] == \
           [(r["stream"], r["slot"], r["ring_wait"], r["waits"]) for r in ref]
    # the ring rule is what makes simulate's AG start times: an AG occupying a
    # recycled slot never starts before its ring_wait task ended
    for p in plan:
        if p.ring_wait >= 0:
            assert case["start"][p.id] >= case["end"][p.ring_wait]
    # every wait refers to an earlier task (issue order soundness)
    for p in plan:
        assert all(w < p.id for w in p.waits)


def test_survey_a2_slots():
    # 2 layers, 2 mb, depth 2 -> AG slots 0,1,0,1,0,1,0,1 | post 0,1
    g = hzp.build_task_graph(hzp.ModelSpec(num_layers=2, params_per_layer=10**6, num_microbatches=2,
                                           flops_per_token_per_layer=6e6, seq_len=1024),
                             hzp.ParallelConfig(dp=8, z1=8, z2=4, z3=4),
                             hzp.CostModel(ranks_per_node=8, intra_bw=1e10, inter_bw=1e10))
    plan = hzp.launch_plan(g, 2, 1)
    assert [p.slot for p in plan if p.kind in (hzp.hzp.AG_PARAM, hzp.hzp.AG_POST_STEP)] == \
           [0, 1, 0, 1, 0, 1, 0, 1, 0, 1]
    assert len(plan) == 25
    assert plan[4].ring_wait == 1  # task 4 reuses slot 0 after task 1 (first consumer of task 0)


def test_census_and_prelaunch_depth():
    # tests/test_sched.cpp:43-56, 121-127
    spec = hzp.ModelSpec(num_layers=4, params_per_layer=10**6, num_microbatches=2, seq_len=1024,
                         flops_per_token_per_layer=6e6)
    g = hzp.build_task_graph(spec, hzp.ParallelConfig(dp=8, z1=8, z2=4, z3=4),
                             hzp.CostModel(ranks_per_node=8, intra_bw=1e10, inter_bw=1e10))
    counts = [g.count(k) for k in range(8)]
    assert counts == [8, 8, 0, 16, 8, 4, 1, 4]
    for c in SCHED["prelaunch_depth"]:
        g8 = hzp.build_task_graph(hzp.ModelSpec(num_layers=c["layers"], params_per_layer=c["ppl"]),
                                  hzp.ParallelConfig(dp=8, z1=8, z2=4, z3=4),
                                  hzp.CostModel(ranks_per_node=8))
        assert hzp.derive_prelaunch_depth(g8, c["budget"]) == c["depth"]


def test_sched_errors():
    spec = hzp.ModelSpec(num_layers=4, params_per_layer=1000)
    cost = hzp.CostModel(ranks_per_node=8)
    with pytest.raises(hzp.SchedError):
        hzp.build_task_graph(spec, hzp.ParallelConfig(dp=8, z1=8, z2=4, z3=4, tp=2), cost)
    with pytest.raises(hzp.SchedError):
        hzp.build_task_graph(spec, hzp.ParallelConfig(dp=8, z1=8, z2=4, z3=4, pp=3), cost)


def test_async_never_worse_than_vanilla():
    # tests/test_sched.cpp:102-119 on the product's simulate
    import random
    rnd = random.Random(101)
    for _ in range(20):
        spec = hzp.ModelSpec(num_layers=1 << rnd.randrange(4), params_per_layer=10**6,
                             num_microbatches=1 + rnd.randrange(4), seq_len=1024,
                             flops_per_token_per_layer=1e6 * (1 + rnd.randrange(100)))
        g = hzp.build_task_graph(spec, hzp.ParallelConfig(dp=8, z1=8, z2=4, z3=4),
                                 hzp.CostModel(ranks_per_node=8, intra_bw=1e10, inter_bw=1e10,
                                               intra_latency=1e-6))
        v = hzp.simulate(g, 2, 1, hzp.VANILLA)
        a = hzp.simulate(g, 2, 1, hzp.ASYNC)
        assert a.compute_idle <= v.compute_idle + 1e-12
        assert a.makespan <= v.makespan + 1e-12
        assert a.compute_busy == v.compute_busy


def test_chrome_trace_matches_reference_format():
    """trace.cpp:33-73 layout: process/thread metadata + one X event per task."""
    from paper_2510_20111_b200 import hzp as H
    from paper_2510_20111_b200.trace import chrome_trace
    g = H.build_task_graph(H.ModelSpec(num_layers=2, params_per_layer=100, num_microbatches=2),
                           H.ParallelConfig(dp=8, z1=8, z2=4, z3=4), H.CostModel())
    tl = H.simulate(g, 2, 1, H.ASYNC)
    tr = chrome_trace(g, tl.start, tl.end, "sim")
    ev = tr["traceEvents"]
    assert ev[0] == {"name": "process_name", "ph": "M", "pid": 1, "tid": 0, "args": {"name": "sim"}}
    assert [e["args"]["name"] for e in ev[1:4]] == ["compute", "all-gather", "reduce-scatter"]
    xs = [e for e in ev if e["ph"] == "X"]
    assert len(xs) == len(g.tasks)
    for t, e in zip(g.tasks, xs):
        assert e["name"] == H.KIND_NAMES[t.kind] and e["args"]["task_id"] == t.id
        assert abs(e["ts"] - tl.start[t.id] * 1e6) < 1e-6 and e["dur"] >= 0
    assert tr["displayTimeUnit"] == "ms"


PIPE = golden("pipeline")


@pytest.mark.parametrize("case", PIPE["graphs"],
                         ids=lambda c: "L{layers}-M{num_mb}-pp{pp}x{vpp}-r{rank}-reuse{reuse}-rc{recompute}-d{defer_rs}".format(**c))
def test_pipeline_reuse_recompute_bit_exact(case):
    """The CLI's graph (hzpsim.cpp:111-127): pipeline order, apply_reuse
    R1/R2/R3 (pipeline.cpp:167-279), recompute_rule (:281-318) — tasks, deps,
    durations, the reuse report and the simulated timeline bit-exact."""
    spec = hzp.ModelSpec(num_layers=case["layers"], params_per_layer=case["ppl"], seq_len=case["seq"],
                         num_microbatches=case["num_mb"], flops_per_token_per_layer=case["flops"])
    cfg = hzp.ParallelConfig(dp=case["dp"], z1=case["z1"], z2=case["z2"], z3=case["z3"], pp=case["pp"],
                             vpp=case["vpp"])
    cost = hzp.CostModel(num_nodes=1, ranks_per_node=case["dp"] * case["pp"], intra_bw=case["intra_bw"],
                         inter_bw=case["intra_bw"], intra_latency=case["intra_lat"],
                         device_flops=case["device_flops"])
    g = hzp.build_task_graph(spec, cfg, cost, defer_rs=case["defer_rs"], rank=case["rank"], pipeline=True,
                             reuse=case["reuse"], recompute=case["recompute"])
    assert [(t.kind, t.layer, t.microbatch, t.pass_, t.bytes, t.deps) for t in g.tasks] == \
           [(b["kind"], b["layer"], b["mb"], b["pass"], b["bytes"], b["deps"]) for b in case["tasks"]]
    assert [t.duration for t in g.tasks] == case["dur"]
    if case["reuse"]:
        for k in ("r1_eliminated_ag", "r2_merged_rs", "r3_eliminated_ag", "extra_cached_bytes"):
            assert g.reuse_report[k] == case["summary"][k], k
    tl = hzp.simulate(g, 2, 1, hzp.ASYNC)
    assert tl.start == case["start"] and tl.end == case["end"]
    assert tl.makespan == case["summary"]["makespan"]
    assert tl.compute_idle == case["summary"]["compute_idle"]


def test_survey_a2_reuse_drops_mb1_forward_ags():
    # with the CLI's reuse at pp=1, R3 removes mb1's forward AGs -> 23 tasks
    g = hzp.build_task_graph(hzp.ModelSpec(num_layers=2, params_per_layer=10**6, num_microbatches=2,
                                           flops_per_token_per_layer=6e6, seq_len=1024),
                             hzp.ParallelConfig(dp=8, z1=8, z2=4, z3=4),
                             hzp.CostModel(ranks_per_node=8, intra_bw=1e10, inter_bw=1e10), reuse=True)
    assert len(g.tasks) == 23
    assert g.reuse_report == {"r1_eliminated_ag": 0, "r2_merged_rs": 0, "r3_eliminated_ag": 2,
                              "extra_cached_bytes": 2 * g.ag_slot_bytes}
    fwd_mb1 = [t for t in g.tasks if t.kind == hzp.hzp.FWD and t.microbatch == 1]
    # each mb1 forward now waits on mb0's forward AG of the same layer
    for t in fwd_mb1:
        ag = g.tasks[t.deps[0]]
        assert (ag.kind, ag.layer, ag.microbatch, ag.pass_) == (hzp.hzp.AG_PARAM, t.layer, 0, 0)


def test_pipeline_order_errors():
    spec = hzp.ModelSpec(num_layers=8, params_per_layer=1000, num_microbatches=3)
    cost = hzp.CostModel(ranks_per_node=8)
    with pytest.raises(N.HzpError):  # interleaved needs microbatches % pp == 0
        hzp.build_task_graph(spec, hzp.ParallelConfig(dp=4, z1=4, z2=2, z3=2, pp=2, vpp=2), cost, pipeline=True)


def test_seeded_span_and_tokens_follow_the_reference_streams(oracle):
    """Product-side seeded_uniform (train.cpp:17-27) and run_case token stream
    (train.cpp:506-507) vs the oracle's restatement, which is pinned to the
    reference (tests/test_oracle.py)."""
    import numpy as np
    from paper_2510_20111_b200.engine import make_tokens, seeded_span
    ref = oracle.seeded_uniform(5000, 2024, np.float32)
    assert np.array_equal(seeded_span(2024, 5000, 0, 5000), ref)
    got = seeded_span(2024, 4321, 1234, 4000, 0.02)
    assert np.array_equal(got[:4321 - 1234], ref[1234:4321] * np.float32(0.02))
    assert not got[4321 - 1234:].any()  # the zero padding past P
    for step, rank, mb in ((0, 0, 0), (3, 5, 1), (9, 2, 3)):
        u = oracle.seeded_uniform(777, oracle.batch_seed(2024, step, rank, mb), np.float64) + 0.5
        assert np.array_equal(make_tokens(2024, step, rank, mb, 777, 50304),
                              np.floor(u * 50304).astype(np.int32))
