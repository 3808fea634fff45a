"""memory_trace / utilization_report / ledger of the drop-in scheduler
(sched.hpp:139-153, memory.hpp:47; reference sched.cpp:389-477,
memory.cpp:35-45) against values the reference itself produced
(tests/golden/{sched,pipeline}.json, make_golden.py), plus the reference's
own unit cases (tests/test_sched.cpp:141-175) on the product, and the
measured-timeline path (same rules applied to externally supplied times)."""
import pytest

from conftest import golden
from test_host import _graph

import paper_2510_20111_b200 as hzp

SCHED = golden("sched")
PIPE = golden("pipeline")


def _spec(case):
    return hzp.ModelSpec(num_layers=case["layers"], params_per_layer=case["ppl"], seq_len=case["seq"],
                         num_microbatches=case["num_mb"], flops_per_token_per_layer=case["flops"])


def _check(g, case, depth, rs_slots, mode, cfg):
    s = case["summary"]
    led = hzp.ledger(_spec(case), cfg)
    assert led["total_static"] == s["total_static"]
    m = hzp.memory_trace(g, depth, rs_slots, mode, static_bytes=led["total_static"])
    assert m["peak_memory"] == s["peak_memory"]
    assert m["peak_bytes"] == s["peak_bytes"]
    assert m["fragmentation"] == s["fragmentation"]
    assert m["peak_grad_buffer_bytes"] == s["peak_grad_buffer_bytes"]
    assert m["n_samples"] == s["n_samples"]
    t_sum, b_sum = 0.0, 0
    for t, b in m["samples"]:  # same summation order as the shim
        t_sum += t
        b_sum += b
    assert t_sum == s["sample_time_sum"] and b_sum == s["sample_bytes_sum"]
    assert hzp.utilization_report(g, case["device_flops"], depth, rs_slots, mode) == s["utilization"]


@pytest.mark.parametrize("case", SCHED["graphs"],
                         ids=lambda c: "L{layers}-M{num_mb}-z{z2}-d{depth}-r{rs_slots}-{defer_rs}-{vanilla}".format(**c))
def test_memory_trace_bit_exact(case):
    g = _graph(case)
    cfg = hzp.ParallelConfig(dp=case["dp"], z1=case["z1"], z2=case["z2"], z3=case["z3"])
    _check(g, case, case["depth"], case["rs_slots"], hzp.VANILLA if case["vanilla"] else hzp.ASYNC, cfg)


@pytest.mark.parametrize("case", PIPE["graphs"],
                         ids=lambda c: "L{layers}-M{num_mb}-pp{pp}x{vpp}-r{rank}-reuse{reuse}-rc{recompute}".format(**c))
def test_memory_trace_pipeline_graphs_bit_exact(case):
    """Reuse R2 merges RSs away: those BWDs hold their buffer until the
    layer's last RS (sched.cpp:430-444)."""
    cfg = hzp.ParallelConfig(dp=case["dp"], z1=case["z1"], z2=case["z2"], z3=case["z3"], pp=case["pp"],
                             vpp=case["vpp"])
    cost = hzp.CostModel(num_nodes=1, ranks_per_node=case["dp"] * case["pp"], intra_bw=case["intra_bw"],
                         inter_bw=case["intra_bw"], intra_latency=case["intra_lat"],
                         device_flops=case["device_flops"])
    g = hzp.build_task_graph(_spec(case), cfg, cost, defer_rs=case["defer_rs"], rank=case["rank"],
                             pipeline=True, reuse=case["reuse"], recompute=case["recompute"])
    _check(g, case, 2, 1, hzp.ASYNC, cfg)


def _sim_graph(layers, mbs, defer=False):
    # tests/test_sched.cpp sim_model / sim_parallel / sim_cost analogues
    spec = hzp.ModelSpec(num_layers=layers, params_per_layer=10**6, seq_len=1024, num_microbatches=mbs,
                         flops_per_token_per_layer=6e6)
    cfg = hzp.ParallelConfig(dp=8, z1=8, z2=4, z3=4)
    cost = hzp.CostModel(num_nodes=1, ranks_per_node=8, intra_bw=1e10, inter_bw=1e10, intra_latency=1e-6,
                         device_flops=1e12)
    return spec, cfg, hzp.build_task_graph(spec, cfg, cost, defer_rs=defer)


def test_deferred_rs_holds_more_gradient_memory():
    # tests/test_sched.cpp:141-159
    spec, cfg, gi = _sim_graph(8, 2)
    _, _, gd = _sim_graph(8, 2, defer=True)
    st = hzp.ledger(spec, cfg)["total_static"]
    mi = hzp.memory_trace(gi, 2, 1, hzp.ASYNC, st)
    md = hzp.memory_trace(gd, 2, 1, hzp.ASYNC, st)
    assert mi["peak_grad_buffer_bytes"] < md["peak_grad_buffer_bytes"]


def test_steady_state_fragmentation_is_zero():
    # tests/test_sched.cpp:161-169
    spec, cfg, g = _sim_graph(8, 4)
    assert hzp.memory_trace(g, 2, 1, hzp.ASYNC, hzp.ledger(spec, cfg)["total_static"])["fragmentation"] == 0.0


def test_utilization_positive_and_bounded():
    # tests/test_sched.cpp:171-178
    _, _, g = _sim_graph(8, 4)
    u = hzp.utilization_report(g, 1e12)
    assert 0.0 < u <= 1.0


def test_ledger_matches_formula():
    # memory.cpp:35-45: 2N/z3 + 4N/z2 + 12N/z1 (ceil shards)
    spec = hzp.ModelSpec(num_layers=3, params_per_layer=1001, embedding_params=7)
    led = hzp.ledger(spec, hzp.ParallelConfig(dp=8, z1=8, z2=4, z3=2))
    n = 3 * 1001 + 7
    s = lambda z: -(-n // z)  # noqa: E731
    assert led["params_bf16"] == 2 * s(2) and led["grads_fp32"] == 4 * s(4)
    assert led["replica_fp32"] == led["momentum_fp32"] == led["variance_fp32"] == 4 * s(8)
    assert led["total_static"] == 2 * s(2) + 4 * s(4) + 12 * s(8)


@pytest.mark.parametrize("case", SCHED["graphs"][::3],
                         ids=lambda c: "L{layers}-M{num_mb}-z{z2}-d{depth}".format(**c))
def test_measured_path_reproduces_simulated(case):
    """Feeding simulate's own start / end times through the measured-timeline
    path gives the same trace (the rules are shared, only the times differ)."""
    g = _graph(case)
    mode = hzp.VANILLA if case["vanilla"] else hzp.ASYNC
    a = hzp.memory_trace(g, case["depth"], case["rs_slots"], mode, 5)
    b = hzp.memory_trace(g, case["depth"], case["rs_slots"], mode, 5, start=case["start"], end=case["end"])
    for k in ("peak_bytes", "fragmentation", "peak_grad_buffer_bytes", "peak_memory", "n_samples", "samples"):
        assert a[k] == b[k], k
