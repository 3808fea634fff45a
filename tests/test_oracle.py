"""Pin the oracle: restatement == reference (golden fixtures + live _ref lib).

Mirrors the reference's own suites: tests/test_train.cpp (equivalence,
mutation control), tests/test_kernels.cpp (bf16 RNE), tests/test_collective.cpp
(RS/AR left-fold order, AG∘RS == AR), tests/test_config.cpp (layout),
tests/test_sched.cpp (census, simulate).
"""
import itertools

import numpy as np
import pytest

from conftest import golden
from oracle import sched_oracle as so

NUM = golden("numerics")
SCHED = golden("sched")
LAYOUT = golden("layout")
KERN = golden("kernels")


@pytest.mark.parametrize("case", NUM["cases"], ids=lambda c: "{dims}-{dp}-{z1}{z2}{z3}-mb{mbs}-{precision}".format(**c))
def test_restatement_matches_reference_golden(oracle, case):
    dt = np.float64 if case["precision"] == "fp64" else np.float32
    st, losses = oracle.run_states(case["dims"], case["dp"], case["z1"], case["z2"], case["z3"],
                                   case["mbs"], case["batch"], case["seed"], case["steps"],
                                   case["precision"] == "mixed", dt)
    h = case["hash"]
    assert (st.P, st.s1, st.s2, st.s3) == (case["P"], case["s1"], case["s2"], case["s3"])
    assert oracle.fnv1a(st.gathered_params()) == h["params"]
    for r in range(case["dp"]):
        assert oracle.fnv1a(st.param[r]) == h["param_shards"][r]
        assert oracle.fnv1a(st.grad[r]) == h["grad_shards"][r]
        assert oracle.fnv1a(st.master[r]) == h["master"][r]
        assert oracle.fnv1a(st.mom[r]) == h["mom"][r]
        assert oracle.fnv1a(st.var[r]) == h["var"][r]
    assert [float(x) for x in losses] == case["losses"]


def test_cpu_config_params_head_matches_survey(oracle):
    # fp32 and mixed p[0..3] after 10 steps, seed 2024
    st, _ = oracle.run_states([12, 20, 8], 4, 4, 2, 2, 1, 4, 2024, 10, False, np.float32)
    assert np.allclose(st.gathered_params()[:4],
                       [0.11059311, 0.285236388, -0.23909162, -0.158302352], rtol=0, atol=1e-8)
    st, _ = oracle.run_states([12, 20, 8], 4, 4, 2, 2, 1, 4, 2024, 10, True, np.float32)
    assert list(st.gathered_params()[:4]) == [np.float32(v) for v in
                                             (0.110839844, 0.28515625, -0.239257812, -0.158203125)]


def test_sharded_equals_baseline_fp64_exact(oracle):
    # tests/test_train.cpp:117-141 / acceptance.cpp:132-155
    for dp in (1, 2, 4):
        divs = [d for d in range(1, dp + 1) if dp % d == 0]
        for z1, z2, z3 in itertools.product(divs, divs, divs):
            dims = [12, 20, 8]
            st = oracle.shard_init(dims, dp, z1, z2, z3, 11, False, np.float64)
            base = oracle.baseline_init(dims, 11, False, np.float64)
            for step in range(2):
                x = oracle.make_inputs(dims, dp, 2, 4, 11, step, np.float64)
                oracle.train_step_hzp(st, x, 4, False)
                oracle.train_step_baseline(base, dims, dp, z2, x, 4, False)
            assert np.array_equal(st.gathered_params(), base["working"])


def test_wrong_reduction_tree_diverges(oracle):
    # mutation control, tests/test_train.cpp:96-115
    dims = [6, 10, 4]
    st = oracle.shard_init(dims, 4, 1, 4, 1, 9, False, np.float64)
    good = oracle.baseline_init(dims, 9, False, np.float64)
    bad = oracle.baseline_init(dims, 9, False, np.float64)
    for step in range(2):
        x = oracle.make_inputs(dims, 4, 2, 4, 9, step, np.float64)
        oracle.train_step_hzp(st, x, 4, False)
        oracle.train_step_baseline(good, dims, 4, 4, x, 4, False)
        oracle.train_step_baseline(bad, dims, 4, 1, x, 4, False)
    assert np.array_equal(st.gathered_params(), good["working"])
    assert not np.array_equal(good["working"], bad["working"])


def test_finite_difference_gradient(oracle):
    # tests/test_train.cpp:45-62
    dims = [6, 10, 4]
    P = sum(dims[i - 1] * dims[i] + dims[i] for i in range(1, len(dims)))
    p = oracle.seeded_uniform(P, 7)
    x = oracle.seeded_uniform(3 * 6, 8)
    loss, g = oracle.mlp_loss_grad(dims, p, x, 3)
    h = 1e-6
    for i in range(0, P, 7):
        up, dn = p.copy(), p.copy()
        up[i] += h
        dn[i] -= h
        fd = (oracle.mlp_loss_grad(dims, up, x, 3)[0] - oracle.mlp_loss_grad(dims, dn, x, 3)[0]) / (2 * h)
        assert abs(g[i] - fd) <= 1e-5 * max(1.0, abs(fd))


def test_restatement_matches_live_reference(oracle, ref):
    rng = np.random.default_rng(3)
    for _ in range(12):
        dp = int(rng.choice([1, 2, 4, 8]))
        divs = [d for d in range(1, dp + 1) if dp % d == 0]
        z1, z2, z3 = (int(rng.choice(divs)) for _ in range(3))
        mbs = int(rng.integers(1, 4))
        dims = [int(rng.integers(3, 17)) for _ in range(int(rng.integers(2, 5)))]
        for prec in ("fp32", "mixed"):
            a, la, _ = ref.run_states(dims, dp, z1, z2, z3, mbs, 4, 5, 3, prec == "mixed")
            b, lb = oracle.run_states(dims, dp, z1, z2, z3, mbs, 4, 5, 3, prec == "mixed")
            for f in ("param", "grad", "master", "mom", "var"):
                assert np.array_equal(getattr(a, f), getattr(b, f)), (dims, dp, z1, z2, z3, f)
            assert np.array_equal(la, lb)


def test_bf16_round_known_answers(oracle):
    # tests/test_kernels.cpp:34-68
    for k, v in KERN["bf16_known"].items():
        assert float(oracle.L.orc_bf16_round(float(k))) == v
    x = np.array(KERN["bf16_bits_in"], dtype=np.uint32).view(np.float32)
    y = oracle.bf16_round(x)
    assert np.array_equal(y.view(np.uint32), np.array(KERN["bf16_bits_out"], dtype=np.uint32))
    assert np.all((y.view(np.uint32) & 0xFFFF) == 0)
    nan = np.array([0x7F800001], dtype=np.uint32).view(np.float32)
    out = oracle.bf16_round(nan).view(np.uint32)[0]
    assert out & 0x00400000 and (out & 0x7F800000) == 0x7F800000


def test_collectives_left_fold(oracle):
    # tests/test_collective.cpp:96-111
    fulls = np.array(KERN["rs_in"], dtype=np.float32).reshape(4, 8)
    assert np.array_equal(oracle.reduce_scatter(fulls).reshape(-1),
                          np.array(KERN["rs_out"], dtype=np.float32))
    assert np.array_equal(oracle.all_reduce(fulls), np.array(KERN["ar_out"], dtype=np.float32))
    acc = fulls[0].copy()
    for r in range(1, 4):
        acc = acc + fulls[r]
    assert np.array_equal(oracle.all_reduce(fulls), acc)


def test_ag_of_rs_equals_ar_fp64(oracle):
    # tests/test_collective.cpp:78-94
    rng = np.random.default_rng(9)
    for _ in range(50):
        g = int(rng.integers(1, 17))
        n = g * int(rng.integers(1, 33))
        fulls = rng.random((g, n)) - 0.5
        rs = oracle.reduce_scatter(fulls)
        assert np.array_equal(oracle.all_gather(rs), oracle.all_reduce(fulls))
    with pytest.raises(ValueError):
        oracle.reduce_scatter(np.zeros((3, 4)))


def test_layout_restatement_matches_golden():
    for c in LAYOUT["groups"]:
        g = so.build_process_groups(c["dp"], c["z1"], c["z2"], c["z3"])
        for k in ("Z1", "Z2", "Z3", "DZP"):
            assert g[k] == c[k]
    for c in LAYOUT["shard_elems"]:
        assert so.shard_elems(c["n"], c["parts"]) == c["s"]
    for c in LAYOUT["validate"]:
        P = c["layers"] * c["ppl"]
        assert so.validate(c["dp"], c["z1"], c["z2"], c["z3"], P, c["dp"]) == c["code"]


@pytest.mark.parametrize("case", SCHED["graphs"], ids=lambda c: "L{layers}-M{num_mb}-z{z2}-d{depth}-r{rs_slots}-{defer_rs}-{vanilla}".format(**c))
def test_sched_restatement_matches_golden(case):
    tasks = so.build_task_graph(case["layers"], case["num_mb"], case["dp"], case["z2"], case["defer_rs"])
    assert len(tasks) == len(case["tasks"])
    for a, b in zip(tasks, case["tasks"]):
        assert (a["kind"], a["layer"], a["mb"], a["pass"], a["deps"]) == \
               (b["kind"], b["layer"], b["mb"], b["pass"], b["deps"])
    start, end, s = so.simulate(tasks, case["dur"], case["depth"], case["rs_slots"], case["vanilla"])
    assert start == case["start"] and end == case["end"]
    assert s["compute_idle"] == case["summary"]["compute_idle"]
    assert s["makespan"] == case["summary"]["makespan"]


def test_task_census_formula():
    # tasks = 5LM + (R>1 ? L : 0) + 1 + L
    for L, M, z2 in itertools.product((1, 4, 24, 32), (1, 2, 4), (1, 2, 4, 8)):
        R = 8 // z2
        n = len(so.build_task_graph(L, M, 8, z2))
        assert n == 5 * L * M + (L if R > 1 else 0) + 1 + L
