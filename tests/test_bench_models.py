"""Host-side models the bench reports against (no GPU): the per-rank NVLink
bytes of the Z1 stage (`bench.z1_link_bytes`, the denominator of
`z1_adam.roofline_ms`), checked against a hand count of the reference layout
(train.cpp:229-249 shard offsets, DZP replicas = same Z2 position in every Z2
group, bf16 pushes to the Z3 owner in every Z3 group of the Z1 group)."""
import importlib.util
import os

import pytest

from conftest import ROOT


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_flat_layout_moves_nothing(bench):
    # z1 = z2 = z3 = N: a rank's Z1 chunk is its own Z2 segment and Z3 shard
    for n in (2, 4, 8):
        eg, ing = bench.z1_link_bytes(n, 1 << 20, n, n, n)
        assert max(eg) == 0 and max(ing) == 0


def test_hierarchical_422_hand_count(bench):
    # dp 4, (z1, z2, z3) = (4, 2, 2), P divisible by 4: per chunk element
    #   chunk 0 (rank 0): replicas at 0, 2 -> 4 B from rank 2; push to 0, 2 -> 2 B to rank 2
    #   chunk 1 (rank 1): replicas at 0, 2 -> 4 B from each; push to 0, 2 -> 2 B to each
    #   chunk 2 (rank 2): replicas at 1, 3 -> 4 B from each; push to 1, 3 -> 2 B to each
    #   chunk 3 (rank 3): replicas at 1, 3 -> 4 B from rank 1; push to 1, 3 -> 2 B to rank 1
    P = 4 * 1000
    s1 = P // 4
    eg, ing = bench.z1_link_bytes(4, P, 4, 2, 2)
    assert [e // s1 for e in eg] == [6, 12, 12, 6]
    assert [i // s1 for i in ing] == [6, 12, 12, 6]
    assert sum(eg) == sum(ing)


def test_fp32_pushes_and_replica_free_groups(bench):
    # (2, 1, 1) at dp 2: z2 = 1 -> every rank holds the whole gradient (two
    # replicas); z3 = 1 -> both ranks own every parameter: 4 B in + 2 B (bf16)
    # or 4 B (fp32) out per chunk element
    P = 2 * 512
    s1 = P // 2
    eg, ing = bench.z1_link_bytes(2, P, 2, 1, 1)
    assert [e // s1 for e in eg] == [6, 6] and [i // s1 for i in ing] == [6, 6]
    eg, _ = bench.z1_link_bytes(2, P, 2, 1, 1, pbytes=4)
    assert [e // s1 for e in eg] == [8, 8]
