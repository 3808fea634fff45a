"""N > 1 host logic on CPU: world_size 2 / 4 gloo process groups, one process
per rank as on a GPU node.  Each rank builds its own LaunchPlan and its P2P
tile tables through the C-ABI (no GPU needed); rank 0 gathers everything and
checks the multi-rank invariants the device kernels rely on:

  * every rank derives the identical launch order / slot plan;
  * AG tiles: rank r pushes exactly the part of each layer inside its own
    Z3 shard (e // s3 == r % z3, train.cpp:229-249); the owners of a Z3
    group together cover each layer exactly once (groups of 2: pull form,
    every reader covers each layer once from the elements' owners);
  * RS tiles of a Z2 group partition (layer ∩ segment) across its members;
  * Z1 tiles of a Z1 group partition [0, P), and every element is pushed to
    exactly the group members q with q % z3 == e // s3 (train.cpp:361-379).
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_20111_b200 import _native as N
from paper_2510_20111_b200 import hzp as H


def _tiles(dp, z1, z2, z3, P, layers, rank, es):
    L = len(layers)
    offs = (C.c_int64 * L)(*[o for o, _ in layers])
    sizes = (C.c_int64 * L)(*[n for _, n in layers])
    par = N.hzp_parallel(dp, z1, z2, z3, 1, 1, 1, 1)
    n = C.c_int()
    N.check(N.lib.hzp_comm_tiles(C.byref(par), P, offs, sizes, L, rank, es, None, 0, C.byref(n),
                                 None, None, None, None))
    out = (N.hzp_comm_tile * max(1, n.value))()
    ag = (C.c_int * (L + 1))()
    rs = (C.c_int * (L + 1))()
    z1o, z1n = C.c_int(), C.c_int()
    N.check(N.lib.hzp_comm_tiles(C.byref(par), P, offs, sizes, L, rank, es, out, n.value, C.byref(n),
                                 ag, rs, C.byref(z1o), C.byref(z1n)))
    t = [(x.a_off, x.b_off, x.c_off, x.mask, x.len, x.src, x.vec) for x in out[: n.value]]
    return {"tiles": t, "ag": list(ag), "rs": list(rs), "z1": (z1o.value, z1n.value)}


def _worker(rank, world, port, z, layers, P, es, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    z1, z2, z3 = z
    g = H.build_task_graph(H.ModelSpec(num_layers=len(layers), params_per_layer=1, num_microbatches=2),
                           H.ParallelConfig(dp=world, z1=z1, z2=z2, z3=z3), H.CostModel(ranks_per_node=world))
    plan = [(p.id, p.kind, p.stream, p.slot, tuple(p.waits)) for p in H.launch_plan(g, 2, 1)]
    mine = {"plan": plan, **_tiles(world, z1, z2, z3, P, layers, rank, es)}
    allv = [None] * world
    dist.all_gather_object(allv, mine)
    if rank == 0:
        q.put(allv)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASES = [
    (2, (2, 2, 2), [12, 20, 8]),
    (2, (2, 1, 2), [12, 20, 8]),
    (4, (4, 2, 2), [12, 20, 8]),
    (4, (2, 4, 4), [64, 128, 128, 64]),
    (4, (4, 4, 1), [96, 200, 40]),
    (4, (4, 2, 2), [64, 128, 128, 64]),
    (4, (4, 1, 2), [5, 3, 2]),
    (4, (2, 2, 2), [12, 20, 8]),
]


@pytest.mark.parametrize("es", [2, 4])
@pytest.mark.parametrize("world,z,dims", CASES, ids=[f"w{c[0]}-z{''.join(map(str, c[1]))}" for c in CASES])
def test_multirank_plans_and_tiles(world, z, dims, es):
    layers, off = [], 0
    for i in range(len(dims) - 1):
        n = dims[i] * dims[i + 1] + dims[i + 1]
        layers.append((off, n))
        off += n
    P = off
    z1, z2, z3 = z
    s1, s2, s3 = (-(-P // k) for k in (z1, z2, z3))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, z, layers, P, es, q))
             for port in [_free_port()] for r in range(world)]
    for p in procs:
        p.start()
    allv = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # identical plans on every rank
    assert all(v["plan"] == allv[0]["plan"] for v in allv)
    if z3 == 2:  # groups of 2: pull form, every reader covers each layer once from the owners
        for r, v in enumerate(allv):
            for l, (lo, ln) in enumerate(layers):
                cov = np.zeros(ln, np.int32)
                for (a, b, c, m, n, src, vec) in v["tiles"][v["ag"][l]:v["ag"][l + 1]]:
                    cov[a:a + n] += 1
                    owner = src - (r - r % z3)
                    assert 0 <= owner < z3 and owner * s3 + b == lo + a
                assert np.all(cov == 1), (r, l)
    for g0 in range(0, world if z3 != 2 else 0, z3):
        for l, (lo, ln) in enumerate(layers):
            cov = np.zeros(ln, np.int32)
            for r in range(g0, g0 + z3):
                v = allv[r]
                for (a, b, c, m, n, src, vec) in v["tiles"][v["ag"][l]:v["ag"][l + 1]]:
                    assert src == r  # the owner pushes its own span
                    cov[a:a + n] += 1
                    assert (r % z3) * s3 + b == lo + a  # offset in the owner's shard
                    if vec:
                        assert (a * es) % 16 == 0 and (b * es) % 16 == 0 and (n * es) % 16 == 0
            assert np.all(cov == 1), (g0, l)
    if z2 > 1:
        for g0 in range(0, world, z2):
            for l, (lo, ln) in enumerate(layers):
                cov = np.zeros(ln, np.int32)
                for r in range(g0, g0 + z2):
                    v = allv[r]
                    for (a, b, c, m, n, src, vec) in v["tiles"][v["rs"][l]:v["rs"][l + 1]]:
                        assert src == g0
                        assert (r % z2) * s2 + a == lo + b  # segment offset <-> layer offset
                        cov[b:b + n] += 1
                assert np.all(cov == 1), (g0, l)
    for g0 in range(0, world, z1):
        cov = np.zeros(P, np.int32)
        pushed = np.zeros((world, P), np.int32)
        for r in range(g0, g0 + z1):
            v = allv[r]
            o, n1 = v["z1"]
            for (a, b, c, m, n, src, vec) in v["tiles"][o:o + n1]:
                e0 = (r % z1) * s1 + a
                assert src * s2 + b == e0 and (e0 // s3) * s3 + c == e0
                cov[e0:e0 + n] += 1
                for qq in range(world):
                    if m >> qq & 1:
                        pushed[qq, e0:e0 + n] += 1
        assert np.all(cov == 1)
        for qq in range(world):
            want = np.zeros(P, np.int32)
            if g0 <= qq < g0 + z1:
                seg = qq % z3
                want[seg * s3:min(P, (seg + 1) * s3)] = 1
            assert np.array_equal(pushed[qq], want), (g0, qq)
