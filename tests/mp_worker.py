"""One rank of the multi-process (one process per GPU) parity run.

Launched by tests/test_gpu_multi.py as
    torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/mp_worker.py <z1> <z2> <z3> <prec>
Each process drives its own GPU and dp rank; peers are wired through CUDA IPC
(handles exchanged over torch.distributed, control plane only).  Every rank
runs the oracle on the CPU for the whole job and checks its own shards.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import load_oracle  # noqa: E402
from paper_2510_20111_b200 import EngineConfig, HzpEngine, ParallelConfig  # noqa: E402


def kernels(z1, z2, z3, prec):
    """Kernel-level multi-process parity: AG and RS through the test entry
    points (host barriers between phases, no device flags)."""
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank))
    dims = [64, 128, 128, 64]
    o = load_oracle()
    st = o.shard_init(dims, world, z1, z2, z3, 7, bool(prec))
    eng = HzpEngine(EngineConfig(model=0, precision=prec, dims=dims, batch=16, num_microbatches=1,
                                 par=ParallelConfig(dp=world, z1=z1, z2=z2, z3=z3), device=local,
                                 my_rank=rank))
    eng.connect()
    eng.load_state(st)
    dist.barrier()
    ok = True
    for l, (off, n) in enumerate(eng.layers if z3 > 1 else []):  # z3 = 1: the AG is the identity
        eng.ag_layer(l, 0)
        g0 = rank - rank % z3
        want = o.all_gather(st.param[g0:g0 + z3])[off:off + n]
        got = eng.ag_slot(rank, 0, n)
        if prec:
            got = (got.astype(np.uint32) << 16).view(np.float32)
        ok &= bool(np.array_equal(got, want))
    if z2 > 1:
        rng = np.random.default_rng(5)
        grads = rng.standard_normal((world, st.s2 * z2)).astype(np.float32)
        eng.zero_grads()
        for l, (off, n) in enumerate(eng.layers):
            eng.wgrad_upload(rank, l, 0, grads[rank, off:off + n])
            torch.cuda.synchronize()
            dist.barrier()
            eng.rs_layer(l, 0)
            torch.cuda.synchronize()
            dist.barrier()
        g0 = rank - rank % z2
        got = eng.download(rank, 1)
        lo = (rank % z2) * st.s2
        nv = max(0, min(st.s2, st.P - lo))
        if prec == 0:  # fp32 wire: ordered pull, bit-exact
            seg = o.reduce_scatter(grads[g0:g0 + z2])[rank % z2]
            ok &= bool(np.array_equal(got[:nv], (0 + seg)[:nv]))
        else:  # bf16 wire: multimem.ld_reduce in the switch vs the unicast model
            from test_gpu_comm import rs_bf16_model
            want = rs_bf16_model(o, grads[g0:g0 + z2])[lo:lo + nv]
            exact = float(np.mean(got[:nv].view(np.uint32) == want.view(np.uint32))) if nv else 1.0
            err = float(np.max(np.abs(got[:nv] - want)) / max(np.max(np.abs(want)), 1e-30)) if nv else 0.0
            print(f"rank {rank}: bf16 multimem RS vs model: exact {exact:.6f} max rel {err:.3g}", flush=True)
            ok &= err <= 2.0 ** -7
    print(f"rank {rank}: {'OK' if ok else 'FAIL'} kernels", flush=True)
    dist.barrier()
    eng.close()
    return ok


def gpt_race(z1, z2, z3):
    """Race check of the device-flag protocol without a sanitizer (closed on
    this pool): the bf16 GPT step (dense GELU and MoE) on every rank, three
    times — async twice, then with HZP_DEBUG_SYNC (every task serialised on
    the device and followed by a cross-rank barrier) — must give bitwise the
    same parameters, optimizer state and losses.  A missing wait anywhere in
    the AG / RS / GradReady / Z1 protocol lets some run read a buffer early."""
    from paper_2510_20111_b200.engine import make_tokens
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank))
    c = dict(layers=3, hidden=256, heads=2, ffn=1024, vocab=512, seq=256, batch=2)
    ok = True
    for experts in (0, 8):
        runs = []
        for mode in ("async", "async", "serial"):
            if mode == "serial":
                os.environ["HZP_DEBUG_SYNC"] = "1"
            eng = HzpEngine(EngineConfig(model=1, precision=1, gpt_layers=c["layers"], gpt_hidden=c["hidden"],
                                         gpt_heads=c["heads"], gpt_ffn=c["ffn"], gpt_vocab=c["vocab"],
                                         gpt_seq=c["seq"], batch=c["batch"], num_microbatches=2,
                                         gpt_experts=experts,
                                         par=ParallelConfig(dp=world, z1=z1, z2=z2, z3=z3), device=local,
                                         my_rank=rank))
            os.environ.pop("HZP_DEBUG_SYNC", None)
            eng.connect()
            eng.init_seeded(2024, 0.02)
            dist.barrier()
            losses = []
            for step in range(3):
                tok = np.stack([make_tokens(2024, step, rank, mb, c["batch"] * (c["seq"] + 1), c["vocab"])
                                .reshape(c["batch"], c["seq"] + 1) for mb in range(2)])[None]
                losses.append(np.asarray(eng.step(np.ascontiguousarray(tok, np.int32))))
            eng.sync()
            runs.append((np.concatenate(losses), eng.param_f32(rank), eng.download(rank, 2),
                         eng.download(rank, 3), eng.download(rank, 4)))
            dist.barrier()
            eng.close()
        same = [all(np.array_equal(a, b) for a, b in zip(runs[0], r)) for r in runs[1:]]
        print(f"rank {rank}: experts {experts}: async == async {same[0]}, async == serialised {same[1]}", flush=True)
        ok &= all(same)
    print(f"rank {rank}: {'OK' if ok else 'FAIL'} gpt race", flush=True)
    return ok


def main():
    z1, z2, z3, prec = (int(x) for x in sys.argv[1:5])
    dist.init_process_group("gloo")
    if len(sys.argv) > 5 and sys.argv[5] == "gpt_race":
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", dist.get_rank())))
        ok = gpt_race(z1, z2, z3)
        dist.destroy_process_group()
        sys.exit(0 if ok else 1)
    if len(sys.argv) > 5 and sys.argv[5] == "kernels":
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", dist.get_rank())))
        ok = kernels(z1, z2, z3, prec)
        dist.destroy_process_group()
        sys.exit(0 if ok else 1)
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dims, mbs, batch, steps = [64, 128, 128, 64], 2, 16, 4
    if os.environ.get("HZP_TEST_DIMS"):  # ragged shards (P not a multiple of the group sizes)
        dims, batch = [int(d) for d in os.environ["HZP_TEST_DIMS"].split(",")], 3
    o = load_oracle()
    st = o.shard_init(dims, world, z1, z2, z3, 2024, bool(prec))
    eng = HzpEngine(EngineConfig(model=0, precision=prec, dims=dims, batch=batch, num_microbatches=mbs,
                                 par=ParallelConfig(dp=world, z1=z1, z2=z2, z3=z3), device=local,
                                 my_rank=rank, reuse=int(os.environ.get("HZP_TEST_REUSE", "0"))))
    eng.connect()
    eng.load_state(st)
    dist.barrier()
    for step in range(steps):
        x = o.make_inputs(dims, world, mbs, batch, 2024, step)
        ref_losses, _ = o.train_step_hzp(st, x, batch, bool(prec))
        losses = eng.step(np.ascontiguousarray(x[rank:rank + 1]))
    eng.sync()
    tol = 0.0 if prec == 0 else 1e-2  # fp32 tier: bitwise (ordered RS, libm tanhf restatement)

    def rel(a, b):
        return float(np.max(np.abs(a.astype(np.float64) - b)) / max(np.max(np.abs(b)), 1e-30))
    errs = {"param": rel(eng.param_f32(rank), st.param[rank]),
            "master": rel(eng.download(rank, 2), st.master[rank]),
            "var": rel(eng.download(rank, 4), st.var[rank]),
            "loss": abs(float(losses[0]) - float(ref_losses[rank])) / abs(float(ref_losses[rank]))}
    ok = all(v <= tol for v in errs.values())
    print(f"rank {rank}: {'OK' if ok else 'FAIL'} {errs}", flush=True)
    dist.barrier()
    eng.close()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
