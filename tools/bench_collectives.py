"""AG / RS sweep over NVLink / NVSwitch (SURVEY §8(d) sweep 4, BASELINE
configs[4]: 1 MB - 1 GB x prefetch depth 1-4 at 2 / 4 / 8 GPUs), one process
per GPU, with an NCCL comparator on the same bytes.

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \
        tools/bench_collectives.py [--sizes-mb 1,4,16,64,256,1024] [--depths 1,2,4]

Two layer placements of the flat ZeRO-3 layout (the kernels are the step's
own: owner multimem.st AG, multimem.ld_reduce RS for the bf16 wire, ordered
pull for fp32):
  balanced     one-layer MLP ctx (dims = [1024, k]): the layer spans all N
               shards, every rank owns 1/N (the nccl-tests shape);
  single-owner 2N equal layers (dims = [k] * (2N + 1)): layer 0 lies inside
               rank 0's shard (the 1.3B / 7B case: a broadcast / a reduce at
               one owner).
Timing: hzp_collective_time (back-to-back on the collective's stream, CUDA
events, one device barrier first), max over ranks.  busbw = (N-1)/N x
bytes / time; owner_link = bytes / time (the owner's NVLink carries the
layer once).  Rank 0 prints one JSON object per row; with --cpu-ref also the
reference's own CPU all_gather / reduce_scatter (collective.cpp:44-115,
oracle/_ref, one host thread, sizes <= 64 MB) on the same bytes.
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2510_20111_b200 import EngineConfig, HzpEngine, ParallelConfig  # noqa: E402

NVLINK_GBPS = 900.0


def cpu_reference(g, mb):
    """The reference's CPU collectives on the same per-call bytes (1 thread)."""
    import time
    import numpy as np
    sys.path.insert(0, ROOT)
    from oracle.numerics import RefLib
    L = RefLib().L
    n = (mb << 20) // 4 // g * g
    full = np.random.default_rng(0).random(n * g, dtype=np.float32)
    out = np.empty(n, np.float32)
    t0 = time.perf_counter()
    L.ref_reduce_scatter_f32(full, g, n, out)
    rs = time.perf_counter() - t0
    nd = (mb << 20) // 8 // g * g
    shards = np.random.default_rng(1).random(nd, dtype=np.float64)
    outd = np.empty(nd * g, np.float64)
    t0 = time.perf_counter()
    L.ref_all_gather_f64(shards, g, nd // g, outd)
    ag = time.perf_counter() - t0
    for op, t, nbytes in (("reference_cpu_reduce_scatter_f32", rs, 4 * n),
                          ("reference_cpu_all_gather_f64", ag, 8 * nd)):
        bw = (g - 1) / g * nbytes / t / 1e9
        print(json.dumps({"op": op, "n_ranks": g, "bytes": nbytes, "ms": round(t * 1e3, 3),
                          "busbw_GBps": round(bw, 2), "cores": 1,
                          "note": "reference collective.cpp over g in-process ranks (incl. its tensor copies)"}),
              flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes-mb", default="1,4,16,64,256,1024")
    ap.add_argument("--depth", type=int, default=2)
    ap.add_argument("--depths", default="1,2,4", help="AG prefetch depths (bf16 wire)")
    ap.add_argument("--precs", default="1,0", help="1 = bf16 wire, 0 = fp32")
    ap.add_argument("--cpu-ref", action="store_true")
    ap.add_argument("--iters", type=int, default=8)
    args = ap.parse_args()
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ["LOCAL_RANK"])
    dist.init_process_group("gloo", init_method="env://")
    torch.cuda.set_device(local)
    nccl = dist.new_group(backend="nccl")
    dev = f"cuda:{local}"

    def mx(x):
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(fn, stream_ptr=None):
        st = torch.cuda.ExternalStream(stream_ptr, device=dev) if stream_ptr else torch.cuda.current_stream()
        for _ in range(2):
            fn(0)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for i in range(args.iters):
            fn(i)
        e1.record(st)
        e1.synchronize()
        return mx(e0.elapsed_time(e1) / args.iters)

    depths = [int(x) for x in args.depths.split(",")]
    for mb in (int(x) for x in args.sizes_mb.split(",")):
        for prec in (int(x) for x in args.precs.split(",")):
            es = 2 if prec else 4
            elems = mb * (1 << 20) // es
            for place in ("balanced", "single-owner"):
                if place == "balanced":
                    k = max(64, (elems // 1025) // 64 * 64)  # shard bounds 16-B aligned up to N = 8
                    dims, n = [1024, k], 1025 * k
                else:
                    k = max(64, int((elems ** 0.5) // 64 * 64))
                    dims, n = [k] * (2 * world + 1), k * k + k
                nbytes = es * n
                for depth in (depths if prec else [args.depth]):
                    eng = HzpEngine(EngineConfig(model=0, precision=prec, dims=dims, batch=8,
                                                 par=ParallelConfig(dp=world, z1=world, z2=world, z3=world),
                                                 prelaunch_depth=depth, device=local, my_rank=rank))
                    eng.connect()
                    eng.init_random()  # values do not matter for timing (device-side, fast)
                    for op in (("ag", "rs") if depth == args.depth else ("ag",)):
                        eng.collective_time(op, 0, 2)
                        ms = mx(eng.collective_time(op, 0, args.iters))
                        bw = (world - 1) / world * nbytes / (ms / 1e3) / 1e9
                        link = nbytes / (ms / 1e3) / 1e9
                        if rank == 0:
                            print(json.dumps({"op": op, "placement": place, "dtype": "bf16" if prec else "f32",
                                              "n_gpus": world, "bytes": nbytes, "depth": depth,
                                              "ms": round(ms, 4), "busbw_GBps": round(bw, 1),
                                              "owner_link_GBps": round(link, 1) if place == "single-owner" else None,
                                              "frac_nvlink": round((link if place == "single-owner" else bw)
                                                                   / NVLINK_GBPS, 3)}), flush=True)
                    eng.close()
        elems = mb * (1 << 20) // 2
        n = 1025 * max(64, (elems // 1025) // 64 * 64)
        if args.cpu_ref and rank == 0 and mb <= 64:
            cpu_reference(world, mb)
        m = n - n % world
        full = torch.empty(m, dtype=torch.bfloat16, device=dev)
        part = torch.empty(m // world, dtype=torch.bfloat16, device=dev)
        for op, fn in (("nccl_all_gather", lambda i: dist.all_gather_into_tensor(full, part, group=nccl)),
                       ("nccl_reduce_scatter", lambda i: dist.reduce_scatter_tensor(part, full, group=nccl))):
            ms = timed(fn)
            bw = (world - 1) / world * 2 * m / (ms / 1e3) / 1e9
            if rank == 0:
                print(json.dumps({"op": op, "n_gpus": world, "bytes": 2 * m, "ms": round(ms, 4),
                                  "busbw_GBps": round(bw, 1), "frac_nvlink": round(bw / NVLINK_GBPS, 3)}),
                      flush=True)
        del full, part
        torch.cuda.empty_cache()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
