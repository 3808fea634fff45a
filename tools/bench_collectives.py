"""AG / RS bus-bandwidth sweep over NVLink (SURVEY §8(d) sweep 4), one process
per GPU, with an NCCL comparator on the same bytes.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \\
        tools/bench_collectives.py [--sizes-mb 1,4,16,64,256,1024] [--depth 2]

Each size is the full (unsharded) layer in the bf16 wire format: a
one-layer MLP ctx (`dims = [1024, k]`, layer = 1025 k elements) in flat
ZeRO-3 over the N ranks.  AG = `hzp_ag_layer` into ring slot `i % depth`
(k back-to-back AGs into k slots); RS = `hzp_rs_layer` from gradient slot 0.
Both legs are measured with the NVLink part on the copy engines (default)
and as SM pull kernels (HZP_AG_CE=0 / HZP_RS_CE=0), in the bf16 wire format
and (--precs 1,0) fp32; the AG additionally at prefetch depths 1-4
(--depths, copy-engine bf16 leg).  busbw = (N-1)/N x bytes / time, CUDA
events on the ctx stream, max over ranks.  Rank 0 prints one JSON object per
(size, op, path, dtype, depth), and with --cpu-ref the reference's own
`all_gather` / `reduce_scatter` (collective.cpp:44-115, oracle/_ref, one
host thread, sizes <= 64 MB) on the same bytes — the CPU baseline of sweep 4.
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
    ap.add_argument("--depths", default="1,2,4", help="AG prefetch depths (copy-engine bf16 leg)")
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
            k = max(64, (elems // 1025) // 64 * 64)  # shard bounds 16-B aligned up to N = 8
            n = 1025 * k
            nbytes = es * n
            for ce in (1, 0):
                for depth in (depths if (ce and prec) else [args.depth]):
                    os.environ["HZP_AG_CE"] = str(ce)
                    os.environ["HZP_RS_CE"] = str(ce)
                    eng = HzpEngine(EngineConfig(model=0, precision=prec, dims=[1024, k], batch=8,
                                                 par=ParallelConfig(dp=world, z1=world, z2=world, z3=world),
                                                 prelaunch_depth=depth, device=local, my_rank=rank))
                    eng.connect()
                    eng.init_random()
                    path = "copy-engine" if ce else "sm-pull"
                    legs = [("ag", lambda i: eng.ag_layer(0, i % depth), 1)]
                    if depth == args.depth:
                        legs.append(("rs", lambda i: eng.rs_layer(0, 0), 2))
                    for op, fn, sid in legs:
                        ms = timed(fn, eng.stream(sid))
                        bw = (world - 1) / world * nbytes / (ms / 1e3) / 1e9
                        if rank == 0:
                            print(json.dumps({"op": op, "path": path, "dtype": "bf16" if prec else "f32",
                                              "n_gpus": world, "bytes": nbytes, "depth": depth,
                                              "ms": round(ms, 4), "busbw_GBps": round(bw, 1),
                                              "frac_nvlink": round(bw / NVLINK_GBPS, 3)}), flush=True)
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
