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

from oracle import load_oracle  # noqa: E402
from paper_2510_20111_b200 import EngineConfig, HzpEngine, ParallelConfig  # noqa: E402


def main():
    z1, z2, z3, prec = (int(x) for x in sys.argv[1:5])
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dims, mbs, batch, steps = [64, 128, 128, 64], 2, 16, 4
    o = load_oracle()
    st = o.shard_init(dims, world, z1, z2, z3, 2024, bool(prec))
    eng = HzpEngine(EngineConfig(model=0, precision=prec, dims=dims, batch=batch, num_microbatches=mbs,
                                 par=ParallelConfig(dp=world, z1=z1, z2=z2, z3=z3), device=local,
                                 my_rank=rank))
    eng.connect()
    eng.load_state(st)
    dist.barrier()
    for step in range(steps):
        x = o.make_inputs(dims, world, mbs, batch, 2024, step)
        ref_losses, _ = o.train_step_hzp(st, x, batch, bool(prec))
        losses = eng.step(np.ascontiguousarray(x[rank:rank + 1]))
    eng.sync()
    tol = 1e-5 if prec == 0 else 1e-2

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
