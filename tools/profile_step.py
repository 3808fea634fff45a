"""Per-GEMM-shape and per-task breakdown of one 1.3B-class GPT step.

    python tools/profile_step.py [--batch 4] [--microbatches 2] [--layers 24]
    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        tools/profile_step.py        # flat ZeRO-3 over N ranks; rank 0 prints
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2510_20111_b200 import EngineConfig, HzpEngine, ParallelConfig  # noqa: E402
from paper_2510_20111_b200 import hzp as H  # noqa: E402
from paper_2510_20111_b200.engine import gemm_profile, gemm_profile_dump  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=4)
    ap.add_argument("--microbatches", type=int, default=2)
    ap.add_argument("--layers", type=int, default=24)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method="env://")
    torch.cuda.set_device(local)
    par = ParallelConfig(dp=world, z1=world, z2=world, z3=world) if world > 1 else ParallelConfig()
    cfg = EngineConfig(model=1, precision=1, gpt_layers=args.layers, gpt_hidden=2048, gpt_heads=16,
                       gpt_ffn=8192, gpt_vocab=50304, gpt_seq=2048, batch=args.batch,
                       num_microbatches=args.microbatches, par=par, my_rank=rank, device=local,
                       timeline=1)
    eng = HzpEngine(cfg)
    if world > 1:
        eng.connect()
    eng.init_random()
    import numpy as np
    tok = torch.from_numpy(np.random.default_rng(rank).integers(
        0, 50304, size=(1, args.microbatches, args.batch, 2049), dtype=np.int32)).cuda()
    for _ in range(2):
        eng.step_async(tok.data_ptr(), True)
    eng.sync()
    eng.step_async(tok.data_ptr(), True)
    eng.sync()
    tl = eng.timeline()
    g = H.build_task_graph(H.ModelSpec(num_layers=args.layers + 2, params_per_layer=1,
                                       num_microbatches=args.microbatches),
                           H.ParallelConfig(dp=world, z1=world, z2=world, z3=world) if world > 1
                           else H.ParallelConfig(), H.CostModel())
    by_kind = {}
    for t in g.tasks:
        d = tl["end_ms"][t.id] - tl["start_ms"][t.id]
        k = H.KIND_NAMES[t.kind] + ("(emb)" if t.layer == 0 else "(head)" if t.layer == args.layers + 1 else "")
        by_kind[k] = by_kind.get(k, 0.0) + d
    if rank != 0:
        gemm_profile(True)
        eng.step_async(tok.data_ptr(), True)
        eng.sync()
        gemm_profile(False)
        eng.close()
        return
    print(json.dumps({"world": world, "makespan_ms": tl["makespan_ms"], "compute_busy_ms": tl["compute_busy_ms"],
                      "compute_idle_ms": tl["compute_idle_ms"],
                      "by_kind_ms": {k: round(v, 3) for k, v in by_kind.items()}}, indent=1))
    order = sorted(range(len(g.tasks)), key=lambda i: tl["end_ms"][i])
    print("last tasks to finish (kind layer start end ms):")
    for i in order[-8:]:
        t = g.tasks[i]
        print(f"  {H.KIND_NAMES[t.kind]:>14} L{t.layer:<3} {tl['start_ms'][i]:9.3f} {tl['end_ms'][i]:9.3f}")
    gemm_profile(True)
    eng.step_async(tok.data_ptr(), True)
    eng.sync()
    gemm_profile(False)
    f, ms, n, table = gemm_profile_dump()
    print(f"GEMM total: {n} launches, {ms:.2f} ms, {f / ms / 1e9:.1f} TFLOP/s")
    print(table)
    eng.close()


if __name__ == "__main__":
    main()
