"""Per-GEMM-shape and per-task breakdown of one 1.3B-class GPT step (N=1).

    python tools/profile_step.py [--batch 4] [--microbatches 2] [--layers 24]
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
    cfg = EngineConfig(model=1, precision=1, gpt_layers=args.layers, gpt_hidden=2048, gpt_heads=16,
                       gpt_ffn=8192, gpt_vocab=50304, gpt_seq=2048, batch=args.batch,
                       num_microbatches=args.microbatches, par=ParallelConfig(), my_rank=0,
                       timeline=1)
    eng = HzpEngine(cfg)
    eng.init_random()
    import numpy as np
    tok = torch.from_numpy(np.random.default_rng(0).integers(
        0, 50304, size=(1, args.microbatches, args.batch, 2049), dtype=np.int32)).cuda()
    for _ in range(2):
        eng.step_async(tok.data_ptr(), True)
    eng.sync()
    eng.step_async(tok.data_ptr(), True)
    eng.sync()
    tl = eng.timeline()
    g = H.build_task_graph(H.ModelSpec(num_layers=args.layers + 2, params_per_layer=1,
                                       num_microbatches=args.microbatches),
                           H.ParallelConfig(), H.CostModel())
    by_kind = {}
    for t in g.tasks:
        d = tl["end_ms"][t.id] - tl["start_ms"][t.id]
        k = H.KIND_NAMES[t.kind] + ("(emb)" if t.layer == 0 else "(head)" if t.layer == args.layers + 1 else "")
        by_kind[k] = by_kind.get(k, 0.0) + d
    print(json.dumps({"makespan_ms": tl["makespan_ms"], "compute_busy_ms": tl["compute_busy_ms"],
                      "compute_idle_ms": tl["compute_idle_ms"],
                      "by_kind_ms": {k: round(v, 3) for k, v in by_kind.items()}}, indent=1))
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
