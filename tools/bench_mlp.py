"""SURVEY §8(d) sweep 2: the reference's own model family (the MLP of
train.cpp) at GPU scale through the same engine — one process, dp = 1, bf16
working copy, `dims = 4096,16384,4096`, 8192 rows x 2 microbatches per step.
Device-timed (CUDA events on the compute stream, inputs resident in HBM).

    python tools/bench_mlp.py [--dims 4096,16384,4096] [--rows 8192] [--microbatches 2]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2510_20111_b200 import EngineConfig, HzpEngine, ParallelConfig  # noqa: E402
from paper_2510_20111_b200.engine import gemm_profile, gemm_profile_read_busy  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", default="4096,16384,4096")
    ap.add_argument("--rows", type=int, default=8192)
    ap.add_argument("--microbatches", type=int, default=2)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    dims = [int(d) for d in args.dims.split(",")]
    eng = HzpEngine(EngineConfig(model=0, precision=1, dims=dims, batch=args.rows,
                                 num_microbatches=args.microbatches, par=ParallelConfig(), my_rank=0))
    eng.init_random(seed=7, scale=0.02)
    x = torch.from_numpy(np.random.default_rng(0).uniform(
        -0.5, 0.5, size=(1, args.microbatches, args.rows, dims[0])).astype(np.float32)).cuda()
    for _ in range(args.warmup):
        eng.step_async(x.data_ptr(), True)
    eng.sync()
    cs = torch.cuda.ExternalStream(eng.stream(0))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(cs)
    for _ in range(args.steps):
        eng.step_async(x.data_ptr(), True)
    e1.record(cs)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    gemm_profile(True)
    eng.step_async(x.data_ptr(), True)
    eng.sync()
    gemm_profile(False)
    gf, gms, gbusy, gn = gemm_profile_read_busy()
    params = sum(a * b + b for a, b in zip(dims[:-1], dims[1:]))
    rows = args.rows * args.microbatches
    print(json.dumps({"workload": "reference MLP (train.cpp) at GPU scale", "dims": dims, "params": params,
                      "rows_per_step": rows, "ms_per_step": round(ms, 3), "rows_per_s": round(rows / ms * 1e3, 1),
                      "model_tflops": round(6.0 * params * rows / ms / 1e9, 1),
                      "gemm": {"launches": gn, "tflops_over_busy": round(gf / gbusy / 1e9, 1) if gbusy else None,
                               "busy_share_of_step": round(gbusy / ms, 3)}}))
    eng.close()


if __name__ == "__main__":
    main()
