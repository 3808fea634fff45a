#!/bin/bash
# Hierarchical-ZeRO benches (z2 = 2, one RS peer) on 4 GPUs: 7B and MoE.
mkdir -p gpurun_out
timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29821 bench.py --gpus 4 --model 7b --no-cpu-baseline > gpurun_out/r01g_bench_7b_n4.jsonl 2> gpurun_out/r01g_bench_7b_n4.err
timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29822 bench.py --gpus 4 --model moe --no-cpu-baseline > gpurun_out/r01g_bench_moe_n4.jsonl 2> gpurun_out/r01g_bench_moe_n4.err
cut -c1-200 gpurun_out/r01g_bench_*.jsonl; tail -3 gpurun_out/r01g_bench_moe_n4.err
