#!/bin/bash
# Round-end validation on 4 GPUs: full GPU suite, collective sweep, 1.3B and 7B benches.
mkdir -p gpurun_out
timeout 1100 python -m pytest tests -m gpu -x -q > gpurun_out/r01c_pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/r01c_pytest_gpu.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29801 tools/bench_collectives.py --sizes-mb 16,64,256,1024 --depths 2 > gpurun_out/r01c_collectives_n4.jsonl 2> gpurun_out/r01c_collectives_n4.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29802 bench.py --gpus 4 > gpurun_out/r01c_bench_n4.jsonl 2> gpurun_out/r01c_bench_n4.err
timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29803 bench.py --gpus 4 --model 7b --no-cpu-baseline > gpurun_out/r01c_bench_7b_n4.jsonl 2> gpurun_out/r01c_bench_7b_n4.err
tail -2 gpurun_out/r01c_pytest_gpu.log; grep '"rs"' gpurun_out/r01c_collectives_n4.jsonl; cut -c1-200 gpurun_out/r01c_bench_n4.jsonl gpurun_out/r01c_bench_7b_n4.jsonl
