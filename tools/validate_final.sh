#!/bin/bash
# Final validation on 4 GPUs: GPU suite, smoke, benches N=1/2/4, RS sweep N=4 and N=2.
mkdir -p gpurun_out
timeout 1100 python -m pytest tests -m gpu -x -q > gpurun_out/r01f_pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/r01f_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r01f_smoke.log 2>&1
timeout 400 python bench.py > gpurun_out/r01f_bench_n1.jsonl 2> gpurun_out/r01f_bench_n1.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29811 bench.py --gpus 2 > gpurun_out/r01f_bench_n2.jsonl 2> gpurun_out/r01f_bench_n2.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29812 bench.py --gpus 4 > gpurun_out/r01f_bench_n4.jsonl 2> gpurun_out/r01f_bench_n4.err
timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29813 tools/bench_collectives.py --sizes-mb 16,64,256,1024 --depths 2 --precs 1 > gpurun_out/r01f_collectives_n4.jsonl 2> gpurun_out/r01f_collectives_n4.err
CUDA_VISIBLE_DEVICES=0,1 timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29814 tools/bench_collectives.py --sizes-mb 16,64,256,1024 --depths 2 --precs 1 > gpurun_out/r01f_collectives_n2.jsonl 2> gpurun_out/r01f_collectives_n2.err
tail -2 gpurun_out/r01f_pytest_gpu.log; tail -1 gpurun_out/r01f_smoke.log; grep -h copy-engine gpurun_out/r01f_collectives_n*.jsonl | cut -c1-200; cut -c1-150 gpurun_out/r01f_bench_n*.jsonl
