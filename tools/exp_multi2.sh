#!/bin/bash
# 4 GPUs: step parity (Z1 prefetch, 16K tiles), the GPT race check, multi-GPU
# parity, then the DZP configs' bench lines.
tag=${1:-x}
source <(sed -n '/^run()/,/^}/p' tools/exp_multi.sh)
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_comm.py tests/test_gpu_layer_table.py -q -x > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/${tag}_tests.log
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/${tag}_multi.log 2>&1; echo "multi rc=$?"; tail -1 gpurun_out/${tag}_multi.log
run moe_n4 4 --model moe
run 7b_n4 4 --model 7b
