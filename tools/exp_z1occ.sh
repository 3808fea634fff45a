#!/bin/bash
# 4 GPUs: Z1 at one float4 per pass / 48 registers on the DZP configs + multi-GPU step parity.
tag=${1:-zo}
source <(sed -n '/^run()/,/^}/p' tools/exp_multi.sh)
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "step" > gpurun_out/${tag}_multi.log 2>&1; echo "multi rc=$?"; tail -1 gpurun_out/${tag}_multi.log
run moe_n4 4 --model moe
run 7b_n4 4 --model 7b
run 13b_n4 4
run 7b_n2 2 --model 7b
