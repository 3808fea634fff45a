#!/bin/bash
# 4 GPUs: multicast RS with the fp32 shard prefetched beside the in-switch reduce.
tag=${1:-rm}
source <(sed -n '/^run()/,/^}/p' tools/exp_multi.sh)
timeout 900 python -m pytest tests/test_gpu_comm.py -q -x > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/${tag}_tests.log
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "4-z3 or kernels" > gpurun_out/${tag}_multi.log 2>&1; echo "multi rc=$?"; tail -1 gpurun_out/${tag}_multi.log
run 13b_n4 4
python -c "
import json; d=json.loads(open('gpurun_out/${tag}_13b_n4.jsonl').read().strip().splitlines()[-1]); c=d['collectives']
print({k: c.get(k) for k in ('rs','nccl_reduce_to_owner')})"
