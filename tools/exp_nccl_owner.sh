#!/bin/bash
# 4 GPUs: bench lines with the NCCL single-owner comparators (broadcast from /
# reduce to the layer's owner, same groups) beside ours.
tag=${1:-no}
source <(sed -n '/^run()/,/^}/p' tools/exp_multi.sh)
run 13b_n4 4
run 13b_n2 2
run moe_n4 4 --model moe
for f in 13b_n4 13b_n2 moe_n4; do python -c "
import json; d=json.loads(open('gpurun_out/${tag}_$f.jsonl').read().strip().splitlines()[-1]); c=d['collectives']
print('$f', {k: c.get(k) for k in ('ag','rs','nccl_all_gather','nccl_reduce_scatter','nccl_broadcast_from_owner','nccl_reduce_to_owner')})"; done
