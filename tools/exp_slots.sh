#!/bin/bash
# 4 GPUs: gradient-ring depth and AG depth (1.3B flat N = 2 / 4, 7B N = 4).
tag=${1:-sl}
source <(sed -n '/^run()/,/^}/p' tools/exp_multi.sh)
run 13b_n4_w2d2 4
run 13b_n4_w3d3 4 --wgrad-slots 3 --depth 3
run 13b_n2_w2d2 2
run 13b_n2_w3d3 2 --wgrad-slots 3 --depth 3
run 7b_n4_w3 4 --model 7b --wgrad-slots 3
run moe_n4_w3 4 --model moe --wgrad-slots 3
