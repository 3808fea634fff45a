#!/bin/bash
# 1 GPU: attention backward with 32-query sub-tiles — parity, kernel timing, N = 1 step.
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_gpt.py -q -x > gpurun_out/at_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/at_tests.log
timeout 600 python tools/bench_kernels.py attn > gpurun_out/at_kernels.jsonl 2>&1; cut -c1-170 gpurun_out/at_kernels.jsonl
for i in a b; do timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/at_13b_$i.jsonl 2> gpurun_out/at_13b_$i.err; python -c "
import json; d=json.loads(open('gpurun_out/at_13b_$i.jsonl').read().strip().splitlines()[-1]); print('$i', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"; done
