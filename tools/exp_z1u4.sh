#!/bin/bash
# 1 GPU: Z1 kernel with 4 float4 per pass (parity + microbench + N = 1 lines), then the final ncu round.
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_comm.py -q -x > gpurun_out/u4_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/u4_tests.log
timeout 600 python tools/bench_kernels.py comm > gpurun_out/u4_kernels_comm.jsonl 2>&1; grep z1 gpurun_out/u4_kernels_comm.jsonl
for m in 1.3b moe 7b; do timeout 900 python bench.py --model $m --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/u4_$m.jsonl 2> gpurun_out/u4_$m.err; python -c "
import json; d=json.loads(open('gpurun_out/u4_$m.jsonl').read().strip().splitlines()[-1]); print('$m', d['value'], d['ms_per_step'], d['z1_adam']['ms'], d['z1_adam']['frac'], d['exposed_comm']['idle_by_next_task_ms'], d['clocks']['sm_mhz'])"; done
tools/ncu_round2.sh r02b
