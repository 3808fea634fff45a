#!/bin/bash
# 1 GPU: fused LayerNorm backward tuning — GPT gradient tests, N = 1 lines, per-launch kernel times.
timeout 900 python -m pytest tests/test_gpu_gpt.py -q -x > gpurun_out/ln_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/ln_tests.log
for i in a b; do timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ln_13b_$i.jsonl 2> gpurun_out/ln_13b_$i.err; python -c "
import json; d=json.loads(open('gpurun_out/ln_13b_$i.jsonl').read().strip().splitlines()[-1]); print('$i', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"; done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ln_bwd|colred|colsum" -c 60 --csv --log-file gpurun_out/ln_ncu.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ln_ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/ln_ncu.csv
