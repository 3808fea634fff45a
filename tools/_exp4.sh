#!/bin/bash
run() { local name=$1 n=$2; shift 2
  env $EXTRA timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n --steps 10 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/exp4_$name.jsonl 2> gpurun_out/exp4_$name.err
  python - gpurun_out/exp4_$name.jsonl <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); e = d["exposed_comm"]
    print(sys.argv[1], d["value"], "ms", d["ms_per_step"], "idle", e["frac"], e.get("idle_by_next_task_ms"), "clk", d["clocks"]["sm_mhz"])
except Exception as ex: print(sys.argv[1], "unparsed", ex)
PY
}
timeout 600 python -m pytest tests/test_gpu_comm.py tests/test_gpu_layer_table.py -q -x > gpurun_out/exp4_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/exp4_tests.log
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "4-z1 or 4-z2 or 4-z3" > gpurun_out/exp4_multi.log 2>&1; echo "multi rc=$?"; tail -1 gpurun_out/exp4_multi.log
EXTRA="HZP_EXP_OPTPRIO=0" run moe_rs_lo 4 --model moe
EXTRA="HZP_EXP_OPTPRIO=1" run moe_rs_mid 4 --model moe
EXTRA="HZP_EXP_OPTPRIO=0 HZP_EXP_PUSHSTREAM=1" run moe_ps_lo 4 --model moe
EXTRA="HZP_EXP_OPTPRIO=1 HZP_EXP_PUSHSTREAM=1" run moe_ps_mid 4 --model moe
EXTRA="HZP_EXP_OPTPRIO=0 HZP_EXP_PUSHSTREAM=1" run 7b_ps_lo 4 --model 7b
EXTRA="HZP_EXP_OPTPRIO=1 HZP_EXP_PUSHSTREAM=1" run 7b_ps_mid 4 --model 7b
EXTRA="HZP_EXP_OPTPRIO=0" run 7b_rs_lo 4 --model 7b
