#!/bin/bash
run() { local name=$1 n=$2; shift 2
  env $EXTRA timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n --steps 10 --warmup 3 "$@" > gpurun_out/exp2_$name.jsonl 2> gpurun_out/exp2_$name.err
  python - gpurun_out/exp2_$name.jsonl <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); e = d["exposed_comm"]; c = d.get("collectives") or {}
    print(sys.argv[1], d["value"], "ms", d["ms_per_step"], "idle", e["frac"], e.get("idle_by_next_task_ms"), "clk", d["clocks"]["sm_mhz"], "ag", (c.get("ag") or {}).get("ms"), "rs", (c.get("rs") or {}).get("ms"))
except Exception as ex: print(sys.argv[1], "unparsed", ex)
PY
}
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "2-" > gpurun_out/exp2_multi.log 2>&1; echo "multi rc=$?"; tail -1 gpurun_out/exp2_multi.log
timeout 600 python -m pytest tests/test_gpu_comm.py tests/test_gpu_layer_table.py -q -x > gpurun_out/exp2_comm.log 2>&1; echo "comm rc=$?"; tail -1 gpurun_out/exp2_comm.log
run 13b_n2 2
run 7b_n4 4 --model 7b
run moe_n4 4 --model moe
EXTRA=HZP_EXP_OPTPRIO=1 run 7b_n4_optmid 4 --model 7b
EXTRA=HZP_EXP_OPTPRIO=1 run 13b_n4_optmid 4
EXTRA=A=1 run 13b_n4 4
