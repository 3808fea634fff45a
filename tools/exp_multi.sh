#!/bin/bash
# Multi-GPU check of a change (run under gpurun --gpus 4): the comm / layer
# table / multi-GPU parity tests, then the N = 2 / 4 bench lines of the
# three BASELINE models.  usage: tools/exp_multi.sh TAG [tests|bench|all]
tag=${1:-exp}; what=${2:-all}
mkdir -p gpurun_out
run() { local name=$1 n=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n --steps 10 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/${tag}_$name.jsonl 2> gpurun_out/${tag}_$name.err
  python - gpurun_out/${tag}_$name.jsonl <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); e = d["exposed_comm"]; c = d.get("collectives") or {}
    print(sys.argv[1], d["value"], "ms", d["ms_per_step"], "idle", e["frac"], e.get("idle_by_next_task_ms"), "clk", d["clocks"]["sm_mhz"], "ag", json.dumps(c.get("ag")), "nccl", (c.get("nccl_all_gather") or {}).get("ms"), "z1", (d.get("z1_adam") or {}).get("ms"))
except Exception as ex: print(sys.argv[1], "unparsed", ex)
PY
}
if [ "$what" != bench ]; then
timeout 900 python -m pytest tests/test_gpu_comm.py tests/test_gpu_layer_table.py tests/test_gpu_step.py tests/test_gpu_gemm.py -q -x > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/${tag}_tests.log
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/${tag}_multi.log 2>&1; echo "multi rc=$?"; tail -1 gpurun_out/${tag}_multi.log
fi
[ "$what" = tests ] && exit 0
run 13b_n2 2
run 7b_n4 4 --model 7b
run moe_n4 4 --model moe
run 13b_n4 4
