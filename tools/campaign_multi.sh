#!/bin/bash
# Multi-GPU measurement campaign (run under gpurun --gpus 4): the three
# BASELINE models at N = 2 and 4, the async / vanilla x prefetch-depth
# ablation (BASELINE configs[4]), the AG / RS sweep, and
# (MULTI_TESTS=1) the multi-GPU parity tests.  Outputs under gpurun_out/<tag>_*.
tag=${1:-r02m}
what=${2:-all}  # all | models (the N = 2 / 4 model lines and the depth-2 / 3 ablation pair only)
mkdir -p gpurun_out
run() {  # run <name> <nproc> <bench args...>
  local name=$1 n=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n --steps 10 --warmup 3 "$@" \
    > gpurun_out/${tag}_$name.jsonl 2> gpurun_out/${tag}_$name.err
  python - gpurun_out/${tag}_$name.jsonl <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    e = d["exposed_comm"]
    print(sys.argv[1], d["value"], "ms", d["ms_per_step"], "idle", e["frac"], e.get("idle_by_next_task_ms"),
          "clk", d["clocks"]["sm_mhz"], "z1", d["z1_adam"]["ms"])
except Exception as ex:
    print(sys.argv[1], "unparsed", ex)
PY
}
[ "${MULTI_TESTS:-0}" = 1 ] && { timeout 1500 python -m pytest tests/test_gpu_multi.py -q > gpurun_out/${tag}_multi.log 2>&1; echo "multi rc=$?"; tail -1 gpurun_out/${tag}_multi.log; }
for n in 2 4; do
  run 13b_n$n $n
  run 7b_n$n $n --model 7b
  run moe_n$n $n --model moe
done
# scheduler ablation (BASELINE configs[4]): async vs vanilla at prefetch
# depth 1 / 2 / 3 (3 = the 1.3B default, the model runs above) / 4, N = 2 and 4
run 13b_n2_async_d2 2 --depth 2
run 13b_n2_vanilla_d2 2 --mode vanilla --depth 2
run 13b_n4_async_d2 4 --depth 2
run 13b_n4_vanilla_d2 4 --mode vanilla --depth 2
run 13b_n4_vanilla_d3 4 --mode vanilla --depth 3
run 7b_n4_vanilla 4 --model 7b --mode vanilla
[ "$what" = models ] && exit 0
run 13b_n4_async_d1 4 --depth 1
run 13b_n4_vanilla_d1 4 --mode vanilla --depth 1
run 13b_n4_async_d4 4 --depth 4
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29950 tools/bench_collectives.py --sizes-mb 64,256,1024 --depths 2 --precs 1,0 \
  > gpurun_out/${tag}_sweep_n4.jsonl 2> gpurun_out/${tag}_sweep_n4.err
echo "sweep n4 rc=$? rows $(wc -l < gpurun_out/${tag}_sweep_n4.jsonl)"
