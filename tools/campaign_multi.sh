#!/bin/bash
# Multi-GPU measurement campaign (run under gpurun --gpus 4): multi-GPU
# parity tests, the three BASELINE models at N = 2 and 4, the async / vanilla
# x prefetch-depth ablation (BASELINE configs[4]), and the
# AG / RS sweep.  Outputs under gpurun_out/<tag>_*.
tag=${1:-r02m}
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
timeout 1200 python -m pytest tests/test_gpu_multi.py -q > gpurun_out/${tag}_multi.log 2>&1; echo "multi rc=$?"; tail -1 gpurun_out/${tag}_multi.log
for n in 2 4; do
  run 13b_n$n $n
  run 7b_n$n $n --model 7b
  run moe_n$n $n --model moe
done
for m in async vanilla; do
  for d in 1 2 4; do run 13b_n4_${m}_d$d 4 --mode $m --depth $d; done
  run 7b_n4_${m} 4 --model 7b --mode $m
done
for n in 2 4; do
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 29950 tools/bench_collectives.py --sizes-mb 1,4,16,64,256,1024 --depths 1,2,4 --precs 1,0 \
    > gpurun_out/${tag}_sweep_n$n.jsonl 2> gpurun_out/${tag}_sweep_n$n.err
  echo "sweep n$n rc=$? rows $(wc -l < gpurun_out/${tag}_sweep_n$n.jsonl)"
done
