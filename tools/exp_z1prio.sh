#!/bin/bash
# EXPERIMENT (1 GPU): optimizer-stream priority vs the optimizer tail at N = 1.
tag=${1:-z1p}
mkdir -p gpurun_out
s() { python - "$1" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); e = d["exposed_comm"]
    print(sys.argv[1], d["value"], "ms", d["ms_per_step"], "idle", e["frac"], e.get("idle_by_next_task_ms"), "clk", d["clocks"]["sm_mhz"], "z1", (d.get("z1_adam") or {}).get("ms"))
except Exception as ex: print(sys.argv[1], "unparsed", ex)
PY
}
for m in 7b 1.3b; do
  for p in 0 1 2; do
    HZP_EXP_OPTPRIO=$p timeout 900 python bench.py --model $m --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_${m}_p$p.jsonl 2> gpurun_out/${tag}_${m}_p$p.err; s gpurun_out/${tag}_${m}_p$p.jsonl
  done
  timeout 900 python bench.py --model $m --steps 5 --warmup 3 --no-cpu-baseline --mode vanilla > gpurun_out/${tag}_${m}_van.jsonl 2> gpurun_out/${tag}_${m}_van.err; s gpurun_out/${tag}_${m}_van.jsonl
done
