#!/bin/bash
# One GPU validation pass (run under gpurun): GPU tests, bench at N GPUs and,
# for N > 1, the N = 1 bench too.
#   tools/gpu_round.sh <tag> <ngpus> [pytest -k expr]
tag=${1:-run}; n=${2:-1}; k=${3:-}
mkdir -p gpurun_out
if [ "$k" != "none" ]; then
  if [ -n "$k" ]; then
    timeout 1200 python -m pytest tests -m gpu -x -q -k "$k" > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?"
  else
    timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?"
  fi
  tail -5 gpurun_out/${tag}_pytest.log
fi
summ() { python - "$1" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    c = d.get("collectives") or {}
    print(sys.argv[1], "value", d["value"], "ms", d["ms_per_step"], "idle", d["exposed_comm"]["frac"],
          "gemm_busy_TF", d["roofline"]["achieved_over_busy"], "clk", d["clocks"]["sm_mhz"],
          "e2e", round(d["e2e"]["value"], 1), "ag", (c.get("ag") or {}).get("ms"), "rs", (c.get("rs") or {}).get("ms"),
          "z1", d["z1_adam"]["ms"])
except Exception as e:
    print(sys.argv[1], "unparsed", e)
PY
}
if [ "$n" -gt 1 ]; then
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29555 \
    bench.py --gpus $n --steps 10 --warmup 3 ${BENCH_ARGS} > gpurun_out/${tag}_bench_n$n.jsonl 2> gpurun_out/${tag}_bench_n$n.err
  echo "bench n$n rc=$?"; summ gpurun_out/${tag}_bench_n$n.jsonl
fi
timeout 900 python bench.py --steps 10 --warmup 3 ${BENCH_ARGS} > gpurun_out/${tag}_bench_n1.jsonl 2> gpurun_out/${tag}_bench_n1.err
echo "bench n1 rc=$?"; summ gpurun_out/${tag}_bench_n1.jsonl
tail -3 gpurun_out/${tag}_bench_n1.err
