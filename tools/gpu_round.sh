#!/bin/bash
# One GPU validation pass (run under gpurun): GPU tests, smoke, bench at N GPUs.
#   tools/gpu_round.sh <tag> <ngpus> [pytest -k expr]
tag=${1:-run}; n=${2:-1}; k=${3:-}
mkdir -p gpurun_out
if [ -n "$k" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$k" > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?"
else
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?"
fi
tail -5 gpurun_out/${tag}_pytest.log
if [ "$n" -gt 1 ]; then
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29555 \
    bench.py --gpus $n --steps 10 --warmup 3 > gpurun_out/${tag}_bench_n$n.jsonl 2> gpurun_out/${tag}_bench_n$n.err
  echo "bench rc=$?"
else
  timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/${tag}_bench_n1.jsonl 2> gpurun_out/${tag}_bench_n1.err
  echo "bench rc=$?"
fi
tail -c 3000 gpurun_out/${tag}_bench_n$n.jsonl; tail -5 gpurun_out/${tag}_bench_n$n.err
