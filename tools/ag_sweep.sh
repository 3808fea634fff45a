#!/bin/bash
# AG copy-engine: one stream (rotated owners) vs one stream per owner (HZP_AG_PAR), N=4
mkdir -p gpurun_out; out=gpurun_out/r01d_ag_sweep_n4.jsonl; : > $out
for par in 0 1; do
  echo "{\"ag_par\": $par}" >> $out
  HZP_AG_PAR=$par timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29900+par)) tools/bench_collectives.py --sizes-mb 16,64,256,1024 --depths 1,2 --precs 1 2>>gpurun_out/r01d_ag_sweep.err | grep '"copy-engine"' >> $out
done
HZP_AG_PAR=1 timeout 600 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/r01d_agpar_multi.log 2>&1; echo rc=$? >> gpurun_out/r01d_agpar_multi.log
HZP_AG_PAR=1 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29910 bench.py --gpus 4 --no-cpu-baseline > gpurun_out/r01d_bench_n4_agpar1.jsonl 2> gpurun_out/r01d_bench_n4_agpar1.err
cat $out; tail -2 gpurun_out/r01d_agpar_multi.log; cut -c1-200 gpurun_out/r01d_bench_n4_agpar1.jsonl
