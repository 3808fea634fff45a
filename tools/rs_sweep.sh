#!/bin/bash
# RS copy-engine chunking / parallel-peer sweep at N=4 (HZP_RS_CHUNKS, HZP_RS_PAR)
out=gpurun_out/r01b_rs_sweep_n4.jsonl; mkdir -p gpurun_out; : > $out
p=29600
for par in 0 1; do for ch in 1 2 4 8; do
  p=$((p+1))
  echo "{\"rs_par\": $par, \"rs_chunks\": $ch}" >> $out
  HZP_RS_PAR=$par HZP_RS_CHUNKS=$ch timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $p tools/bench_collectives.py --sizes-mb 64,1024 --depths 2 --precs 1 2>>gpurun_out/r01b_rs_sweep.err | grep '"rs", "path": "copy-engine"' >> $out
done; done
HZP_RS_PAR=1 timeout 600 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/r01b_rspar_multi.log 2>&1; echo rc=$? >> gpurun_out/r01b_rspar_multi.log
for par in 0 1; do
  HZP_RS_PAR=$par timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700+par)) bench.py --gpus 4 --no-cpu-baseline > gpurun_out/r01b_bench_n4_rspar$par.jsonl 2> gpurun_out/r01b_bench_n4_rspar$par.err
done
cat $out; tail -2 gpurun_out/r01b_rspar_multi.log; cat gpurun_out/r01b_bench_n4_rspar*.jsonl | cut -c1-300
