#!/bin/bash
# RS chunk floor at N=2 (one peer): HZP_RS_MIN_CHUNK_MB 64 (default) vs 8 (old 4 M-element floor)
mkdir -p gpurun_out; out=gpurun_out/r01e_rs_chunk_n2.jsonl; : > $out
for mb in 64 8; do
  echo "{\"rs_min_chunk_mb\": $mb}" >> $out
  HZP_RS_MIN_CHUNK_MB=$mb timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29950+mb)) tools/bench_collectives.py --sizes-mb 16,64,256,1024 --depths 2 --precs 1 2>>gpurun_out/r01e_rs_chunk_n2.err | grep '"rs", "path": "copy-engine"' >> $out
  HZP_RS_MIN_CHUNK_MB=$mb timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29970+mb)) bench.py --gpus 2 --no-cpu-baseline > gpurun_out/r01e_bench_n2_minchunk$mb.jsonl 2> gpurun_out/r01e_bench_n2_minchunk$mb.err
done
cat $out; cut -c1-160 gpurun_out/r01e_bench_n2_minchunk*.jsonl
