#!/bin/bash
# ncu evidence for the N = 1 step (run under gpurun, 1 GPU): the plain run
# first (must exit 0), then the serialised launch list of one step and full
# captures of the top kernels.  B200_PROFILING.md recipe.
tag=${1:-r02}
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/${tag}_ncu_plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/${tag}_ncu_plain.log; exit 1; }
# one step = the warm-up step's launches after init: skip init + 1 step, list ~1 step
ncu --metrics gpu__time_duration.sum --clock-control none -s 1800 -c 1800 --csv \
    --log-file gpurun_out/${tag}_ncu_launches.csv $CMD > gpurun_out/${tag}_ncu_launches.log 2>&1
echo "launch list rc=$?"
for k in "gemm_tc_kernel:300" "attn_fwd2_kernel:10" "attn_bwd_kernel:10" "z1_adam_kernel:30" "ln_bwd_dx_kernel:10" "colred_kernel:10"; do
  name=${k%%:*}; skip=${k##*:}
  ncu --set full --clock-control none --import-source on -k regex:$name -s $skip -c 1 \
      -o gpurun_out/${tag}_ncu_$name $CMD > gpurun_out/${tag}_ncu_$name.log 2>&1
  echo "$name rc=$?"
done
# GEMM DRAM traffic per launch (bench.py roofline.traffic): per-shape launch
# counts of one step + ncu DRAM bytes of every gemm_tc launch of that step
python tools/gemm_traffic.py shapes gpurun_out/${tag}_gemm_shapes.json > /dev/null 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:gemm_tc --csv --log-file gpurun_out/${tag}_gemm_dram.csv python tools/gemm_traffic.py run \
    > gpurun_out/${tag}_gemm_dram.log 2>&1
echo "gemm dram rc=$?"
