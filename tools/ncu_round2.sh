#!/bin/bash
# ncu evidence for the final N = 1 step (run under gpurun, 1 GPU): the plain
# run first (must exit 0), the serialised launch list of about one step, and
# full captures of the kernels changed in round 2's second half.
tag=${1:-r02b}
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/${tag}_ncu_plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/${tag}_ncu_plain.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -s 1800 -c 1800 --csv \
    --log-file gpurun_out/${tag}_ncu_launches.csv $CMD > gpurun_out/${tag}_ncu_launches.log 2>&1
echo "launch list rc=$?"
for k in "attn_bwd_kernel:10" "attn_fwd2_kernel:10" "ln_bwd_fused_kernel:10" "z1_adam_kernel:30"; do
  name=${k%%:*}; skip=${k##*:}
  ncu --set full --clock-control none --import-source on -k regex:$name -s $skip -c 1 \
      -o gpurun_out/${tag}_ncu_$name $CMD > gpurun_out/${tag}_ncu_$name.log 2>&1
  echo "$name rc=$?"
done
