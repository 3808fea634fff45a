#!/bin/bash
# One compute-sanitizer tool per gpurun call (B200_PROFILING.md):
#   gpurun [--gpus 2] -- tools/sanitize.sh memcheck|racecheck|synccheck TAG
# 1 GPU: the emulated 2-rank step (every kernel incl. AG / RS / Z1 unicast
# models); 2 GPUs: the 2-process step (NVLS collectives + the flag protocol).
tool=$1; tag=${2:-r02}
mkdir -p gpurun_out
HZP_SANITIZER=$tool HZP_SANITIZER_LOG=gpurun_out/${tag}_sanitizer_${tool}.txt \
  timeout 1500 python -m pytest tests/test_gpu_sanitizer.py -q -x > gpurun_out/${tag}_sanitizer_${tool}.pytest 2>&1
echo "$tool rc=$?"; tail -1 gpurun_out/${tag}_sanitizer_${tool}.pytest
grep -E "ERROR SUMMARY|sanitized step ok|rank .*: OK" gpurun_out/${tag}_sanitizer_${tool}.txt | head -5
