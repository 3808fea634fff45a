#!/bin/bash
# Final 1-GPU check of the shipped tree: the GPU test suite, smoke, the default bench line.
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/fc_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/fc_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fc_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/fc_bench.jsonl 2> gpurun_out/fc_bench.err; echo "bench rc=$?"; tail -c 400 gpurun_out/fc_bench.jsonl
