#!/bin/bash
# Single-GPU measurement campaign (run under gpurun): the GPU test suite,
# smoke, the N = 1 headline (twice), the 7B / MoE configs at N = 1, the
# same-config lines of both arms, the reference arm, kernel microbenches.
tag=${1:-r02s}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${tag}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"
summ() { python - "$1" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], d["value"], d.get("unit"), "ms", d.get("ms_per_step"), "e2e", (d.get("e2e") or {}).get("value"),
          "clk", (d.get("clocks") or {}).get("sm_mhz"), "roof", (d.get("roofline") or {}).get("frac"))
except Exception as ex:
    print(sys.argv[1], "unparsed", ex)
PY
}
b() { local name=$1; shift; timeout 1200 python bench.py "$@" > gpurun_out/${tag}_$name.jsonl 2> gpurun_out/${tag}_$name.err; summ gpurun_out/${tag}_$name.jsonl; }
b n1_a --steps 20 --warmup 5
b n1_b --steps 20 --warmup 5
b n1_vanilla --steps 20 --warmup 5 --mode vanilla --no-cpu-baseline
b 7b_n1 --model 7b --steps 5 --warmup 3 --no-cpu-baseline
b moe_n1 --model moe --steps 5 --warmup 3 --no-cpu-baseline
b mlp --model mlp
b mlp_ref --model mlp --impl reference
b mlpslice --model mlp-slice
b mlpslice_ref --model mlp-slice --impl reference
b ref --impl reference --steps 2 --warmup 1
timeout 600 python tools/bench_kernels.py attn > gpurun_out/${tag}_kernels_attn.jsonl 2>&1
timeout 600 python tools/bench_kernels.py comm > gpurun_out/${tag}_kernels_comm.jsonl 2>&1
cat gpurun_out/${tag}_kernels_attn.jsonl gpurun_out/${tag}_kernels_comm.jsonl | cut -c1-200
