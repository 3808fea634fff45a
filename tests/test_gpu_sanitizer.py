"""compute-sanitizer over the engine's step (race / sync / memory
checking of the device-flag protocol and the kernels).

Opt-in: one tool per run, selected with HZP_SANITIZER=memcheck|racecheck|
synccheck (B200_PROFILING.md: at most one sanitizer tool per GPU session;
several in one call have left a GPU unusable).  With >= 2 GPUs the tool wraps
a 2-process step (multicast AG / RS, GradReady / AgReady / RsDone flags,
fused Z1 over NVLink); on one GPU it wraps the emulated 2-rank step.
Round 2: compute-sanitizer is closed on this GPU pool (the first memcheck call
was refused, profiles/r02_sanitizer_closed.txt); the flag protocol's race
check is test_gpu_multi.py::test_multiprocess_gpt_async_equals_serialised
(async vs fully serialised runs, bitwise), and memory safety rests on the
bitwise parity tests against the oracle (every shard, ragged sizes)."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

TOOL = os.environ.get("HZP_SANITIZER", "")

EMULATED = r"""
import sys, numpy as np
sys.path.insert(0, %r)
from oracle import load_oracle
from paper_2510_20111_b200 import EngineConfig, HzpEngine, ParallelConfig
o = load_oracle()
dims, dp = [64, 128, 64], 2
for prec in (0, 1):
    st = o.shard_init(dims, dp, 2, 2, 2, 2024, bool(prec))
    e = HzpEngine(EngineConfig(model=0, precision=prec, dims=dims, batch=16, num_microbatches=2,
                               par=ParallelConfig(dp=dp, z1=2, z2=2, z3=2)))
    e.load_state(st)
    for step in range(2):
        e.step(o.make_inputs(dims, dp, 2, 16, 2024, step))
    e.close()
print("sanitized step ok")
"""


def _ngpu():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.skipif(TOOL not in ("memcheck", "racecheck", "synccheck"),
                    reason="opt-in: HZP_SANITIZER=memcheck|racecheck|synccheck (one tool per GPU session)")
def test_step_under_compute_sanitizer(gpu, tmp_path):
    san = ["compute-sanitizer", "--tool", TOOL, "--error-exitcode", "9", "--print-limit", "50"]
    if _ngpu() >= 2:
        cmd = san + ["--target-processes", "all", sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                     "--nproc-per-node=2", "--master-addr", "127.0.0.1", "--master-port", "29680",
                     os.path.join(ROOT, "tests", "mp_worker.py"), "2", "2", "2", "1"]
    else:
        script = tmp_path / "emulated.py"
        script.write_text(EMULATED % ROOT)
        cmd = san + [sys.executable, str(script)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1800)
    log = r.stdout[-20000:] + "\n" + r.stderr[-20000:]
    out = os.environ.get("HZP_SANITIZER_LOG")
    if out:
        with open(out, "w") as fh:
            fh.write(" ".join(cmd) + "\n" + log)
    print(log[-4000:])
    assert r.returncode == 0, log[-4000:]
    assert "ERROR SUMMARY: 0 errors" in log
