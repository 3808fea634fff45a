"""Multi-GPU (one process per GPU; peer arenas mapped over NVLink, AG / RS
through NVLS multicast) parity runs.
Skipped unless the box has >= 2 GPUs; the host-side logic of the same path
is covered on CPU by tests/test_multiproc_cpu.py (gloo, world_size 2)."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def _ngpu():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.parametrize("n,z", [(2, (2, 2, 2)), (2, (2, 2, 1)), (4, (4, 2, 2)), (4, (4, 4, 4))])
@pytest.mark.parametrize("prec", [0, 1])
def test_multiprocess_kernels_match_oracle(n, z, prec):
    if _ngpu() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + n * 10 + prec),
           os.path.join(ROOT, "tests", "mp_worker.py"), *map(str, z), str(prec), "kernels"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0
    assert r.stdout.count(": OK") == n


@pytest.mark.parametrize("n,z,reuse", [(2, (2, 2, 2), 0), (2, (2, 1, 2), 0), (2, (2, 2, 1), 0), (4, (4, 2, 2), 0),
                                       (4, (4, 4, 4), 0), (4, (2, 4, 2), 0), (2, (2, 2, 2), 1), (4, (4, 2, 2), 1)])
@pytest.mark.parametrize("prec", [0, 1])
def test_multiprocess_step_matches_oracle(n, z, reuse, prec):
    """reuse=1: the CLI's R3 reuse (microbatch 1's forward reads microbatch 0's
    gathered layers from the side cache) over real NVLink peers."""
    if _ngpu() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + n * 10 + prec + 4 * reuse),
           os.path.join(ROOT, "tests", "mp_worker.py"), *map(str, z), str(prec)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300,
                       env=dict(os.environ, HZP_TEST_REUSE=str(reuse)))
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0
    assert r.stdout.count(": OK") == n


@pytest.mark.parametrize("n,z", [(2, (2, 2, 2)), (4, (4, 2, 2))])
def test_multiprocess_ragged_shards_match_oracle(n, z):
    """P = 23 over 2 / 4 ranks: padded Z3 / Z1 shards, a layer smaller than a
    shard, unaligned spans of a few elements (unicast element stores beside
    the multicast vectors)."""
    if _ngpu() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29640 + n),
           os.path.join(ROOT, "tests", "mp_worker.py"), *map(str, z), "0"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300,
                       env=dict(os.environ, HZP_TEST_DIMS="5,3,2"))
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0
    assert r.stdout.count(": OK") == n


@pytest.mark.parametrize("n,z", [(2, (2, 2, 2)), (4, (4, 2, 2)), (4, (4, 4, 4))])
def test_multiprocess_gpt_async_equals_serialised(n, z):
    """Race check of the cross-GPU flag protocol (compute-sanitizer is closed
    on this pool): the bf16 GPT step, dense and MoE, async twice and fully
    serialised (HZP_DEBUG_SYNC) once — bitwise the same parameters, Adam state
    and losses on every rank (tests/mp_worker.py gpt_race)."""
    if _ngpu() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29700 + n * 10 + z[1]),
           os.path.join(ROOT, "tests", "mp_worker.py"), *map(str, z), "1", "gpt_race"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0
    assert r.stdout.count("OK gpt race") == n
