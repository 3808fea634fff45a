"""Probe the box: multicast (NVLS) support, handle types, NVLink topology and
whether torch symmetric memory exposes a multicast pointer.  Run under
torchrun with 2+ ranks (diagnostic only; not part of the product)."""
import ctypes
import os
import subprocess

import torch
import torch.distributed as dist
from cuda.bindings import driver as d


def main():
    rank = int(os.environ.get("RANK", "0"))
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl")
    d.cuInit(0)
    _, dev = d.cuDeviceGet(rank)
    A = d.CUdevice_attribute
    attrs = {}
    for n in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED",
              "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED"):
        attrs[n] = d.cuDeviceGetAttribute(getattr(A, n), dev)
    print(f"rank {rank}: {attrs}", flush=True)
    # pidfd_getfd availability (syscall 438)
    libc = ctypes.CDLL(None, use_errno=True)
    pfd = libc.syscall(434, os.getpid(), 0)  # pidfd_open
    fd2 = libc.syscall(438, pfd, 1, 0) if pfd >= 0 else -1
    print(f"rank {rank}: pidfd_open={pfd} pidfd_getfd={fd2} errno={ctypes.get_errno()}", flush=True)
    try:
        import torch.distributed._symmetric_memory as sm
        t = sm.empty(1 << 20, dtype=torch.bfloat16, device=f"cuda:{rank}")
        h = sm.rendezvous(t, dist.group.WORLD.group_name)
        print(f"rank {rank}: symm mem ok, multicast_ptr={getattr(h, 'multicast_ptr', None)}", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"rank {rank}: symm mem failed: {e!r}", flush=True)
    x = torch.ones(1 << 26, device=f"cuda:{rank}", dtype=torch.bfloat16)
    dist.all_reduce(x)
    torch.cuda.synchronize()
    dist.barrier()
    if rank == 0:
        print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout, flush=True)
        print(subprocess.run(["nvidia-smi", "-q", "-d", "FABRIC"], capture_output=True, text=True).stdout[:3000],
              flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
