"""Probe (diagnostic, not product): can a multicast object be shared across
processes on this box, via a FABRIC handle (bytes) and/or a POSIX fd passed
with pidfd_getfd?  torchrun with 2 ranks."""
import ctypes
import os

import torch
import torch.distributed as dist
from cuda.bindings import driver as d


def chk(r):
    if isinstance(r, tuple):
        err, *rest = r
    else:
        err, rest = r, []
    if err != d.CUresult.CUDA_SUCCESS:
        raise RuntimeError(str(err))
    return rest[0] if len(rest) == 1 else rest


def main():
    rank = int(os.environ["RANK"])
    ws = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo")
    torch.zeros(1, device="cuda")
    chk(d.cuInit(0))
    dev = chk(d.cuDeviceGet(rank))
    for name, ht in (("fabric", d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_FABRIC),
                     ("posix_fd", d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR)):
        res = "ok"
        try:
            prop = d.CUmulticastObjectProp()
            prop.numDevices = ws
            prop.size = 2 << 20
            prop.handleTypes = ht
            blob = None
            if rank == 0:
                mc = chk(d.cuMulticastCreate(prop))
                if name == "fabric":
                    h = chk(d.cuMemExportToShareableHandle(mc, ht, 0))
                    blob = bytes(h.data)
                else:
                    fd = chk(d.cuMemExportToShareableHandle(mc, ht, 0))
                    blob = (os.getpid(), int(fd))
            objs = [None] * ws
            dist.all_gather_object(objs, blob)
            if rank != 0:
                if name == "fabric":
                    fh = d.CUmemFabricHandle()
                    fh.data = objs[0]
                    mc = chk(d.cuMemImportFromShareableHandle(fh, ht))
                else:
                    libc = ctypes.CDLL(None, use_errno=True)
                    pid, fd = objs[0]
                    pfd = libc.syscall(434, pid, 0)
                    lfd = libc.syscall(438, pfd, fd, 0)
                    if pfd < 0 or lfd < 0:
                        raise RuntimeError(f"pidfd {pfd} getfd {lfd} errno {ctypes.get_errno()}")
                    mc = chk(d.cuMemImportFromShareableHandle(lfd, ht))
            chk(d.cuMulticastAddDevice(mc, dev))
            dist.barrier()
            ap = d.CUmemAllocationProp()
            ap.type = d.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
            ap.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
            ap.location.id = rank
            ap.requestedHandleTypes = ht
            mem = chk(d.cuMemCreate(2 << 20, ap, 0))
            chk(d.cuMulticastBindMem(mc, 0, mem, 0, 2 << 20, 0))
            va = chk(d.cuMemAddressReserve(2 << 20, 0, 0, 0))
            chk(d.cuMemMap(va, 2 << 20, 0, mc, 0))
            acc = d.CUmemAccessDesc()
            acc.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
            acc.location.id = rank
            acc.flags = d.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
            chk(d.cuMemSetAccess(va, 2 << 20, [acc], 1))
            dist.barrier()
        except Exception as e:  # noqa: BLE001
            res = f"FAIL {e!r}"
        print(f"rank {rank}: {name}: {res}", flush=True)
        dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
