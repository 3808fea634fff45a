"""Raw NVLink peer-copy ceilings on this box (one process, 2+ GPUs visible):
copy-engine cudaMemcpyPeer (torch cross-device copy_) one and both
directions, to calibrate the AG / RS bus-bandwidth fractions."""
import json
import torch

def timeit(fn, iters=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize(0); torch.cuda.synchronize(1)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(torch.cuda.current_stream(0))
    for _ in range(iters):
        fn()
    e1.record(torch.cuda.current_stream(0))
    torch.cuda.synchronize(0); torch.cuda.synchronize(1)
    return e0.elapsed_time(e1) / iters

for mb in (64, 256, 1024):
    n = mb * (1 << 20)
    a0 = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    a1 = torch.empty(n, dtype=torch.uint8, device="cuda:1")
    b0 = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    b1 = torch.empty(n, dtype=torch.uint8, device="cuda:1")
    with torch.cuda.device(0):
        ms = timeit(lambda: a0.copy_(a1, non_blocking=True))  # pull 1 -> 0
    print(json.dumps({"op": "ce_pull_1to0", "MB": mb, "ms": round(ms, 4), "GBps": round(n / ms / 1e6, 1)}))
    s1 = torch.cuda.Stream(device=1)
    def both():
        a0.copy_(a1, non_blocking=True)
        with torch.cuda.stream(s1):
            b1.copy_(b0, non_blocking=True)
    with torch.cuda.device(0):
        ms = timeit(both)
    print(json.dumps({"op": "ce_bidir", "MB": mb, "ms": round(ms, 4), "GBps_per_dir": round(n / ms / 1e6, 1)}))
