"""Run one tcgen05 GEMM layout a few times (for ncu captures).

    python tools/gemm_one.py M N K a_mn b_mn [iters]
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2510_20111_b200.engine import gemm_bf16  # noqa: E402


def main():
    M, N, K, a_mn, b_mn = (int(x) for x in sys.argv[1:6])
    iters = int(sys.argv[6]) if len(sys.argv) > 6 else 3
    dev = torch.device("cuda:0")
    A = (torch.randn(K, M, device=dev) if a_mn else torch.randn(M, K, device=dev)).to(torch.bfloat16)
    B = (torch.randn(K, N, device=dev) if b_mn else torch.randn(N, K, device=dev)).to(torch.bfloat16)
    C = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    for _ in range(iters):
        gemm_bf16(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, M if a_mn else K, N if b_mn else K, N,
                  a_mn, b_mn, 0, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
