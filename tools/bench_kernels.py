"""Kernel microbenchmarks (CUDA-event timed, warm, inputs > L2 where it matters).

  python tools/bench_kernels.py gemm        # tcgen05 GEMM TFLOP/s per layout
  python tools/bench_kernels.py comm        # AG/RS/Z1 GB/s (emulated ranks = HBM)
Prints one JSON object per line.
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2510_20111_b200.engine import gemm_bf16  # noqa: E402


def timeit(fn, iters=20, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def bench_gemm():
    dev = torch.device("cuda:0")
    if os.environ.get("HZP_GEMM_QUICK"):
        shapes_q = [(8192, 8192, 2048), (8192, 2048, 8192)]
        for (M, N, K) in shapes_q:
            A = torch.randn(M, K, device=dev).to(torch.bfloat16)
            B = torch.randn(N, K, device=dev).to(torch.bfloat16)
            C = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
            ms = timeit(lambda: gemm_bf16(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, K, K, N, 0, 0, 0,
                                          torch.cuda.current_stream().cuda_stream))
            print(json.dumps({"kernel": "gemm_tc_bf16", "M": M, "N": N, "K": K, "ms": round(ms, 4),
                              "tflops": round(2 * M * N * K / ms / 1e9, 1)}), flush=True)
        return
    shapes = [(8192, 8192, 8192), (8192, 6144, 2048), (8192, 2048, 2048), (8192, 8192, 2048),
              (8192, 2048, 8192), (2048, 8192, 8192), (6144, 2048, 8192)]
    for (M, N, K) in shapes:
        for a_mn, b_mn in ((0, 0), (0, 1), (1, 1)):
            A = torch.randn(K, M, device=dev).to(torch.bfloat16) if a_mn else torch.randn(M, K, device=dev).to(torch.bfloat16)
            B = torch.randn(K, N, device=dev).to(torch.bfloat16) if b_mn else torch.randn(N, K, device=dev).to(torch.bfloat16)
            C = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
            lda = M if a_mn else K
            ldb = N if b_mn else K
            ms = timeit(lambda: gemm_bf16(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, lda, ldb, N,
                                          a_mn, b_mn, 0, torch.cuda.current_stream().cuda_stream))
            At = A.t() if a_mn else A
            Bt = B if b_mn else B.t()
            ms_t = timeit(lambda: torch.matmul(At, Bt))
            tf = 2 * M * N * K / ms / 1e9
            print(json.dumps({"kernel": "gemm_tc_bf16", "M": M, "N": N, "K": K, "a_mn": a_mn,
                              "b_mn": b_mn, "ms": round(ms, 4), "tflops": round(tf, 1),
                              "cublas_tflops": round(2 * M * N * K / ms_t / 1e9, 1)}), flush=True)


def bench_comm():
    from paper_2510_20111_b200 import EngineConfig, HzpEngine, ParallelConfig
    # emulated dp ranks on one GPU (the unicast model of the NVLS kernels: the
    # owner stores into every member's slot, the reducer sums the members'
    # slots in order), so this measures HBM-side efficiency, not NVLink
    for dims, dp in (([4096, 16384, 4096], 4), ([4096, 16384, 4096], 8)):
        eng = HzpEngine(EngineConfig(model=0, precision=1, dims=dims, batch=8,
                                     par=ParallelConfig(dp=dp, z1=dp, z2=dp, z3=dp)))
        eng.init_random()
        off, n = eng.layers[0]
        for op in ("ag", "rs", "z1"):
            if op == "z1":
                ms = timeit(eng.z1_adam_step, iters=5)
                gbs = eng.s1 * dp * 30 / ms / 1e6  # 30 B / element of every driven rank's chunk
            else:
                ms = eng.collective_time(op, 0, 10)
                # AG: layer read once per owner span + written dp times; RS: dp
                # bf16 reads + 8 B fp32 grad read-modify-write per element
                gbs = (n * 2 * (1 + dp) if op == "ag" else n * (2 * dp + 8)) / ms / 1e6
            print(json.dumps({"kernel": op, "dp": dp, "layer_elems": n, "ms": round(ms, 4),
                              "GBps_hbm": round(gbs, 1)}), flush=True)
        eng.close()


def bench_epi():
    """The step's epilogue variants on their real shapes (8 warps, TMA store)."""
    import ctypes as C
    from paper_2510_20111_b200 import _native as N
    dev = torch.device("cuda:0")
    p = lambda t: C.c_void_p(t.data_ptr() if t is not None else 0)  # noqa: E731

    def ex(A, B, Cm, M, N_, K, act=0, bias=None, aux=None, resid=None, out_bf16=1, mode=0, b_mn=0):
        N.check(N.lib.hzp_gemm_bf16_ex(p(A), p(B), p(Cm), M, N_, K, K, N_ if b_mn else K, N_, 0, b_mn, mode,
                                       out_bf16, act, p(bias), p(aux), N_ if aux is not None else 0, p(resid),
                                       N_ if resid is not None else 0, None, 1.0,
                                       C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    for (M, N_, K, what) in ((8192, 8192, 2048, "plain"), (8192, 8192, 2048, "bias"), (8192, 8192, 2048, "gelu"),
                             (8192, 8192, 2048, "gelugrad"), (8192, 6144, 2048, "bias"),
                             (8192, 2048, 2048, "bias+resid"), (8192, 2048, 8192, "bias+resid")):
        A = torch.randn(M, K, device=dev).to(torch.bfloat16)
        B = torch.randn(N_, K, device=dev).to(torch.bfloat16)
        Cm = torch.empty(M, N_, device=dev, dtype=torch.bfloat16)
        bias = torch.randn(N_, device=dev).to(torch.bfloat16)
        aux = torch.randn(M, N_, device=dev).to(torch.bfloat16)
        kw = {"plain": {}, "bias": dict(bias=bias), "gelu": dict(act=2, bias=bias, aux=aux),
              "gelugrad": dict(act=4, aux=aux), "bias+resid": dict(bias=bias, resid=aux)}[what]
        ms = timeit(lambda: ex(A, B, Cm, M, N_, K, **kw))
        print(json.dumps({"kernel": "gemm_epi", "M": M, "N": N_, "K": K, "epilogue": what, "ms": round(ms, 4),
                          "tflops": round(2 * M * N_ * K / ms / 1e9, 1)}), flush=True)


def bench_attn():
    import ctypes as C
    from paper_2510_20111_b200 import _native as N
    dev = torch.device("cuda:0")
    b, nh, S, hd = 4, 16, 2048, 128
    h = nh * hd
    qkv = (torch.randn(b, S, 3 * h, device=dev) * 0.5).to(torch.bfloat16)
    do = (torch.randn(b, S, h, device=dev) * 0.1).to(torch.bfloat16)
    O = torch.zeros(b, S, h, device=dev, dtype=torch.bfloat16)
    lse = torch.zeros(b * nh, S, device=dev)
    D = torch.zeros(2, b * nh, S, device=dev)
    dqkv = torch.zeros(b, S, 3 * h, device=dev, dtype=torch.bfloat16)
    dsT = torch.zeros(b * nh, S, S, device=dev, dtype=torch.bfloat16)
    p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    fwd = lambda: N.check(N.lib.hzp_attention_fwd(p(qkv), p(O), p(lse), b, nh, S, h, st))  # noqa: E731
    bwd = lambda: N.check(N.lib.hzp_attention_bwd(p(qkv), p(O), p(do), p(lse), p(D), p(dqkv), None,  # noqa: E731
                                                  b, nh, S, h, st))
    bwd_legacy = lambda: N.check(N.lib.hzp_attention_bwd(p(qkv), p(O), p(do), p(lse), p(D), p(dqkv),  # noqa: E731
                                                         p(dsT), b, nh, S, h, st))
    flops_fwd = 4.0 * b * nh * S * S * hd / 2  # causal QK^T + PV
    # backward algorithmic FLOPs: S^T, dP^T, dV, dK, dQ = 2.5 x forward (the
    # dQ pass's recomputed S / dP products are not counted)
    for name, fn, fl in (("attn_fwd", fwd, flops_fwd),
                         ("attn_bwd (rowdot + dK/dV + dQ pass, P/dS in TMEM)", bwd, 2.5 * flops_fwd),
                         ("attn_bwd legacy (rowdot + dK/dV + dS^T in HBM + dQ GEMM)", bwd_legacy, 2.5 * flops_fwd)):
        ms = timeit(fn)
        print(json.dumps({"kernel": name, "b": b, "nh": nh, "S": S, "ms": round(ms, 4),
                          "tflops_causal": round(fl / ms / 1e9, 1)}), flush=True)
    ms = timeit(lambda: torch.nn.functional.scaled_dot_product_attention(
        qkv[..., :h].view(b, S, nh, hd).transpose(1, 2), qkv[..., h:2 * h].view(b, S, nh, hd).transpose(1, 2),
        qkv[..., 2 * h:].view(b, S, nh, hd).transpose(1, 2), is_causal=True))
    print(json.dumps({"kernel": "torch_sdpa_fwd (comparator)", "ms": round(ms, 4),
                      "tflops_causal": round(flops_fwd / ms / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "gemm"
    {"gemm": bench_gemm, "comm": bench_comm, "attn": bench_attn, "epi": bench_epi}[what]()
