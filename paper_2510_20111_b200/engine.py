"""Device engine API — the B200 replacement for the reference's numerical
workflow (shard_init / train_step_hzp / gather_params, train.hpp:105-135).

``HzpEngine`` wraps one ``hzp_ctx``: one GPU, driving either every dp rank
(emulation: all ranks' buffers on one device, used for single-GPU parity) or
exactly one rank (``my_rank``; one process per GPU, peers wired through CUDA
IPC after an all-gather of handles over torch.distributed).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _native as N
from .hzp import ParallelConfig

MLP, GPT = 0, 1
FP32, BF16 = 0, 1
F_PARAM, F_GRAD, F_MASTER, F_MOM, F_VAR = range(5)


@dataclass
class EngineConfig:
    model: int = MLP
    precision: int = FP32
    dims: List[int] = field(default_factory=lambda: [12, 20, 8])
    gpt_layers: int = 0
    gpt_hidden: int = 0
    gpt_heads: int = 0
    gpt_ffn: int = 0
    gpt_vocab: int = 0
    gpt_seq: int = 0
    batch: int = 4
    num_microbatches: int = 1
    par: ParallelConfig = field(default_factory=ParallelConfig)
    prelaunch_depth: int = 2   # hzpsim.cpp:95 default
    rs_slots: int = 1          # hzpsim.cpp:96 default
    wgrad_slots: int = 2
    mode: int = 1              # async
    lr: float = 1e-3           # AdamParams defaults (train.hpp:22-27)
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    grad_scale: float = 1.0
    device: int = 0
    my_rank: int = -1          # -1: emulate all dp ranks on `device`
    timeline: int = 0
    gpt_experts: int = 0       # GPT: MoE feed-forward with this many experts (0 = dense)
    gpt_topk: int = 2
    gpt_capacity: int = 0      # slots per expert per microbatch (0 = auto)
    reuse: int = 0             # CLI parameter reuse (R3 side cache for later forwards)
    recompute: int = 0         # activation recomputation (FWD-recompute before each BWD)
    gpt_swiglu: int = 0        # GPT: SwiGLU feed-forward (dense blocks and MoE experts)

    def c(self) -> N.hzp_engine_config:
        c = N.hzp_engine_config()
        c.model, c.precision = self.model, self.precision
        c.num_dims = len(self.dims)
        for i, d in enumerate(self.dims):
            c.dims[i] = d
        c.gpt_layers, c.gpt_hidden, c.gpt_heads = self.gpt_layers, self.gpt_hidden, self.gpt_heads
        c.gpt_ffn, c.gpt_vocab, c.gpt_seq = self.gpt_ffn, self.gpt_vocab, self.gpt_seq
        c.batch, c.num_microbatches = self.batch, self.num_microbatches
        c.par = self.par.c()
        c.prelaunch_depth, c.rs_slots, c.wgrad_slots = self.prelaunch_depth, self.rs_slots, self.wgrad_slots
        c.mode = self.mode
        c.lr, c.beta1, c.beta2, c.eps = self.lr, self.beta1, self.beta2, self.eps
        c.grad_scale, c.device, c.my_rank, c.timeline = self.grad_scale, self.device, self.my_rank, self.timeline
        c.gpt_experts, c.gpt_topk, c.gpt_capacity = self.gpt_experts, self.gpt_topk, self.gpt_capacity
        c.reuse = self.reuse
        c.recompute = self.recompute
        c.gpt_swiglu = self.gpt_swiglu
        return c


class HzpEngine:
    def __init__(self, cfg: EngineConfig):
        self.cfg = cfg
        h = C.c_void_p()
        N.check(N.lib.hzp_ctx_create(C.byref(cfg.c()), C.byref(h)))
        self._h = h
        P, s1, s2, s3 = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        nl = C.c_int()
        N.check(N.lib.hzp_ctx_layout(h, C.byref(P), C.byref(s1), C.byref(s2), C.byref(s3), C.byref(nl)))
        self.P, self.s1, self.s2, self.s3 = P.value, s1.value, s2.value, s3.value
        self.num_layers = nl.value
        self.layers = []
        for l in range(self.num_layers):
            o, n = C.c_int64(), C.c_int64()
            N.check(N.lib.hzp_ctx_layer_range(h, l, C.byref(o), C.byref(n)))
            self.layers.append((o.value, n.value))
        self.local_ranks = list(range(cfg.par.dp)) if cfg.my_rank < 0 else [cfg.my_rank]

    def close(self):
        if getattr(self, "_h", None):
            N.lib.hzp_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    # ---- multi-process wiring -------------------------------------------------
    def ipc_handle(self) -> bytes:
        buf = (C.c_char * 256)()
        n = C.c_size_t(256)
        N.check(N.lib.hzp_ctx_ipc_handle(self._h, buf, C.byref(n)))
        return bytes(buf[: n.value])

    def open_peers(self, handles: List[bytes]) -> None:
        hl = len(handles[0])
        blob = b"".join(handles)
        N.check(N.lib.hzp_ctx_open_peers(self._h, blob, hl, len(handles)))

    def connect(self, group=None) -> None:
        """Exchange IPC handles over torch.distributed (control plane only)."""
        import torch.distributed as dist
        mine = self.ipc_handle()
        allh: List[Optional[bytes]] = [None] * dist.get_world_size(group)
        dist.all_gather_object(allh, mine, group=group)
        self.open_peers(allh)
        dist.barrier(group=group)

    # ---- ShardedState mirror ---------------------------------------------------
    def _field_shape(self, f):
        if f == F_PARAM:
            return self.s3, (np.uint16 if self.cfg.precision == BF16 else np.float32)
        if f == F_GRAD:
            return self.s2, np.float32
        return self.s1, np.float32

    def upload(self, rank: int, f: int, arr: np.ndarray) -> None:
        n, dt = self._field_shape(f)
        a = np.ascontiguousarray(arr, dtype=dt)
        assert a.size == n, (a.size, n)
        N.check(N.lib.hzp_state_upload(self._h, rank, f, a.ctypes.data, n))

    def download(self, rank: int, f: int) -> np.ndarray:
        n, dt = self._field_shape(f)
        a = np.empty(n, dtype=dt)
        N.check(N.lib.hzp_state_download(self._h, rank, f, a.ctypes.data, n))
        return a

    def set_step(self, rank: int, step: int) -> None:
        N.check(N.lib.hzp_state_set_step(self._h, rank, step))

    def get_step(self, rank: int) -> int:
        v = C.c_int()
        N.check(N.lib.hzp_state_get_step(self._h, rank, C.byref(v)))
        return v.value

    # ---- checkpoint (save / restore ShardedState per rank) ------------
    def driven_ranks(self) -> List[int]:
        if self.cfg.my_rank >= 0:
            return [self.cfg.my_rank]
        return list(range(self.cfg.par.dp))

    def save_checkpoint(self, path: str) -> None:
        """One .npz per driven rank: param (working dtype), grad, master, m, v
        shards and the Adam step — the reference's ShardedState (train.hpp:73-83).

        ``grad`` is this rank's Z2 shard as the reduce-scatter left it.  With
        DZP replicas (dp / z2 > 1) the reference all-reduces it across the
        replicas (train.cpp:326-341); here that sum is formed only inside the
        fused Z1 kernel (registers), so the saved ``grad`` is the per-replica
        shard, not the reference's all-reduced one.  Resuming is unaffected:
        the first reduce-scatter of the next step overwrites it."""
        import os
        os.makedirs(path, exist_ok=True)
        for r in self.driven_ranks():
            np.savez(os.path.join(path, f"rank{r}.npz"), param=self.download(r, F_PARAM),
                     grad=self.download(r, F_GRAD), master=self.download(r, F_MASTER),
                     mom=self.download(r, F_MOM), var=self.download(r, F_VAR),
                     adam_step=np.int64(self.get_step(r)), P=np.int64(self.P),
                     layout=np.array([self.cfg.par.dp, self.cfg.par.z1, self.cfg.par.z2, self.cfg.par.z3]),
                     precision=np.int64(self.cfg.precision), model=np.int64(self.cfg.model),
                     layers=np.array(self.layers, dtype=np.int64).reshape(-1, 2))

    def load_checkpoint(self, path: str) -> None:
        import os
        for r in self.driven_ranks():
            z = np.load(os.path.join(path, f"rank{r}.npz"))
            if int(z["P"]) != self.P or list(z["layout"]) != [self.cfg.par.dp, self.cfg.par.z1,
                                                              self.cfg.par.z2, self.cfg.par.z3]:
                raise ValueError("checkpoint layout does not match this ctx")
            if "precision" not in z or int(z["precision"]) != self.cfg.precision:
                raise ValueError("checkpoint precision does not match this ctx "
                                 "(a bf16 working copy would be reinterpreted as fp32 or truncated)")
            if int(z["model"]) != self.cfg.model or [tuple(x) for x in z["layers"]] != \
                    [tuple(x) for x in self.layers]:
                raise ValueError("checkpoint model / layer table does not match this ctx")
            if z["param"].dtype != self._field_shape(F_PARAM)[1]:
                raise ValueError("checkpoint param dtype does not match the working precision")
            self.upload(r, F_PARAM, z["param"])
            self.upload(r, F_GRAD, z["grad"])
            self.upload(r, F_MASTER, z["master"])
            self.upload(r, F_MOM, z["mom"])
            self.upload(r, F_VAR, z["var"])
            self.set_step(r, int(z["adam_step"]))

    def init_seeded(self, seed: int = 2024, scale: float = 1.0) -> None:
        """shard_init (train.cpp:224-253) on the device: master / working copy
        = seeded_uniform(P, seed) * scale, sharded (scale 1: bitwise the
        reference's)."""
        N.check(N.lib.hzp_state_init_seeded(self._h, seed, scale))

    def init_random(self, seed: int = 1234, scale: float = 0.04) -> None:
        N.check(N.lib.hzp_state_init_random(self._h, seed, scale))

    def load_state(self, st) -> None:
        """Upload an oracle HzpState (flat per-rank arrays) for the driven ranks."""
        for r in self.local_ranks:
            p = st.param[r]
            if self.cfg.precision == BF16:
                p = (np.ascontiguousarray(p, dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)
            self.upload(r, F_PARAM, p)
            self.upload(r, F_GRAD, st.grad[r])
            self.upload(r, F_MASTER, st.master[r])
            self.upload(r, F_MOM, st.mom[r])
            self.upload(r, F_VAR, st.var[r])
            self.set_step(r, int(st.adam_step[r]))

    def param_f32(self, rank: int) -> np.ndarray:
        p = self.download(rank, F_PARAM)
        if p.dtype == np.uint16:
            p = (p.astype(np.uint32) << 16).view(np.float32)
        return p

    # ---- the step ---------------------------------------------------------------
    def step(self, inputs, on_device: bool = False) -> np.ndarray:
        """train_step_hzp on the device; inputs [local][mb][...]; returns losses."""
        losses = (C.c_float * len(self.local_ranks))()
        if on_device:
            ptr = inputs.data_ptr() if hasattr(inputs, "data_ptr") else int(inputs)
            N.check(N.lib.hzp_step(self._h, C.c_void_p(ptr), 1, losses))
        else:
            a = np.ascontiguousarray(inputs)
            N.check(N.lib.hzp_step(self._h, C.c_void_p(a.ctypes.data), 0, losses))
        return np.array(list(losses), dtype=np.float32)

    def step_async(self, ptr: int, on_device: bool) -> None:
        N.check(N.lib.hzp_step(self._h, C.c_void_p(ptr), int(on_device), None))

    def sync(self) -> None:
        N.check(N.lib.hzp_sync(self._h))

    def launch_log(self):
        n = C.c_int()
        N.check(N.lib.hzp_launch_log(self._h, None, 0, C.byref(n)))
        recs = (N.hzp_launch_rec * max(1, n.value))()
        N.check(N.lib.hzp_launch_log(self._h, recs, n.value, C.byref(n)))
        return [(r.task_id, r.kind, r.layer, r.microbatch, r.stream, r.slot, r.covered_first,
                 r.covered_last) for r in recs[: n.value]]

    def timeline(self):
        n = C.c_int()
        cap = 1 << 16
        s, e = (C.c_double * cap)(), (C.c_double * cap)()
        idle, busy, mk = C.c_double(), C.c_double(), C.c_double()
        N.check(N.lib.hzp_timeline(self._h, s, e, cap, C.byref(n), C.byref(idle), C.byref(busy),
                                   C.byref(mk)))
        return {"start_ms": list(s)[: n.value], "end_ms": list(e)[: n.value],
                "compute_idle_ms": idle.value, "compute_busy_ms": busy.value,
                "makespan_ms": mk.value}

    def z1_timeline(self):
        """Per-layer optimizer times of the last recorded step (async mode):
        ready / start / end ms from step start (hzp_z1_timeline)."""
        n = C.c_int()
        cap = 4096
        a, b, c = (C.c_double * cap)(), (C.c_double * cap)(), (C.c_double * cap)()
        N.check(N.lib.hzp_z1_timeline(self._h, a, b, c, cap, C.byref(n)))
        k = min(n.value, cap)
        return {"ready_ms": list(a)[:k], "start_ms": list(b)[:k], "end_ms": list(c)[:k]}

    def set_timeline(self, on: bool) -> None:
        N.check(N.lib.hzp_set_timeline(self._h, 1 if on else 0))

    def stream(self, which: int = 0) -> int:
        p = C.c_void_p()
        N.check(N.lib.hzp_ctx_stream(self._h, which, C.byref(p)))
        return p.value or 0

    def launch_count(self) -> int:
        k = C.c_int64()
        N.check(N.lib.hzp_ctx_launch_count(self._h, C.byref(k)))
        return k.value

    # ---- kernel-level entry points ------------------------------------------------
    def ag_layer(self, layer: int, slot: int) -> None:
        N.check(N.lib.hzp_ag_layer(self._h, layer, slot))

    def ag_slot(self, rank: int, slot: int, n: int) -> np.ndarray:
        dt = np.uint16 if self.cfg.precision == BF16 else np.float32
        a = np.empty(n, dtype=dt)
        N.check(N.lib.hzp_ag_slot_download(self._h, rank, slot, a.ctypes.data, n))
        return a

    def wgrad_upload(self, rank: int, layer: int, wslot: int, g: np.ndarray) -> None:
        a = np.ascontiguousarray(g, dtype=np.float32)
        N.check(N.lib.hzp_wgrad_upload(self._h, rank, layer, wslot,
                                       a.ctypes.data_as(C.POINTER(C.c_float)), a.size))

    def rs_layer(self, layer: int, wslot: int) -> None:
        N.check(N.lib.hzp_rs_layer(self._h, layer, wslot))

    def collective_time(self, kind: str, layer: int, iters: int = 5) -> float:
        """ms per back-to-back AG ("ag") or RS ("rs") of `layer`, CUDA-event timed."""
        v = C.c_double()
        N.check(N.lib.hzp_collective_time(self._h, {"ag": 0, "rs": 1}[kind], layer, iters, C.byref(v)))
        return v.value

    def z1_adam_step(self) -> None:
        N.check(N.lib.hzp_z1_adam_step(self._h))

    def zero_grads(self) -> None:
        N.check(N.lib.hzp_zero_grads(self._h))

    def barrier(self) -> None:
        N.check(N.lib.hzp_barrier(self._h))


def seeded_span(seed: int, P: int, first: int, n: int, scale: float = 1.0) -> np.ndarray:
    out = np.empty(n, np.float32)
    N.check(N.lib.hzp_seeded_span(seed, P, first, n, scale, out.ctypes.data_as(C.POINTER(C.c_float))))
    return out


def make_tokens(seed: int, step: int, rank: int, mb: int, n: int, vocab: int) -> np.ndarray:
    """run_case's per-(step, rank, microbatch) token stream (train.cpp:506-507)."""
    out = np.empty(n, np.int32)
    N.check(N.lib.hzp_make_tokens(seed, step, rank, mb, n, vocab, out.ctypes.data_as(C.POINTER(C.c_int32))))
    return out


def kernel_launches() -> int:
    return int(N.lib.hzp_kernel_launches())


def gemm_profile(on: bool) -> None:
    N.check(N.lib.hzp_gemm_profile(int(on)))


def gemm_profile_read():
    f, ms, n = C.c_double(), C.c_double(), C.c_int()
    N.check(N.lib.hzp_gemm_profile_read(C.byref(f), C.byref(ms), C.byref(n)))
    return f.value, ms.value, n.value


def gemm_profile_read_busy():
    """(flops, summed launch ms, union-of-launches ms, launches); clears."""
    f, ms, busy, n = C.c_double(), C.c_double(), C.c_double(), C.c_int()
    N.check(N.lib.hzp_gemm_profile_read_busy(C.byref(f), C.byref(ms), C.byref(busy), C.byref(n)))
    return f.value, ms.value, busy.value, n.value


def gemm_profile_dump():
    f, ms, n = C.c_double(), C.c_double(), C.c_int()
    buf = C.create_string_buffer(1 << 16)
    N.check(N.lib.hzp_gemm_profile_dump(C.byref(f), C.byref(ms), C.byref(n), buf, 1 << 16))
    return f.value, ms.value, n.value, buf.value.decode()


def gemm_bf16(A, B, C_, M, N_, K, lda, ldb, ldc, a_mn=0, b_mn=0, epi=0, stream=0):
    """Standalone tcgen05 GEMM on raw device pointers (tests / benches)."""
    N.check(N.lib.hzp_gemm_bf16(C.c_void_p(A), C.c_void_p(B), C.c_void_p(C_), M, N_, K, lda, ldb,
                                ldc, a_mn, b_mn, epi, C.c_void_p(stream)))


def gemm_f32(A, B, C_, M, N_, K, lda, ldb, ldc, a_mn=0, b_mn=0, epi=0, stream=0):
    N.check(N.lib.hzp_gemm_f32(C.c_void_p(A), C.c_void_p(B), C.c_void_p(C_), M, N_, K, lda, ldb,
                               ldc, a_mn, b_mn, epi, C.c_void_p(stream)))
