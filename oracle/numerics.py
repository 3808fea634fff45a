"""ctypes front-ends for the oracle libraries (TEST INFRASTRUCTURE ONLY).

``Oracle`` wraps our C restatement ``_build/libhzp_oracle.so`` (hzp_oracle.c);
``RefLib`` wraps the reference library ``_ref/libhzpref.so`` built from the
reference's own sources.  Both expose the same few entry points so tests can
check restatement == reference and GPU == restatement on identical inputs.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libhzp_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libhzpref.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")


def build_oracle() -> None:
    """Compile the restatement (and the reference lib when its sources exist)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def shard_elems(n: int, parts: int) -> int:
    """shard_elems (src/memory.cpp:13-15)."""
    return (n + parts - 1) // parts


def mlp_param_count(dims) -> int:
    """MlpShape::param_count (include/hzp/train.hpp:36-42)."""
    return sum(dims[i - 1] * dims[i] + dims[i] for i in range(1, len(dims)))


@dataclass
class HzpState:
    """Flat per-rank ShardedState (include/hzp/train.hpp:73-83)."""

    dims: list
    dp: int
    z1: int
    z2: int
    z3: int
    dtype: type
    param: np.ndarray = field(default=None)   # [dp, s3]
    grad: np.ndarray = field(default=None)    # [dp, s2]
    master: np.ndarray = field(default=None)  # [dp, s1]
    mom: np.ndarray = field(default=None)
    var: np.ndarray = field(default=None)
    adam_step: np.ndarray = field(default=None)  # [dp] int32

    @property
    def P(self) -> int:
        return mlp_param_count(self.dims)

    @property
    def s1(self) -> int:
        return shard_elems(self.P, self.z1)

    @property
    def s2(self) -> int:
        return shard_elems(self.P, self.z2)

    @property
    def s3(self) -> int:
        return shard_elems(self.P, self.z3)

    def copy(self) -> "HzpState":
        return HzpState(self.dims, self.dp, self.z1, self.z2, self.z3, self.dtype,
                        self.param.copy(), self.grad.copy(), self.master.copy(),
                        self.mom.copy(), self.var.copy(), self.adam_step.copy())

    def gathered_params(self) -> np.ndarray:
        """gather_params (src/train.cpp:255-265): first Z3 group, truncated to P."""
        return self.param[: self.z3].reshape(-1)[: self.P].copy()


class Oracle:
    """Our C restatement of the reference numerics (hzp_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build_oracle()
        L = C.CDLL(path)
        self.L = L
        u64 = C.c_uint64
        L.orc_seeded_uniform_f64.argtypes = [_f64p, C.c_size_t, u64]
        L.orc_seeded_uniform_f32.argtypes = [_f32p, C.c_size_t, u64]
        L.orc_batch_seed.argtypes = [u64, C.c_int, C.c_int, C.c_int]
        L.orc_batch_seed.restype = u64
        L.orc_bf16_round.argtypes = [C.c_float]
        L.orc_bf16_round.restype = C.c_float
        L.orc_bf16_round_vec.argtypes = [_f32p, C.c_size_t]
        L.orc_tanhf_vec.argtypes = [_f32p, _f32p, C.c_size_t]
        L.orc_fnv1a.argtypes = [C.c_void_p, C.c_size_t]
        L.orc_fnv1a.restype = u64
        for sfx, p in (("f32", _f32p), ("f64", _f64p)):
            fn = getattr(L, f"orc_mlp_loss_grad_{sfx}")
            fn.argtypes = [_i32p, C.c_int, p, p, C.c_int, p]
            fn.restype = C.c_float if sfx == "f32" else C.c_double
            getattr(L, f"orc_adam_update_{sfx}").argtypes = [
                p, p, p, p, C.c_int64, C.c_int, C.c_double, C.c_double, C.c_double, C.c_double]
            getattr(L, f"orc_reduce_scatter_{sfx}").argtypes = [p, C.c_int, C.c_int64, p]
            getattr(L, f"orc_all_reduce_{sfx}").argtypes = [p, C.c_int, C.c_int64, p]
            getattr(L, f"orc_all_gather_{sfx}").argtypes = [p, C.c_int, C.c_int64, p]
            getattr(L, f"orc_shard_init_{sfx}").argtypes = [
                _i32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, u64, C.c_int,
                p, p, p, p, p, _i32p]
            getattr(L, f"orc_train_step_hzp_{sfx}").argtypes = [
                _i32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, p,
                C.c_double, C.c_double, C.c_double, C.c_double, C.c_int,
                p, p, p, p, p, _i32p, p, C.c_void_p]
            getattr(L, f"orc_train_step_baseline_{sfx}").argtypes = [
                _i32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, p,
                C.c_double, C.c_double, C.c_double, C.c_double, C.c_int,
                p, p, p, p, _i32p, p]
            getattr(L, f"orc_make_inputs_{sfx}").argtypes = [
                _i32p, C.c_int, C.c_int, C.c_int, u64, C.c_int, p]

    @staticmethod
    def _sfx(dtype) -> str:
        return "f32" if np.dtype(dtype) == np.float32 else "f64"

    def seeded_uniform(self, n: int, seed: int, dtype=np.float64) -> np.ndarray:
        out = np.empty(n, dtype=dtype)
        getattr(self.L, f"orc_seeded_uniform_{self._sfx(dtype)}")(out, n, seed)
        return out

    def batch_seed(self, seed: int, step: int, rank: int, mb: int) -> int:
        return int(self.L.orc_batch_seed(seed, step, rank, mb))

    def bf16_round(self, x: np.ndarray) -> np.ndarray:
        out = np.ascontiguousarray(x, dtype=np.float32).copy()
        self.L.orc_bf16_round_vec(out, out.size)
        return out

    def tanhf(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float32)
        out = np.empty_like(x)
        self.L.orc_tanhf_vec(x, out, x.size)
        return out

    def fnv1a(self, a: np.ndarray) -> str:
        a = np.ascontiguousarray(a)
        return "%016x" % self.L.orc_fnv1a(a.ctypes.data, a.nbytes)

    def mlp_loss_grad(self, dims, params, inputs, batch):
        dt = params.dtype
        d = np.asarray(dims, dtype=np.int32)
        g = np.zeros(mlp_param_count(dims), dtype=dt)
        loss = getattr(self.L, f"orc_mlp_loss_grad_{self._sfx(dt)}")(
            d, len(dims) - 1, np.ascontiguousarray(params), np.ascontiguousarray(inputs), batch, g)
        return loss, g

    def adam_update(self, master, m, v, g, step, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8):
        getattr(self.L, f"orc_adam_update_{self._sfx(master.dtype)}")(
            master, m, v, np.ascontiguousarray(g), master.size, step, lr, b1, b2, eps)

    def reduce_scatter(self, fulls: np.ndarray) -> np.ndarray:
        g, total = fulls.shape
        out = np.empty(total, dtype=fulls.dtype)
        rc = getattr(self.L, f"orc_reduce_scatter_{self._sfx(fulls.dtype)}")(
            np.ascontiguousarray(fulls), g, total, out)
        if rc:
            raise ValueError("tensor length not divisible by group size")
        return out.reshape(g, total // g)

    def all_reduce(self, ts: np.ndarray) -> np.ndarray:
        g, n = ts.shape
        out = np.empty(n, dtype=ts.dtype)
        getattr(self.L, f"orc_all_reduce_{self._sfx(ts.dtype)}")(np.ascontiguousarray(ts), g, n, out)
        return out

    def all_gather(self, shards: np.ndarray) -> np.ndarray:
        g, per = shards.shape
        out = np.empty(g * per, dtype=shards.dtype)
        getattr(self.L, f"orc_all_gather_{self._sfx(shards.dtype)}")(
            np.ascontiguousarray(shards), g, per, out)
        return out

    def shard_init(self, dims, dp, z1, z2, z3, seed, bf16_working, dtype=np.float32) -> HzpState:
        st = HzpState(list(dims), dp, z1, z2, z3, dtype)
        st.param = np.zeros((dp, st.s3), dtype=dtype)
        st.grad = np.zeros((dp, st.s2), dtype=dtype)
        st.master = np.zeros((dp, st.s1), dtype=dtype)
        st.mom = np.zeros((dp, st.s1), dtype=dtype)
        st.var = np.zeros((dp, st.s1), dtype=dtype)
        st.adam_step = np.zeros(dp, dtype=np.int32)
        getattr(self.L, f"orc_shard_init_{self._sfx(dtype)}")(
            np.asarray(dims, dtype=np.int32), len(dims) - 1, dp, z1, z2, z3, seed,
            int(bf16_working), st.param, st.grad, st.master, st.mom, st.var, st.adam_step)
        return st

    def make_inputs(self, dims, dp, num_mb, batch, seed, step, dtype=np.float32) -> np.ndarray:
        out = np.empty((dp, num_mb, batch, dims[0]), dtype=dtype)
        getattr(self.L, f"orc_make_inputs_{self._sfx(dtype)}")(
            np.asarray(dims, dtype=np.int32), dp, num_mb, batch, seed, step, out)
        return out

    def train_step_hzp(self, st: HzpState, inputs: np.ndarray, batch: int, bf16_working: bool,
                       lr=1e-3, b1=0.9, b2=0.999, eps=1e-8, want_rank_grads=False):
        """One train_step_hzp (src/train.cpp:267-381); mutates st in place.

        Returns (losses[dp], rank_grads[num_mb, dp, s2*z2] or None)."""
        num_mb = inputs.shape[1]
        losses = np.zeros(st.dp, dtype=st.dtype)
        rg = None
        ptr = None
        if want_rank_grads:
            rg = np.zeros((num_mb, st.dp, st.s2 * st.z2), dtype=st.dtype)
            ptr = rg.ctypes.data
        getattr(self.L, f"orc_train_step_hzp_{self._sfx(st.dtype)}")(
            np.asarray(st.dims, dtype=np.int32), len(st.dims) - 1, st.dp, st.z1, st.z2, st.z3,
            num_mb, batch, np.ascontiguousarray(inputs, dtype=st.dtype), lr, b1, b2, eps,
            int(bf16_working), st.param, st.grad, st.master, st.mom, st.var, st.adam_step,
            losses, ptr)
        return losses, rg

    def baseline_init(self, dims, seed, bf16_working, dtype=np.float32):
        """baseline_init (src/train.cpp:212-222)."""
        P = mlp_param_count(dims)
        master = self.seeded_uniform(P, seed, dtype)
        working = self.bf16_round(master) if (bf16_working and dtype == np.float32) else master.copy()
        return {"working": working, "master": master, "mom": np.zeros(P, dtype),
                "var": np.zeros(P, dtype), "adam_step": np.zeros(1, np.int32)}

    def train_step_baseline(self, base, dims, dp, z2, inputs, batch, bf16_working,
                            lr=1e-3, b1=0.9, b2=0.999, eps=1e-8):
        dt = base["master"].dtype
        losses = np.zeros(dp, dtype=dt)
        getattr(self.L, f"orc_train_step_baseline_{self._sfx(dt)}")(
            np.asarray(dims, dtype=np.int32), len(dims) - 1, dp, z2, inputs.shape[1], batch,
            np.ascontiguousarray(inputs, dtype=dt), lr, b1, b2, eps, int(bf16_working),
            base["working"], base["master"], base["mom"], base["var"], base["adam_step"], losses)
        return losses

    def run_states(self, dims, dp, z1, z2, z3, mbs, batch, seed, steps, bf16_working,
                   dtype=np.float32):
        """shard_init + `steps` train_step_hzp with run_case inputs (train.cpp:484-508)."""
        st = self.shard_init(dims, dp, z1, z2, z3, seed, bf16_working, dtype)
        losses = None
        for step in range(steps):
            x = self.make_inputs(dims, dp, mbs, batch, seed, step, dtype)
            losses, _ = self.train_step_hzp(st, x, batch, bf16_working)
        return st, losses


class RefLib:
    """The reference library itself (oracle/_ref/libhzpref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        self.L = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_shard_elems.argtypes = [C.c_longlong, C.c_longlong]
        L.ref_shard_elems.restype = C.c_longlong
        L.ref_bf16_round.argtypes = [C.c_float]
        L.ref_bf16_round.restype = C.c_float
        L.ref_bf16_round_vec.argtypes = [_f32p, C.c_longlong, C.c_int]
        L.ref_seeded_uniform_f64.argtypes = [_f64p, C.c_longlong, C.c_ulonglong]
        L.ref_seeded_uniform_f32.argtypes = [_f32p, C.c_longlong, C.c_ulonglong]
        L.ref_run_states_f32.argtypes = [_i32p] + [C.c_int] * 7 + [C.c_ulonglong, C.c_int, C.c_int] + [_f32p] * 7
        L.ref_run_states_f64.argtypes = [_i32p] + [C.c_int] * 7 + [C.c_ulonglong, C.c_int] + [_f64p] * 7
        L.ref_mlp_loss_grad_f32.argtypes = [_i32p, C.c_int, _f32p, _f32p, C.c_int, _f32p]
        L.ref_mlp_loss_grad_f32.restype = C.c_float
        L.ref_groups.argtypes = [C.c_int] * 5 + [_i32p]
        L.ref_validate.argtypes = [C.c_longlong, C.c_longlong] + [C.c_int] * 5
        L.ref_all_gather_f64.argtypes = [_f64p, C.c_int, C.c_longlong, _f64p]
        L.ref_reduce_scatter_f32.argtypes = [_f32p, C.c_int, C.c_longlong, _f32p]
        L.ref_all_reduce_f32.argtypes = [_f32p, C.c_int, C.c_longlong, _f32p]
        L.ref_derive_prelaunch_depth.argtypes = [C.c_longlong, C.c_longlong] + [C.c_int] * 4 + [C.c_longlong]
        L.ref_time_train_step_f32.argtypes = [_i32p] + [C.c_int] * 7 + [C.c_ulonglong, C.c_int]
        L.ref_time_train_step_f32.restype = C.c_double
        L.ref_time_steps_f32.argtypes = [_i32p] + [C.c_int] * 7 + [C.c_ulonglong, C.c_int, C.c_int, _f32p]
        L.ref_time_steps_f32.restype = C.c_double

    def run_states(self, dims, dp, z1, z2, z3, mbs, batch, seed, steps, bf16_working,
                   dtype=np.float32):
        P = mlp_param_count(dims)
        st = HzpState(list(dims), dp, z1, z2, z3, dtype)
        st.param = np.zeros((dp, st.s3), dtype=dtype)
        st.grad = np.zeros((dp, st.s2), dtype=dtype)
        st.master = np.zeros((dp, st.s1), dtype=dtype)
        st.mom = np.zeros((dp, st.s1), dtype=dtype)
        st.var = np.zeros((dp, st.s1), dtype=dtype)
        st.adam_step = np.full(dp, steps, dtype=np.int32)
        losses = np.zeros(dp, dtype=dtype)
        base = np.zeros(P, dtype=dtype)
        d = np.asarray(dims, dtype=np.int32)
        if dtype == np.float32:
            rc = self.L.ref_run_states_f32(d, len(dims) - 1, dp, z1, z2, z3, mbs, batch, seed, steps,
                                           int(bf16_working), st.param, st.grad, st.master, st.mom,
                                           st.var, losses, base)
        else:
            rc = self.L.ref_run_states_f64(d, len(dims) - 1, dp, z1, z2, z3, mbs, batch, seed, steps,
                                           st.param, st.grad, st.master, st.mom, st.var, losses, base)
        if rc:
            raise RuntimeError(self.L.ref_last_error().decode())
        return st, losses, base

    def groups(self, dp, z1, z2, z3, kind: int):
        out = np.zeros(dp, dtype=np.int32)
        n = self.L.ref_groups(dp, z1, z2, z3, kind, out)
        return [list(map(int, g)) for g in out.reshape(n, -1)]

    def task_graph(self, layers, ppl, seq=1024, mbsize=1, num_mb=1, flops=6e6, dp=8, z1=8, z2=4,
                   z3=4, pp=1, vpp=1, intra_bw=1e10, intra_lat=1e-6, device_flops=1e12,
                   defer_rs=False, rank=0, with_reuse=False, depth=2, rs_slots=1, vanilla=False,
                   recompute=False):
        class Sim(C.Structure):
            _fields_ = [("makespan", C.c_double), ("compute_idle", C.c_double),
                        ("compute_busy", C.c_double), ("peak_memory", C.c_longlong),
                        ("fragmentation", C.c_double), ("peak_grad_buffer_bytes", C.c_longlong),
                        ("ag_slot_count", C.c_int), ("rs_slot_count", C.c_int),
                        ("ag_slot_bytes", C.c_longlong), ("rs_slot_bytes", C.c_longlong),
                        ("r1_eliminated_ag", C.c_int), ("r2_merged_rs", C.c_int),
                        ("r3_eliminated_ag", C.c_int), ("extra_cached_bytes", C.c_longlong),
                        ("total_static", C.c_longlong), ("peak_bytes", C.c_longlong),
                        ("utilization", C.c_double), ("n_samples", C.c_int),
                        ("sample_time_sum", C.c_double), ("sample_bytes_sum", C.c_longlong)]
        cap = 6 * layers * num_mb * max(1, vpp) + 4 * layers + 8
        ints = lambda: np.zeros(cap, dtype=np.int32)  # noqa: E731
        dbl = lambda: np.zeros(cap, dtype=np.float64)  # noqa: E731
        kind, layer, mb, pas = ints(), ints(), ints(), ints()
        nbytes = np.zeros(cap, dtype=np.int64)
        dur, start, end, rel = dbl(), dbl(), dbl(), dbl()
        dep_off = np.zeros(cap + 1, dtype=np.int32)
        dep_cap = cap * 8
        deps = np.zeros(dep_cap, dtype=np.int32)
        sim = Sim()
        L = self.L
        L.ref_task_graph.argtypes = (
            [C.c_longlong] * 5 + [C.c_double] + [C.c_int] * 6 + [C.c_double] * 3 + [C.c_int] * 8
            + [_i32p] * 4 + [_i64p] + [_f64p] * 4 + [_i32p, _i32p, C.c_int, C.POINTER(Sim)])
        n = L.ref_task_graph(layers, ppl, seq, mbsize, num_mb, flops, dp, z1, z2, z3, pp, vpp,
                             intra_bw, intra_lat, device_flops, int(defer_rs), rank,
                             int(with_reuse), int(recompute), depth, rs_slots, int(vanilla), cap, kind, layer, mb,
                             pas, nbytes, dur, start, end, rel, dep_off, deps, dep_cap,
                             C.byref(sim))
        if n < 0:
            raise RuntimeError(L.ref_last_error().decode())
        tasks = []
        for i in range(n):
            tasks.append({"id": i, "kind": int(kind[i]), "layer": int(layer[i]), "mb": int(mb[i]),
                          "pass": int(pas[i]), "bytes": int(nbytes[i]), "dur": float(dur[i]),
                          "start": float(start[i]), "end": float(end[i]),
                          "pool_release": float(rel[i]),
                          "deps": [int(x) for x in deps[dep_off[i]:dep_off[i + 1]]]})
        summary = {f: getattr(sim, f) for f, _ in Sim._fields_}
        return tasks, summary


def load_oracle() -> Oracle:
    return Oracle()


def load_ref() -> RefLib | None:
    try:
        return RefLib()
    except (FileNotFoundError, OSError):
        return None
