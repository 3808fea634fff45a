"""Partition + scheduler API — Python mirror of the reference's hzp:: namespace.

Every function calls the C-ABI (libhzp_b200.so, which runs the C++ drop-in in
csrc/hzp/).  Names, argument meaning and error behaviour follow
/root/reference/proj/include/hzp/{config,memory,sched}.hpp:

  ParallelConfig, ModelSpec, Topology/CostModel  (config.hpp:16-54)
  validate_config        -> raises ValidationError  (config.hpp:89-91)
  build_process_groups   -> {kind: [[ranks], ...]}  (config.hpp:96-97)
  shard_elems                                     (memory.hpp:37-38)
  build_task_graph       -> TaskGraph              (sched.hpp:90-91)
  make_pools / derive_prelaunch_depth              (sched.hpp:108-112)
  simulate               -> Timeline               (sched.hpp:137)
  launch_plan            -> [PlanEntry]  (new: the executor's issue records)
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List

from . import _native as N
from ._native import SchedError, ValidationError  # noqa: F401

# TaskKind / StreamId / SchedMode (sched.hpp:20-29, 93-95)
FWD, BWD, FWD_RECOMPUTE, AG_PARAM, RS_GRAD, AR_DZP, OPT_STEP, AG_POST_STEP = range(8)
KIND_NAMES = ["FWD", "BWD", "FWD-recompute", "AG-param", "RS-grad", "AR-dzp", "OPT-step",
              "AG-post-step"]
COMPUTE, AG, RS = 0, 1, 2
VANILLA, ASYNC = 0, 1
GROUP_KINDS = {"Z1": 0, "Z2": 1, "Z3": 2, "DZP": 3}


@dataclass
class ParallelConfig:
    dp: int = 1
    z1: int = 1
    z2: int = 1
    z3: int = 1
    pp: int = 1
    vpp: int = 1
    cp: int = 1
    tp: int = 1

    def c(self) -> N.hzp_parallel:
        return N.hzp_parallel(self.dp, self.z1, self.z2, self.z3, self.pp, self.vpp, self.cp, self.tp)


@dataclass
class ModelSpec:
    num_layers: int = 0
    params_per_layer: int = 0
    embedding_params: int = 0
    seq_len: int = 1
    micro_batch_size: int = 1
    num_microbatches: int = 1
    flops_per_token_per_layer: float = 0.0
    hidden_size: int = 0

    def c(self) -> N.hzp_model_spec:
        return N.hzp_model_spec(self.num_layers, self.params_per_layer, self.embedding_params,
                                self.seq_len, self.micro_batch_size, self.num_microbatches,
                                self.flops_per_token_per_layer, self.hidden_size)


@dataclass
class CostModel:
    """Topology + CostModel::device_flops (config.hpp:44-54, collective.hpp:63-67)."""
    num_nodes: int = 1
    ranks_per_node: int = 1
    intra_bw: float = 1.0
    inter_bw: float = 1.0
    intra_latency: float = 0.0
    inter_latency: float = 0.0
    device_flops: float = 1e12

    def c(self) -> N.hzp_cost:
        return N.hzp_cost(self.num_nodes, self.ranks_per_node, self.intra_bw, self.inter_bw,
                          self.intra_latency, self.inter_latency, self.device_flops)


def shard_elems(n: int, parts: int) -> int:
    return int(N.lib.hzp_shard_elems(n, parts))


def validate_config(spec: ModelSpec, cfg: ParallelConfig, topo: CostModel) -> None:
    N.check(N.lib.hzp_validate(C.byref(spec.c()), C.byref(cfg.c()), C.byref(topo.c())))


def build_process_groups(cfg: ParallelConfig) -> dict:
    out = {}
    world = cfg.dp * cfg.pp * cfg.cp * cfg.tp
    buf = (C.c_int * world)()
    gsz, ng = C.c_int(), C.c_int()
    for name, k in GROUP_KINDS.items():
        N.check(N.lib.hzp_groups(C.byref(cfg.c()), k, buf, world, C.byref(gsz), C.byref(ng)))
        flat = list(buf)[: gsz.value * ng.value]
        out[name] = [flat[i * gsz.value:(i + 1) * gsz.value] for i in range(ng.value)]
    return out


@dataclass
class Task:
    id: int
    kind: int
    layer: int
    microbatch: int
    virtual_stage: int
    pass_: int
    duration: float
    bytes: int
    deps: List[int] = field(default_factory=list)


class TaskGraph:
    """build_task_graph result (sched.hpp:78-88); owns the native graph."""

    def __init__(self, spec: ModelSpec, cfg: ParallelConfig, cost: CostModel,
                 defer_rs: bool = False, rank: int = 0, pipeline: bool = False, reuse: bool = False,
                 recompute: bool = False):
        h = C.c_void_p()
        self.reuse_report = None
        if pipeline or reuse or recompute:
            # the CLI's graph: pipeline slot order, then reuse, then recompute
            rep = N.hzp_reuse_report()
            N.check(N.lib.hzp_graph_build_pipeline(C.byref(spec.c()), C.byref(cfg.c()), C.byref(cost.c()),
                                                   int(defer_rs), rank, int(reuse), int(recompute),
                                                   C.byref(rep), C.byref(h)))
            if reuse:
                self.reuse_report = {"r1_eliminated_ag": rep.r1_eliminated_ag, "r2_merged_rs": rep.r2_merged_rs,
                                     "r3_eliminated_ag": rep.r3_eliminated_ag,
                                     "extra_cached_bytes": rep.extra_cached_bytes}
        else:
            N.check(N.lib.hzp_graph_build(C.byref(spec.c()), C.byref(cfg.c()), C.byref(cost.c()),
                                          int(defer_rs), rank, C.byref(h)))
        self._h = h
        self.spec, self.cfg = spec, cfg
        t = N.hzp_task()
        self.tasks: List[Task] = []
        for i in range(N.lib.hzp_graph_size(h)):
            N.check(N.lib.hzp_graph_task(h, i, C.byref(t)))
            self.tasks.append(Task(t.id, t.kind, t.layer, t.microbatch, t.virtual_stage, t.pass_,
                                   t.duration, t.bytes, [t.deps[j] for j in range(t.num_deps)]))
        self.ag_slot_bytes = int(N.lib.hzp_graph_ag_slot_bytes(h))
        self.grad_buf_bytes = int(N.lib.hzp_graph_grad_buf_bytes(h))

    def count(self, kind: int) -> int:
        return sum(1 for t in self.tasks if t.kind == kind)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            N.lib.hzp_graph_destroy(h)
            self._h = None


def build_task_graph(spec, cfg, cost, defer_rs=False, rank=0, pipeline=False, reuse=False,
                     recompute=False) -> TaskGraph:
    """build_task_graph (sched.hpp:90-91); with pipeline/reuse/recompute, the
    CLI's graph (hzpsim.cpp:111-127): the rank's pipeline schedule order, then
    apply_reuse, then recompute_rule."""
    return TaskGraph(spec, cfg, cost, defer_rs, rank, pipeline, reuse, recompute)


def make_pools(graph: TaskGraph, prelaunch_depth: int, rs_slots: int):
    ag, rs = N.hzp_pool(), N.hzp_pool()
    N.check(N.lib.hzp_make_pools(graph._h, prelaunch_depth, rs_slots, C.byref(ag), C.byref(rs)))
    return ({"capacity": ag.capacity, "slot_count": ag.slot_count, "slot_bytes": ag.slot_bytes},
            {"capacity": rs.capacity, "slot_count": rs.slot_count, "slot_bytes": rs.slot_bytes})


def derive_prelaunch_depth(graph: TaskGraph, free_budget: int) -> int:
    return int(N.lib.hzp_derive_prelaunch_depth(graph._h, free_budget))


@dataclass
class Timeline:
    start: list
    end: list
    makespan: float
    compute_idle: float
    compute_busy: float


def simulate(graph: TaskGraph, depth: int = 2, rs_slots: int = 1, mode: int = ASYNC) -> Timeline:
    n = len(graph.tasks)
    s, e = (C.c_double * max(1, n))(), (C.c_double * max(1, n))()
    summ = N.hzp_sim_summary()
    N.check(N.lib.hzp_simulate(graph._h, depth, rs_slots, mode, s, e, C.byref(summ)))
    return Timeline(list(s)[:n], list(e)[:n], summ.makespan, summ.compute_idle, summ.compute_busy)


def ledger(spec: ModelSpec, cfg: ParallelConfig) -> dict:
    """Per-rank static bytes of the sharded states (memory.hpp:47)."""
    m = N.hzp_ledger()
    N.check(N.lib.hzp_memory_ledger(C.byref(spec.c()), C.byref(cfg.c()), C.byref(m)))
    return {f: getattr(m, f) for f, _ in N.hzp_ledger._fields_}


def _times(graph, start, end):
    if start is None:
        return None, None
    n = len(graph.tasks)
    if len(start) != n or len(end) != n:
        raise ValueError("one start / end time per task")
    return (C.c_double * n)(*start), (C.c_double * n)(*end)


def memory_trace(graph: TaskGraph, depth: int = 2, rs_slots: int = 1, mode: int = ASYNC,
                 static_bytes: int = 0, start=None, end=None) -> dict:
    """memory_trace (sched.hpp:139-149) of simulate(graph, ...) or, with
    start / end, of a measured timeline: peak bytes (static + dynamic), pool
    fragmentation, peak gradient-buffer bytes and the (time, bytes) samples."""
    s, e = _times(graph, start, end)
    out = N.hzp_memory_report()
    N.check(N.lib.hzp_memory_trace(graph._h, depth, rs_slots, mode, s, e, static_bytes, C.byref(out),
                                   None, None, 0))
    cap = max(1, out.n_samples)
    ts, bs = (C.c_double * cap)(), (C.c_int64 * cap)()
    N.check(N.lib.hzp_memory_trace(graph._h, depth, rs_slots, mode, s, e, static_bytes, C.byref(out),
                                   ts, bs, cap))
    r = {f: getattr(out, f) for f, _ in N.hzp_memory_report._fields_}
    r["samples"] = list(zip(list(ts)[: out.n_samples], list(bs)[: out.n_samples]))
    return r


def utilization_report(graph: TaskGraph, peak_flops: float, depth: int = 2, rs_slots: int = 1,
                       mode: int = ASYNC, start=None, end=None) -> float:
    """Model FLOPs / (makespan x peak) (sched.hpp:151-152)."""
    s, e = _times(graph, start, end)
    v = C.c_double()
    N.check(N.lib.hzp_utilization_report(graph._h, depth, rs_slots, mode, s, e, peak_flops, C.byref(v)))
    return v.value


@dataclass
class PlanEntry:
    id: int
    kind: int
    layer: int
    microbatch: int
    stream: int
    slot: int
    ring_wait: int
    waits: List[int]


def launch_plan(graph: TaskGraph, depth: int = 2, rs_slots: int = 1) -> List[PlanEntry]:
    out, e = [], N.hzp_plan_entry()
    for i in range(len(graph.tasks)):
        N.check(N.lib.hzp_plan_entry_get(graph._h, depth, rs_slots, i, C.byref(e)))
        out.append(PlanEntry(e.id, e.kind, e.layer, e.microbatch, e.stream, e.slot, e.ring_wait,
                             [e.waits[j] for j in range(e.num_waits)]))
    return out
