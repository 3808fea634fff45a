"""Chrome-trace export of simulated and measured step timelines, in the
reference's format (trace.cpp:33-73: process / thread-name metadata, one
complete "X" event per task on its stream's track, ts / dur in µs, args
task_id / layer / microbatch / bytes)."""
from __future__ import annotations

import json
from typing import Optional, Sequence

from .hzp import KIND_NAMES, TaskGraph, launch_plan

STREAM_NAMES = ("compute", "all-gather", "reduce-scatter")  # trace.cpp stream_name()


def chrome_trace(graph: TaskGraph, start_s: Sequence[float], end_s: Sequence[float],
                 process_name: str = "hzp", depth: int = 2, rs_slots: int = 1) -> dict:
    """Trace dict for per-task [start, end) times in seconds (hzp.simulate's
    Timeline, or a measured engine timeline converted from ms)."""
    plan = launch_plan(graph, depth, rs_slots)
    ev = [{"name": "process_name", "ph": "M", "pid": 1, "tid": 0, "args": {"name": process_name}}]
    for tid, name in enumerate(STREAM_NAMES):
        ev.append({"name": "thread_name", "ph": "M", "pid": 1, "tid": tid, "args": {"name": name}})
    for t, p in zip(graph.tasks, plan):
        args = {"task_id": t.id}
        if t.layer >= 0:
            args["layer"] = t.layer
        if t.microbatch >= 0:
            args["microbatch"] = t.microbatch
        if t.bytes > 0:
            args["bytes"] = t.bytes
        ev.append({"name": KIND_NAMES[t.kind], "cat": "task", "ph": "X", "pid": 1, "tid": int(p.stream),
                   "ts": start_s[t.id] * 1e6, "dur": (end_s[t.id] - start_s[t.id]) * 1e6, "args": args})
    return {"traceEvents": ev, "displayTimeUnit": "ms"}


def write_chrome_trace(path: str, graph: TaskGraph, start_s: Sequence[float], end_s: Sequence[float],
                       process_name: str = "hzp", depth: int = 2, rs_slots: int = 1) -> None:
    with open(path, "w") as fh:
        json.dump(chrome_trace(graph, start_s, end_s, process_name, depth, rs_slots), fh, indent=2)
        fh.write("\n")


def measured_trace(engine, graph: TaskGraph, process_name: Optional[str] = None) -> dict:
    """Trace of the engine's last recorded step (hzp_set_timeline(1) + a step)."""
    tl = engine.timeline()
    return chrome_trace(graph, [x / 1e3 for x in tl["start_ms"]], [x / 1e3 for x in tl["end_ms"]],
                        process_name or "hzp_b200 measured", engine.cfg.prelaunch_depth, engine.cfg.rs_slots)
