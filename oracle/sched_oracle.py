"""Pure-Python restatement of the reference's layout + scheduler (TEST ONLY).

Integer layout (process groups, shard offsets) and the launch-order / ring-slot
rules of the AsyncHZP scheduler.  Used to check the product's C++ host code
(layout, task graph, LaunchPlan) bit-exactly.  Citations are to
/root/reference/proj.
"""
from __future__ import annotations

# TaskKind order (include/hzp/sched.hpp:20-29)
FWD, BWD, FWD_RECOMPUTE, AG_PARAM, RS_GRAD, AR_DZP, OPT_STEP, AG_POST = range(8)
KIND_NAMES = ["FWD", "BWD", "FWD-recompute", "AG-param", "RS-grad", "AR-dzp", "OPT-step",
              "AG-post-step"]
FORWARD, BACKWARD, NONE = 0, 1, 2  # Pass (sched.hpp:31)
COMPUTE, AG, RS = 0, 1, 2          # StreamId (sched.hpp:95)


def shard_elems(n: int, parts: int) -> int:
    """src/memory.cpp:13-15."""
    return (n + parts - 1) // parts


def build_process_groups(dp, z1, z2, z3, pp=1, cp=1, tp=1):
    """src/config.cpp:127-146: contiguous Z1/Z2/Z3 ranges, strided DZP groups."""
    outer = pp * cp * tp
    out = {}
    for name, z in (("Z1", z1), ("Z2", z2), ("Z3", z3)):
        out[name] = [[b * dp + s + i for i in range(z)]
                     for b in range(outer) for s in range(0, dp, z)]
    reps = dp // z2
    out["DZP"] = [[b * dp + r * z2 + i for r in range(reps)]
                  for b in range(outer) for i in range(z2)]
    return out


def validate(dp, z1, z2, z3, total_params, ranks):
    """validate_config's divisibility rules (src/config.cpp:36-94).

    Returns 0 ok, 1 NonDivisible, 2 EmptyModel (error codes mirror
    ValidationError::Code + 1)."""
    if total_params <= 0:
        return 2
    for z in (z1, z2, z3):
        if not (z >= 1 and dp % z == 0):
            return 1
    if dp != ranks:
        return 1
    return 0


def stream_of(kind):
    """src/sched.cpp:36-51."""
    if kind in (FWD, BWD, FWD_RECOMPUTE, OPT_STEP):
        return COMPUTE
    if kind in (AG_PARAM, AG_POST):
        return AG
    return RS


def uses_ag_pool(kind):
    """src/sched.cpp:58-60."""
    return kind in (AG_PARAM, AG_POST)


def build_task_graph(num_layers, num_mb, dp, z2, defer_rs=False):
    """build_task_graph (src/sched.cpp:75-222), pp=1, default F/B slot order.

    Returns a list of dicts {id, kind, layer, mb, pass, deps} (durations are
    not part of the launch contract and are omitted)."""
    tasks = []

    def add(kind, layer, mb, pas, deps):
        tasks.append({"id": len(tasks), "kind": kind, "layer": layer, "mb": mb, "pass": pas,
                      "deps": list(deps)})
        return len(tasks) - 1

    prev = -1
    rs_ids, rs_by_layer, pending = [], {}, []
    last_bwd = -1
    for mb in range(num_mb):
        for l in range(num_layers):                       # F slot (sched.cpp:155-165)
            ag = add(AG_PARAM, l, mb, FORWARD, [])
            prev = add(FWD, l, mb, FORWARD, [ag] + ([prev] if prev >= 0 else []))
        for l in reversed(range(num_layers)):             # B slot (sched.cpp:166-188)
            ag = add(AG_PARAM, l, mb, BACKWARD, [])
            prev = add(BWD, l, mb, BACKWARD, [ag] + ([prev] if prev >= 0 else []))
            last_bwd = prev
            if defer_rs:
                pending.append((l, mb, prev))
            else:
                rs = add(RS_GRAD, l, mb, BACKWARD, [prev])
                rs_ids.append(rs)
                rs_by_layer.setdefault(l, []).append(rs)
    for l, mb, bwd in pending:                            # sched.cpp:192-200
        deps = [bwd] + ([last_bwd] if last_bwd >= 0 and last_bwd != bwd else [])
        rs = add(RS_GRAD, l, mb, BACKWARD, deps)
        rs_ids.append(rs)
        rs_by_layer.setdefault(l, []).append(rs)
    if dp // z2 > 1:                                      # sched.cpp:203-211
        opt_deps = [add(AR_DZP, l, -1, NONE, rs_by_layer[l]) for l in sorted(rs_by_layer)]
    else:
        opt_deps = rs_ids
    opt = add(OPT_STEP, -1, -1, NONE, opt_deps)          # sched.cpp:215
    for l in sorted(rs_by_layer):                         # sched.cpp:217-220
        add(AG_POST, l, -1, NONE, [opt])
    return tasks


def launch_plan(tasks, depth, rs_slots):
    """Per-task (stream, slot, wait-list) from simulate's ring rules.

    AG-pool task k takes slot k % depth and, once k >= depth, waits for the
    first consumer (in id order) of AG-pool task k-depth (src/sched.cpp:285-301);
    RS task k takes slot k % rs_slots and waits for RS task k-rs_slots
    (src/sched.cpp:302-309).  Waits = deps + that ring predecessor."""
    n = len(tasks)
    first_consumer = [-1] * n
    for t in tasks:
        for d in t["deps"]:
            if first_consumer[d] < 0:
                first_consumer[d] = t["id"]
    ag_order, rs_order, plan = [], [], []
    for t in tasks:
        slot, ring_wait = -1, -1
        if uses_ag_pool(t["kind"]):
            k = len(ag_order)
            slot = k % depth
            if k >= depth:
                blocking = ag_order[k - depth]
                c = first_consumer[blocking]
                ring_wait = c if c >= 0 else blocking
            ag_order.append(t["id"])
        elif t["kind"] == RS_GRAD:
            k = len(rs_order)
            slot = k % rs_slots
            if k >= rs_slots:
                ring_wait = rs_order[k - rs_slots]
            rs_order.append(t["id"])
        waits = list(t["deps"])
        if ring_wait >= 0 and ring_wait not in waits:
            waits.append(ring_wait)
        plan.append({"id": t["id"], "stream": stream_of(t["kind"]), "slot": slot,
                     "ring_wait": ring_wait, "waits": waits})
    return plan


def simulate(tasks, durations, depth, rs_slots, vanilla=False):
    """simulate's start/end times (src/sched.cpp:242-350) given per-task durations."""
    n = len(tasks)
    first_consumer = [-1] * n
    for t in tasks:
        for d in t["deps"]:
            if first_consumer[d] < 0:
                first_consumer[d] = t["id"]
    start, end = [0.0] * n, [0.0] * n
    free = [0.0, 0.0, 0.0]
    comm_block = 0.0
    ag_order, rs_order = [], []
    for t in tasks:
        i = t["id"]
        s = stream_of(t["kind"])
        at = free[s]
        for d in t["deps"]:
            at = max(at, end[d])
        if vanilla and s == COMPUTE:
            at = max(at, comm_block)
        if uses_ag_pool(t["kind"]):
            k = len(ag_order)
            if k >= depth:
                blocking = ag_order[k - depth]
                c = first_consumer[blocking]
                at = max(at, end[c] if c >= 0 else end[blocking])
            ag_order.append(i)
        if t["kind"] == RS_GRAD:
            k = len(rs_order)
            if k >= rs_slots:
                at = max(at, end[rs_order[k - rs_slots]])
            rs_order.append(i)
        start[i] = at
        end[i] = at + durations[i]
        free[s] = end[i]
        if vanilla and t["kind"] in (AG_PARAM, RS_GRAD, AR_DZP, AG_POST):
            comm_block = max(comm_block, end[i])
    busy = 0.0
    for t in tasks:  # plain left fold (Python's sum() is compensated since 3.12)
        if stream_of(t["kind"]) == COMPUTE:
            busy += durations[t["id"]]
    last = max([end[t["id"]] for t in tasks if stream_of(t["kind"]) == COMPUTE] + [0.0])
    return start, end, {"makespan": max(end + [0.0]), "compute_busy": busy,
                        "compute_idle": last - busy}


def ag_runs(layer_off, layer_len, s3, z3):
    """Owner spans of one layer's all-gather: [(dst_off, owner_idx, src_off, len)].

    Element e of the flat working copy lives on Z3 group member e // s3 at
    offset e % s3 (src/train.cpp:229-249, collective.cpp:44-67)."""
    runs, e, end = [], layer_off, layer_off + layer_len
    while e < end:
        owner = e // s3
        stop = min(end, (owner + 1) * s3)
        runs.append((e - layer_off, owner, e - owner * s3, stop - e))
        e = stop
    return runs
