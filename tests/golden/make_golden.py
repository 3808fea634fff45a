"""Generate tests/golden/*.json from the REFERENCE ITSELF (oracle/_ref/libhzpref.so).

Run in the build container (where /root/reference exists and `make -C oracle`
has built the reference library):

    python tests/golden/make_golden.py

The fixtures pin the oracle restatement and the product's host code.  Every
value below is produced by calling the reference's own functions
(train_step_hzp, build_task_graph, simulate, build_process_groups,
bf16_round, collectives) through oracle/ref_shim.cpp.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.numerics import RefLib, Oracle  # noqa: E402

SEED = 2024


def fnv(o: Oracle, a: np.ndarray) -> str:
    return o.fnv1a(np.ascontiguousarray(a))


def numerics_cases(ref: RefLib, o: Oracle):
    cases = []
    grid = [
        # (dims, dp, z1, z2, z3, mbs, batch, steps)  — CPU config first
        ([12, 20, 8], 4, 4, 2, 2, 1, 4, 10),
        ([12, 20, 8], 4, 4, 2, 2, 2, 4, 10),
        ([12, 20, 8], 4, 2, 2, 2, 1, 4, 10),
        ([12, 20, 8], 8, 8, 4, 4, 2, 4, 3),
        ([12, 20, 8], 8, 8, 2, 2, 2, 4, 3),
        ([12, 20, 8], 8, 2, 4, 8, 1, 4, 3),
        ([12, 20, 8], 8, 4, 8, 2, 2, 4, 3),
        ([6, 10, 4], 4, 2, 4, 2, 2, 4, 2),
        ([16, 32, 32, 8], 8, 8, 4, 4, 2, 8, 4),
    ]
    for dims, dp, z1, z2, z3, mbs, batch, steps in grid:
        for prec in ("fp32", "mixed", "fp64"):
            dt = np.float64 if prec == "fp64" else np.float32
            st, losses, base = ref.run_states(dims, dp, z1, z2, z3, mbs, batch, SEED, steps,
                                              prec == "mixed", dt)
            cases.append({
                "dims": dims, "dp": dp, "z1": z1, "z2": z2, "z3": z3, "mbs": mbs,
                "batch": batch, "steps": steps, "seed": SEED, "precision": prec,
                "P": st.P, "s1": st.s1, "s2": st.s2, "s3": st.s3,
                "params_head": [float(x) for x in st.gathered_params()[:4]],
                "hash": {
                    "params": fnv(o, st.gathered_params()),
                    "param_shards": [fnv(o, st.param[r]) for r in range(dp)],
                    "grad_shards": [fnv(o, st.grad[r]) for r in range(dp)],
                    "master": [fnv(o, st.master[r]) for r in range(dp)],
                    "mom": [fnv(o, st.mom[r]) for r in range(dp)],
                    "var": [fnv(o, st.var[r]) for r in range(dp)],
                    "baseline_working": fnv(o, base),
                },
                "losses": [float(x) for x in losses],
                "max_abs_vs_baseline": float(np.max(np.abs(
                    st.gathered_params().astype(np.float64) - base.astype(np.float64)))),
            })
    # full arrays for the CPU config, mixed + fp32: lets GPU tests compare
    # element-wise without re-running the oracle
    full = {}
    for prec in ("fp32", "mixed"):
        st, losses, base = ref.run_states([12, 20, 8], 4, 4, 2, 2, 1, 4, SEED, 10,
                                          prec == "mixed", np.float32)
        full[prec] = {"params": [float(x) for x in st.gathered_params()],
                      "master": [float(x) for x in st.master.reshape(-1)],
                      "losses": [float(x) for x in losses]}
    return {"cases": cases, "cpu_config_full": full}


def sched_cases(ref: RefLib):
    out = []
    grid = [
        # (layers, num_mb, dp, z1, z2, z3, depth, rs_slots, defer)
        (2, 2, 8, 8, 4, 4, 2, 1, False),
        (4, 2, 8, 8, 4, 4, 2, 1, False),   # tests/test_sched.cpp census
        (8, 4, 8, 8, 4, 4, 2, 1, False),
        (8, 2, 8, 8, 4, 4, 1, 1, False),
        (8, 2, 8, 8, 4, 4, 4, 2, False),
        (8, 2, 8, 8, 4, 4, 2, 1, True),
        (24, 1, 8, 8, 8, 8, 2, 1, False),  # 1.3B flat
        (24, 2, 8, 8, 8, 8, 2, 1, False),
        (32, 2, 8, 8, 4, 4, 2, 1, False),  # 7B
        (16, 4, 8, 8, 2, 2, 2, 1, False),  # MoE
        (2, 1, 4, 4, 2, 2, 2, 1, False),   # CPU config
        (2, 2, 4, 4, 2, 2, 2, 1, False),
    ]
    for L, M, dp, z1, z2, z3, depth, rss, defer in grid:
        for vanilla in (False, True):
            tasks, summ = ref.task_graph(L, 1000000, seq=1024, num_mb=M, flops=6e6, dp=dp, z1=z1,
                                         z2=z2, z3=z3, intra_bw=1e10, intra_lat=1e-6,
                                         device_flops=1e12, defer_rs=defer, depth=depth,
                                         rs_slots=rss, vanilla=vanilla)
            out.append({
                "layers": L, "num_mb": M, "dp": dp, "z1": z1, "z2": z2, "z3": z3,
                "depth": depth, "rs_slots": rss, "defer_rs": defer, "vanilla": vanilla,
                "ppl": 1000000, "seq": 1024, "flops": 6e6, "intra_bw": 1e10,
                "intra_lat": 1e-6, "device_flops": 1e12,
                "tasks": [{k: t[k] for k in ("kind", "layer", "mb", "pass", "bytes", "deps")}
                          for t in tasks],
                "dur": [t["dur"] for t in tasks],
                "start": [t["start"] for t in tasks],
                "end": [t["end"] for t in tasks],
                "pool_release": [t["pool_release"] for t in tasks],
                "summary": summ,
            })
    depth = [{"layers": 8, "ppl": 1000000, "budget": b,
              "depth": ref.L.ref_derive_prelaunch_depth(8, 1000000, 8, 8, 4, 4, b)}
             for b in (0, 2000000, 6000000, 6999999, 200000000)]
    return {"graphs": out, "prelaunch_depth": depth}


def pipeline_cases(ref: RefLib):
    """The CLI's graph (hzpsim.cpp:111-127): pipeline order for `rank`, then
    apply_reuse (mode 1) or not (mode 2), then recompute_rule."""
    out = []
    grid = [
        # (layers, num_mb, dp, z1, z2, z3, pp, vpp, rank, mode, recompute, defer)
        (2, 2, 8, 8, 4, 4, 1, 1, 0, 1, False, False),   # SURVEY App. A-2 with reuse: 23 tasks
        (4, 4, 8, 8, 4, 4, 1, 1, 0, 1, False, False),
        (8, 2, 8, 8, 8, 8, 1, 1, 0, 1, True, False),
        (8, 4, 4, 4, 2, 2, 2, 1, 0, 1, False, False),   # 1F1B warm-up on rank 0
        (8, 4, 4, 4, 2, 2, 2, 1, 1, 1, False, False),
        (8, 4, 4, 4, 2, 2, 2, 1, 0, 2, False, False),
        (8, 4, 4, 4, 2, 2, 2, 1, 0, 1, True, False),
        (8, 4, 4, 4, 2, 2, 2, 1, 0, 1, False, True),
        (8, 4, 4, 4, 2, 2, 2, 2, 0, 1, False, False),   # interleaved
        (8, 4, 4, 4, 2, 2, 2, 2, 1, 1, True, False),
        (12, 6, 2, 2, 2, 2, 3, 2, 2, 1, False, False),
        (12, 6, 2, 2, 2, 2, 3, 2, 1, 2, True, True),
        (4, 3, 8, 8, 4, 4, 4, 1, 3, 1, False, False),
    ]
    for L, M, dp, z1, z2, z3, pp, vpp, rank, mode, rec, defer in grid:
        tasks, summ = ref.task_graph(L, 1000000, seq=1024, num_mb=M, flops=6e6, dp=dp, z1=z1, z2=z2,
                                     z3=z3, pp=pp, vpp=vpp, intra_bw=1e10, intra_lat=1e-6,
                                     device_flops=1e12, defer_rs=defer, rank=rank, with_reuse=mode,
                                     recompute=rec, depth=2, rs_slots=1)
        out.append({
            "layers": L, "num_mb": M, "dp": dp, "z1": z1, "z2": z2, "z3": z3, "pp": pp, "vpp": vpp,
            "rank": rank, "reuse": mode == 1, "recompute": rec, "defer_rs": defer,
            "ppl": 1000000, "seq": 1024, "flops": 6e6, "intra_bw": 1e10, "intra_lat": 1e-6,
            "device_flops": 1e12,
            "tasks": [{k: t[k] for k in ("kind", "layer", "mb", "pass", "bytes", "deps")} for t in tasks],
            "dur": [t["dur"] for t in tasks],
            "start": [t["start"] for t in tasks],
            "end": [t["end"] for t in tasks],
            "summary": summ,
        })
    return {"graphs": out}


def layout_cases(ref: RefLib):
    out = []
    for dp in (1, 2, 4, 8):
        divs = [d for d in range(1, dp + 1) if dp % d == 0]
        for z1 in divs:
            for z2 in divs:
                for z3 in divs:
                    out.append({"dp": dp, "z1": z1, "z2": z2, "z3": z3,
                                "Z1": ref.groups(dp, z1, z2, z3, 0),
                                "Z2": ref.groups(dp, z1, z2, z3, 1),
                                "Z3": ref.groups(dp, z1, z2, z3, 2),
                                "DZP": ref.groups(dp, z1, z2, z3, 3)})
    se = [{"n": n, "parts": p, "s": int(ref.L.ref_shard_elems(n, p))}
          for n, p in ((10, 2), (10, 3), (1, 8), (0, 4), (428, 2), (428, 4), (1000, 8),
                       (1310000000, 8), (6610000000, 4), (6610000000, 8))]
    val = [{"dp": dp, "z1": z1, "z2": z2, "z3": z3, "layers": L, "ppl": ppl,
            "code": ref.L.ref_validate(L, ppl, dp, z1, z2, z3, dp)}
           for dp, z1, z2, z3, L, ppl in ((8, 8, 4, 2, 4, 1000), (8, 8, 3, 2, 4, 1000),
                                          (8, 1, 1, 1, 0, 0), (6, 3, 2, 6, 2, 10),
                                          (6, 4, 2, 6, 2, 10))]
    return {"groups": out, "shard_elems": se, "validate": val}


def kernel_cases(ref: RefLib, o: Oracle):
    rng = np.random.default_rng(21)
    raw = rng.integers(0, 2**32, size=4099, dtype=np.uint64).astype(np.uint32)
    # keep NaN payloads out; they are tested separately
    f = raw.view(np.float32).copy()
    f = f[~np.isnan(f)]
    r = f.copy()
    ref.L.ref_bf16_round_vec(r, r.size, 0)
    known = {str(x): float(ref.L.ref_bf16_round(x)) for x in
             (1.0, -2.0, 0.0, 1.0078125, 1.00390625, 1.01171875, 1.005, -1.005)}
    # RS / AR known answers, fp32 left fold (tests/test_collective.cpp:96-111)
    fulls = o.seeded_uniform(4 * 8, 77, np.float32).reshape(4, 8)
    rs = np.zeros(8, dtype=np.float32)
    ref.L.ref_reduce_scatter_f32(np.ascontiguousarray(fulls), 4, 8, rs)
    ar = np.zeros(8, dtype=np.float32)
    ref.L.ref_all_reduce_f32(np.ascontiguousarray(fulls), 4, 8, ar)
    return {
        "bf16_bits_in": [int(x) for x in f.view(np.uint32)],
        "bf16_bits_out": [int(x) for x in r.view(np.uint32)],
        "bf16_known": known,
        "rs_in": [float(x) for x in fulls.reshape(-1)],
        "rs_out": [float(x) for x in rs.reshape(-1)],
        "ar_out": [float(x) for x in ar],
    }


def main():
    ref = RefLib()
    o = Oracle()
    for name, payload in (("numerics", numerics_cases(ref, o)), ("sched", sched_cases(ref)),
                          ("layout", layout_cases(ref)),
                          ("pipeline", pipeline_cases(ref)), ("kernels", kernel_cases(ref, o))):
        path = os.path.join(HERE, f"{name}.json")
        with open(path, "w") as fh:
            json.dump(payload, fh, indent=None, separators=(",", ":"))
        print(path, os.path.getsize(path))


if __name__ == "__main__":
    main()
