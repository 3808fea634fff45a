"""DRAM traffic of the tcgen05 GEMM launches of one 1.3B-class step (N=1) vs
their algorithmic bytes -> profiles/*gemm_dram_traffic.json (bench.py's
roofline.traffic).

    python tools/gemm_traffic.py run            # one step; prints nothing (ncu target)
    python tools/gemm_traffic.py shapes OUT     # per-shape launch counts of one step
    python tools/gemm_traffic.py combine NCU.csv SHAPES.json OUT.json

ncu recipe (one GPU):
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \\
        --clock-control none -k regex:gemm_tc --csv --log-file g.csv python tools/gemm_traffic.py run

Algorithmic bytes per launch = A + B + C written (+ C read for an fp32
accumulate, + GELU aux written, + the side input read), each once.
"""
import collections
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one_step(profile):
    import numpy as np
    import torch
    from paper_2510_20111_b200 import EngineConfig, HzpEngine
    from paper_2510_20111_b200.engine import gemm_profile, gemm_profile_dump
    eng = HzpEngine(EngineConfig(model=1, precision=1, gpt_layers=24, gpt_hidden=2048, gpt_heads=16,
                                 gpt_ffn=8192, gpt_vocab=50304, gpt_seq=2048, batch=4, num_microbatches=2,
                                 my_rank=0))
    eng.init_random()
    tok = torch.from_numpy(np.random.default_rng(0).integers(0, 50304, size=(1, 2, 4, 2049),
                                                             dtype=np.int32)).cuda()
    if profile:
        gemm_profile(True)
    eng.step_async(tok.data_ptr(), True)
    eng.sync()
    out = None
    if profile:
        gemm_profile(False)
        out = gemm_profile_dump()[3]
    eng.close()
    return out


def shape_bytes(line):
    # "MxNxK zZ mnAB cC actE bfF"
    m = re.match(r"(\d+)x(\d+)x(\d+) z(\d+) mn(\d)(\d) c(\d) act(\d+) bf(\d)", line)
    M, N, K, Z, _, _, causal, act, bf = (int(x) for x in m.groups())
    a, b = 2 * M * K, 2 * N * K
    c = M * N * (2 if bf else 8)  # fp32 accumulate: read + write
    extra = 2 * M * N if act in (2, 4) else 0  # GELU aux out / aux in
    if causal:
        a //= 2  # only the causal half of the A operand is read
    return Z * (a + b + c + extra)


def main():
    mode = sys.argv[1]
    if mode == "run":
        one_step(False)
    elif mode == "shapes":
        text = one_step(True)
        counts = {}
        for line in text.strip().splitlines():
            key, n = line[:48].strip(), int(float(re.search(r"n=\s*(\d+)", line).group(1)))
            counts[key] = n
        json.dump(counts, open(sys.argv[2], "w"), indent=1)
    elif mode == "combine":
        rows = [r for r in csv.reader(open(sys.argv[2])) if len(r) > 10]
        h = rows[0]
        ki, mi, vi, ui, idi = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit",
                                                     "ID"))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        per = collections.defaultdict(dict)
        for r in rows[1:]:
            if "gemm_tc" in r[ki]:
                per[r[idi]][r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
        rd = sum(d.get("dram__bytes_read.sum", 0) for d in per.values())
        wr = sum(d.get("dram__bytes_write.sum", 0) for d in per.values())
        counts = json.load(open(sys.argv[3]))
        n = sum(counts.values())
        alg = sum(c * shape_bytes(k) for k, c in counts.items())
        out = {"source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over the gemm_tc launches of "
                         "one bench-config step (N=1), tools/gemm_traffic.py",
               "launches": len(per), "launches_from_profile": n, "dram_read_bytes": rd, "dram_write_bytes": wr,
               "dram_bytes_per_launch": (rd + wr) / max(1, len(per)),
               "algorithmic_bytes_per_launch": alg / max(1, n), "ratio": (rd + wr) / max(1.0, alg),
               "note": "algorithmic = A + B + C (+ C read for fp32 accumulate, + GELU aux) per launch"}
        json.dump(out, open(sys.argv[4], "w"), indent=1)
        print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
