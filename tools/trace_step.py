"""Chrome trace (trace.cpp's format) of one measured 1.3B-class step next to
the reference simulator's timeline of the same task graph.

    python tools/trace_step.py OUT_PREFIX       # OUT_PREFIX_measured.json, OUT_PREFIX_simulated.json
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2510_20111_b200 import EngineConfig, HzpEngine  # noqa: E402
from paper_2510_20111_b200 import hzp as H  # noqa: E402
from paper_2510_20111_b200.trace import chrome_trace, measured_trace  # noqa: E402


def main():
    import json
    out = sys.argv[1]
    L, M = 24, 2
    eng = HzpEngine(EngineConfig(model=1, precision=1, gpt_layers=L, gpt_hidden=2048, gpt_heads=16, gpt_ffn=8192,
                                 gpt_vocab=50304, gpt_seq=2048, batch=4, num_microbatches=M, my_rank=0))
    eng.init_random()
    tok = torch.from_numpy(np.random.default_rng(0).integers(0, 50304, size=(1, M, 4, 2049),
                                                             dtype=np.int32)).cuda()
    for _ in range(3):
        eng.step_async(tok.data_ptr(), True)
    eng.sync()
    eng.set_timeline(True)
    eng.step_async(tok.data_ptr(), True)
    eng.sync()
    g = H.build_task_graph(H.ModelSpec(num_layers=L + 2, params_per_layer=1, num_microbatches=M),
                           H.ParallelConfig(), H.CostModel())
    with open(out + "_measured.json", "w") as fh:
        json.dump(measured_trace(eng, g, "hzp_b200 measured step (1.3B, N=1)"), fh)
    # the reference simulator's view of the same graph (its unit cost model)
    tl = eng.timeline()
    sim = H.simulate(g, 2, 1, H.ASYNC)
    with open(out + "_simulated.json", "w") as fh:
        json.dump(chrome_trace(g, sim.start, sim.end, "reference simulate() (unit cost model)"), fh)
    print("makespan_ms", tl["makespan_ms"], "compute_idle_ms", tl["compute_idle_ms"])
    eng.close()


if __name__ == "__main__":
    main()
