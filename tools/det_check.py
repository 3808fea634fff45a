"""Run-to-run determinism of the GPT engine step, and bitwise neutrality of
parameter reuse / activation recomputation (dense and MoE, dp = 1 and dp = 2
emulated).  Prints, per variant, whether the losses match the plain run and
the max |difference| of the updated parameters and of the gradient shards.

    python tools/det_check.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, ROOT)

from test_gpu_gpt import CFG, _engine  # noqa: E402


def main():
    c = dict(CFG, layers=3)
    tok = np.random.default_rng(5).integers(0, c["vocab"], size=(2, 2, c["batch"], c["seq"] + 1), dtype=np.int32)
    for experts in (0, 8):
        for dp, z in ((2, (2, 2, 2)), (1, (1, 1, 1))):
            t = tok if dp == 2 else tok[:1]
            out = {}
            for key in ((0, 0), (0, 0, "again"), (1, 0), (0, 1), (1, 1)):
                e = _engine(c, dp=dp, z=z, mbs=2, reuse=key[0], recompute=key[1], gpt_experts=experts)
                e.init_random(seed=11, scale=0.04)
                losses = [np.asarray(e.step(t)) for _ in range(2)]
                out[key] = (losses, [e.param_f32(r) for r in range(dp)], [e.download(r, 1) for r in range(dp)])
                e.close()
            base = out[(0, 0)]
            for k, v in out.items():
                print(experts, dp, k, "loss", [np.array_equal(x, y) for x, y in zip(v[0], base[0])],
                      "param", [float(np.abs(x - y).max()) for x, y in zip(v[1], base[1])],
                      "grad", [float(np.abs(x - y).max()) for x, y in zip(v[2], base[2])], flush=True)


if __name__ == "__main__":
    main()
