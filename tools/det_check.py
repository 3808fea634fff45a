import sys, numpy as np
import os; R = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, os.path.join(R, "tests")); sys.path.insert(0, R)
from test_gpu_gpt import CFG, _engine
c = dict(CFG, layers=3)
rng = np.random.default_rng(5)
tok = rng.integers(0, c["vocab"], size=(2, 2, c["batch"], c["seq"] + 1), dtype=np.int32)
for experts in (0, 8):
  for dp, z in ((2, (2, 2, 2)), (1, (1, 1, 1))):
    t = tok if dp == 2 else tok[:1]
    out = {}
    for key in ((0, 0), (0, 0, "again"), (1, 0), (0, 1), (1, 1)):
        e = _engine(c, dp=dp, z=z, mbs=2, reuse=key[0], recompute=key[1], gpt_experts=experts)
        e.init_random(seed=11, scale=0.04)
        ls = [np.asarray(e.step(t)) for _ in range(2)]
        out[key] = (ls, [e.param_f32(r) for r in range(dp)], [e.download(r, 1) for r in range(dp)])
        e.close()
    b = out[(0, 0)]
    for k, v in out.items():
        print(experts, dp, k, "loss", [np.array_equal(x, y) for x, y in zip(v[0], b[0])],
              "param", [float(np.abs(x - y).max()) for x, y in zip(v[1], b[1])],
              "grad", [float(np.abs(x - y).max()) for x, y in zip(v[2], b[2])], flush=True)
