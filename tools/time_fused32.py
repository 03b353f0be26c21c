"""Fused fp32 (tcgen05) Gram timings on cfg3 / cfg4 / cfg5 and E3 fp32 (library event hooks).

    python tools/time_fused32.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2503_18118_b200 as xl  # noqa: E402
from paper_2503_18118_b200 import parallel  # noqa: E402
from workloads import CONFIGS  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    xl._L.xlmimo_timing_enable(1)
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    xl._L.xlmimo_timing_enable(0)
    return {k: round(v[1] / reps, 3) for k, v in parallel.read_kernel_times(xl).items()}


out = {}
for c, D in [(3, 10000), (4, 1000), (5, 32)]:
    w = CONFIGS[c]
    arr = xl.Array.ula(w.n_y, w.fc_hz) if w.kind == "ula" else xl.Array.upa(w.n_y, w.n_z, w.fc_hz)
    pos = xl.gen_drops(xl.Users.polar(w.r, w.az, w.el), w.K, D, seed=w.seed)
    out[f"cfg{c}"] = timed(lambda: xl.gram_exact(arr, pos, precision=xl.FP32))
a = xl.Array.ula(35000, 100e9)
pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), 1000, 148, seed=2)
out["E3"] = timed(lambda: xl.gram_exact(a, pos, precision=xl.FP32), reps=1)
print(json.dumps(out))
