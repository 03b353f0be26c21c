"""Per-kernel timings (library event hooks) of the fp32 materialised / fused-pair paths for
A/B builds (tools/variants.py names; "product" = the package build).

    python tools/ab_paths.py NAME...
"""
import importlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

from variants import load  # noqa: E402
from workloads import CONFIGS  # noqa: E402


def timed(xl, fn, reps=3):
    fn()
    torch.cuda.synchronize()
    xl._L.xlmimo_timing_enable(1)
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    xl._L.xlmimo_timing_enable(0)
    par = importlib.import_module(xl.__name__ + ".parallel")
    return {k: round(v[1] / reps, 3) for k, v in par.read_kernel_times(xl).items()}


for name in sys.argv[1:]:
    xl = load(name)
    out = {}
    w = CONFIGS[5]
    arr = xl.Array.ula(w.n_y, w.fc_hz)
    pos = xl.gen_drops(xl.Users.polar(w.r, w.az), w.K, 32, seed=w.seed)
    out["cfg5 mat32 D=32"] = timed(xl, lambda: xl.gram_exact(arr, pos, precision=xl.FP32, mode=xl.MATERIALIZED))
    a = xl.Array.ula(65536, 100e9)
    pos = xl.gen_drops(xl.Users.polar((2.0, 20.0), (-60.0, 60.0)), 100, 296, seed=3)
    out["K100 fp32 fused N=65536 D=296"] = timed(xl, lambda: xl.gram_exact(a, pos, precision=xl.FP32))
    w = CONFIGS[4]
    arr = xl.Array.upa(w.n_y, w.n_z, w.fc_hz)
    pos = xl.gen_drops(xl.Users.polar(w.r, w.az, w.el), w.K, 256, seed=w.seed)
    out["cfg4 mat32 D=256"] = timed(xl, lambda: xl.gram_exact(arr, pos, precision=xl.FP32, mode=xl.MATERIALIZED))
    print(name, json.dumps(out), flush=True)
