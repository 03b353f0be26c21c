"""Receivers (CAP + ZF + MMSE) for 64 < K <= 160 on A/B builds: the shared-memory Cholesky
vs the tiled DMMA one (tools/variants.py names).

    python tools/ab_chol.py NAME...
"""
import importlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

from variants import load  # noqa: E402

KS = [(72, 1000), (100, 1000), (128, 1000), (160, 1000)]
if os.environ.get("AB_CHOL_LARGE"):
    KS = [(256, 296), (512, 148), (1000, 148)]
for name in sys.argv[1:]:
    xl = load(name)
    par = importlib.import_module(xl.__name__ + ".parallel")
    a = xl.Array.ula(4096, 100e9)
    for K, D in KS:
        pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, D, seed=13)
        G = xl.gram_exact(a, pos)
        r0, _ = xl.sum_rate(G, [10.0], xl.RECV_ZF | xl.RECV_MMSE | xl.RECV_CAP)
        torch.cuda.synchronize()
        par.read_kernel_times(xl)
        xl._L.xlmimo_timing_enable(1)
        for _ in range(3):
            r, _ = xl.sum_rate(G, [10.0], xl.RECV_ZF | xl.RECV_MMSE | xl.RECV_CAP)
        torch.cuda.synchronize()
        xl._L.xlmimo_timing_enable(0)
        t = {k: round(v[1] / 3, 3) for k, v in par.read_kernel_times(xl).items() if "gram" not in k}
        print(name, K, t, float(r[0, 0, 0]), flush=True)
