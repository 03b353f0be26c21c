"""fp64 Gram for K > 128 (h_chunk + DMMA SYRK) on A/B builds: time and normalised
difference from the first build named, on the E3 user field (35 000 elements, 100 GHz).

    python tools/ab_syrk.py NAME...
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from tests._util import normalized_err  # noqa: E402
from variants import load  # noqa: E402

refs = {}
for name in sys.argv[1:]:
    xl = load(name)
    a = xl.Array.ula(35000, 100e9)
    for K, D in ((160, 500), (256, 148), (1000, 16)):
        pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, D, seed=13)
        G = xl.gram_exact(a, pos)
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            G = xl.gram_exact(a, pos)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        Gn = G.cpu().numpy()
        err = normalized_err(Gn, refs[K]) if K in refs else 0.0
        refs.setdefault(K, Gn)
        print(f"{name:8s} K {K:5d} D {D:4d}: {statistics.median(ts):9.3f} ms  diff {err:.2e}", flush=True)
