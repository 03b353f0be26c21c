"""A/B of MT2 variants across K on the E1 field (35 000 elements, 1000 drops):
    python tools/ab_mt2k.py "K1,K2,..." VARIANT...   (tuning experiment, GPU box)"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402
from variants import load  # noqa: E402

Ks = [int(k) for k in sys.argv[1].split(",")]
for name in sys.argv[2:]:
    xl = load(name)
    a = xl.Array.ula(35000, 100e9)
    for K in Ks:
        pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, 1000, seed=13)
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
        print(f"{name:10s} K={K:4d} {statistics.median(ts):9.3f} ms  G00={float(G[0, 0, 0].real):.9e}", flush=True)
