"""fp32 Gram for 128 < K <= 256: the fused kernel's wide / cross / narrow launches (default up
to kFusedTcMaxK) vs the TMA-fed pair stream (XLMIMO_OPT_PAIR = 2), E1 field, 35 000 elements,
with the normalised difference to the fp64 Gram on 4 drops.

    python tools/ab_cross.py
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2503_18118_b200 as xl  # noqa: E402
from tests._util import normalized_err  # noqa: E402

a = xl.Array.ula(35000, 100e9)
for K, D in ((100, 1000), (129, 500), (160, 500), (192, 300), (200, 300), (256, 148), (320, 148)):
    pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, D, seed=13)
    G64 = xl.gram_exact(a, pos[:4]).cpu().numpy()
    row = []
    for o in (0, 2):
        with xl.option(xl.OPT_PAIR, o):
            G = xl.gram_exact(a, pos, precision=xl.FP32)
            ts = []
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                G = xl.gram_exact(a, pos, precision=xl.FP32)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            row.append(f"opt{o} {statistics.median(ts) * 1000 / D:8.3f} ms/1000 drops err {normalized_err(G[:4].cpu().numpy(), G64):.2e}")
    print(f"K {K:4d}: " + " | ".join(row), flush=True)
