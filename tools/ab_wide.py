"""fp32 Gram for 64 < K <= 128: the fused kernel's wide + narrow launches (default) vs the
block-pair kernel (XLMIMO_OPT_PAIR = 1) vs the TMA-fed pair stream (2), E1 field, with the
normalised difference to the fp64 Gram.

    python tools/ab_wide.py
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
for K, D in ((65, 1000), (80, 1000), (100, 1000), (128, 1000)):
    pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, D, seed=13)
    G64 = xl.gram_exact(a, pos[:8]).cpu().numpy()
    row = []
    for o in (0, 1, 2):
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
            row.append(f"opt{o} {statistics.median(ts):7.3f} ms err {normalized_err(G[:8].cpu().numpy(), G64):.2e}")
    print(f"K {K:4d} D {D}: " + " | ".join(row), flush=True)
