"""fp32 K > 64 Gram: in-kernel generation (XLMIMO_OPT_PAIR = 1) vs TMA-fed fp16 chunks (2),
timed on the E1/E3 user field at 35 000 elements (tuning the crossover kStreamPairMinK)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2503_18118_b200 as xl  # noqa: E402

a = xl.Array.ula(35000, 100e9)
for K, D in [(65, 1000), (100, 1000), (160, 500), (200, 300), (256, 148), (320, 148), (352, 148)]:
    pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, D, seed=13)
    row = [K, D]
    for o in (1, 2):
        with xl.option(xl.OPT_PAIR, o):
            xl.gram_exact(a, pos, precision=xl.FP32)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            xl.gram_exact(a, pos, precision=xl.FP32)
            e1.record()
            torch.cuda.synchronize()
            row.append(round(e0.elapsed_time(e1), 3))
    print("K %d D %d  gen %.3f ms  stream %.3f ms" % tuple(row), flush=True)
