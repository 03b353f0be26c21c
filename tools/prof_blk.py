"""One large-K gram_exact call (block-pair DMMA kernel, or the chunked SYRK for K > 128)
for ncu captures.

    python tools/prof_blk.py <K> <N> <drops>
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2503_18118_b200 as xl  # noqa: E402

K, N, D = (int(a) for a in sys.argv[1:4])
pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, D, seed=2)
a = xl.Array.ula(N, 100e9)
for _ in range(2):
    G = xl.gram_exact(a, pos)
torch.cuda.synchronize()
print("ok", G.shape, float(G[0, 0, 0].real))
