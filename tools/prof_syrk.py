"""One fp64 Gram at K > 128 (SYRK path: h_chunk + DMMA SYRK) on the E3 field, for ncu.

    python tools/prof_syrk.py K DROPS [N]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2503_18118_b200 as xl  # noqa: E402

K = int(sys.argv[1])
D = int(sys.argv[2])
N = int(sys.argv[3]) if len(sys.argv) > 3 else 35000
a = xl.Array.ula(N, 100e9)
pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, D, seed=13)
for _ in range(2):
    G = xl.gram_exact(a, pos)
torch.cuda.synchronize()
print("ok", G.shape)
