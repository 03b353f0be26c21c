"""One cfg1 steady-state Gram launch (10^6 drops, kernel W) for ncu captures.

    python tools/prof_steady.py [n_drops]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2503_18118_b200 as xl  # noqa: E402
from workloads import CONFIGS  # noqa: E402

w = CONFIGS[1]
D = int(sys.argv[1]) if len(sys.argv) > 1 else 10 ** 6
arr = xl.Array.ula(w.n_y, w.fc_hz)
pos = xl.gen_drops(xl.Users.polar(w.r, w.az), w.K, D, seed=w.seed)
for _ in range(2):
    G = xl.gram_exact(arr, pos)
torch.cuda.synchronize()
print("ok", G.shape)
