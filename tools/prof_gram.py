"""One gram_exact call on a config (for ncu captures).

    python tools/prof_gram.py <cfg> <fp64|fp32|mat32> <drops>
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2503_18118_b200 as xl  # noqa: E402
from workloads import CONFIGS  # noqa: E402

w = CONFIGS[int(sys.argv[1])]
prec = sys.argv[2] if len(sys.argv) > 2 else "fp64"
D = int(sys.argv[3]) if len(sys.argv) > 3 else 100
arr = xl.Array.ula(w.n_y, w.fc_hz) if w.kind == "ula" else xl.Array.upa(w.n_y, w.n_z, w.fc_hz)
pos = xl.gen_drops(xl.Users.polar(w.r, w.az, w.el), w.K, D, seed=w.seed)
for _ in range(2):
    G = xl.gram_exact(arr, pos, precision=xl.FP64 if prec == "fp64" else xl.FP32,
                      mode=xl.MATERIALIZED if prec == "mat32" else xl.FUSED)
torch.cuda.synchronize()
print("ok", G.shape, float(G[0, 0, 0].real))
