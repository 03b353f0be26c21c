"""One cfg2 saturation sweep (reduced drop count) for ncu captures.

    python tools/prof_sweep.py [n_drops] [precision fp64|fp32] [K]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2503_18118_b200 as xl  # noqa: E402
from workloads import CONFIGS  # noqa: E402

W = CONFIGS[2]
D = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
prec = xl.FP32 if len(sys.argv) > 2 and sys.argv[2] == "fp32" else xl.FP64
K = int(sys.argv[3]) if len(sys.argv) > 3 else W.K
arr = xl.Array.ula(W.n_y, W.fc_hz)
users = xl.Users.polar(W.r, W.az)
for rep in range(2):
    res = xl.saturation_sweep(arr, W.n_list, K, D, W.snr_db, W.receivers, users=users, seed=rep, precision=prec)
torch.cuda.synchronize()
print("M_sat", res["sat"][2], "launches", xl.launch_count())
