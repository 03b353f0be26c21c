"""A/B timing of fused fp64 Gram kernel options on a config (tuning; prints, asserts parity)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2503_18118_b200 as xl  # noqa: E402
from tests._util import normalized_err  # noqa: E402
from workloads import CONFIGS  # noqa: E402

cfg, D = int(sys.argv[1]), int(sys.argv[2])
opts = [int(o) for o in sys.argv[3:]] or [0]
w = CONFIGS[cfg]
arr = xl.Array.ula(w.n_y, w.fc_hz) if w.kind == "ula" else xl.Array.upa(w.n_y, w.n_z, w.fc_hz)
pos = xl.gen_drops(xl.Users.polar(w.r, w.az, w.el), w.K, D, seed=w.seed)
ref = None
for o in opts:
    with xl.option(xl.OPT_GRAM_KERNEL, o):
        G = xl.gram_exact(arr, pos)
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            G = xl.gram_exact(arr, pos)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
    g = G.cpu().numpy()
    if ref is None:
        ref = g
    print(f"cfg{cfg} D={D} option {o}: {min(ts):.3f} ms  vs first: {normalized_err(g, ref):.2e}", flush=True)
