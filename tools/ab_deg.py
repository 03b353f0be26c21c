"""A/B of an fp64-generator variant against the product (tuning experiment, GPU box):
time gram_exact (fused fp64) per config and report the variant's max normalised Gram
difference |dG_ij| / sqrt(G_ii G_jj) from the product on the same drops.

    python tools/ab_deg.py VARIANT
"""
import statistics
import sys

import torch

import os  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from variants import load  # noqa: E402
from workloads import CONFIGS  # noqa: E402


def run(xl, cfg, drops, reps=5):
    w = CONFIGS[cfg]
    arr = xl.Array.ula(w.n_y, w.fc_hz) if w.kind == "ula" else xl.Array.upa(w.n_y, w.n_z, w.fc_hz)
    if cfg == 2:
        arr = xl.Array.ula(max(w.n_list), w.fc_hz)
    pos = xl.gen_drops(xl.Users.polar(w.r, w.az, w.el), w.K, drops, seed=w.seed)
    G = xl.gram_exact(arr, pos, precision=xl.FP64)
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        xl.gram_exact(arr, pos, precision=xl.FP64)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts), G


name = sys.argv[1]
prod, var = load("product"), load(name)
for cfg, drops in ((5, 296), (4, 1000), (3, 10000), (2, 2000), (1, 100000)):
    tp, Gp = run(prod, cfg, drops)
    tv, Gv = run(var, cfg, drops)
    d = torch.diagonal(Gp, dim1=1, dim2=2).real
    nrm = torch.sqrt(d[:, :, None] * d[:, None, :])
    err = float(((Gv - Gp).abs() / nrm).max())
    print(f"cfg{cfg} D={drops}: product {tp:.3f} ms  {name} {tv:.3f} ms  ({100 * (tv / tp - 1):+.2f} %)  "
          f"max norm diff {err:.2e}", flush=True)
