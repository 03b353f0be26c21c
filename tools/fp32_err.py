"""Normalised error of the fp32 (TF32 tensor-core) Gram paths against the oracle on a few
geometries, printed (margin check for the 1e-4 tier; tests assert, this prints)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as orc  # noqa: E402
import paper_2503_18118_b200 as xl  # noqa: E402
from tests._util import normalized_err  # noqa: E402

orc.build()
rng = np.random.default_rng(5)
p = np.zeros((2, 16, 3))
p[..., 0] = rng.uniform(0.3, 0.6, (2, 16))
p[..., 1] = rng.uniform(-5.0, 5.0, (2, 16))
cases = [("close 0.3-0.6 m, K16, N8192", xl.Array.ula(8192, 100e9), orc.array("ula", n_y=8192, fc_hz=100e9),
          torch.tensor(p, device="cuda"))]
for name, kind, n_y, n_z, fc, K, r, az, el, D in [("cfg3", "ula", 16384, 1, 100e9, 16, (2, 20), (-75, 75), (0, 0), 8),
                                                  ("cfg4", "upa", 256, 256, 100e9, 32, (2, 20), (-60, 60), (-30, 30), 4),
                                                  ("ula K40", "ula", 5000, 1, 140e9, 40, (5, 100), (-60, 60), (0, 0), 4)]:
    a = xl.Array.ula(n_y, fc) if kind == "ula" else xl.Array.upa(n_y, n_z, fc)
    ao = orc.array(kind, n_y=n_y, n_z=n_z, fc_hz=fc)
    cases.append((name, a, ao, xl.gen_drops(xl.Users.polar(r, az, el), K, D, seed=3)))
for name, a, ao, pos in cases:
    Go = orc.gram_exact(ao, pos.cpu().numpy())
    for mode, tag in ((xl.FUSED, "fused"), (xl.MATERIALIZED, "mat")):
        G = xl.gram_exact(a, pos, precision=xl.FP32, mode=mode).cpu().numpy()
        d = np.real(np.diagonal(Go, axis1=1, axis2=2))
        bias = float(np.mean(np.real(np.diagonal(G, axis1=1, axis2=2)) / d - 1))
        print(f"{name:28s} {tag:6s} err {normalized_err(G, Go):.3e}  diag bias {bias:+.2e}", flush=True)
