"""fp32 fused Gram error of A/B builds (tools/variants.py names) against the product's fp64
Gram (itself 1e-12 from the oracle): normalised error and mean diagonal bias, on cfg3/cfg4/
cfg5 geometries and users close to the array, plus the cfg5 rates' worst deviation.

    python tools/fp32_err_var.py NAME...
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from tests._util import normalized_err  # noqa: E402
from variants import load  # noqa: E402
from workloads import CONFIGS  # noqa: E402

ref = load("product")
rng = np.random.default_rng(5)
p = np.zeros((8, 16, 3))
p[..., 0] = rng.uniform(0.3, 0.6, (8, 16))
p[..., 1] = rng.uniform(-5.0, 5.0, (8, 16))
cases = [("close K16 N8192", ("ula", 8192, 1, 100e9), torch.tensor(p, device="cuda"))]
for c, D in ((3, 200), (4, 16), (5, 8)):
    w = CONFIGS[c]
    cases.append((f"cfg{c}", (w.kind, w.n_y, w.n_z, w.fc_hz),
                  ref.gen_drops(ref.Users.polar(w.r, w.az, w.el), w.K, D, seed=3)))
for name in sys.argv[1:]:
    xl = load(name)
    for tag, (kind, n_y, n_z, fc), pos in cases:
        a = xl.Array.ula(n_y, fc) if kind == "ula" else xl.Array.upa(n_y, n_z, fc)
        ar = ref.Array.ula(n_y, fc) if kind == "ula" else ref.Array.upa(n_y, n_z, fc)
        Go = ref.gram_exact(ar, pos).cpu().numpy()
        Gt = xl.gram_exact(a, pos, precision=xl.FP32)
        G = Gt.cpu().numpy()
        d = np.real(np.diagonal(Go, axis1=1, axis2=2))
        bias = float(np.mean(np.real(np.diagonal(G, axis1=1, axis2=2)) / d - 1))
        line = f"{name:10s} {tag:18s} err {normalized_err(G, Go):.3e}  diag bias {bias:+.2e}"
        if tag == "cfg5":
            recv = ref.RECV_ZF | ref.RECV_MMSE | ref.RECV_CAP
            r64, _ = ref.sum_rate(ref.gram_exact(ar, pos), [10.0], recv)
            r32, _ = ref.sum_rate(torch.as_tensor(G, device="cuda"), [10.0], recv)
            line += f"  rates max|d| {float((r32 - r64).abs().max()):.2e} mean d {float((r32 - r64).mean()):+.2e}"
        print(line, flush=True)
