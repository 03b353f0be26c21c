"""Small invocations of every kernel path, for compute-sanitizer (one tool per run).

    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2503_18118_b200 as xl  # noqa: E402

u = xl.Users.polar((2.0, 20.0), (-60.0, 60.0))
for K, N, prec, mode in [(8, 1000, xl.FP64, xl.FUSED), (4, 999, xl.FP64, xl.FUSED), (3, 777, xl.FP64, xl.FUSED),
                         (16, 2048, xl.FP64, xl.FUSED), (33, 1500, xl.FP64, xl.FUSED),
                         (4, 512, xl.FP32, xl.FUSED), (16, 4096, xl.FP32, xl.FUSED), (40, 1024, xl.FP32, xl.FUSED),
                         (16, 4096, xl.FP32, xl.MATERIALIZED), (5, 1001, xl.FP32, xl.MATERIALIZED)]:
    a = xl.Array.ula(N, 100e9)
    pos = xl.gen_drops(u, K, 3, seed=K)
    G = xl.gram_exact(a, pos, precision=prec, mode=mode)
    r, f = xl.sum_rate(G, [0.0, 10.0], 15)
    if mode == xl.FUSED and prec == xl.FP64:
        Gc, fl = xl.gram_closed_form(a, pos)
upa = xl.Array.upa(16, 12, 100e9)
pos = xl.gen_drops(xl.Users.polar((2.0, 20.0), (-60, 60), (-30, 30)), 12, 2, seed=1)
xl.gram_exact(upa, pos)
xl.gram_exact(upa, pos, precision=xl.FP32)
res = xl.saturation_sweep(xl.Array.ula(1024, 28e9), [256, 512, 1024], 8, 5, [0.0, 10.0], 7, users=u, per_drop=True)
res = xl.saturation_sweep(xl.Array.ula(1024, 28e9), [256, 512, 1024], 8, 5, [0.0, 10.0], 15, users=u,
                          gram_kind=xl.GRAM_CLOSED_FORM)
torch.cuda.synchronize()
print("sanitize smoke ok", res["sat"])
