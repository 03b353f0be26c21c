"""Kernel-variant options on the configs that use them (tuning experiment, GPU box):
cfg3 fp64 Gram (10^5 drops) across XLMIMO_OPT_DMMA_VARIANT 0..3 and the cfg2 exact sweep
(10^4 drops, 9 nested N) across XLMIMO_OPT_SPLIT_NT.
    python tools/ab_opts.py"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_18118_b200 as xl  # noqa: E402
from workloads import CONFIGS  # noqa: E402


def tm(fn, reps=5):
    fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


w = CONFIGS[3]
a = xl.Array.ula(w.n_y, w.fc_hz)
pos = xl.gen_drops(xl.Users.polar(w.r, w.az), w.K, w.n_drops, seed=3)
for v in range(4):
    with xl.option(xl.OPT_DMMA_VARIANT, v):
        print(f"cfg3 fp64 DMMA variant {v}: {tm(lambda: xl.gram_exact(a, pos)):.3f} ms", flush=True)
w = CONFIGS[2]
a = xl.Array.ula(max(w.n_list), w.fc_hz)
pos = xl.gen_drops(xl.Users.polar(w.r, w.az), w.K, w.n_drops, seed=3)
for nt in (0, 64, 128, 192, 256):
    with xl.option(xl.OPT_SPLIT_NT, nt):
        t = tm(lambda: xl.saturation_sweep(a, list(w.n_list), w.K, w.n_drops, list(w.snr_db), w.receivers, pos=pos))
        print(f"cfg2 sweep split variant {nt}: {t:.3f} ms", flush=True)
