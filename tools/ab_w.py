"""A/B of kernel W variants on cfg1's steady state (10^6 drops; tuning experiment, GPU box):
    python tools/ab_w.py VARIANT..."""
import sys, statistics
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tools')
import torch
from variants import load
from workloads import CONFIGS
w = CONFIGS[1]
for name in sys.argv[1:]:
    xl = load(name)
    a = xl.Array.ula(w.n_y, w.fc_hz)
    pos = xl.gen_drops(xl.Users.polar(w.r, w.az), w.K, 10**6, seed=3)
    G = xl.gram_exact(a, pos)
    ts = []
    for _ in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record(); G = xl.gram_exact(a, pos); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(name, round(statistics.median(ts), 4), float(G[5, 1, 2].real), flush=True)
