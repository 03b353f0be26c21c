import sys, statistics
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tools')
import torch
from variants import load
for name in sys.argv[1:]:
    xl = load(name)
    a = xl.Array.ula(35000, 100e9)
    for K in (120, 128):
        pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, 1000, seed=13)
        G = xl.gram_exact(a, pos)
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); e0.record(); G = xl.gram_exact(a, pos); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(name, K, round(statistics.median(ts), 2), float(G[0, 0, 0].real), float(G[0, 0, K - 1].imag), flush=True)
