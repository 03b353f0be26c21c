import sys, statistics
sys.path.insert(0, '/root/repo')
import torch, paper_2503_18118_b200 as xl
a = xl.Array.ula(35000, 100e9)
for K in (128, 129, 136, 144, 152, 160, 161, 192):
    pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, 1000, seed=13)
    G = xl.gram_exact(a, pos)
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record(); G = xl.gram_exact(a, pos); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(K, round(statistics.median(ts), 2), flush=True)
