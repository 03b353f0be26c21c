import sys; sys.path.insert(0,'/root/repo')
import torch, paper_2503_18118_b200 as xl
from paper_2503_18118_b200 import parallel
a = xl.Array.ula(35000, 100e9)
for K in (64, 100, 160, 256):
    pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, 1000, seed=13)
    G = xl.gram_exact(a, pos)
    xl.sum_rate(G, [10.0], xl.RECV_ZF | xl.RECV_MMSE | xl.RECV_CAP)
    torch.cuda.synchronize()
    xl._L.xlmimo_timing_enable(1)
    for _ in range(3):
        xl.gram_exact(a, pos)
        xl.sum_rate(G, [10.0], xl.RECV_ZF | xl.RECV_MMSE | xl.RECV_CAP)
    torch.cuda.synchronize()
    xl._L.xlmimo_timing_enable(0)
    print(K, {k: round(v[1]/3, 3) for k, v in parallel.read_kernel_times(xl).items()}, flush=True)
