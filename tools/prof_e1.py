"""One exact fp64 Gram on the paper's E1 user field (for ncu captures): 100 GHz ULA of 35 000
elements, users x ~ U[1,10] m, y ~ U[-7.5,7.5] m.

    python tools/prof_e1.py <K> <drops>
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2503_18118_b200 as xl  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 100
D = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
a = xl.Array.ula(35000, 100e9)
pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, D, seed=13)
for _ in range(2):
    G = xl.gram_exact(a, pos)
torch.cuda.synchronize()
print("ok", tuple(G.shape), float(G[0, 0, 0].real))
