"""MT2 tile buffers across K on the E1 field (tuning experiment, GPU box): default vs
XLMIMO_OPT_MT2_BUFFERS = 2 and 3.
    python tools/ab_mt2buf.py "K1,K2,..." """
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_18118_b200 as xl  # noqa: E402

a = xl.Array.ula(35000, 100e9)
for K in [int(k) for k in sys.argv[1].split(",")]:
    pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, 1000, seed=13)
    for nb in (0, 2, 3):
        with xl.option(xl.OPT_MT2_BUFFERS, nb):
            G = xl.gram_exact(a, pos)
            ts = []
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                G = xl.gram_exact(a, pos)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
        print(f"K={K:4d} buffers={nb}: {statistics.median(ts):9.3f} ms", flush=True)
