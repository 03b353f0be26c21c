"""Large-K Cholesky timings (library event hooks) on random PD Grams.

    python tools/time_chol.py [K] [drops]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2503_18118_b200 as xl  # noqa: E402
from paper_2503_18118_b200 import parallel  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    xl._L.xlmimo_timing_enable(1)
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    xl._L.xlmimo_timing_enable(0)
    return {k: round(v[1] / reps, 3) for k, v in parallel.read_kernel_times(xl).items()}


K = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
D = int(sys.argv[2]) if len(sys.argv) > 2 else 148
g = torch.Generator(device="cuda").manual_seed(K)
H = torch.randn((D, 2 * K, K), dtype=torch.complex128, device="cuda", generator=g)
G = (H.conj().transpose(1, 2) @ H).contiguous()
allr = xl.RECV_CAP | xl.RECV_ZF | xl.RECV_MMSE | xl.RECV_MRC
print(json.dumps({"K": K, "drops": D, "app_a": timed(lambda: xl.app_a_bounds(G, [0.0])),
                  "receivers": timed(lambda: xl.sum_rate(G, [10.0], allr))}))
