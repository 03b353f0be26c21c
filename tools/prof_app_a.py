"""One Appendix A call at large K (Cholesky kernels) for ncu captures.

    python tools/prof_app_a.py <K> <drops>
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2503_18118_b200 as xl  # noqa: E402

K, D = int(sys.argv[1]), int(sys.argv[2])
g = torch.Generator(device="cuda").manual_seed(K)
H = torch.randn((D, 2 * K, K), dtype=torch.complex128, device="cuda", generator=g)
G = (H.conj().transpose(1, 2) @ H).contiguous()
for _ in range(2):
    rs, bo, _, fl = xl.app_a_bounds(G, [0.0])
torch.cuda.synchronize()
print("ok", float(rs[0, 1]))
