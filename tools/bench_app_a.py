"""Appendix A (NEXT-3) and large-K receiver timings on one GPU (library event hooks).

    python tools/bench_app_a.py

Grams: exact fp64 (E1/E3 user field, 100 GHz); K > 64 through the block-pair DMMA
kernel (K <= 128) or the chunked DMMA SYRK (K > 128; XLMIMO_LARGE_K=blk|syrk overrides).  Work per drop for the Cholesky path: (1 + n_snr) K^3/6 complex MACs.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2503_18118_b200 as xl  # noqa: E402
from paper_2503_18118_b200 import parallel  # noqa: E402

PEAK_FP64 = 148 * 64 * 1965e6


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    xl._L.xlmimo_timing_enable(1)
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    xl._L.xlmimo_timing_enable(0)
    return {k: v[1] / reps for k, v in parallel.read_kernel_times(xl).items()}


def main():
    snr = [0.0]
    for K, N, D in [(8, 4096, 10000), (32, 4096, 10000), (64, 8192, 2000)]:
        pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, D, seed=1)
        G = xl.gram_exact(xl.Array.ula(N, 100e9), pos)
        t = timed(lambda: xl.app_a_bounds(G, snr))
        te = timed(lambda: xl.app_a_bounds(G, snr, eig=True), reps=1)
        print(json.dumps({"K": K, "drops": D, "app_a_ms": t, "with_eig_ms": te}), flush=True)
    for K, N, D in [(100, 35000, 1000), (256, 35000, 148), (1000, 35000, 148)]:
        pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, D, seed=2)
        a = xl.Array.ula(N, 100e9)
        tg = timed(lambda: xl.gram_exact(a, pos), reps=1)
        G = xl.gram_exact(a, pos)
        t = timed(lambda: xl.app_a_bounds(G, snr))
        chol = t.get("chol_logdet", float("nan"))
        cmac = D * 2 * K ** 3 / 6
        gk = sum(v for k, v in tg.items() if k.startswith("gram"))  # all kernels of the exact Gram
        gcmac = D * N * K * (K + 1) / 2
        nb = (K + 63) // 64
        if any(k.startswith("gram_syrk") for k in tg):  # 32x32 tile pairs in the 3M form (3 real
            nt = (K + 31) // 32                           # products per complex one), H generated once
            ops = D * N * (nt * (nt + 1) // 2 * 32 * 32 * 3 + nt * 32 * 29)
        elif K <= 128:  # MT2: G(G+1)/2 8x8 plane blocks, 3 DMMAs (3M) each, 29 + 1 (partner plane)
            g = (K + 7) // 8  # FP64 ops per generated coefficient (G = 16: two launches, each generating all)
            ops = D * N * (g * (g + 1) // 2 * 64 * 3 + (2 if g == 16 else 1) * 8 * g * 30)
        else:  # 64-user block pairs, both blocks generated per pair
            ops = D * N * (nb * (nb + 1) // 2 * 64 * 64 * 4 + (nb * nb) * 64 * 29)
        print(json.dumps({"K": K, "N": N, "drops": D, "gram_ms": tg, "gram_cmac_per_s": gcmac / (gk * 1e-3),
                          "gram_frac_fp64_useful": 4 * gcmac / (gk * 1e-3) / PEAK_FP64,
                          "gram_frac_fp64_issued_model": ops / (gk * 1e-3) / PEAK_FP64,
                          "app_a_ms": t, "chol_cmac_per_s": cmac / (chol * 1e-3),
                          "chol_frac_fp64_nominal": 4 * cmac / (chol * 1e-3) / PEAK_FP64,
                          "gap_mean": float(xl.app_a_bounds(G, snr)[0][:, 1].mean())}), flush=True)
        allr = xl.RECV_CAP | xl.RECV_ZF | xl.RECV_MMSE | xl.RECV_MRC
        tr = timed(lambda: xl.sum_rate(G, snr, allr), reps=1)
        print(json.dumps({"K": K, "drops": D, "sum_rate_all_receivers_ms": tr}), flush=True)


if __name__ == "__main__":
    main()
