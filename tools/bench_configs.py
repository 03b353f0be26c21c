"""Per-config, per-path timings on one GPU (secondary to bench.py, which times cfg2).

    python tools/bench_configs.py [cfgs...]      e.g. 1 3 4 5

For each config: fused fp64 Gram, fused fp32 Gram, materialised (K4a write + K4b
stream) where applicable, closed form (ULA), receivers.  Kernel device times come
from the library's event hooks; HBM GB/s for the streaming kernel counts the
algorithmic bytes 8 N K per drop.  Drop counts are reduced for the big configs
(stated in the output).  Prints one JSON object per line.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2503_18118_b200 as xl  # noqa: E402
from paper_2503_18118_b200 import parallel  # noqa: E402
from workloads import CONFIGS  # noqa: E402

DROPS = {1: 1000, 2: 10000, 3: 10000, 4: 1000, 5: 32}
PEAK_FP64 = 148 * 64 * 1965e6
HBM = 6547.8e9


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    xl._L.xlmimo_timing_enable(1)
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    xl._L.xlmimo_timing_enable(0)
    kt = parallel.read_kernel_times(xl)
    return {k: v[1] / reps for k, v in kt.items()}


def main(cfgs):
    for c in cfgs:
        w = CONFIGS[c]
        D = DROPS[c]
        arr = xl.Array.ula(w.n_y, w.fc_hz) if w.kind == "ula" else xl.Array.upa(w.n_y, w.n_z, w.fc_hz)
        pos = xl.gen_drops(xl.Users.polar(w.r, w.az, w.el), w.K, D, seed=w.seed)
        N, K = w.N, w.K
        coef = N * K * D
        ops = D * N * (K * 31 + 4 * K * (K - 1) // 2 + 2 * K)  # bench.py FP64_OPS_PER_COEF model
        cmac = D * N * K * (K + 1) // 2
        res = {"cfg": c, "workload": w.name, "drops_timed": D, "drops_config": w.n_drops}
        t = timed(lambda: xl.gram_exact(arr, pos, precision=xl.FP64))
        k = max((k for k in t if k.startswith("gram_fused")), key=lambda k: t[k])
        res["fused_fp64"] = {"kernel": k, "ms": t[k], "cmac_per_s": cmac / (t[k] * 1e-3),
                             "fp64_frac_of_nominal": ops / (t[k] * 1e-3) / PEAK_FP64}
        t = timed(lambda: xl.gram_exact(arr, pos, precision=xl.FP32))
        k = max((k for k in t if k.startswith("gram_fused")), key=lambda k: t[k])
        res["fused_fp32"] = {"kernel": k, "ms": t[k], "cmac_per_s": cmac / (t[k] * 1e-3)}
        t = timed(lambda: xl.gram_exact(arr, pos, precision=xl.FP32, mode=xl.MATERIALIZED), reps=2)
        bytes_h = 8 * N * K * D
        ks = [k for k in t if k.startswith("gram_stream")]
        if ks:
            res["materialised"] = {"write_ms": t.get("h_materialise"), "stream_kernel": ks[0], "stream_ms": t[ks[0]],
                                   "stream_gbs": bytes_h / (t[ks[0]] * 1e-3) / 1e9,
                                   "stream_frac_hbm_measured_copy": bytes_h / (t[ks[0]] * 1e-3) / HBM,
                                   "write_gbs": bytes_h / (t["h_materialise"] * 1e-3) / 1e9}
        if w.kind == "ula":
            t = timed(lambda: xl.gram_closed_form(arr, pos))
            res["closed_form_ms"] = t.get("closed_form")
        G = xl.gram_exact(arr, pos, precision=xl.FP64)
        t = timed(lambda: xl.sum_rate(G, list(w.snr_db), w.receivers))
        res["sum_rate_ms"] = t.get("sum_rate")
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [1, 3, 4, 5])
