"""Per-config, per-path timings on one GPU (secondary to bench.py and its sub-records).

    python tools/bench_configs.py [cfgs...]      e.g. 1 3 4 5

For each config: fused fp64 Gram, fused fp32 Gram, materialised (K4a write + K4b
stream) where applicable, closed form (ULA), receivers.  Kernel device times come
from the library's event hooks; HBM GB/s for the streaming kernel counts the
algorithmic bytes 8 N K per drop.  Drop counts are reduced for the big configs
(stated in the output).  Prints one JSON object per line.
"""
import json
import statistics
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


def timed(fn, reps=5):
    """Per-kernel device ms: the median of `reps` separately timed calls after one untimed
    call (median of >= 5 runs)."""
    fn()
    torch.cuda.synchronize()
    runs = []
    for _ in range(reps):
        xl._L.xlmimo_timing_enable(1)
        fn()
        torch.cuda.synchronize()
        xl._L.xlmimo_timing_enable(0)
        runs.append({k: v[1] for k, v in parallel.read_kernel_times(xl).items()})
    return {k: statistics.median(r.get(k, 0.0) for r in runs) for k in runs[0]}


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
        t = timed(lambda: xl.gram_exact(arr, pos, precision=xl.FP32, mode=xl.MATERIALIZED))
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


def steady_cfg1(D=10 ** 6):
    """cfg1 in a steady-state batch: 10^6 drops through drops -> exact fp64 Gram
    -> closed-form Gram -> CAP/ZF/MMSE/MRC, per-kernel device times (one drop is too small to
    time on its own: the 1000-drop config is launch-bound)."""
    w = CONFIGS[1]
    arr = xl.Array.ula(w.n_y, w.fc_hz)
    users = xl.Users.polar(w.r, w.az)
    pos = xl.gen_drops(users, w.K, D, seed=w.seed)
    allr = xl.RECV_CAP | xl.RECV_ZF | xl.RECV_MMSE | xl.RECV_MRC

    def path():
        xl.gen_drops(users, w.K, D, seed=w.seed, out=pos)
        G = xl.gram_exact(arr, pos)
        Gt, fl = xl.gram_closed_form(arr, pos)
        xl.sum_rate(G, list(w.snr_db), allr)
        xl.sum_rate(Gt, list(w.snr_db), allr, flags=fl)
    t = timed(path)
    tot = sum(t.values())
    cmac = D * w.N * w.K * (w.K + 1) // 2
    print(json.dumps({"cfg": "1-steady", "workload": w.name + " (steady-state batch)", "drops_timed": D,
                      "kernel_ms": t, "total_kernel_ms": tot, "drops_per_s": D / (tot * 1e-3),
                      "gram_cmac_per_s": cmac / (t.get("gram_fused_split_fp64", float("nan")) * 1e-3)}), flush=True)


def full_size(cfgs=(1, 3, 4, 5)):
    """Every config at its own full drop count through the whole per-drop path on one GPU:
    drops -> exact Gram (fused fp64; for cfg3 also fused fp32 and materialised) -> the
    config's receivers (-> closed form + receivers where the config asks for it), all drops
    in one batch.  Whole-job device time (CUDA events) and drops/s."""
    for c in cfgs:
        w = CONFIGS[c]
        arr = xl.Array.ula(w.n_y, w.fc_hz) if w.kind == "ula" else xl.Array.upa(w.n_y, w.n_z, w.fc_hz)
        users = xl.Users.polar(w.r, w.az, w.el)
        B = w.n_drops  # one batch: every path's workspace fits (cfg3 fused fp32: 1.7 GB)
        paths = ["fp64"] + (["fp32", "mat32"] if c in (3, 5) else []) + (["closed"] if w.kind == "ula" else [])
        out = {"cfg": c, "workload": w.name, "drops": w.n_drops, "batch": B}
        for path in paths:
            pos = torch.empty((B, w.K, 3), dtype=torch.float64, device="cuda")
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for warm in (True, False):  # one untimed batch first (module load, workspace, attributes)
              torch.cuda.synchronize()
              e0.record()
              for d0 in range(0, B if warm else w.n_drops, B):
                nb = min(B, w.n_drops - d0)
                p = xl.gen_drops(users, w.K, nb, seed=w.seed, first_drop=d0, out=pos[:nb])
                if path == "closed":
                    G, fl = xl.gram_closed_form(arr, p)
                    xl.sum_rate(G, list(w.snr_db), w.receivers, flags=fl)
                else:
                    G = xl.gram_exact(arr, p, precision=xl.FP64 if path == "fp64" else xl.FP32,
                                      mode=xl.MATERIALIZED if path == "mat32" else xl.FUSED)
                    xl.sum_rate(G, list(w.snr_db), w.receivers)
              e1.record()
              torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            cmac = w.n_drops * w.N * w.K * (w.K + 1) // 2
            out[path] = {"ms": ms, "drops_per_s": w.n_drops / (ms * 1e-3),
                         "gram_cmac_per_s": None if path == "closed" else cmac / (ms * 1e-3)}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    if sys.argv[1:] == ["full"]:
        full_size()
        sys.exit(0)
    args = sys.argv[1:]
    if "1s" in args:
        steady_cfg1()
        args = [a for a in args if a != "1s"]
    if args or "1s" not in sys.argv[1:]:
        main([int(a) for a in args] or [1, 3, 4, 5])
