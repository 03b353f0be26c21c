"""bench.py -- the driver's benchmark contract for the XL-MIMO Monte Carlo engine.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Headline workload: BASELINE.json configs[4] (cfg5), the largest single-GPU config --
ULA N = 2^20, 140 GHz, K = 64 users, r ~ U[5, 100] m, az ~ U[-60, 60] deg, SNR 10 dB,
1000 seeded drops, fp64.  One step = the whole hot path on one batch: draw the drops
(a1), the fused exact Gram H^H H with H never materialised (a2+a3, DMMA on the FP64
pipe), CAP + ZF + MMSE per drop (a5), the ergodic means and saturation statistics (a6),
and the same receivers through the closed-form ("modified ZF") Gram of Eqs. (4)/(6)/
(22)/(23) on the same drops (a4).  Each step draws fresh drops (new seed) and a 256 MiB
buffer is written before it to flush L2 (126 MB).

Sub-records (same run, same clock sampling, each its own W warm-up + K timed steps):
  cfg5_materialised  the complex64 H written to HBM (K4a) and streamed back by TMA into
                     tcgen05 (K4b): HBM roofline of the streaming kernel;
  cfg5_fused_fp32    the fused TF32 tcgen05 Gram (generator in shared memory): MUFU roofline;
  cfg1_steady        cfg1 in a 10^6-drop steady-state batch (drops, fused fp64 Gram, closed
                     form, CAP/ZF/MMSE/MRC on both);
  cfg2_sweep         the capacity-vs-N saturation sweep (10^4 drops, nine nested N, three
                     SNRs, exact + closed form) -- round 1's headline;
  cfg3, cfg4         full drop counts (10^5, 10^4), fused fp64 Gram + the config's receivers,
                     and the fused fp32 Gram.
N > 1 (torchrun): weak scaling of the headline, each rank its own 1000 drops (first_drop =
rank * 1000) and one NCCL all-reduce per step of the ergodic sums/counts -- the only
exchange the method has; the sub-records and the CPU baseline run at N = 1 only.

metric: Gram complex MACs per second, N K(K+1)/2 per drop.

--impl reference: the CPU oracle (oracle/, plain fp64 C) on this box's host cores, on
cfg5 drops, each step a bounded sample (the tier's reference arm; a deliberately slow
program -- parity and the roofline fraction are the headline).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from workloads import CONFIGS, cmac_per_drop  # noqa: E402

W = CONFIGS[5]
# FP64-pipe work model per channel coefficient: the cheapest fp64
# evaluation found (coef_fast): distance^2 2, 1/r 5, r 1, quarter-cycle reduction 3,
# sin+cos minimax 10 (degree 4 each, |err| <= 4.7e-11: xl_common.cuh), r^{-3/2} 6, phasor 2
# (MUFU seeds and the quadrant F2I are off the FP64 pipe); then 4 FP64-pipe ops per off-diagonal complex MAC (DFMA, or a quarter of
# the four real m8n8k4 DMMAs per 2x2 plane block), 2 per diagonal one.
FP64_OPS_PER_COEF = 29
MUFU_PER_COEF_FP32 = 2   # the fused fp32 generator: MUFU sin + cos per coefficient
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
HBM_FALLBACK_GBS = 6545.3   # B200_PROFILING.md / MEASURED_PEAKS.json copy bandwidth
READ_PEAK_GBS = 7140.0      # read-only stream, tools/peaks.cu (profiles/r01/microbench_peaks.json)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sub", action="store_true", help="headline only (no per-config sub-records)")
    ap.add_argument("--cpu-sample-seconds", type=float, default=15.0)
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def hbm_peak():
    try:
        d = json.load(open(PEAKS_FILE))
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy, read+write bytes)"
    except (OSError, ValueError, KeyError):
        return HBM_FALLBACK_GBS, "B200_PROFILING.md fallback"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling DURING the timed regions (B200_PROFILING.md clocks line)."""

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self._stop = threading.Event()
        self._proc = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self._proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                           "-i", str(self.idx), "-lms", "100"], stdout=subprocess.PIPE,
                                          stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self._proc = None
            return
        self._t = threading.Thread(target=self._read, daemon=True)
        self._t.start()

    def _read(self):
        for line in self._proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])
            if self._stop.is_set():
                break

    def stop(self):
        self._stop.set()
        if self._proc:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except Exception:
                self._proc.kill()
        sm = []
        mx = None
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for n, v in zip(names, r[4:8]):
                    if v.strip().lower() == "active":
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def ncu_traffic(kname: str, launch: str, drops: float | None = None):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of a kernel from the newest
    committed `ncu --set full` capture of the same launch (profiles/r*/ncu_traffic_*.json),
    or None.  With `drops`, the captured launch's bytes are scaled to that many drops (the
    materialised stream's launches hold 16 drops but the last of a batch fewer)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "ncu_traffic_*.json")))
    for f in reversed(files):
        try:
            d = json.load(open(f))
        except (OSError, ValueError):
            continue
        for e in (d if isinstance(d, list) else [d]):
            if e.get("kernel") == kname and e.get("launch_key") == launch:
                b = int(e["dram_bytes_read"]) + int(e["dram_bytes_write"])
                return int(b * drops / e["drops"]) if drops and e.get("drops") else b
    return None


# ----------------------------------------------------------------------------- oracle timing
ORACLE_SUB_N = 2 ** 16   # the oracle's cost is linear in N: it runs cfg5 drops on the centred 2^16-element sub-array


def oracle_sample(n_drops_sample: int, seed: int, nthreads: int = 0):
    """Time the oracle (as it stands) on a bounded sample of the headline workload: cfg5 drops
    (K = 64, 140 GHz, same user law), the exact Gram, CAP/ZF/MMSE, ergodic reduction and the
    closed-form path, on the centred ORACLE_SUB_N-element sub-array.  Returns (seconds, cMACs)."""
    import oracle
    oracle.build()
    u = oracle.users(r=W.r, az=W.az)
    pos = oracle.gen_drops(u, W.K, n_drops_sample, seed=seed)
    a = oracle.array("ula", n_y=ORACLE_SUB_N, fc_hz=W.fc_hz)
    t0 = time.perf_counter()
    oracle.saturation_sweep(a, [ORACLE_SUB_N], pos, W.snr_db, W.receivers, t=W.t, nthreads=nthreads)
    oracle.saturation_sweep(a, [ORACLE_SUB_N], pos, W.snr_db, W.receivers, gram_kind=1, t=W.t, nthreads=nthreads)
    return time.perf_counter() - t0, ORACLE_SUB_N * W.K * (W.K + 1) // 2 * n_drops_sample


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


SAMPLE_TEXT = (f"cfg5 drops (K = 64, 140 GHz, r ~ U[5,100] m) on the centred {ORACLE_SUB_N}-element sub-array "
               f"of the 2^20 ULA (the oracle's cost is linear in N): exact fp64 Gram + CAP/ZF/MMSE + ergodic "
               f"reduction + closed-form Gram and receivers")


def cpu_baseline(target_s: float):
    cores = cpu_threads()
    t1, _ = oracle_sample(cores, seed=999)               # one drop per thread: calibration
    rounds = max(1, int(target_s / max(t1, 1e-3)))
    n = cores * rounds
    t, cm = oracle_sample(n, seed=1000)
    n1 = max(1, int(target_s / 3 / max(t1, 1e-3)))
    t_1, cm1 = oracle_sample(n1, seed=2000, nthreads=1)
    return {"value": cm / t, "unit": "cMAC/s", "cores": cores, "kind": "oracle",
            "sample": f"{n} {SAMPLE_TEXT}; {t:.1f} s wall on {cores} OpenMP threads (over drops)",
            "single_thread": {"value": cm1 / t_1, "unit": "cMAC/s", "cores": 1,
                              "sample": f"{n1} drops, {t_1:.1f} s wall on 1 thread"}}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    cores = cpu_threads()
    t_cal, _ = oracle_sample(cores, seed=999)
    budget = 150.0 / max(1, args.steps + args.warmup)    # (warmup + steps) in ~150 s
    n_step = max(cores, cores * int(max(1.0, budget / max(t_cal, 1e-3))))
    for w in range(args.warmup):
        oracle_sample(n_step, seed=10 + w)
    ts, cm = [], 0
    for k in range(args.steps):
        t, c = oracle_sample(n_step, seed=100 + k)
        ts.append(t)
        cm += c
    t = sum(ts)
    value = cm / t
    line = {"metric": "gram_cmac_per_s", "value": value, "unit": "cMAC/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": W.name, "n_drops_per_step": n_step, "K": W.K, "N": ORACLE_SUB_N,
                       "step": "drops + exact fp64 Gram + CAP/ZF/MMSE + ergodic + closed-form path",
                       "snr_db": list(W.snr_db), "fc_hz": W.fc_hz},
            "cpu_baseline": {"value": value, "unit": "cMAC/s", "cores": cores, "kind": "oracle",
                             "sample": f"{n_step} {SAMPLE_TEXT} per step"},
            "e2e": {"value": value, "unit": "cMAC/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "drops_per_s": n_step * args.steps / t}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- ours
def fp64_ops(D, N, K):
    """FP64-pipe operations of the fused exact Gram (work model above)."""
    return D * N * (K * FP64_OPS_PER_COEF + 4 * (K * (K - 1) // 2) + 2 * K)


def run_ours(args):
    import numpy as np
    import torch

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    import importlib.util
    spec = importlib.util.spec_from_file_location("_xl_build", os.path.join(ROOT, "paper_2503_18118_b200", "build.py"))
    bmod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bmod)
    if rank == 0:
        bmod.build()
    if dist:
        dist.barrier()
    import paper_2503_18118_b200 as xl
    from paper_2503_18118_b200 import parallel

    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    hbm_gbs, hbm_src = hbm_peak()

    def timed(step, steps, warmup):
        """W untimed + K timed steps (L2 flushed before each), CUDA events on the launching
        stream; per-kernel device times from the library's event hooks."""
        for k in range(warmup):
            flush.fill_(k & 0xFF)
            step(k)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        n0 = xl.launch_count()
        xl._L.xlmimo_timing_enable(1)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        out = None
        ms_flush = 0.0
        e0.record(stream)
        for k in range(steps):
            flush.fill_((warmup + k) & 0xFF)
            out = step(warmup + k)
        e1.record(stream)
        torch.cuda.synchronize()
        xl._L.xlmimo_timing_enable(0)
        kt = parallel.read_kernel_times(xl)
        t_ms = e0.elapsed_time(e1)
        # the flush writes are not part of the step: time them alone and subtract
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for k in range(steps):
            flush.fill_(k & 0xFF)
        f1.record(stream)
        torch.cuda.synchronize()
        ms_flush = f0.elapsed_time(f1)
        return max(t_ms - ms_flush, 1e-6), kt, xl.launch_count() - n0, out

    def fp64_roof(kt, names, D, N, K, clk):
        ks = [k for k in kt if k in names]
        if not ks:
            return None
        kname = max(ks, key=lambda k: kt[k][1])
        cnt, ms = kt[kname]
        per_launch = ms / cnt
        ach = fp64_ops(D, N, K) / (per_launch * 1e-3) / 1e12
        peak = 148 * 64 * clk * 1e6 / 1e12
        return {"bound": "alu", "achieved": ach, "peak": peak, "unit": "FP64 Top/s", "frac": ach / peak,
                "kernel": kname, "launch_ms": per_launch, "launches": cnt,
                "work_model": f"{FP64_OPS_PER_COEF} FP64-pipe ops per element-user coefficient + 4 per off-diagonal "
                              f"cMAC + 2 per diagonal, x {D} drops x N = {N} per launch; peak = 148 SM x 64 FP64 "
                              f"lanes/clk x sm_max clock (B200_PROFILING.md unit counts)"}

    # ------------------------------------------------------------------ headline: cfg5 fp64 step
    D = W.n_drops
    N = W.N
    arr = xl.Array.ula(N, W.fc_hz)
    users = xl.Users.polar(W.r, W.az)
    snr = list(W.snr_db)
    nl = [N]
    ws_bytes = max(xl.sweep_workspace_bytes(arr, nl, W.K, D, len(snr), W.receivers),
                   xl.sweep_workspace_bytes(arr, nl, W.K, D, len(snr), W.receivers,
                                            gram_kind=xl.GRAM_CLOSED_FORM))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    pos = torch.empty((D, W.K, 3), dtype=torch.float64, device=dev)

    def step(k):
        xl.gen_drops(users, W.K, D, seed=1000 + k, first_drop=rank * D, out=pos)
        res = xl.saturation_sweep(arr, nl, W.K, D, snr, W.receivers, pos=pos, t=W.t, ws=ws)
        res_cf = xl.saturation_sweep(arr, nl, W.K, D, snr, W.receivers, pos=pos, t=W.t, ws=ws,
                                     gram_kind=xl.GRAM_CLOSED_FORM)
        if dist:
            pitch = 0.5 * 299792458.0 / W.fc_hz
            res = parallel.allreduce_sweep(res, D, dist, dev, pitch=pitch)
            res_cf = parallel.allreduce_sweep(res_cf, D, dist, dev, pitch=pitch)
        return res, res_cf

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    t_ms, ktimes, launches, (res, res_cf) = timed(step, args.steps, args.warmup)
    if dist:
        tt = torch.tensor([t_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
    clk_guess = 1965.0

    # ------------------------------------------------------------------ e2e: host-buffer C-ABI entry
    pos_host = torch.empty((D, W.K, 3), dtype=torch.float64).pin_memory()
    pos_host.copy_(xl.gen_drops(users, W.K, D, seed=77, first_drop=rank * D).cpu())

    def step_host(k):
        r = xl.saturation_sweep_host(arr, nl, pos_host, snr, W.receivers, t=W.t, ws=ws)
        xl.saturation_sweep_host(arr, nl, pos_host, snr, W.receivers, t=W.t, ws=ws, gram_kind=xl.GRAM_CLOSED_FORM)
        return r

    t0 = time.perf_counter()
    e2e_ms, _, _, _ = timed(step_host, args.steps, min(args.warmup, 1))
    e2e_wall = (time.perf_counter() - t0) * 1e3 * args.steps / (args.steps + min(args.warmup, 1))
    e2e_ms = max(e2e_ms, 0.0)
    if dist:
        tt = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    R = xl.n_recv(W.receivers)
    h2d = 2 * D * W.K * 3 * 8            # positions, once per sweep (exact, closed form)
    n_out = len(nl) * len(snr) * R
    d2h = 2 * (n_out * 8 * 2 + n_out * 8 + 4 * 8)   # ergodic, ergodic_valid, n_valid, sat per sweep

    # ------------------------------------------------------------------ sub-records (N = 1)
    sub = {}
    if world == 1 and not args.no_sub:
        sub = run_subrecords(xl, torch, np, dev, timed, fp64_roof, args, hbm_gbs, hbm_src, clk_guess)
    ck = clocks.stop()
    clk = ck.get("sm_max_mhz") or clk_guess

    # ------------------------------------------------------------------ headline roofline
    roof = fp64_roof(ktimes, ("gram_fused_dmma_tiled_fp64", "gram_fused_dmma_fp64", "gram_fused_split_fp64"),
                     D, N, W.K, clk)
    if roof:
        roof["share_of_step"] = ktimes[roof["kernel"]][1] / t_ms
        roof["traffic"] = ncu_traffic(roof["kernel"], f"cfg5 fp64 D={D}")
    cmac_step = cmac_per_drop(W) * D
    out = None
    if rank == 0:
        value = cmac_step * world * args.steps / (t_ms * 1e-3)
        out = {"metric": "gram_cmac_per_s", "value": value, "unit": "cMAC/s", "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": "weak",
               "vs_baseline": None, "dtype": "f64", "data": "synthetic",
               "config": {"workload": W.name, "n_drops_per_rank": D, "N": N, "K": W.K, "snr_db": snr,
                          "fc_hz": W.fc_hz, "r_m": list(W.r), "az_deg": list(W.az), "receivers": "CAP+ZF+MMSE",
                          "precision": "fp64", "gram": "fused (H never materialised), DMMA on the FP64 pipe",
                          "cmac_per_drop": cmac_per_drop(W),
                          "l2": "flushed before every timed step (256 MiB write, its time subtracted)",
                          "step": "drops + exact fp64 Gram + CAP/ZF/MMSE + ergodic/saturation reduce + closed-form "
                                  "Gram and receivers on the same drops",
                          "parallelism": f"dp{world} (drops)"},
               "drops_per_s": D * world * args.steps / (t_ms * 1e-3),
               "e2e": {"value": cmac_step * world * args.steps / (e2e_ms * 1e-3), "unit": "cMAC/s",
                       "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                       "entry": "xlmimo_saturation_sweep_host (exact + closed form), host positions in, host "
                                "results out", "wall_ms_per_step": e2e_wall / args.steps},
               "gpu_launches": int(launches), "clocks": ck, "roofline": roof,
               "kernel_ms_per_step": {k: v[1] / args.steps for k, v in ktimes.items()},
               "results_last_step": {"ergodic_bits": np.asarray(res["ergodic"]).ravel().tolist(),
                                     "n_valid": np.asarray(res["n_valid"]).ravel().tolist(),
                                     "closed_form_ergodic_bits": np.asarray(res_cf["ergodic"]).ravel().tolist(),
                                     "closed_form_n_valid": np.asarray(res_cf["n_valid"]).ravel().tolist(),
                                     "M_sat": float(res["sat"][2])},
               "sub": sub,
               "run": {"gpu": torch.cuda.get_device_name(dev),
                       "seeds": f"1000 + step (drops of rank r from {D} r)", "hbm_peak_source": hbm_src}}
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        out["cpu_baseline"] = cpu_baseline(args.cpu_sample_seconds)
    if rank == 0:
        print(json.dumps(out), flush=True)
    return 0


def run_subrecords(xl, torch, np, dev, timed, fp64_roof, args, hbm_gbs, hbm_src, clk):
    sub = {}
    K_, W_ = args.steps, args.warmup

    def rec(w, D, ms, kt, launches, extra):
        cm = cmac_per_drop(w) * D
        r = {"workload": w.name, "drops_per_step": D, "ms_per_step": ms / K_, "cmac_per_s": cm * K_ / (ms * 1e-3),
             "drops_per_s": D * K_ / (ms * 1e-3), "gpu_launches": int(launches),
             "kernel_ms_per_step": {k: v[1] / K_ for k, v in kt.items()}}
        r.update(extra)
        return r

    # ---- cfg5 materialised: K4a write + K4b TMA -> tcgen05 stream, then the receivers
    w = CONFIGS[5]
    D = w.n_drops
    arr = xl.Array.ula(w.N, w.fc_hz)
    users = xl.Users.polar(w.r, w.az)
    pos = torch.empty((D, w.K, 3), dtype=torch.float64, device=dev)
    ws = torch.empty(xl.gram_workspace_bytes(arr, w.K, D, xl.FP32, xl.MATERIALIZED),
                     dtype=torch.uint8, device=dev)
    G = torch.empty((D, w.K, w.K, 2), dtype=torch.float64, device=dev)

    def s_mat(k):
        xl.gen_drops(users, w.K, D, seed=3000 + k, out=pos)
        g = xl.gram_exact(arr, pos, precision=xl.FP32, mode=xl.MATERIALIZED, out=G, ws=ws)
        return xl.sum_rate(g, list(w.snr_db), w.receivers)
    ms, kt, nl_, _ = timed(s_mat, K_, W_)
    st = kt.get("gram_stream_tc_tf32")
    wr = kt.get("h_materialise")
    extra = {"precision": "fp32 (complex64 H, TF32 tensor cores, fp64 across chunks)"}
    if st:
        per_launch = st[1] / st[0]
        drops_per_launch = D * K_ / st[0]
        bytes_launch = 8 * w.N * w.K * drops_per_launch
        ach = bytes_launch / (per_launch * 1e-3) / 1e9
        extra["roofline"] = {"bound": "hbm", "achieved": ach, "peak": hbm_gbs, "unit": "GB/s", "frac": ach / hbm_gbs,
                             "traffic": ncu_traffic("gram_stream_tc_tf32", "cfg5 mat32", drops_per_launch),
                             "frac_of_read_peak": ach / READ_PEAK_GBS,
                             "read_peak_source": "profiles/r01/microbench_peaks.json (read-only stream, 7.14 TB/s; "
                                                 "the copy figure above counts read + write)",
                             "kernel": "gram_stream_tc_tf32", "launch_ms": per_launch, "launches": st[0],
                             "algorithmic_bytes_per_launch": bytes_launch,
                             "work_model": "8 N K bytes per drop (complex64 H read once) x drops per launch",
                             "peak_source": hbm_src, "share_of_step": st[1] / ms}
    if wr:
        per_launch = wr[1] / wr[0]
        bytes_launch = 8 * w.N * w.K * D * K_ / wr[0]
        extra["writer"] = {"kernel": "h_materialise (K4a)", "launch_ms": per_launch,
                           "gbs": bytes_launch / (per_launch * 1e-3) / 1e9,
                           "frac_of_hbm_peak": bytes_launch / (per_launch * 1e-3) / 1e9 / hbm_gbs,
                           "traffic": ncu_traffic("h_materialise", "cfg5 mat32 writer", D * K_ / wr[0])}
    sub["cfg5_materialised"] = rec(w, D, ms, kt, nl_, extra)
    del ws

    # ---- cfg5 fused fp32 (TF32 tcgen05, generator writes the operand tiles in shared memory)
    ws = torch.empty(xl.gram_workspace_bytes(arr, w.K, D, xl.FP32, xl.FUSED),
                     dtype=torch.uint8, device=dev)

    def s_f32(k):
        xl.gen_drops(users, w.K, D, seed=4000 + k, out=pos)
        g = xl.gram_exact(arr, pos, precision=xl.FP32, out=G, ws=ws)
        return xl.sum_rate(g, list(w.snr_db), w.receivers)
    ms, kt, nl_, _ = timed(s_f32, K_, W_)
    extra = {"precision": "fp32 tier (fp32 phasors from fp64 anchors, fp16 operands = 11 significant bits like TF32, tcgen05 kind::f16, fp32 accumulation, fp64 across chunks)"}
    tc = kt.get("gram_fused_tc_f16")
    if tc:
        per_launch = tc[1] / tc[0]
        coefs = w.N * w.K * D * K_ / tc[0]
        ach = MUFU_PER_COEF_FP32 * coefs / (per_launch * 1e-3) / 1e12
        peak = 148 * 16 * clk * 1e6 / 1e12
        extra["roofline"] = {"bound": "alu", "achieved": ach, "peak": peak, "unit": "MUFU Top/s", "frac": ach / peak,
                             "kernel": "gram_fused_tc_f16", "launch_ms": per_launch, "launches": tc[0],
                             "coefficients_per_clk_per_sm": coefs / (per_launch * 1e-3) / (clk * 1e6) / 148,
                             "traffic": ncu_traffic("gram_fused_tc_f16", f"cfg5 fp32 D={int(D * K_ / tc[0])}"),
                             "work_model": "2 MUFU (sin, cos) per element-user coefficient; peak = 148 SM x 16 MUFU "
                                           "lanes/clk x sm_max clock", "share_of_step": tc[1] / ms}
    sub["cfg5_fused_fp32"] = rec(w, D, ms, kt, nl_, extra)
    del ws, G, pos

    # ---- cfg1 steady state: 10^6 drops through the whole per-drop path (exact and closed form)
    w = CONFIGS[1]
    D = 10 ** 6
    arr = xl.Array.ula(w.N, w.fc_hz)
    users = xl.Users.polar(w.r, w.az)
    pos = torch.empty((D, w.K, 3), dtype=torch.float64, device=dev)
    allr = xl.RECV_CAP | xl.RECV_ZF | xl.RECV_MMSE | xl.RECV_MRC
    G = torch.empty((D, w.K, w.K, 2), dtype=torch.float64, device=dev)
    ws = torch.empty(max(1, xl.gram_workspace_bytes(arr, w.K, D, xl.FP64, xl.FUSED)),
                     dtype=torch.uint8, device=dev)

    def s_c1(k):
        xl.gen_drops(users, w.K, D, seed=5000 + k, out=pos)
        g = xl.gram_exact(arr, pos, out=G, ws=ws)
        gt, fl = xl.gram_closed_form(arr, pos)
        xl.sum_rate(g, list(w.snr_db), allr)
        return xl.sum_rate(gt, list(w.snr_db), allr, flags=fl)
    ms, kt, nl_, _ = timed(s_c1, K_, W_)
    roof = fp64_roof(kt, ("gram_fused_split_fp64", "gram_fused_dmma_fp64", "gram_fused_small_fp64",
                          "gram_fused_warp_fp64"), D, w.N, w.K, clk)
    if roof:
        roof["traffic"] = ncu_traffic(roof["kernel"], f"cfg1 steady D={D}")
    sub["cfg1_steady"] = rec(w, D, ms, kt, nl_, {
        "step": "10^6 drops: drops + fused fp64 Gram + closed-form Gram + CAP/ZF/MMSE/MRC on both", "roofline": roof})
    del pos, G, ws

    # ---- cfg2: the saturation sweep (round 1's headline)
    w = CONFIGS[2]
    D = w.n_drops
    arr = xl.Array.ula(w.n_y, w.fc_hz)
    users = xl.Users.polar(w.r, w.az)
    snr = list(w.snr_db)
    ws = torch.empty(max(xl.sweep_workspace_bytes(arr, w.n_list, w.K, D, len(snr), w.receivers),
                         xl.sweep_workspace_bytes(arr, w.n_list, w.K, D, len(snr), w.receivers,
                                                  gram_kind=xl.GRAM_CLOSED_FORM)), dtype=torch.uint8, device=dev)
    pos = torch.empty((D, w.K, 3), dtype=torch.float64, device=dev)

    def s_c2(k):
        xl.gen_drops(users, w.K, D, seed=6000 + k, out=pos)
        r = xl.saturation_sweep(arr, w.n_list, w.K, D, snr, w.receivers, pos=pos, t=w.t, ws=ws)
        xl.saturation_sweep(arr, w.n_list, w.K, D, snr, w.receivers, pos=pos, t=w.t, ws=ws,
                            gram_kind=xl.GRAM_CLOSED_FORM)
        return r
    ms, kt, nl_, r = timed(s_c2, K_, W_)
    roof = fp64_roof(kt, ("gram_fused_split_fp64",), D, max(w.n_list), w.K, clk)
    if roof:
        roof["traffic"] = ncu_traffic(roof["kernel"], f"cfg2 sweep D={D}")
    sub["cfg2_sweep"] = rec(w, D, ms, kt, nl_, {
        "step": "drops + exact fp64 sweep (9 nested N, 3 SNR, CAP/ZF/MMSE) + closed-form sweep", "roofline": roof,
        "M_sat": float(r["sat"][2])})
    del ws, pos

    # ---- cfg3, cfg4: full drop counts, fused fp64 Gram + the config's receivers; fused fp32 Gram
    for c in (3, 4):
        w = CONFIGS[c]
        D = w.n_drops
        arr = xl.Array.ula(w.n_y, w.fc_hz) if w.kind == "ula" else xl.Array.upa(w.n_y, w.n_z, w.fc_hz)
        users = xl.Users.polar(w.r, w.az, w.el)
        pos = torch.empty((D, w.K, 3), dtype=torch.float64, device=dev)
        G = torch.empty((D, w.K, w.K, 2), dtype=torch.float64, device=dev)
        for prec, tag in ((xl.FP64, "fp64"), (xl.FP32, "fp32")):
            ws = torch.empty(max(1, xl.gram_workspace_bytes(arr, w.K, D, prec,
                                                                         xl.FUSED)), dtype=torch.uint8, device=dev)

            def s_c(k):
                xl.gen_drops(users, w.K, D, seed=7000 + k, out=pos)
                g = xl.gram_exact(arr, pos, precision=prec, out=G, ws=ws)
                return xl.sum_rate(g, list(w.snr_db), w.receivers)
            ms, kt, nl_, _ = timed(s_c, K_, W_)
            extra = {"precision": tag, "step": "drops + fused exact Gram + " +
                     "+".join(n for n, b in (("CAP", 1), ("ZF", 2), ("MMSE", 4)) if w.receivers & b)}
            if prec == xl.FP64:
                extra["roofline"] = fp64_roof(kt, ("gram_fused_dmma_fp64", "gram_fused_dmma_tiled_fp64"), D, w.N,
                                              w.K, clk)
            else:
                tc = kt.get("gram_fused_tc_f16")
                if tc:
                    per_launch = tc[1] / tc[0]
                    coefs = w.N * w.K * D * K_ / tc[0]
                    ach = MUFU_PER_COEF_FP32 * coefs / (per_launch * 1e-3) / 1e12
                    peak = 148 * 16 * clk * 1e6 / 1e12
                    extra["roofline"] = {"bound": "alu", "achieved": ach, "peak": peak, "unit": "MUFU Top/s",
                                         "frac": ach / peak, "kernel": "gram_fused_tc_f16", "launch_ms": per_launch,
                                         "coefficients_per_clk_per_sm": coefs / (per_launch * 1e-3) / (clk * 1e6) / 148}
            sub[f"cfg{c}_{tag}"] = rec(w, D, ms, kt, nl_, extra)
            del ws
        del pos, G
    torch.cuda.empty_cache()
    return sub


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
