"""bench.py -- the driver's benchmark contract for the XL-MIMO Monte Carlo engine.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1], the config its metric is quoted on): the
capacity-vs-N saturation sweep -- ULA N = 2^8..2^16, 28 GHz, K = 8 users,
r ~ U[3, 30] m, az ~ U[-60, 60] deg, SNR 0/10/20 dB, 10^4 seeded drops, fp64,
CAP + ZF + MMSE.  One step = the whole hot path on one batch: draw the drops
(a1), fused exact Gram with nested-N snapshots (a2+a3), per-(drop, N) receivers
(a5), ergodic means + saturation statistics (a6), and the same sweep on the same drops
through the closed-form ("modified ZF") Gram (a4: Eqs. (4)/(6)/(22)/(23)), results to
host.  Each step
uses a fresh seed (new drops), and a 256 MiB buffer is written between steps to
flush L2 (126 MB).  N > 1 (torchrun): weak scaling, each rank its own 10^4
drops (first_drop = rank * 10^4) and a per-step NCCL all-reduce of the ergodic
sums/counts -- the only exchange the method has.

metric: Gram complex MACs per second, cMAC = N_max K(K+1)/2 per drop (nested
shells: the algorithmic count of the largest array).

--impl reference: the CPU oracle (oracle/, plain fp64 C) on this box's host
cores, same workload, each step a bounded sample of drops (the tier's reference
arm; a deliberately slow program -- parity and roofline are the headline).
"""
from __future__ import annotations

import argparse
import json
import math
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

W = CONFIGS[2]
# FP64-pipe work model per channel coefficient ("Roofline"): the cheapest fp64
# evaluation found (coef_fast): distance^2 2, 1/r 5, r 1, quarter-cycle reduction 3,
# sin+cos minimax 12, r^{-3/2} 6, phasor 2 (MUFU seeds and the quadrant F2I are off the
# FP64 pipe).  With this model frac ~ the FP64 pipe utilisation against the nominal peak.
FP64_OPS_PER_COEF = 31


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-seconds", type=float, default=15.0)
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

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


def ncu_traffic(kname: str, n_drops: int):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel from the
    newest committed ncu --set full capture of the same launch (profiles/r*/ncu_traffic_bench.json),
    or None.  The fused kernel is ALU-bound: this is positions in + Gram partials out."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "ncu_traffic_bench.json")))
    for f in reversed(files):
        try:
            d = json.load(open(f))
        except (OSError, ValueError):
            continue
        if d.get("kernel") == kname and d.get("n_drops") == n_drops:
            return int(d["dram_bytes_read"]) + int(d["dram_bytes_write"])
    return None


# ----------------------------------------------------------------------------- oracle timing
def oracle_sample(n_drops_sample: int, seed: int, nthreads: int = 0):
    """Time the oracle (as it stands) on a bounded sample of the workload."""
    import oracle
    oracle.build()
    u = oracle.users(r=W.r, az=W.az)
    pos = oracle.gen_drops(u, W.K, n_drops_sample, seed=seed)
    a = oracle.array("ula", n_y=W.n_y, fc_hz=W.fc_hz)
    t0 = time.perf_counter()
    oracle.saturation_sweep(a, W.n_list, pos, W.snr_db, W.receivers, t=W.t, nthreads=nthreads)
    oracle.saturation_sweep(a, W.n_list, pos, W.snr_db, W.receivers, gram_kind=1, t=W.t, nthreads=nthreads)
    return time.perf_counter() - t0


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_baseline(target_s: float):
    cores = cpu_threads()
    # calibrate on one drop per thread, then size the sample to ~target_s
    t1 = oracle_sample(cores, seed=999)
    per_round = max(t1, 1e-3)
    rounds = max(1, int(target_s / per_round))
    n = cores * rounds
    t = oracle_sample(n, seed=1000)
    value = cmac_per_drop(W) * n / t
    # the same oracle on one thread (SURVEY 8(d) oracle timing plan): t1 ~ one drop on one core
    n1 = max(1, int(target_s / 3 / per_round))
    t_1 = oracle_sample(n1, seed=2000, nthreads=1)
    return {"value": value, "unit": "cMAC/s", "cores": cores, "kind": "oracle",
            "sample": f"{n} drops of cfg2 (all 9 N, 3 SNR, CAP+ZF+MMSE, exact and closed-form sweeps; the oracle "
                      f"computes every N independently), "
                      f"{t:.1f} s wall on {cores} OpenMP threads",
            "drops_per_s": n / t,
            "single_thread": {"value": cmac_per_drop(W) * n1 / t_1, "unit": "cMAC/s", "cores": 1,
                              "sample": f"{n1} drops, {t_1:.1f} s wall on 1 thread"}}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    cores = cpu_threads()
    t_cal = oracle_sample(cores, seed=999)
    # size each step so (warmup + steps) fit in ~150 s
    budget = 150.0 / max(1, args.steps + args.warmup)
    n_step = max(cores, int(cores * max(1.0, budget / max(t_cal, 1e-3))))
    for w in range(args.warmup):
        oracle_sample(n_step, seed=10 + w)
    ts = []
    for k in range(args.steps):
        ts.append(oracle_sample(n_step, seed=100 + k))
    t = sum(ts)
    value = cmac_per_drop(W) * n_step * args.steps / t
    line = {"metric": "gram_cmac_per_s", "value": value, "unit": "cMAC/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": W.name, "n_drops_per_step": n_step, "K": W.K, "n_list": list(W.n_list),
                       "step": "drops + exact fp64 sweep + closed-form sweep on the same drops",
                       "snr_db": list(W.snr_db), "fc_hz": W.fc_hz},
            "cpu_baseline": {"value": value, "unit": "cMAC/s", "cores": cores, "kind": "oracle",
                             "sample": f"{n_step} drops per step (of the 10^4-drop workload)"},
            "e2e": {"value": value, "unit": "cMAC/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "drops_per_s": n_step * args.steps / t}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- ours
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
    sys.path.insert(0, ROOT)
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

    D = W.n_drops
    arr = xl.Array.ula(W.n_y, W.fc_hz)
    users = xl.Users.polar(W.r, W.az)
    snr = list(W.snr_db)
    R = xl.n_recv(W.receivers)
    ws_bytes = max(xl.sweep_workspace_bytes(arr, W.n_list, W.K, D, len(snr), W.receivers),
                   xl.sweep_workspace_bytes(arr, W.n_list, W.K, D, len(snr), W.receivers,
                                            gram_kind=xl.GRAM_CLOSED_FORM))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)  # the two sweeps run in turn on one stream
    pos = torch.empty((D, W.K, 3), dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def step(k):
        flush.fill_(k & 0xFF)                                      # L2 flush between steps
        xl.gen_drops(users, W.K, D, seed=1000 + k, first_drop=rank * D, out=pos)
        res = xl.saturation_sweep(arr, W.n_list, W.K, D, snr, W.receivers, pos=pos, t=W.t, ws=ws)
        res_cf = xl.saturation_sweep(arr, W.n_list, W.K, D, snr, W.receivers, pos=pos, t=W.t, ws=ws,
                                     gram_kind=xl.GRAM_CLOSED_FORM)
        if dist:
            pitch = 0.5 * 299792458.0 / W.fc_hz
            res = parallel.allreduce_sweep(res, D, dist, dev, pitch=pitch)
            res_cf = parallel.allreduce_sweep(res_cf, D, dist, dev, pitch=pitch)
        return res, res_cf

    for k in range(args.warmup):
        step(k)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    n0 = xl.launch_count()
    xl._L.xlmimo_timing_enable(1)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(args.steps):
        res, res_cf = step(args.warmup + k)
    e1.record(stream)
    torch.cuda.synchronize()
    xl._L.xlmimo_timing_enable(0)
    launches = xl.launch_count() - n0
    t_ms = e0.elapsed_time(e1)
    if dist:
        tt = torch.tensor([t_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
    ck = clocks.stop()
    ktimes = parallel.read_kernel_times(xl)

    # ---- e2e: the host-buffer C-ABI entry, H2D of positions + D2H of the result every step
    pos_host = torch.empty((D, W.K, 3), dtype=torch.float64).pin_memory()
    pos_host.copy_(xl.gen_drops(users, W.K, D, seed=77, first_drop=rank * D).cpu())
    def step_host():
        r = xl.saturation_sweep_host(arr, W.n_list, pos_host, snr, W.receivers, t=W.t, ws=ws)
        xl.saturation_sweep_host(arr, W.n_list, pos_host, snr, W.receivers, t=W.t, ws=ws,
                                 gram_kind=xl.GRAM_CLOSED_FORM)
        return r

    for _ in range(max(1, args.warmup)):
        step_host()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    f0 = torch.cuda.Event(enable_timing=True)
    f1 = torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for k in range(args.steps):
        flush.fill_(k & 0xFF)
        step_host()
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = f0.elapsed_time(f1)
    e2e_wall = (time.perf_counter() - t0) * 1e3
    e2e_ms = max(e2e_ms, e2e_wall)
    if dist:
        tt = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    h2d = 2 * D * W.K * 3 * 8  # positions, once per sweep (exact, closed form)
    n_out = len(W.n_list) * len(snr) * R
    d2h = 2 * (n_out * 8 + n_out * 8 + 4 * 8)

    # ---- roofline of the dominant kernel (fused fp64 Gram, FP64 pipe bound)
    cmac_step = cmac_per_drop(W) * D            # per rank
    N = max(W.n_list)
    gram_k = [k for k in ktimes if k.startswith("gram_fused")]
    kname = max(gram_k, key=lambda k: ktimes[k][1]) if gram_k else "gram_fused"
    kcount, kms = ktimes.get(kname, (0, 0.0))
    roof = None
    if kcount:
        per_launch_ms = kms / kcount
        tri_off = W.K * (W.K - 1) // 2
        ops = D * N * (W.K * FP64_OPS_PER_COEF + 4 * tri_off + 2 * W.K)   # FP64-pipe ops per launch
        achieved = ops / (per_launch_ms * 1e-3) / 1e12
        clk = ck.get("sm_max_mhz") or 1965.0
        peak = 148 * 64 * clk * 1e6 / 1e12
        roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "FP64 Top/s", "frac": achieved / peak,
                "traffic": ncu_traffic(kname, D), "kernel": kname, "launch_ms": per_launch_ms,
                "work_model": f"per element-user coefficient {FP64_OPS_PER_COEF} FP64 ops, 4 DFMA per off-diagonal "
                              "cMAC, 2 per diagonal; peak = 148 SM x 64 FP64 lanes/clk x sm_max clock",
                "share_of_step": kms / t_ms}
    out = None
    if rank == 0:
        value = cmac_step * world * args.steps / (t_ms * 1e-3)
        out = {"metric": "gram_cmac_per_s", "value": value, "unit": "cMAC/s", "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": "weak",
               "vs_baseline": None, "dtype": "f64", "data": "synthetic",
               "config": {"workload": W.name, "n_drops_per_rank": D, "K": W.K, "n_list": list(W.n_list),
                          "snr_db": snr, "fc_hz": W.fc_hz, "receivers": "CAP+ZF+MMSE", "precision": "fp64",
                          "cmac_per_drop": cmac_per_drop(W), "l2": "flushed between steps (256 MiB write)",
                          "step": "drops + exact fp64 sweep + closed-form sweep on the same drops",
                          "parallelism": f"dp{world} (drops)"},
               "drops_per_s": D * world * args.steps / (t_ms * 1e-3),
               "e2e": {"value": cmac_step * world * args.steps / (e2e_ms * 1e-3), "unit": "cMAC/s",
                       "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
               "gpu_launches": int(launches), "clocks": ck, "roofline": roof,
               "kernel_ms_per_step": {k: v[1] / args.steps for k, v in ktimes.items()},
               "sat_M": float(res["sat"][2]),
               "run": {"gpu": torch.cuda.get_device_name(dev), "seeds": f"1000 + step (drops of rank r from {D} r)",
                       "nan_rates_last_step": int(np.asarray(res["n_valid"]).size * D * world
                                                  - int(np.asarray(res["n_valid"]).sum())),
                       "closed_form_nan_rates_last_step": int(np.asarray(res_cf["n_valid"]).size * D * world
                                                              - int(np.asarray(res_cf["n_valid"]).sum()))}}
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        out["cpu_baseline"] = cpu_baseline(args.cpu_sample_seconds)
    if rank == 0:
        print(json.dumps(out), flush=True)
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
