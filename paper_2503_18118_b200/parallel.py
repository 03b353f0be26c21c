"""Multi-GPU plumbing for the Monte Carlo sweep (one process per GPU).

The path shards by drops: drops are independent and the counter-based draws make
any partition reproduce the same drops (rank r takes first_drop = r * D).  The
only exchange the method has is the final ergodic combination: per (N, SNR,
receiver) sums and valid counts, and the saturation statistics.  That is one
small all-reduce per step (NCCL over NVLink on GPUs; gloo in the CPU tests).

Host logic only (no method arithmetic beyond combining means): the per-drop
path runs in the library's kernels on every rank.
"""
from __future__ import annotations

import ctypes
import math

import numpy as np


def shard_range(total_drops: int, rank: int, world: int):
    """Contiguous [first_drop, first_drop + n) of `total_drops` for `rank` (strong scaling split)."""
    base, rem = divmod(total_drops, world)
    n = base + (1 if rank < rem else 0)
    first = rank * base + min(rank, rem)
    return first, n


def pack_sweep(res: dict, n_drops: int, pitch: float) -> np.ndarray:
    """Per-rank partial sums: [sum_k (mean*count) ..., counts ..., D, D*E_up, D*E_dn,
    sum of extent/pitch, sum of (extent/pitch)^2]."""
    erg = np.nan_to_num(np.asarray(res["ergodic_valid"], dtype=np.float64), nan=0.0).ravel()
    cnt = np.asarray(res["n_valid"], dtype=np.float64).ravel()
    sat = np.asarray(res["sat"], dtype=np.float64)
    D = float(n_drops)
    me = (sat[0] - sat[1]) / pitch
    var = (sat[3] * math.sqrt(D)) ** 2
    s2 = var * (D - 1.0) + D * me * me
    return np.concatenate([erg * cnt, cnt, [D, D * sat[0], D * sat[1], D * me, s2]])


def unpack_sweep(v: np.ndarray, shape, pitch: float) -> dict:
    n = int(np.prod(shape))
    sums, cnt = v[:n], v[n:2 * n]
    D, su, sd, se, s2 = v[2 * n:2 * n + 5]
    with np.errstate(invalid="ignore", divide="ignore"):
        ergv = np.where(cnt > 0, sums / np.maximum(cnt, 1), np.nan)
    erg = np.where(cnt == D, ergv, np.nan)      # R10: ergodic only when every drop of every rank is valid
    eu, ed, me = su / D, sd / D, se / D
    var = (s2 - D * me * me) / (D - 1.0) if D > 1 else 0.0
    sat = np.array([eu, ed, math.ceil((eu - ed) / pitch), math.sqrt(max(var, 0.0)) / math.sqrt(D)])
    return {"ergodic": erg.reshape(shape), "ergodic_valid": ergv.reshape(shape),
            "n_valid": cnt.reshape(shape).astype(np.int64), "sat": sat}


def allreduce_sweep(res: dict, n_drops: int, dist, device, pitch: float | None = None) -> dict:
    """Combine per-rank sweep results into the all-drop ergodic table (one all-reduce)."""
    import torch
    if pitch is None:
        pitch = res.get("pitch", 1.0)
    shape = np.asarray(res["ergodic"]).shape
    v = torch.tensor(pack_sweep(res, n_drops, pitch), dtype=torch.float64, device=device)
    dist.all_reduce(v)
    return unpack_sweep(v.cpu().numpy(), shape, pitch)


def read_kernel_times(xl, max_entries: int = 64) -> dict:
    """{kernel name: (launches, summed device ms)} from the library's event hooks."""
    names = ctypes.create_string_buffer(64 * max_entries)
    counts = (ctypes.c_int64 * max_entries)()
    ms = (ctypes.c_double * max_entries)()
    n = xl._L.xlmimo_timing_read(max_entries, names, counts, ms)
    out = {}
    for i in range(max(n, 0)):
        nm = names.raw[64 * i:64 * (i + 1)].split(b"\0", 1)[0].decode()
        out[nm] = (int(counts[i]), float(ms[i]))
    return out
