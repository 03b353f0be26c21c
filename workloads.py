"""The five synthetic workloads of BASELINE.json (``configs``), as plain data.

This module holds NO arithmetic of the method: it only names array / user-law /
drop-count / SNR parameters.  It is the one module both the product path
(bench.py, tests through the C ABI) and the oracle (tests) read, as the seeded
input recipe ("Inputs").  Positions themselves are drawn by each side
from the same counter-based generator (Philox4x64-10, key = (seed, 0),
counter = (drop, user, 0, 0)), so no position array is shared either.

Base seed 0 for every config (the configs name none; R19).
"""
from __future__ import annotations

from dataclasses import dataclass, field

RECV_CAP, RECV_ZF, RECV_MMSE, RECV_MRC = 1, 2, 4, 8


@dataclass(frozen=True)
class Workload:
    name: str
    kind: str            # "ula" | "upa"
    n_y: int             # ULA: N
    n_z: int             # UPA second axis (1 for ULA)
    fc_hz: float
    K: int
    r: tuple             # (r_min, r_max) m, uniform in r
    az: tuple            # (az_min, az_max) deg from broadside
    el: tuple            # (el_min, el_max) deg (UPA only)
    n_drops: int
    snr_db: tuple
    receivers: int
    precision: str = "fp64"
    n_list: tuple = field(default_factory=tuple)   # saturation sweep grid
    t: float = 0.9
    seed: int = 0
    spacing_wl: float = 0.5
    beta0: float = 1.0

    @property
    def N(self) -> int:
        return self.n_y * self.n_z


CONFIGS = {
    # BASELINE.json configs[0]
    1: Workload("cfg1_ula256_28GHz_K4", "ula", 256, 1, 28e9, 4, (5.0, 50.0), (-60.0, 60.0), (0.0, 0.0),
                1000, (10.0,), RECV_ZF | RECV_MMSE | RECV_CAP),
    # configs[1]: the saturation sweep (the bench workload)
    2: Workload("cfg2_sweep_ula2^8..2^16_28GHz_K8", "ula", 65536, 1, 28e9, 8, (3.0, 30.0), (-60.0, 60.0),
                (0.0, 0.0), 10000, (0.0, 10.0, 20.0), RECV_CAP | RECV_ZF | RECV_MMSE,
                n_list=tuple(2 ** k for k in range(8, 17))),
    # configs[2]
    3: Workload("cfg3_ula16384_100GHz_K16", "ula", 16384, 1, 100e9, 16, (2.0, 20.0), (-75.0, 75.0), (0.0, 0.0),
                100000, (10.0,), RECV_MMSE),
    # configs[3]
    4: Workload("cfg4_upa256x256_100GHz_K32", "upa", 256, 256, 100e9, 32, (2.0, 20.0), (-60.0, 60.0),
                (-30.0, 30.0), 10000, (10.0,), RECV_ZF | RECV_MMSE),
    # configs[4]
    5: Workload("cfg5_ula2^20_140GHz_K64", "ula", 2 ** 20, 1, 140e9, 64, (5.0, 100.0), (-60.0, 60.0),
                (0.0, 0.0), 1000, (10.0,), RECV_ZF | RECV_MMSE | RECV_CAP),
}


def cmac_per_drop(w: Workload, nested: bool = True) -> int:
    """Algorithmic complex MACs per drop: N * K(K+1)/2 (upper triangle incl. diagonal).
    For the sweep, nested = the largest N only (shells are shared)."""
    tri = w.K * (w.K + 1) // 2
    if w.n_list:
        return (max(w.n_list) if nested else sum(w.n_list)) * tri
    return w.N * tri
