"""CPU oracle for the near-field XL-MIMO Monte Carlo hot path (arXiv 2503.18118).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product (``paper_2503_18118_b200``) never imports it, and it
never imports the product: the two share no code ("Oracle").

* ``xlmimo_oracle.c`` (-> ``liboracle.so``): plain fp64 loops for the per-drop
  path -- Philox draws, Eq. (3) channel, exact Gram, Eqs. (4)/(6)/(22)/(23)
  closed-form Gram, Cholesky receivers, Eqs. (13)-(16) saturation coordinates,
  the capacity-vs-N sweep.
* this module: ctypes marshalling for the above, plus the analytic ergodic
  saturation point of PAPER.md Appendix B, evaluated by
  quadrature for the rectangle law of the paper and for the polar user law of
  the configs (reading R15).

Parity status: every function here is pinned in ``tests/test_oracle_pins.py``
(nothing is "parity unpinned"; the weakest pin, the UPA off-diagonal, is pinned
by mpmath brute force on tiny arrays and the solid-angle diagonal only).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "xlmimo_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
C_LIGHT = 299792458.0  # exact

RECV_CAP, RECV_ZF, RECV_MMSE, RECV_MRC = 1, 2, 4, 8


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C99 + OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-fopenmp",
                               "-ffp-contract=off", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class OrArray(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("n_y", ctypes.c_int64), ("n_z", ctypes.c_int64),
                ("fc_hz", ctypes.c_double), ("spacing_wl", ctypes.c_double), ("beta0", ctypes.c_double)]


class OrUsers(ctypes.Structure):
    _fields_ = [("r_min_m", ctypes.c_double), ("r_max_m", ctypes.c_double),
                ("az_min_deg", ctypes.c_double), ("az_max_deg", ctypes.c_double),
                ("el_min_deg", ctypes.c_double), ("el_max_deg", ctypes.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        P = ctypes.POINTER
        d, i32, i64, u32, u64 = ctypes.c_double, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64
        vp = ctypes.c_void_p
        L.or_philox4x64_10.argtypes = [vp, vp, vp]
        L.or_gen_drops.argtypes = [P(OrUsers), i32, i64, u64, u64, vp]
        L.or_wavelength.argtypes = [P(OrArray)]
        L.or_wavelength.restype = d
        L.or_element_pos.argtypes = [P(OrArray), i64, P(d), P(d)]
        L.or_channel_coef.argtypes = [P(OrArray), vp, i64, P(d), P(d)]
        L.or_channel_matrix.argtypes = [P(OrArray), vp, i32, vp]
        L.or_gram_exact.argtypes = [P(OrArray), vp, i32, i64, vp, i32]
        L.or_gram_closed_form.argtypes = [P(OrArray), vp, i32, i64, vp, vp]
        L.or_power_eq4.argtypes = [d, d, d, d, d]
        L.or_power_eq4.restype = d
        L.or_power_limit_eq5.argtypes = [d, d, d]
        L.or_power_limit_eq5.restype = d
        L.or_corr_eq6.argtypes = [d, d, d, d, d, d, P(d), P(d)]
        L.or_corr_limit_eq8.argtypes = [d, d, d, d, d, P(d), P(d)]
        L.or_sum_rate.argtypes = [vp, i32, i64, vp, i32, u32, vp, vp]
        L.or_saturation_coords.argtypes = [vp, i32, i64, d, vp, vp]
        L.or_sum_rate_mismatched.argtypes = [vp, vp, i32, i64, vp, i32, vp, vp]
        L.or_bounds_app_a.argtypes = [vp, i32, i64, vp, i32, vp, vp, vp, vp, i32]
        L.or_gen_drops_rect.argtypes = [d, d, d, d, i32, i64, u64, u64, vp]
        L.or_saturation_sweep.argtypes = [P(OrArray), vp, i32, vp, i32, i64, vp, i32, u32, i32, d,
                                          vp, vp, vp, vp, vp, i32]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def array(kind="ula", n_y=256, n_z=1, fc_hz=28e9, spacing_wl=0.5, beta0=1.0) -> OrArray:
    return OrArray(0 if kind == "ula" else 1, int(n_y), int(n_z), float(fc_hz), float(spacing_wl), float(beta0))


def users(r=(5.0, 50.0), az=(-60.0, 60.0), el=(0.0, 0.0)) -> OrUsers:
    return OrUsers(float(r[0]), float(r[1]), float(az[0]), float(az[1]), float(el[0]), float(el[1]))


def wavelength(arr: OrArray) -> float:
    return lib().or_wavelength(ctypes.byref(arr))


def n_recv(receivers: int) -> int:
    return bin(receivers & 15).count("1")


# --------------------------------------------------------------------------- per-drop path
def philox4x64_10(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint64)
    k = np.ascontiguousarray(key, dtype=np.uint64)
    out = np.zeros(4, dtype=np.uint64)
    lib().or_philox4x64_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def gen_drops(u: OrUsers, K: int, n_drops: int, seed: int = 0, first_drop: int = 0) -> np.ndarray:
    pos = np.zeros((n_drops, K, 3), dtype=np.float64)
    lib().or_gen_drops(ctypes.byref(u), K, n_drops, seed, first_drop, _ptr(pos))
    return pos


def element_pos(arr: OrArray, m: int):
    y, z = ctypes.c_double(), ctypes.c_double()
    lib().or_element_pos(ctypes.byref(arr), m, ctypes.byref(y), ctypes.byref(z))
    return y.value, z.value


def channel_coef(arr: OrArray, p, m: int) -> complex:
    p = np.ascontiguousarray(p, dtype=np.float64)
    re, im = ctypes.c_double(), ctypes.c_double()
    lib().or_channel_coef(ctypes.byref(arr), _ptr(p), m, ctypes.byref(re), ctypes.byref(im))
    return complex(re.value, im.value)


def channel_matrix(arr: OrArray, pos_drop) -> np.ndarray:
    """H as an (M, K) complex matrix, column i = h_i (Eq. 2)."""
    pos_drop = np.ascontiguousarray(pos_drop, dtype=np.float64)
    K = pos_drop.shape[0]
    M = arr.n_y * (arr.n_z if arr.kind == 1 else 1)
    H = np.zeros((K, M, 2), dtype=np.float64)
    lib().or_channel_matrix(ctypes.byref(arr), _ptr(pos_drop), K, _ptr(H))
    return (H[..., 0] + 1j * H[..., 1]).T.copy()


def gram_exact(arr: OrArray, pos: np.ndarray, nthreads: int = 0) -> np.ndarray:
    pos = np.ascontiguousarray(pos, dtype=np.float64)
    D, K, _ = pos.shape
    g = np.zeros((D, K, K, 2), dtype=np.float64)
    lib().or_gram_exact(ctypes.byref(arr), _ptr(pos), K, D, _ptr(g), nthreads)
    return g[..., 0] + 1j * g[..., 1]


def gram_closed_form(arr: OrArray, pos: np.ndarray):
    pos = np.ascontiguousarray(pos, dtype=np.float64)
    D, K, _ = pos.shape
    g = np.zeros((D, K, K, 2), dtype=np.float64)
    fl = np.zeros(D, dtype=np.uint32)
    lib().or_gram_closed_form(ctypes.byref(arr), _ptr(pos), K, D, _ptr(g), _ptr(fl))
    return g[..., 0] + 1j * g[..., 1], fl


def power_eq4(M, lam, beta0, x, y) -> float:
    return lib().or_power_eq4(float(M), lam, beta0, x, y)


def power_limit_eq5(lam, beta0, x) -> float:
    return lib().or_power_limit_eq5(lam, beta0, x)


def corr_eq6(M, lam, xi, yi, xj, yj) -> complex:
    re, im = ctypes.c_double(), ctypes.c_double()
    lib().or_corr_eq6(float(M), lam, xi, yi, xj, yj, ctypes.byref(re), ctypes.byref(im))
    return complex(re.value, im.value)


def corr_limit_eq8(lam, xi, yi, xj, yj) -> complex:
    re, im = ctypes.c_double(), ctypes.c_double()
    lib().or_corr_limit_eq8(lam, xi, yi, xj, yj, ctypes.byref(re), ctypes.byref(im))
    return complex(re.value, im.value)


def sum_rate(gram: np.ndarray, snr_db, receivers: int, flags_in=None):
    """gram: (D, K, K) complex.  Returns rates (D, S, R) and flags (D,)."""
    g = np.ascontiguousarray(np.stack([gram.real, gram.imag], axis=-1), dtype=np.float64)
    D, K = g.shape[0], g.shape[1]
    snr = np.ascontiguousarray(np.atleast_1d(snr_db), dtype=np.float64)
    R = n_recv(receivers)
    rates = np.zeros((D, snr.size, R), dtype=np.float64)
    fl = np.zeros(D, dtype=np.uint32) if flags_in is None else np.array(flags_in, dtype=np.uint32)
    lib().or_sum_rate(_ptr(g), K, D, _ptr(snr), snr.size, receivers, _ptr(rates), _ptr(fl))
    return rates, fl


def sum_rate_mismatched(gram: np.ndarray, gram_model: np.ndarray, snr_db):
    """Effective rate of the modified-ZF equalizer G~^{-1} H^H on the true channel (NEXT-1).
    Returns rates (D, S) and flags (D,) (bit 5: G~ singular)."""
    g = np.ascontiguousarray(np.stack([gram.real, gram.imag], axis=-1), dtype=np.float64)
    gm = np.ascontiguousarray(np.stack([gram_model.real, gram_model.imag], axis=-1), dtype=np.float64)
    D, K = g.shape[0], g.shape[1]
    snr = np.ascontiguousarray(np.atleast_1d(snr_db), dtype=np.float64)
    rates = np.zeros((D, snr.size))
    fl = np.zeros(D, dtype=np.uint32)
    lib().or_sum_rate_mismatched(_ptr(g), _ptr(gm), K, D, _ptr(snr), snr.size, _ptr(rates), _ptr(fl))
    return rates, fl


def gram_exact_blas(arr: OrArray, pos: np.ndarray) -> np.ndarray:
    """Exact Gram for large K (Appendix A at K up to 1000): H from the oracle's own
    Eq. (3) coefficients (channel_matrix), then G = H^H H by one library matmul
    (PAPER.md:74).  Same definition as gram_exact (pinned equal at small sizes);
    only the summation order differs."""
    pos = np.ascontiguousarray(pos, dtype=np.float64)
    out = []
    for d in range(pos.shape[0]):
        H = channel_matrix(arr, pos[d])
        G = H.conj().T @ H
        G = 0.5 * (G + G.conj().T)  # exact Hermitian symmetry (R20); Im diag = 0
        np.fill_diagonal(G, G.diagonal().real)
        out.append(G)
    return np.stack(out)


def bounds_app_a(gram: np.ndarray, snr_db, eig: bool = False, nthreads: int = 0):
    """Appendix A per drop, NEXT-3.
    Returns rstat (D, 2) = (log2 det R, gap = -(1/K) log2 det R), bounds (D, S, 3) =
    (log2 U, log2 det(I + rho G), log2 L), eigenvalues of R (D, K) ascending (cyclic
    Jacobi) or None, flags (D,)."""
    g = np.ascontiguousarray(np.stack([gram.real, gram.imag], axis=-1), dtype=np.float64)
    D, K = g.shape[0], g.shape[1]
    snr = np.ascontiguousarray(np.atleast_1d(snr_db), dtype=np.float64)
    rstat = np.zeros((D, 2))
    bounds = np.zeros((D, snr.size, 3))
    ev = np.zeros((D, K)) if eig else None
    fl = np.zeros(D, dtype=np.uint32)
    lib().or_bounds_app_a(_ptr(g), K, D, _ptr(snr), snr.size, _ptr(rstat), _ptr(bounds),
                          _ptr(ev) if ev is not None else None, _ptr(fl), nthreads)
    return rstat, bounds, ev, fl


def gen_drops_rect(x, y, K: int, n_drops: int, seed: int = 0, first_drop: int = 0) -> np.ndarray:
    """The paper's rectangle user field x ~ U[x0, x1], y ~ U[y0, y1]."""
    pos = np.zeros((n_drops, K, 3), dtype=np.float64)
    lib().or_gen_drops_rect(float(x[0]), float(x[1]), float(y[0]), float(y[1]), K, n_drops, seed, first_drop,
                            _ptr(pos))
    return pos


def saturation_coords(pos: np.ndarray, t: float):
    pos = np.ascontiguousarray(pos, dtype=np.float64)
    D, K, _ = pos.shape
    up, dn = np.zeros(D), np.zeros(D)
    lib().or_saturation_coords(_ptr(pos), K, D, t, _ptr(up), _ptr(dn))
    return up, dn


def saturation_sweep(arr: OrArray, n_list, pos: np.ndarray, snr_db, receivers: int, gram_kind: int = 0,
                     t: float = 0.9, per_drop: bool = False, nthreads: int = 0, valid_mean: bool = False):
    """(ergodic, n_valid, sat, per_drop) -- plus ergodic_valid (the mean over the valid drops
    only) when valid_mean.  ergodic is NaN for a column with any NaN drop (R10)."""
    pos = np.ascontiguousarray(pos, dtype=np.float64)
    D, K, _ = pos.shape
    nl = np.ascontiguousarray(n_list, dtype=np.int64)
    snr = np.ascontiguousarray(np.atleast_1d(snr_db), dtype=np.float64)
    R = n_recv(receivers)
    erg = np.zeros((nl.size, snr.size, R))
    nv = np.zeros((nl.size, snr.size, R), dtype=np.int64)
    sat = np.zeros(4)
    pd = np.zeros((D, nl.size, snr.size, R)) if per_drop else None
    ergv = np.zeros((nl.size, snr.size, R))
    lib().or_saturation_sweep(ctypes.byref(arr), _ptr(nl), nl.size, _ptr(pos), K, D, _ptr(snr), snr.size,
                              receivers, gram_kind, t, _ptr(erg), _ptr(nv), _ptr(ergv), _ptr(sat),
                              _ptr(pd) if pd is not None else None, nthreads)
    if valid_mean:
        return erg, nv, sat, pd, ergv
    return erg, nv, sat, pd


# --------------------------------------------------------------------------- Appendix B
def slope(t: float) -> float:
    """t / sqrt(1 - t^2), the slope of Eqs. (12)-(16)."""
    return t / math.sqrt(1.0 - t * t)


def trapezoid_breakpoints(x_min, x_max, y_min, y_max, t):
    """L1, R1, L2, R2 of Eq. (17)'s definitions."""
    s = slope(t)
    L1 = x_min * s + y_min
    R1 = min(x_min * s + y_max, x_max * s + y_min)
    L2 = max(x_min * s + y_max, x_max * s + y_min)
    R2 = x_max * s + y_max
    return L1, R1, L2, R2


def trapezoid_cdf(z, L1, R1, L2, R2):
    """F_{z_i}(z) of Appendix B, D1 = L2-R1+R2-L1, D2 = R1-L1."""
    D1 = L2 - R1 + R2 - L1
    D2 = R1 - L1
    if z < L1:
        return 0.0
    if z < R1:
        return (z - L1) ** 2 / (D1 * D2)
    if z < L2:
        return (R1 - L1) / D1 + 2.0 / D1 * (z - R1)
    if z < R2:
        return 1.0 - (z - R2) ** 2 / (D1 * D2)
    return 1.0


def ergodic_y_up_rect(x_min, x_max, y_min, y_max, t, K):
    """E[y_up] of Appendix B: int y d(F_z(y)^K) over [L1, R2],
    evaluated by parts as R2 - int_{L1}^{R2} F_z(y)^K dy with quadrature split at
    the kinks R1, L2."""
    from scipy.integrate import quad
    L1, R1, L2, R2 = trapezoid_breakpoints(x_min, x_max, y_min, y_max, t)
    f = lambda z: trapezoid_cdf(z, L1, R1, L2, R2) ** K
    tot = 0.0
    for a, b in ((L1, R1), (R1, L2), (L2, R2)):
        if b > a:
            tot += quad(f, a, b, epsabs=1e-13, epsrel=1e-13, limit=400)[0]
    return R2 - tot


def ergodic_y_down_rect(x_min, x_max, y_min, y_max, t, K):
    """Eq. (18): E[y_down] = y_min + y_max - E[y_up]."""
    return y_min + y_max - ergodic_y_up_rect(x_min, x_max, y_min, y_max, t, K)


def _polar_cdf(z, r_min, r_max, az_min, az_max, c_x, c_y):
    """P(c_x * x + c_y * y <= z) for x = r cos(az), y = r sin(az), r ~ U[r_min, r_max],
    az ~ U[az_min, az_max] (degrees), by quadrature over az (R15)."""
    from scipy.integrate import quad
    a0, a1 = math.radians(az_min), math.radians(az_max)

    def frac(az):
        g = c_x * math.cos(az) + c_y * math.sin(az)
        if g > 0:
            return min(max((z / g - r_min) / (r_max - r_min), 0.0), 1.0)
        if g < 0:
            return 1.0 - min(max((z / g - r_min) / (r_max - r_min), 0.0), 1.0)
        return 1.0 if z >= 0 else 0.0

    return quad(frac, a0, a1, epsabs=1e-12, epsrel=1e-11, limit=400)[0] / (a1 - a0)


def ergodic_saturation_polar(r_min, r_max, az_min, az_max, t, K, pitch):
    """Analytic ergodic saturation point for the polar user law of the configs
    (reading R15): Appendix B's pipeline, E[y_up] = z_hi - int F_z(z)^K dz with
    z = x t/sqrt(1-t^2) + y, E[y_down] = w_lo + int (1 - F_w(w))^K dw with
    w = -x t/sqrt(1-t^2) + y, and M_sat = ceil((E[y_up] - E[y_down]) / pitch)."""
    from scipy.integrate import quad
    s = slope(t)

    def support(cx, cy):
        vals = []
        azs = np.linspace(math.radians(az_min), math.radians(az_max), 20001)
        g = cx * np.cos(azs) + cy * np.sin(azs)
        for r in (r_min, r_max):
            vals.extend((r * g).tolist())
        # the extremum of g over az may be interior
        return min(vals), max(vals)

    zlo, zhi = support(s, 1.0)
    Fz = lambda z: _polar_cdf(z, r_min, r_max, az_min, az_max, s, 1.0)
    Eup = zhi - quad(lambda z: Fz(z) ** K, zlo, zhi, epsabs=1e-10, epsrel=1e-10, limit=400)[0]
    wlo, whi = support(-s, 1.0)
    Fw = lambda w: _polar_cdf(w, r_min, r_max, az_min, az_max, -s, 1.0)
    Edn = wlo + quad(lambda w: (1.0 - Fw(w)) ** K, wlo, whi, epsabs=1e-10, epsrel=1e-10, limit=400)[0]
    return Eup, Edn, math.ceil((Eup - Edn) / pitch)
