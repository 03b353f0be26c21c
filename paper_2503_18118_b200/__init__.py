"""B200 (sm_100a) Monte Carlo engine for near-field XL-MIMO uplink sum capacity
(Cui, Park, Alouini, arXiv 2503.18118).

Thin Python binding over the C ABI of ``libxlmimo.so`` (``include/xlmimo.h``):
argument marshalling only.  Every step of the path -- drops, channel, Gram,
closed-form Gram, receivers, ergodic reduction, saturation statistics -- runs
in the library's CUDA kernels.  PyTorch provides device memory and streams.
There is no CPU fallback: importing this package without the built library,
or calling it without a CUDA device, raises.

Function names follow the ABI: gen_drops, gram_exact, gram_closed_form,
sum_rate, saturation_sweep (+ saturation_sweep_host, the host-buffer entry),
and the widened rows sum_rate_mismatched (NEXT-1), app_a_bounds (NEXT-3),
gen_drops_rect (NEXT-4).
"""
from __future__ import annotations

import ctypes
import os

import torch

__all__ = ["Array", "Users", "gen_drops", "draw_words", "gram_workspace_bytes", "sweep_workspace_bytes", "gram_exact", "gram_closed_form", "sum_rate", "sum_rate_mismatched",
           "gen_drops_rect", "app_a_bounds", "saturation_sweep",
           "saturation_sweep_host", "launch_count", "lib_path", "XlmimoError",
           "ULA", "UPA", "FP64", "FP32", "FUSED", "MATERIALIZED", "GRAM_EXACT", "GRAM_CLOSED_FORM",
           "RECV_CAP", "RECV_ZF", "RECV_MMSE", "RECV_MRC", "n_recv", "option", "set_option", "get_option",
           "OPT_LARGE_K", "OPT_PAIR", "OPT_GRAM_KERNEL", "OPT_SPLIT_NT", "OPT_DMMA_VARIANT", "OPT_MT2_BUFFERS",
           "OPT_STREAM"]

ULA, UPA = 0, 1
FP64, FP32 = 0, 1
FUSED, MATERIALIZED = 0, 1
GRAM_EXACT, GRAM_CLOSED_FORM = 0, 1
RECV_CAP, RECV_ZF, RECV_MMSE, RECV_MRC = 1, 2, 4, 8
(OPT_LARGE_K, OPT_PAIR, OPT_GRAM_KERNEL, OPT_SPLIT_NT, OPT_DMMA_VARIANT, OPT_MT2_BUFFERS,
 OPT_STREAM) = range(7)
FLAG_G_NOT_PD, FLAG_A_NOT_PD, FLAG_MRC_UNDEF, FLAG_DEGENERATE, FLAG_NONFINITE = 1, 2, 4, 8, 16

_HERE = os.path.dirname(os.path.abspath(__file__))
lib_path = os.path.join(_HERE, "libxlmimo.so")

if not os.path.exists(lib_path):
    raise ImportError(f"libxlmimo.so not built ({lib_path}); run `python -m paper_2503_18118_b200.build` "
                      "(there is no CPU fallback)")


class Array(ctypes.Structure):
    """xlmimo_array_t: ULA (n_y = N, n_z = 1) or UPA (n_y x n_z), pitch spacing_wl * lambda."""
    _fields_ = [("kind", ctypes.c_int32), ("n_y", ctypes.c_int64), ("n_z", ctypes.c_int64),
                ("fc_hz", ctypes.c_double), ("spacing_wl", ctypes.c_double), ("beta0", ctypes.c_double)]

    @classmethod
    def ula(cls, N, fc_hz, spacing_wl=0.5, beta0=1.0):
        return cls(ULA, int(N), 1, float(fc_hz), float(spacing_wl), float(beta0))

    @classmethod
    def upa(cls, n_y, n_z, fc_hz, spacing_wl=0.5, beta0=1.0):
        return cls(UPA, int(n_y), int(n_z), float(fc_hz), float(spacing_wl), float(beta0))

    @property
    def N(self):
        return self.n_y * (self.n_z if self.kind == UPA else 1)


class Users(ctypes.Structure):
    """xlmimo_users_t: r ~ U[r_min, r_max] from the array centre, az/el uniform (degrees)."""
    _fields_ = [("r_min_m", ctypes.c_double), ("r_max_m", ctypes.c_double),
                ("az_min_deg", ctypes.c_double), ("az_max_deg", ctypes.c_double),
                ("el_min_deg", ctypes.c_double), ("el_max_deg", ctypes.c_double)]

    @classmethod
    def polar(cls, r, az, el=(0.0, 0.0)):
        return cls(float(r[0]), float(r[1]), float(az[0]), float(az[1]), float(el[0]), float(el[1]))


class XlmimoError(RuntimeError):
    pass


def _load():
    L = ctypes.CDLL(lib_path)
    P, vp = ctypes.POINTER, ctypes.c_void_p
    i32, i64, u32, u64, d, sz = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64,
                                 ctypes.c_double, ctypes.c_size_t)
    L.xlmimo_gen_drops.argtypes = [P(Users), i32, i64, u64, u64, vp, vp]
    L.xlmimo_draw_words.argtypes = [i32, i64, u64, u64, vp, vp]
    L.xlmimo_draw_words.restype = ctypes.c_int
    L.xlmimo_gram_exact_workspace.argtypes = [P(Array), i32, i64, i32, i32]
    L.xlmimo_gram_exact_workspace.restype = sz
    L.xlmimo_gram_exact.argtypes = [P(Array), vp, i32, i64, i32, i32, vp, vp, sz, vp]
    L.xlmimo_gram_closed_form.argtypes = [P(Array), vp, i32, i64, vp, vp, vp]
    L.xlmimo_sum_rate.argtypes = [vp, i32, i64, vp, i32, u32, vp, vp, vp]
    L.xlmimo_sum_rate_workspace.argtypes = [i32, i64, i32, u32]
    L.xlmimo_sum_rate_workspace.restype = sz
    L.xlmimo_sum_rate_ws.argtypes = [vp, i32, i64, vp, i32, u32, vp, vp, vp, sz, vp]
    L.xlmimo_app_a_bounds_workspace.argtypes = [i32, i64, i32, i32]
    L.xlmimo_app_a_bounds_workspace.restype = sz
    L.xlmimo_app_a_bounds.argtypes = [vp, i32, i64, vp, i32, vp, vp, vp, vp, vp, sz, vp]
    L.xlmimo_saturation_sweep_workspace.argtypes = [P(Array), vp, i32, i32, i64, i32, u32, i32, i32]
    L.xlmimo_saturation_sweep_workspace.restype = sz
    L.xlmimo_saturation_sweep.argtypes = [P(Array), vp, i32, P(Users), vp, i32, i64, u64, vp, i32, u32, i32, i32, d,
                                          vp, vp, vp, vp, vp, vp, sz, vp]
    L.xlmimo_saturation_sweep_host.argtypes = [P(Array), vp, i32, vp, i32, i64, vp, i32, u32, i32, i32, d,
                                               vp, vp, vp, vp, vp, sz, vp]
    L.xlmimo_sum_rate_mismatched.argtypes = [vp, vp, i32, i64, vp, i32, vp, vp, vp]
    L.xlmimo_sum_rate_mismatched.restype = ctypes.c_int
    L.xlmimo_gen_drops_rect.argtypes = [d, d, d, d, i32, i64, u64, u64, vp, vp]
    L.xlmimo_gen_drops_rect.restype = ctypes.c_int
    L.xlmimo_set_option.argtypes = [i32, i64]
    L.xlmimo_set_option.restype = ctypes.c_int
    L.xlmimo_get_option.argtypes = [i32]
    L.xlmimo_get_option.restype = i64
    L.xlmimo_timing_enable.argtypes = [i32]
    L.xlmimo_timing_read.argtypes = [i32, ctypes.c_char_p, vp, vp]
    L.xlmimo_last_error.restype = ctypes.c_char_p
    L.xlmimo_launch_count.restype = u64
    for name in ("xlmimo_gen_drops", "xlmimo_gram_exact", "xlmimo_gram_closed_form", "xlmimo_sum_rate",
                 "xlmimo_sum_rate_ws", "xlmimo_app_a_bounds", "xlmimo_saturation_sweep",
                 "xlmimo_saturation_sweep_host"):
        getattr(L, name).restype = ctypes.c_int
    return L


_L = _load()


def _check(rc: int, what: str):
    if rc != 0:
        raise XlmimoError(f"{what} failed ({rc}): {_L.xlmimo_last_error().decode()}")


def _need_cuda():
    if not torch.cuda.is_available():
        raise XlmimoError("xlmimo needs a CUDA device (B200, sm_100a); there is no CPU fallback")


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _dptr(t: torch.Tensor):
    assert t.is_cuda and t.is_contiguous()
    return ctypes.c_void_p(t.data_ptr())


def _check_tensor(t: torch.Tensor, what: str, dtype, shape):
    """Argument checks before a device pointer crosses the ABI (a wrong dtype or a short
    tensor would make the kernels read or write out of bounds)."""
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise XlmimoError(f"{what}: expected a CUDA tensor")
    if t.dtype not in (dtype if isinstance(dtype, tuple) else (dtype,)):
        raise XlmimoError(f"{what}: dtype {t.dtype}, expected {dtype}")
    if tuple(t.shape) != tuple(shape):
        raise XlmimoError(f"{what}: shape {tuple(t.shape)}, expected {tuple(shape)}")
    if not t.is_contiguous():
        raise XlmimoError(f"{what}: must be contiguous")


def _check_pos(pos: torch.Tensor, K: int, n_drops: int):
    _check_tensor(pos, "pos", torch.float64, (n_drops, K, 3))


def _check_flags(fl: torch.Tensor, n_drops: int):
    _check_tensor(fl, "flags", (torch.int32, torch.uint32), (n_drops,))


def _gram_arg(gram: torch.Tensor, what: str = "gram") -> torch.Tensor:
    """[D, K, K] complex128 or [D, K, K, 2] float64 -> the contiguous interleaved float64 view."""
    g = torch.view_as_real(gram) if gram.is_complex() else gram
    if g.dim() != 4 or g.shape[1] != g.shape[2] or g.shape[3] != 2:
        raise XlmimoError(f"{what}: shape {tuple(gram.shape)}, expected [D, K, K] complex or [D, K, K, 2]")
    g = g.contiguous()
    _check_tensor(g, what, torch.float64, tuple(g.shape))
    return g


def _hptr(a):
    return ctypes.c_void_p(a.data_ptr()) if isinstance(a, torch.Tensor) else a.ctypes.data_as(ctypes.c_void_p)


def _f64_host(x):
    import numpy as np
    return np.ascontiguousarray(np.atleast_1d(x), dtype=np.float64)


def n_recv(receivers: int) -> int:
    return bin(int(receivers) & 15).count("1")


def set_option(opt: int, value: int):
    """Kernel-path override (include/xlmimo.h, "path options"); 0 = automatic."""
    _check(_L.xlmimo_set_option(opt, int(value)), "xlmimo_set_option")


def get_option(opt: int) -> int:
    return int(_L.xlmimo_get_option(opt))


class option:
    """``with option(OPT_LARGE_K, 2): ...`` -- set a path override for a block, then restore it."""

    def __init__(self, opt: int, value: int):
        self.opt, self.value = opt, value

    def __enter__(self):
        self.prev = get_option(self.opt)
        set_option(self.opt, self.value)
        return self

    def __exit__(self, *exc):
        set_option(self.opt, self.prev)
        return False


def launch_count() -> int:
    """Kernels launched by libxlmimo in this process (monotone)."""
    return int(_L.xlmimo_launch_count())


def _workspace(nbytes: int, device):
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)


# --------------------------------------------------------------------------- a1
def gen_drops(users: Users, K: int, n_drops: int, seed: int = 0, first_drop: int = 0, device=None,
              out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Seeded drops -> positions [n_drops, K, 3] fp64 (metres) on the device."""
    _need_cuda()
    dev = device or torch.device("cuda", torch.cuda.current_device())
    pos = out if out is not None else torch.empty((n_drops, K, 3), dtype=torch.float64, device=dev)
    _check_pos(pos, K, n_drops)
    _check(_L.xlmimo_gen_drops(ctypes.byref(users), K, n_drops, seed, first_drop, _dptr(pos), _stream(stream)),
           "xlmimo_gen_drops")
    return pos


def draw_words(K: int, n_drops: int, seed: int = 0, first_drop: int = 0, device=None, stream=None) -> torch.Tensor:
    """The raw Philox4x64-10 words behind gen_drops: [n_drops, K, 4] uint64 on the device."""
    _need_cuda()
    dev = device or torch.device("cuda", torch.cuda.current_device())
    w = torch.empty((n_drops, K, 4), dtype=torch.uint64, device=dev)
    _check(_L.xlmimo_draw_words(K, n_drops, seed, first_drop, _dptr(w), _stream(stream)), "xlmimo_draw_words")
    return w


# --------------------------------------------------------------------------- a2 + a3
def gram_workspace_bytes(array: Array, K: int, n_drops: int, precision: int = FP64, mode: int = FUSED) -> int:
    """xlmimo_gram_exact_workspace: scratch bytes gram_exact needs for this shape (0 = none)."""
    return int(_L.xlmimo_gram_exact_workspace(ctypes.byref(array), K, n_drops, precision, mode))


def gram_exact(array: Array, pos: torch.Tensor, precision: int = FP64, mode: int = FUSED,
               out: torch.Tensor | None = None, ws: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Exact Gram H^H H, complex128 [n_drops, K, K]."""
    _need_cuda()
    D, K, _ = pos.shape
    _check_pos(pos, K, D)
    g = out if out is not None else torch.empty((D, K, K, 2), dtype=torch.float64, device=pos.device)
    _check_tensor(g, "out", torch.float64, (D, K, K, 2))
    need = _L.xlmimo_gram_exact_workspace(ctypes.byref(array), K, D, precision, mode)
    if ws is None or ws.numel() < need:
        ws = _workspace(need, pos.device)
    _check(_L.xlmimo_gram_exact(ctypes.byref(array), _dptr(pos), K, D, precision, mode, _dptr(g), _dptr(ws),
                                ws.numel(), _stream(stream)), "xlmimo_gram_exact")
    return torch.view_as_complex(g)


# --------------------------------------------------------------------------- a4
def gram_closed_form(array: Array, pos: torch.Tensor, stream=None):
    """Closed-form (modified-ZF) Gram complex128 [D, K, K] and per-drop flags (uint32 as int32)."""
    _need_cuda()
    D, K, _ = pos.shape
    _check_pos(pos, K, D)
    g = torch.empty((D, K, K, 2), dtype=torch.float64, device=pos.device)
    fl = torch.zeros(D, dtype=torch.int32, device=pos.device)
    _check(_L.xlmimo_gram_closed_form(ctypes.byref(array), _dptr(pos), K, D, _dptr(g), _dptr(fl), _stream(stream)),
           "xlmimo_gram_closed_form")
    return torch.view_as_complex(g), fl


# --------------------------------------------------------------------------- a5
def sum_rate(gram: torch.Tensor, snr_db, receivers: int, flags: torch.Tensor | None = None,
             ws: torch.Tensor | None = None, stream=None):
    """Receivers per drop: rates [D, n_snr, n_recv] (bits/s/Hz) and flags [D] (OR-ed into `flags`).
    K <= 64: warp Cholesky per drop; 64 < K <= 1024: all receivers through a CTA or tiled DMMA
    Cholesky and blocked inverse in a workspace."""
    _need_cuda()
    g = _gram_arg(gram)
    D, K = g.shape[0], g.shape[1]
    snr = _f64_host(snr_db)
    rates = torch.empty((D, snr.size, n_recv(receivers)), dtype=torch.float64, device=g.device)
    fl = flags if flags is not None else torch.zeros(D, dtype=torch.int32, device=g.device)
    _check_flags(fl, D)
    need = int(_L.xlmimo_sum_rate_workspace(K, D, snr.size, receivers))
    if need and (ws is None or ws.numel() < need):
        ws = _workspace(need, g.device)
    _check(_L.xlmimo_sum_rate_ws(_dptr(g), K, D, _hptr(snr), snr.size, receivers, _dptr(rates), _dptr(fl),
                                 _dptr(ws) if need else None, ws.numel() if need else 0, _stream(stream)),
           "xlmimo_sum_rate_ws")
    return rates, fl


def app_a_bounds(gram: torch.Tensor, snr_db, eig: bool = False, ws: torch.Tensor | None = None, stream=None):
    """NEXT-3, Appendix A per drop.  Returns rstat [D, 2] = (log2 det R,
    gap = -log2 det(R)/K), bounds [D, n_snr, 3] = (log2 U, log2 det(I + rho G), log2 L),
    eigenvalues of R [D, K] ascending (Jacobi for K <= 64, Householder + bisection above) or
    None, flags [D]."""
    _need_cuda()
    g = _gram_arg(gram)
    D, K = g.shape[0], g.shape[1]
    snr = _f64_host(snr_db)
    rstat = torch.empty((D, 2), dtype=torch.float64, device=g.device)
    bounds = torch.empty((D, snr.size, 3), dtype=torch.float64, device=g.device)
    ev = torch.empty((D, K), dtype=torch.float64, device=g.device) if eig else None
    fl = torch.zeros(D, dtype=torch.int32, device=g.device)
    need = int(_L.xlmimo_app_a_bounds_workspace(K, D, snr.size, 1 if eig else 0))
    if need and (ws is None or ws.numel() < need):
        ws = _workspace(need, g.device)
    _check(_L.xlmimo_app_a_bounds(_dptr(g), K, D, _hptr(snr), snr.size, _dptr(rstat), _dptr(bounds),
                                  _dptr(ev) if ev is not None else None, _dptr(fl), _dptr(ws) if need else None,
                                  ws.numel() if need else 0, _stream(stream)), "xlmimo_app_a_bounds")
    return rstat, bounds, ev, fl


def sum_rate_mismatched(gram: torch.Tensor, gram_model: torch.Tensor, snr_db, flags: torch.Tensor | None = None,
                        stream=None):
    """NEXT-1: effective rate of the modified-ZF equalizer G~^{-1} H^H on the true channel.
    Returns rates [D, n_snr] and flags [D] (bit 5: G~ singular)."""
    _need_cuda()
    g = _gram_arg(gram)
    gm = _gram_arg(gram_model, "gram_model")
    if gm.shape != g.shape:
        raise XlmimoError(f"gram_model: shape {tuple(gm.shape)} != gram {tuple(g.shape)}")
    D, K = g.shape[0], g.shape[1]
    snr = _f64_host(snr_db)
    rates = torch.empty((D, snr.size), dtype=torch.float64, device=g.device)
    fl = flags if flags is not None else torch.zeros(D, dtype=torch.int32, device=g.device)
    _check_flags(fl, D)
    _check(_L.xlmimo_sum_rate_mismatched(_dptr(g), _dptr(gm), K, D, _hptr(snr), snr.size, _dptr(rates), _dptr(fl),
                                         _stream(stream)), "xlmimo_sum_rate_mismatched")
    return rates, fl


def gen_drops_rect(x, y, K: int, n_drops: int, seed: int = 0, first_drop: int = 0, device=None,
                   out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """NEXT-4: drops from the paper's rectangle user field x ~ U[x0,x1], y ~ U[y0,y1]."""
    _need_cuda()
    dev = device or torch.device("cuda", torch.cuda.current_device())
    pos = out if out is not None else torch.empty((n_drops, K, 3), dtype=torch.float64, device=dev)
    _check_pos(pos, K, n_drops)
    _check(_L.xlmimo_gen_drops_rect(float(x[0]), float(x[1]), float(y[0]), float(y[1]), K, n_drops, seed,
                                    first_drop, _dptr(pos), _stream(stream)), "xlmimo_gen_drops_rect")
    return pos


# --------------------------------------------------------------------------- a1..a6
def sweep_workspace_bytes(array: Array, n_list, K, n_drops, n_snr, receivers, gram_kind=GRAM_EXACT,
                          precision=FP64) -> int:
    import numpy as np
    nl = np.ascontiguousarray(n_list, dtype=np.int64)
    return int(_L.xlmimo_saturation_sweep_workspace(ctypes.byref(array), _hptr(nl), nl.size, K, n_drops, n_snr,
                                                    receivers, gram_kind, precision))


def saturation_sweep(array: Array, n_list, K: int, n_drops: int, snr_db, receivers: int, *, users: Users | None = None,
                     pos: torch.Tensor | None = None, seed: int = 0, gram_kind: int = GRAM_EXACT,
                     precision: int = FP64, t: float = 0.9, per_drop: bool = False, ws: torch.Tensor | None = None,
                     stream=None, device=None):
    """Capacity-vs-N sweep over nested centred ULAs.  Returns a dict with host numpy arrays
    ergodic [n_n, n_snr, n_recv] (NaN for a column with any NaN drop, R10), n_valid (same),
    ergodic_valid (same: the mean over the valid drops), sat [4] and (optionally) the device
    per_drop [n_drops, n_n, n_snr, n_recv]."""
    import numpy as np
    _need_cuda()
    dev = pos.device if pos is not None else (device or torch.device("cuda", torch.cuda.current_device()))
    nl = np.ascontiguousarray(n_list, dtype=np.int64)
    snr = _f64_host(snr_db)
    R = n_recv(receivers)
    if pos is not None:
        _check_pos(pos, K, n_drops)
    erg = np.zeros((nl.size, snr.size, R))
    ergv = np.zeros((nl.size, snr.size, R))
    nv = np.zeros((nl.size, snr.size, R), dtype=np.int64)
    sat = np.zeros(4)
    pd = torch.empty((n_drops, nl.size, snr.size, R), dtype=torch.float64, device=dev) if per_drop else None
    need = sweep_workspace_bytes(array, nl, K, n_drops, snr.size, receivers, gram_kind, precision)
    if ws is None or ws.numel() < need:
        ws = _workspace(need, dev)
    _check(_L.xlmimo_saturation_sweep(ctypes.byref(array), _hptr(nl), nl.size,
                                      ctypes.byref(users) if users is not None else None,
                                      _dptr(pos) if pos is not None else None, K, n_drops, seed, _hptr(snr),
                                      snr.size, receivers, gram_kind, precision, t, _hptr(erg), _hptr(nv),
                                      _hptr(ergv), _hptr(sat), _dptr(pd) if pd is not None else None, _dptr(ws),
                                      ws.numel(), _stream(stream)), "xlmimo_saturation_sweep")
    return {"ergodic": erg, "n_valid": nv, "ergodic_valid": ergv, "sat": sat, "per_drop": pd}


def saturation_sweep_host(array: Array, n_list, pos_host: torch.Tensor, snr_db, receivers: int, *,
                          gram_kind: int = GRAM_EXACT, precision: int = FP64, t: float = 0.9,
                          ws: torch.Tensor | None = None, stream=None, device=None):
    """The end-to-end entry: HOST positions (pin them for speed) in, host results out."""
    import numpy as np
    _need_cuda()
    if pos_host.is_cuda or pos_host.dtype != torch.float64 or not pos_host.is_contiguous() or pos_host.dim() != 3 \
            or pos_host.shape[2] != 3:
        raise XlmimoError("pos_host: expected a contiguous host float64 tensor [n_drops, K, 3]")
    dev = device or torch.device("cuda", torch.cuda.current_device())
    n_drops, K, _ = pos_host.shape
    nl = np.ascontiguousarray(n_list, dtype=np.int64)
    snr = _f64_host(snr_db)
    R = n_recv(receivers)
    erg = np.zeros((nl.size, snr.size, R))
    ergv = np.zeros((nl.size, snr.size, R))
    nv = np.zeros((nl.size, snr.size, R), dtype=np.int64)
    sat = np.zeros(4)
    need = sweep_workspace_bytes(array, nl, K, n_drops, snr.size, receivers, gram_kind, precision)
    if ws is None or ws.numel() < need:
        ws = _workspace(need, dev)
    _check(_L.xlmimo_saturation_sweep_host(ctypes.byref(array), _hptr(nl), nl.size, _hptr(pos_host), K, n_drops,
                                           _hptr(snr), snr.size, receivers, gram_kind, precision, t, _hptr(erg),
                                           _hptr(nv), _hptr(ergv), _hptr(sat), _dptr(ws), ws.numel(),
                                           _stream(stream)),
           "xlmimo_saturation_sweep_host")
    return {"ergodic": erg, "n_valid": nv, "ergodic_valid": ergv, "sat": sat}
