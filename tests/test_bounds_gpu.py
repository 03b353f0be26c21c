"""Out-of-bounds write guard (compute-sanitizer is not available on the GPU pool):
every entry point writes into outputs and workspaces that sit between guard bands
filled with a sentinel bit pattern; after the call (and a synchronize) the guard
bands must be untouched.  Shapes include ragged tails and the large-K paths."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

GUARD = 4096                      # doubles on each side
SENT = -1.2345678901234567e300    # sentinel value


@pytest.fixture(scope="module")
def xl():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from tests.conftest import build_product
    build_product()
    import paper_2503_18118_b200 as xl
    return xl


class Guarded:
    """A float64 device buffer of n elements between two sentinel guard bands."""

    def __init__(self, n, dtype=torch.float64):
        self.n = n
        self.big = torch.full((n + 2 * GUARD,), SENT, dtype=torch.float64, device="cuda")
        self.view = self.big[GUARD:GUARD + n]
        if dtype != torch.float64:
            self.view = self.view.view(dtype)

    def ptr(self):
        return ctypes.c_void_p(self.big.data_ptr() + 8 * GUARD)

    def check(self):
        torch.cuda.synchronize()
        assert torch.all(self.big[:GUARD] == SENT), "write before the buffer"
        assert torch.all(self.big[GUARD + self.n:] == SENT), "write past the buffer"


def _ws(nbytes):
    return Guarded(max(1, (int(nbytes) + 7) // 8))


@pytest.mark.parametrize("K,N,prec,mode,kind", [(8, 1000, 0, 0, "ula"), (4, 999, 0, 0, "ula"), (3, 777, 0, 0, "ula"),
                                                (16, 2050, 0, 0, "ula"), (33, 1501, 0, 0, "ula"), (64, 700, 0, 0, "ula"),
                                                (100, 333, 0, 0, "ula"), (200, 129, 0, 0, "ula"),
                                                (5, 513, 1, 0, "ula"), (16, 4099, 1, 0, "ula"), (40, 1030, 1, 0, "ula"),
                                                (16, 4096, 1, 1, "ula"), (5, 1001, 1, 1, "ula"), (12, 300, 0, 0, "upa"),
                                                (12, 300, 1, 0, "upa"), (70, 300, 0, 0, "upa"),
                                                (130, 1100, 1, 0, "ula"), (150, 1030, 0, 0, "ula"),
                                                (100, 2048, 1, 0, "ula"), (200, 2048, 1, 0, "ula"),
                                                (256, 1100, 1, 0, "ula"), (300, 1100, 1, 0, "ula"),
                                                (100, 2048, 1, 1, "ula"), (128, 1000, 0, 0, "ula"),
                                                # MT2's variable-size star plans (G = 7, 10, 12, 14, 13 UPA)
                                                (56, 700, 0, 0, "ula"), (80, 333, 0, 0, "ula"),
                                                (96, 333, 0, 0, "ula"), (112, 333, 0, 0, "ula"),
                                                (104, 300, 0, 0, "upa")])
def test_gram_exact_writes_in_bounds(xl, K, N, prec, mode, kind):
    D = 3
    if kind == "ula":
        a = xl.Array.ula(N, 100e9)
        pos = xl.gen_drops(xl.Users.polar((2.0, 20.0), (-60, 60)), K, D, seed=K)
    else:
        a = xl.Array.upa(20, N // 20, 100e9)
        pos = xl.gen_drops(xl.Users.polar((2.0, 20.0), (-60, 60), (-30, 30)), K, D, seed=K)
    g = Guarded(D * K * K * 2)
    need = xl._L.xlmimo_gram_exact_workspace(ctypes.byref(a), K, D, prec, mode)
    ws = _ws(need)
    rc = xl._L.xlmimo_gram_exact(ctypes.byref(a), ctypes.c_void_p(pos.data_ptr()), K, D, prec, mode, g.ptr(),
                                 ws.ptr() if need else None, need, None)
    assert rc == 0, xl._L.xlmimo_last_error()
    g.check()
    ws.check()
    assert torch.isfinite(g.view).all()


@pytest.mark.parametrize("K", [3, 8, 16, 33, 64, 100, 161, 250])
def test_receivers_and_bounds_write_in_bounds(xl, K):
    D, S = 5, 2
    snr = np.array([0.0, 10.0])
    sp = snr.ctypes.data_as(ctypes.c_void_p)
    a = xl.Array.ula(max(4 * K, 300), 100e9)
    pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, D, seed=K)
    G = torch.view_as_real(xl.gram_exact(a, pos)).contiguous()
    gp = ctypes.c_void_p(G.data_ptr())
    allr = 15
    rates = Guarded(D * S * 4)
    flags = Guarded((D + 1) // 2, torch.int32)
    flags.view.zero_()
    need = xl._L.xlmimo_sum_rate_workspace(K, D, S, allr)
    ws = _ws(need)
    rc = xl._L.xlmimo_sum_rate_ws(gp, K, D, sp, S, allr, rates.ptr(), flags.ptr(), ws.ptr() if need else None,
                                  need, None)
    assert rc == 0, xl._L.xlmimo_last_error()
    for b in (rates, flags, ws):
        b.check()
    rst = Guarded(D * 2)
    bo = Guarded(D * S * 3)
    ev = Guarded(D * K)
    need = xl._L.xlmimo_app_a_bounds_workspace(K, D, S, 1)
    ws2 = _ws(need)
    rc = xl._L.xlmimo_app_a_bounds(gp, K, D, sp, S, rst.ptr(), bo.ptr(), ev.ptr() if ev else None, None,
                                   ws2.ptr() if need else None, need, None)
    assert rc == 0, xl._L.xlmimo_last_error()
    for b in (rst, bo, ws2) + ((ev,) if ev else ()):
        b.check()
    if K <= 64:
        mis = Guarded(D * S)
        rc = xl._L.xlmimo_sum_rate_mismatched(gp, gp, K, D, sp, S, mis.ptr(), None, None)
        assert rc == 0
        mis.check()


def test_drops_closed_form_and_sweep_write_in_bounds(xl):
    K, D = 8, 37
    p = Guarded(D * K * 3)
    u = xl.Users.polar((3.0, 30.0), (-60, 60))
    assert xl._L.xlmimo_gen_drops(ctypes.byref(u), K, D, 0, 5, p.ptr(), None) == 0
    p.check()
    pr = Guarded(D * K * 3)
    assert xl._L.xlmimo_gen_drops_rect(1.0, 2.0, -7.5, 7.5, K, D, 0, 0, pr.ptr(), None) == 0
    pr.check()
    a = xl.Array.ula(1025, 28e9)
    g = Guarded(D * K * K * 2)
    fl = Guarded((D + 1) // 2, torch.int32)
    assert xl._L.xlmimo_gram_closed_form(ctypes.byref(a), p.ptr(), K, D, g.ptr(), fl.ptr(), None) == 0
    g.check()
    fl.check()
    nl = np.array([255, 513, 1025], dtype=np.int64)
    snr = np.array([0.0, 10.0, 20.0])
    R = 3
    erg = np.zeros(3 * 3 * R)
    nv = np.zeros(3 * 3 * R, dtype=np.int64)
    sat = np.zeros(4)
    pd = Guarded(D * 3 * 3 * R)
    need = xl.sweep_workspace_bytes(a, nl, K, D, 3, 7)
    ws = _ws(need)
    f = lambda arr: arr.ctypes.data_as(ctypes.c_void_p)
    rc = xl._L.xlmimo_saturation_sweep(ctypes.byref(a), f(nl), 3, None, p.ptr(), K, D, 0, f(snr), 3, 7, 0, 0, 0.9,
                                       f(erg), f(nv), None, f(sat), pd.ptr(), ws.ptr(), need, None)
    assert rc == 0, xl._L.xlmimo_last_error()
    pd.check()
    ws.check()
