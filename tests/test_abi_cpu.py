"""CPU-side checks of the C ABI boundary (no GPU, no compute calls):
the library loads, exports every symbol include/xlmimo.h declares, and rejects
invalid arguments with the documented status codes before touching the device."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "xlmimo.h")
LIB = os.path.join(ROOT, "paper_2503_18118_b200", "libxlmimo.so")


def declared_functions():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(xlmimo_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from tests.conftest import build_product
    build_product()
    return ctypes.CDLL(LIB)


def test_header_declares_the_north_star_entry_points():
    fns = declared_functions()
    for f in ("xlmimo_gen_drops", "xlmimo_gram_exact", "xlmimo_gram_closed_form", "xlmimo_sum_rate",
              "xlmimo_saturation_sweep", "xlmimo_last_error"):
        assert f in fns


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = set(line.split()[-1] for line in out.splitlines() if line.strip())
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing
    for f in declared_functions():
        getattr(lib, f)
    # nothing but the ABI is exported (hidden visibility for internals)
    extra = [s for s in exported if s.startswith("xl") and s not in declared_functions()]
    assert not extra, extra


def test_library_is_sm100a_cubin():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_invalid_arguments_are_rejected_without_a_device(lib):
    import paper_2503_18118_b200 as xl
    L = xl._L
    bad_users = xl.Users.polar((0.0, 10.0), (-60, 60))
    assert L.xlmimo_gen_drops(ctypes.byref(bad_users), 4, 10, 0, 0, ctypes.c_void_p(8), None) == -1
    assert b"user law" in L.xlmimo_last_error()
    u = xl.Users.polar((5.0, 50.0), (-95, 60))
    assert L.xlmimo_gen_drops(ctypes.byref(u), 4, 10, 0, 0, ctypes.c_void_p(8), None) == -1
    u = xl.Users.polar((5.0, 50.0), (-60, 60))
    assert L.xlmimo_gen_drops(ctypes.byref(u), 0, 10, 0, 0, ctypes.c_void_p(8), None) == -1
    upa = xl.Array.upa(8, 8, 100e9)
    assert L.xlmimo_gram_closed_form(ctypes.byref(upa), ctypes.c_void_p(8), 4, 1, ctypes.c_void_p(8), None, None) == -2
    ula_wide = xl.Array.ula(256, 28e9, spacing_wl=0.7)   # Eq. (4) is the lambda/2 array's
    assert L.xlmimo_gram_closed_form(ctypes.byref(ula_wide), ctypes.c_void_p(8), 4, 1, ctypes.c_void_p(8), None,
                                     None) == -2
    assert b"lambda/2" in L.xlmimo_last_error()
    ula = xl.Array.ula(256, 28e9)
    assert L.xlmimo_gram_exact(ctypes.byref(ula), ctypes.c_void_p(8), 1025, 1, 0, 0, ctypes.c_void_p(8), None, 0,
                               None) == -2
    assert L.xlmimo_gram_exact(ctypes.byref(ula), ctypes.c_void_p(8), 65, 1, 0, 1, ctypes.c_void_p(8), None, 0,
                               None) == -2  # materialised is complex64 (fp32) only
    assert L.xlmimo_gram_exact(ctypes.byref(ula), ctypes.c_void_p(8), 65, 1, 0, 0, ctypes.c_void_p(8), None, 0,
                               None) == -3  # needs its workspace
    bad = xl.Array.ula(256, -1.0)
    assert L.xlmimo_gram_exact(ctypes.byref(bad), ctypes.c_void_p(8), 4, 1, 0, 0, ctypes.c_void_p(8), None, 0,
                               None) == -1
    import numpy as np
    snr = np.zeros(1)
    assert L.xlmimo_sum_rate(ctypes.c_void_p(8), 4, 1, snr.ctypes.data_as(ctypes.c_void_p), 1, 0,
                             ctypes.c_void_p(8), None, None) == -1  # no receivers
    # Appendix A / large K: K <= 1024, workspace for K > 64 (Cholesky slots, Householder slots)
    rs = ctypes.c_void_p(8)
    assert L.xlmimo_app_a_bounds(rs, 65, 1, snr.ctypes.data_as(ctypes.c_void_p), 1, rs, rs, rs, None, None, 0,
                                 None) == -3  # K > 64 eigenvalues: Householder slots in the workspace
    assert L.xlmimo_app_a_bounds(rs, 1025, 1, snr.ctypes.data_as(ctypes.c_void_p), 1, rs, rs, None, None, None, 0,
                                 None) == -2
    assert L.xlmimo_app_a_bounds(rs, 100, 1, snr.ctypes.data_as(ctypes.c_void_p), 1, rs, rs, None, None, None, 0,
                                 None) == -3
    assert L.xlmimo_app_a_bounds(rs, 8, 1, None, 1, rs, rs, None, None, None, 0, None) == -1
    assert L.xlmimo_app_a_bounds_workspace(8, 100, 1, 0) == 0 < L.xlmimo_app_a_bounds_workspace(100, 100, 1, 0)
    assert L.xlmimo_app_a_bounds_workspace(8, 100, 1, 1) == 0  # K <= 64: Jacobi in shared memory
    assert L.xlmimo_app_a_bounds_workspace(100, 100, 1, 1) > L.xlmimo_app_a_bounds_workspace(100, 100, 1, 0)
    assert L.xlmimo_sum_rate(rs, 1025, 1, snr.ctypes.data_as(ctypes.c_void_p), 1, 2, rs, None, None) == -2  # K>1024
    assert L.xlmimo_sum_rate(rs, 333, 1, snr.ctypes.data_as(ctypes.c_void_p), 1, 2, rs, None, None) == -3  # ZF: ws
    assert L.xlmimo_sum_rate(rs, 100, 1, snr.ctypes.data_as(ctypes.c_void_p), 1, 2, rs, None, None) == -3  # ZF: ws
    assert L.xlmimo_sum_rate(rs, 100, 1, snr.ctypes.data_as(ctypes.c_void_p), 1, 1, rs, None, None) == -3  # CAP: ws
    assert L.xlmimo_sum_rate_workspace(100, 4, 1, 8) == 0 < L.xlmimo_sum_rate_workspace(100, 4, 1, 1)
    assert L.xlmimo_sum_rate_workspace(100, 4, 1, 1) < L.xlmimo_sum_rate_workspace(100, 4, 1, 7)  # + inverse diagonals
    nl = np.array([256, 512, 1023], dtype=np.int64)  # mixed parity
    erg = np.zeros(16)
    nv = np.zeros(16, dtype=np.int64)
    sat = np.zeros(4)
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    assert L.xlmimo_saturation_sweep(ctypes.byref(ula), p(nl), 3, ctypes.byref(u), None, 4, 10, 0, p(snr), 1, 1, 0, 0,
                                     0.9, p(erg), p(nv), None, p(sat), None, None, 0, None) == -1
    nl = np.array([512, 256], dtype=np.int64)  # not ascending
    assert L.xlmimo_saturation_sweep(ctypes.byref(ula), p(nl), 2, ctypes.byref(u), None, 4, 10, 0, p(snr), 1, 1, 0, 0,
                                     0.9, p(erg), p(nv), None, p(sat), None, None, 0, None) == -1
    nl = np.array([256, 512], dtype=np.int64)
    assert L.xlmimo_saturation_sweep(ctypes.byref(ula), p(nl), 2, ctypes.byref(u), None, 4, 10, 0, p(snr), 1, 1, 0, 0,
                                     1.0, p(erg), p(nv), None, p(sat), None, None, 0, None) == -1  # t not in (0,1)
    assert L.xlmimo_saturation_sweep(ctypes.byref(ula), p(nl), 2, ctypes.byref(u), None, 4, 10, 0, p(snr), 1, 1, 0, 0,
                                     0.9, p(erg), p(nv), None, p(sat), None, None, 0, None) == -3  # no workspace
    assert xl.sweep_workspace_bytes(ula, nl, 4, 10, 1, 1) > 0
    # the size query validates like the call: bad arguments size to 0, never to a wrapped value
    assert xl.sweep_workspace_bytes(ula, nl, 4, 10, -1, 1) == 0          # n_snr < 1
    assert xl.sweep_workspace_bytes(ula, nl, 4, 10, 17, 1) == 0          # n_snr > 16
    assert xl.sweep_workspace_bytes(ula, nl, 4, 10, 1, 0) == 0           # no receiver
    assert xl.sweep_workspace_bytes(ula, nl, 4, 10, 1, 16) == 0          # unknown receiver bit
    assert xl.sweep_workspace_bytes(ula, nl, 4, 10, 1, 1, gram_kind=7) == 0
    assert xl.sweep_workspace_bytes(ula, nl, 4, 10, 1, 1, precision=5) == 0


def test_workspace_queries_are_pure(lib):
    import paper_2503_18118_b200 as xl
    a = xl.Array.ula(2 ** 20, 140e9)
    w1 = xl._L.xlmimo_gram_exact_workspace(ctypes.byref(a), 64, 1000, 0, 0)
    w2 = xl._L.xlmimo_gram_exact_workspace(ctypes.byref(a), 64, 1000, 0, 0)
    assert w1 == w2 > 0
    assert xl._L.xlmimo_gram_exact_workspace(ctypes.byref(a), 1025, 1000, 0, 0) == 0
    assert xl._L.xlmimo_gram_exact_workspace(ctypes.byref(a), 65, 1000, 0, 1) == 0  # fp64 materialised
    assert xl._L.xlmimo_gram_exact_workspace(ctypes.byref(a), 65, 1000, 1, 1) > 0  # fp32 materialised pairs
    assert xl._L.xlmimo_gram_exact_workspace(ctypes.byref(a), 65, 1000, 1, 0) > 0
    assert xl._L.xlmimo_gram_exact_workspace(ctypes.byref(a), 65, 1000, 0, 0) > 0


def test_product_path_has_no_oracle_dependency():
    """The product (package + csrc + include + bench kernels) never references oracle/."""
    pkg = os.path.join(ROOT, "paper_2503_18118_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "liboracle" not in txt, f
                assert "or_gram" not in txt and "xlmimo_oracle" not in txt, f
    assert "oracle" not in open(HDR).read().lower()


def test_path_options_are_an_abi_knob_not_the_environment(lib):
    """Kernel-path overrides are the documented xlmimo_set_option knob (include/xlmimo.h);
    the product sources read no environment variable, so production behaviour cannot change
    silently."""
    import glob
    import paper_2503_18118_b200 as xl
    for src in glob.glob(os.path.join(os.path.dirname(LIB), "csrc", "*")):
        assert "getenv" not in open(src).read(), src
    for opt in range(7):
        assert xl.get_option(opt) == 0
    with xl.option(xl.OPT_LARGE_K, 2):
        assert xl.get_option(xl.OPT_LARGE_K) == 2
    assert xl.get_option(xl.OPT_LARGE_K) == 0
    assert xl._L.xlmimo_set_option(7, 1) == -1 and xl._L.xlmimo_set_option(-1, 1) == -1
    assert xl._L.xlmimo_get_option(99) == 0
