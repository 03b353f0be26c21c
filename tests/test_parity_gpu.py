"""GPU parity: the CUDA path through the C ABI vs the CPU oracle, on the same
seeded inputs (oracle consumes the GPU-drawn positions for Gram/rate parity;
the draws themselves are compared separately).

Tolerances (north_star): Gram normalized error
|dG_ij| / sqrt(G_ii G_jj) <= 1e-9 (fp64) / 1e-4 (fp32); per-drop rates <= 1e-6
bits/s/Hz (fp64) / 1e-3 (fp32); flags and integer outputs exact.
"""
import math

import numpy as np
import pytest

from tests._util import normalized_err
from workloads import CONFIGS

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def xl():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from tests.conftest import build_product
    build_product()
    import paper_2503_18118_b200 as xl
    return xl


def _arr(xl, orc, kind, n_y, n_z, fc):
    if kind == "ula":
        return xl.Array.ula(n_y, fc), orc.array("ula", n_y=n_y, fc_hz=fc)
    return xl.Array.upa(n_y, n_z, fc), orc.array("upa", n_y=n_y, n_z=n_z, fc_hz=fc)


def _users(xl, orc, r, az, el=(0.0, 0.0)):
    return xl.Users.polar(r, az, el), orc.users(r=r, az=az, el=el)


# --------------------------------------------------------------------------- a1
@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_drops_match_oracle(xl, orc, cfg):
    w = CONFIGS[cfg]
    ug, uo = _users(xl, orc, w.r, w.az, w.el)
    n = min(w.n_drops, 2000)
    pg = xl.gen_drops(ug, w.K, n, seed=w.seed).cpu().numpy()
    po = orc.gen_drops(uo, w.K, n, seed=w.seed)
    assert np.max(np.abs(pg - po)) <= 4e-15 * max(1.0, w.r[1])
    # first_drop addressing
    pg2 = xl.gen_drops(ug, w.K, 10, seed=w.seed, first_drop=n - 10).cpu().numpy()
    assert np.array_equal(pg2, pg[n - 10:])


def test_drops_empty(xl):
    u = xl.Users.polar((5.0, 50.0), (-60, 60))
    assert xl.gen_drops(u, 4, 0).shape == (0, 4, 3)


# --------------------------------------------------------------------------- a2 + a3
CASES = [
    # kind, n_y, n_z, fc, K, drops, r, az, el
    ("ula", 256, 1, 28e9, 4, 1000, (5.0, 50.0), (-60.0, 60.0), (0.0, 0.0)),     # cfg1 all drops
    ("ula", 1000, 1, 28e9, 8, 7, (3.0, 30.0), (-60.0, 60.0), (0.0, 0.0)),       # ragged even N, K=8
    ("ula", 999, 1, 100e9, 5, 5, (2.0, 20.0), (-75.0, 75.0), (0.0, 0.0)),       # odd N
    ("ula", 1, 1, 28e9, 3, 3, (5.0, 50.0), (-60.0, 60.0), (0.0, 0.0)),          # N = 1
    ("ula", 777, 1, 100e9, 1, 4, (2.0, 20.0), (-75.0, 75.0), (0.0, 0.0)),       # K = 1
    ("ula", 4133, 1, 100e9, 9, 3, (2.0, 20.0), (-75.0, 75.0), (0.0, 0.0)),      # K = 9 (tiled, padded)
    ("ula", 16384, 1, 100e9, 16, 6, (2.0, 20.0), (-75.0, 75.0), (0.0, 0.0)),    # cfg3 geometry
    ("ula", 3001, 1, 140e9, 33, 2, (5.0, 100.0), (-60.0, 60.0), (0.0, 0.0)),    # K = 33 (KP = 48)
    ("ula", 5000, 1, 140e9, 64, 2, (5.0, 100.0), (-60.0, 60.0), (0.0, 0.0)),    # K = 64
    ("upa", 37, 23, 100e9, 6, 3, (2.0, 20.0), (-60.0, 60.0), (-30.0, 30.0)),    # UPA ragged, small K
    ("upa", 64, 64, 100e9, 32, 2, (2.0, 20.0), (-60.0, 60.0), (-30.0, 30.0)),   # UPA K = 32
    ("ula", 2049, 1, 100e9, 20, 3, (2.0, 20.0), (-75.0, 75.0), (0.0, 0.0)),     # K = 20 (3 groups, odd N)
    ("upa", 51, 29, 100e9, 45, 2, (2.0, 20.0), (-60.0, 60.0), (-30.0, 30.0)),   # K = 45 (6 groups, ragged UPA)
    ("ula", 1500, 1, 140e9, 52, 2, (5.0, 100.0), (-60.0, 60.0), (0.0, 0.0)),    # K = 52 (7 groups)
    ("upa", 12, 10, 100e9, 16, 2, (2.0, 20.0), (-60.0, 60.0), (-30.0, 30.0)),   # UPA rows not a multiple of 8
    ("upa", 24, 11, 100e9, 12, 2, (2.0, 20.0), (-60.0, 60.0), (-30.0, 30.0)),   # UPA rows a multiple of 8
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}{c[1]}x{c[2]}_K{c[4]}_D{c[5]}")
@pytest.mark.parametrize("prec", ["fp64", "fp32", "mat32"])
def test_gram_exact_parity(xl, orc, case, prec):
    kind, n_y, n_z, fc, K, D, r, az, el = case
    ag, ao = _arr(xl, orc, kind, n_y, n_z, fc)
    ug, _ = _users(xl, orc, r, az, el)
    pos = xl.gen_drops(ug, K, D, seed=17)
    mode = xl.MATERIALIZED if prec == "mat32" else xl.FUSED
    G = xl.gram_exact(ag, pos, precision=xl.FP64 if prec == "fp64" else xl.FP32, mode=mode).cpu().numpy()
    Go = orc.gram_exact(ao, pos.cpu().numpy())
    tol = 1e-9 if prec == "fp64" else 1e-4
    assert normalized_err(G, Go) <= tol
    assert np.array_equal(G, np.conj(np.swapaxes(G, 1, 2)))   # exactly Hermitian
    assert np.all(np.imag(np.diagonal(G, axis1=1, axis2=2)) == 0)


def test_gram_exact_empty_and_determinism(xl):
    a = xl.Array.ula(4096, 100e9)
    u = xl.Users.polar((2.0, 20.0), (-75, 75))
    assert xl.gram_exact(a, xl.gen_drops(u, 16, 0)).shape == (0, 16, 16)
    pos = xl.gen_drops(u, 16, 33, seed=3)
    g1 = xl.gram_exact(a, pos)
    g2 = xl.gram_exact(a, pos)
    assert torch.equal(g1, g2)


def test_gram_cfg5_full_size_sampled(xl, orc):
    """cfg5 at full size (N = 2^20, K = 64) in the bench launch configuration; the oracle
    recomputes sampled user pairs one by one (a K=2 Gram of the pair)."""
    w = CONFIGS[5]
    ag, ao = _arr(xl, orc, "ula", w.n_y, 1, w.fc_hz)
    ug, _ = _users(xl, orc, w.r, w.az)
    pos = xl.gen_drops(ug, w.K, 4, seed=w.seed)
    G = xl.gram_exact(ag, pos).cpu().numpy()
    P = pos.cpu().numpy()
    rng = np.random.default_rng(0)
    for _ in range(3):
        d = int(rng.integers(4))
        i, j = (int(v) for v in rng.choice(w.K, 2, replace=False))
        sub = P[d:d + 1, [i, j]]
        Go = orc.gram_exact(ao, sub)[0]
        Gs = G[d][np.ix_([i, j], [i, j])]
        assert normalized_err(Gs, Go) <= 1e-9
    # properties at any size: PSD, |rho| <= 1, diag vs Eq. (4) (P1: <= 3e-11 for N >= 65536)
    lam = 299792458.0 / w.fc_hz
    for d in range(4):
        ev = np.linalg.eigvalsh(G[d])
        assert ev.min() > 0
        for i in range(w.K):
            x, y = P[d, i, 0], P[d, i, 1]
            assert abs(G[d, i, i].real / orc.power_eq4(w.n_y, lam, 1.0, x, y) - 1) < 1e-9


def test_gram_cfg5_materialised_and_fp32_full_size(xl, orc):
    """cfg5 full size: the materialised complex64 H path and the fused fp32 path vs the
    oracle on sampled pairs (1e-4 normalized, fp32 tolerance)."""
    w = CONFIGS[5]
    ag, ao = _arr(xl, orc, "ula", w.n_y, 1, w.fc_hz)
    pos = xl.gen_drops(xl.Users.polar(w.r, w.az), w.K, 2, seed=w.seed)
    P = pos.cpu().numpy()
    Gm = xl.gram_exact(ag, pos, precision=xl.FP32, mode=xl.MATERIALIZED).cpu().numpy()
    Gf = xl.gram_exact(ag, pos, precision=xl.FP32).cpu().numpy()
    for d, (i, j) in [(0, (3, 41)), (1, (0, 63)), (1, (17, 18))]:
        Go = orc.gram_exact(ao, P[d:d + 1, [i, j]])[0]
        for G in (Gm, Gf):
            assert normalized_err(G[d][np.ix_([i, j], [i, j])], Go) <= 1e-4


# --------------------------------------------------------------------------- a4
@pytest.mark.parametrize("cfg", [1, 3, 5])
def test_closed_form_parity(xl, orc, cfg):
    w = CONFIGS[cfg]
    ag, ao = _arr(xl, orc, "ula", w.n_y, 1, w.fc_hz)
    ug, _ = _users(xl, orc, w.r, w.az)
    D = min(w.n_drops, 1000)
    pos = xl.gen_drops(ug, w.K, D, seed=w.seed)
    G, fl = xl.gram_closed_form(ag, pos)
    Go, flo = orc.gram_closed_form(ao, pos.cpu().numpy())
    assert normalized_err(G.cpu().numpy(), Go) <= 1e-9
    assert np.array_equal(fl.cpu().numpy().astype(np.uint32), flo)


def test_closed_form_upa_unsupported(xl):
    a = xl.Array.upa(8, 8, 100e9)
    pos = xl.gen_drops(xl.Users.polar((2, 20), (-60, 60)), 4, 2)
    with pytest.raises(xl.XlmimoError):
        xl.gram_closed_form(a, pos)


# --------------------------------------------------------------------------- a5
@pytest.mark.parametrize("which", ["exact_cfg1", "closed_cfg1", "exact_K16", "exact_K64", "singular"])
def test_sum_rate_parity(xl, orc, which):
    allr = xl.RECV_CAP | xl.RECV_ZF | xl.RECV_MMSE | xl.RECV_MRC
    snr = [0.0, 10.0, 20.0]
    if which.endswith("cfg1"):
        w = CONFIGS[1]
        a = xl.Array.ula(w.n_y, w.fc_hz)
        pos = xl.gen_drops(xl.Users.polar(w.r, w.az), w.K, w.n_drops, seed=w.seed)
        if which.startswith("exact"):
            G = xl.gram_exact(a, pos)
            fl0 = None
        else:
            G, fl0 = xl.gram_closed_form(a, pos)   # ~40 % of drops not PD (R10)
    elif which == "singular":
        a = xl.Array.ula(64, 28e9)
        p = np.array([[[3.0, 1.0, 0.0], [3.0, 1.0, 0.0], [5.0, -2.0, 0.0]]] * 3)
        pos = torch.tensor(p, device="cuda")
        G = xl.gram_exact(a, pos)
        fl0 = None
    else:
        K = 16 if which == "exact_K16" else 64
        a = xl.Array.ula(2048, 100e9)
        pos = xl.gen_drops(xl.Users.polar((2.0, 20.0), (-75, 75)), K, 20, seed=5)
        G = xl.gram_exact(a, pos)
        fl0 = None
    Gh = G.cpu().numpy()
    rates, fl = xl.sum_rate(G, snr, allr, flags=fl0.clone() if fl0 is not None else None)
    ro, flo = orc.sum_rate(Gh, snr, allr, flags_in=fl0.cpu().numpy() if fl0 is not None else None)
    rg = rates.cpu().numpy()
    assert np.array_equal(np.isnan(rg), np.isnan(ro))
    ok = ~np.isnan(ro)
    assert np.max(np.abs(rg[ok] - ro[ok]), initial=0.0) <= 1e-6
    assert np.array_equal(fl.cpu().numpy().astype(np.uint32), flo)
    if which == "closed_cfg1":
        assert np.any(flo & 1) and np.any(flo & 8)   # the flags really fire here


# --------------------------------------------------------------------------- a1..a6 sweep
def test_sweep_parity_reduced_cfg2(xl, orc):
    """cfg2 grid, SNRs and receivers on the first 48 drops: ergodic means, counts, M_sat and
    per-drop rates vs the oracle, which computes every N independently (no shells)."""
    w = CONFIGS[2]
    D = 48
    ag = xl.Array.ula(w.n_y, w.fc_hz)
    ao = orc.array("ula", n_y=w.n_y, fc_hz=w.fc_hz)
    ug = xl.Users.polar(w.r, w.az)
    res = xl.saturation_sweep(ag, w.n_list, w.K, D, w.snr_db, w.receivers, users=ug, seed=w.seed, per_drop=True)
    pos = xl.gen_drops(ug, w.K, D, seed=w.seed).cpu().numpy()
    erg, nv, sat, pd = orc.saturation_sweep(ao, w.n_list, pos, w.snr_db, w.receivers, per_drop=True)
    assert np.max(np.abs(res["per_drop"].cpu().numpy() - pd)) <= 1e-6
    assert np.max(np.abs(res["ergodic"] - erg)) <= 1e-6
    assert np.array_equal(res["n_valid"], nv)
    assert res["sat"][2] == sat[2]
    assert np.allclose(res["sat"][[0, 1, 3]], sat[[0, 1, 3]], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("K", [24, 40])
def test_sweep_parity_many_users(xl, orc, K):
    """Nested levels on the K > 16 DMMA kernel (level ends inside tiles, ring carried
    across levels): per-drop rates vs the oracle's independent per-N Grams."""
    n_list = [96, 200, 1000, 1536, 4000]
    ag, ao = xl.Array.ula(4000, 100e9), orc.array("ula", n_y=4000, fc_hz=100e9)
    ug = xl.Users.polar((2.0, 20.0), (-60.0, 60.0))
    res = xl.saturation_sweep(ag, n_list, K, 4, [10.0], xl.RECV_CAP | xl.RECV_ZF | xl.RECV_MMSE, users=ug, seed=5,
                              per_drop=True)
    pos = xl.gen_drops(ug, K, 4, seed=5).cpu().numpy()
    _, nv, _, pd = orc.saturation_sweep(ao, n_list, pos, [10.0], xl.RECV_CAP | xl.RECV_ZF | xl.RECV_MMSE, per_drop=True)
    got = res["per_drop"].cpu().numpy()
    both = np.isfinite(pd)
    assert np.array_equal(np.isfinite(got), both) and np.array_equal(res["n_valid"], nv)
    assert np.max(np.abs(got[both] - pd[both])) <= 1e-6


def test_sweep_closed_form_parity(xl, orc):
    w = CONFIGS[2]
    D = 200
    ag = xl.Array.ula(w.n_y, w.fc_hz)
    ao = orc.array("ula", n_y=w.n_y, fc_hz=w.fc_hz)
    ug = xl.Users.polar(w.r, w.az)
    res = xl.saturation_sweep(ag, w.n_list, w.K, D, w.snr_db, 15, users=ug, seed=1, gram_kind=xl.GRAM_CLOSED_FORM,
                              per_drop=True)
    pos = xl.gen_drops(ug, w.K, D, seed=1).cpu().numpy()
    erg, nv, sat, pd, ergv = orc.saturation_sweep(ao, w.n_list, pos, w.snr_db, 15, gram_kind=1, per_drop=True,
                                                  valid_mean=True)
    g = res["per_drop"].cpu().numpy()
    assert np.array_equal(np.isnan(g), np.isnan(pd))
    ok = ~np.isnan(pd)
    assert np.max(np.abs(g[ok] - pd[ok])) <= 1e-6
    assert np.array_equal(res["n_valid"], nv)
    assert np.array_equal(np.isnan(res["ergodic"]), np.isnan(erg))          # R10: NaN iff some drop is NaN
    assert np.array_equal(np.isnan(res["ergodic"]), nv < D)
    assert np.allclose(res["ergodic"], erg, atol=1e-6, equal_nan=True)
    assert np.allclose(res["ergodic_valid"], ergv, atol=1e-6, equal_nan=True)


def test_sweep_full_cfg2_properties_and_sampled_drops(xl, orc):
    """Full cfg2 (10^4 drops, N = 2^8..2^16) in the bench configuration: capacity per drop
    non-decreasing in N, saturated at the analytic point (P8), M_sat identical to the oracle's
    per-drop Eqs. (13)-(16) on the same drops and within 1 % of the Appendix B quadrature (R15);
    sampled drops recomputed by the oracle."""
    w = CONFIGS[2]
    ag = xl.Array.ula(w.n_y, w.fc_hz)
    ug = xl.Users.polar(w.r, w.az)
    res = xl.saturation_sweep(ag, w.n_list, w.K, w.n_drops, w.snr_db, w.receivers, users=ug, seed=w.seed,
                              per_drop=True)
    pd = res["per_drop"].cpu().numpy()          # [D, nN, S, R], R = CAP, ZF, MMSE
    cap = pd[..., 0]
    assert np.all(np.diff(cap, axis=1) >= -1e-9)
    norm = res["ergodic"][:, :, 0] / res["ergodic"][-1:, :, 0]
    Ms = res["sat"][2]
    for n, N in enumerate(w.n_list):
        if N >= Ms:
            assert np.all(norm[n] >= 0.99)
        if N <= Ms / 5:
            assert np.all(norm[n] <= 0.95)
    lam = 299792458.0 / w.fc_hz
    _, _, Mq = orc.ergodic_saturation_polar(w.r[0], w.r[1], w.az[0], w.az[1], w.t, w.K, lam / 2)
    assert abs(Ms - Mq) / Mq < 0.01
    pos = xl.gen_drops(ug, w.K, w.n_drops, seed=w.seed).cpu().numpy()
    up, dn = orc.saturation_coords(pos, w.t)
    assert Ms == math.ceil((up.mean() - dn.mean()) / (lam / 2))
    idx = np.array([0, 1234, 5678, 9999])
    ao = orc.array("ula", n_y=w.n_y, fc_hz=w.fc_hz)
    _, _, _, pdo = orc.saturation_sweep(ao, w.n_list, pos[idx], w.snr_db, w.receivers, per_drop=True)
    assert np.max(np.abs(pd[idx] - pdo)) <= 1e-6
    # host-buffer entry == device entry on the same drops (bitwise)
    ph = torch.tensor(pos).pin_memory()
    rh = xl.saturation_sweep_host(ag, w.n_list, ph, w.snr_db, w.receivers)
    assert np.array_equal(rh["ergodic"], res["ergodic"]) and np.array_equal(rh["sat"], res["sat"])


def test_sweep_fp32_parity(xl, orc):
    """The fp32 sweep (fp32 phasors, fp64 accumulation) vs the fp64 oracle: rates within the
    fp32 tolerance 1e-3 bits/s/Hz (north_star)."""
    w = CONFIGS[2]
    D = 24
    ag = xl.Array.ula(w.n_y, w.fc_hz)
    ao = orc.array("ula", n_y=w.n_y, fc_hz=w.fc_hz)
    ug = xl.Users.polar(w.r, w.az)
    res = xl.saturation_sweep(ag, w.n_list, w.K, D, w.snr_db, w.receivers, users=ug, seed=3, precision=xl.FP32,
                              per_drop=True)
    pos = xl.gen_drops(ug, w.K, D, seed=3).cpu().numpy()
    _, nv, sat, pd = orc.saturation_sweep(ao, w.n_list, pos, w.snr_db, w.receivers, per_drop=True)
    assert np.max(np.abs(res["per_drop"].cpu().numpy() - pd)) <= 1e-3
    assert np.array_equal(res["n_valid"], nv) and res["sat"][2] == sat[2]


@pytest.mark.parametrize("K,N,prec,mode", [(8, 1000, "fp64", "fused"), (16, 2048, "fp64", "fused"),
                                           (33, 1500, "fp64", "fused"), (16, 4096, "fp32", "fused"),
                                           (40, 1024, "fp32", "fused"), (16, 4096, "fp32", "mat"),
                                           (5, 1001, "fp32", "mat")])
def test_determinism_all_paths(xl, K, N, prec, mode):
    """T3: identical inputs give bitwise-identical outputs on every path (fixed reduction
    orders, static work assignment in the persistent tensor-core kernels, no float atomics)."""
    a = xl.Array.ula(N, 100e9)
    pos = xl.gen_drops(xl.Users.polar((2.0, 20.0), (-60.0, 60.0)), K, 7, seed=K)
    kw = dict(precision=xl.FP64 if prec == "fp64" else xl.FP32, mode=xl.MATERIALIZED if mode == "mat" else xl.FUSED)
    g1 = xl.gram_exact(a, pos, **kw)
    g2 = xl.gram_exact(a, pos, **kw)
    assert torch.equal(g1, g2)
    r1, f1 = xl.sum_rate(g1, [0.0, 10.0], 15)
    r2, f2 = xl.sum_rate(g2, [0.0, 10.0], 15)
    assert torch.equal(r1.view(torch.int64), r2.view(torch.int64)) and torch.equal(f1, f2)


def test_launch_counter_moves(xl):
    n0 = xl.launch_count()
    xl.gen_drops(xl.Users.polar((5, 50), (-60, 60)), 4, 8)
    assert xl.launch_count() > n0


# --------------------------------------------------------------------------- NEXT-1 / NEXT-4
def test_gen_drops_rect_matches_oracle(xl, orc):
    pg = xl.gen_drops_rect((1.0, 2.0), (-7.5, 7.5), 10, 500, seed=9).cpu().numpy()
    po = orc.gen_drops_rect((1.0, 2.0), (-7.5, 7.5), 10, 500, seed=9)
    # affine map of the same 53-bit uniforms; the GPU contracts it into one FMA (1 ulp)
    assert np.max(np.abs(pg - po)) <= 2e-15 * 7.5


@pytest.mark.parametrize("K,N,fc", [(10, 256, 100e9), (10, 25000, 100e9), (4, 256, 28e9), (33, 4096, 140e9),
                                    (64, 8192, 140e9)])
def test_sum_rate_mismatched_parity(xl, orc, K, N, fc):
    """Modified-ZF effective rate (NEXT-1) on GPU exact + closed-form Grams vs the oracle on the
    same Grams: 1e-6 bits/s/Hz; NaN/flag pattern identical."""
    a = xl.Array.ula(N, fc)
    pos = xl.gen_drops_rect((1.0, 2.0), (-7.5, 7.5), K, 16, seed=K) if K == 10 else \
        xl.gen_drops(xl.Users.polar((5.0, 50.0), (-60, 60)), K, 16, seed=K)
    G = xl.gram_exact(a, pos)
    Gt, _ = xl.gram_closed_form(a, pos)
    snr = [3.51, 10.0, 30.0]
    r, fl = xl.sum_rate_mismatched(G, Gt, snr)
    ro, flo = orc.sum_rate_mismatched(G.cpu().numpy(), Gt.cpu().numpy(), snr)
    rg = r.cpu().numpy()
    assert np.array_equal(np.isnan(rg), np.isnan(ro))
    ok = ~np.isnan(ro)
    assert np.max(np.abs(rg[ok] - ro[ok]), initial=0.0) <= 1e-6
    assert np.array_equal(fl.cpu().numpy().astype(np.uint32), flo)
    # G~ = G reduces to ZF
    rz, _ = xl.sum_rate_mismatched(G, G, snr)
    zf, _ = xl.sum_rate(G, snr, xl.RECV_ZF)
    assert torch.allclose(rz, zf[..., 0], rtol=1e-10, atol=1e-10)


def test_resume_by_first_drop_equals_one_run(xl):
    """Checkpoint/resume: drops are addressed by (seed, drop index), so a sweep
    run as two batches (first_drop = 0 and D/2) and combined with the multi-rank combine
    (paper_2503_18118_b200.parallel) reproduces the one-batch sweep."""
    from paper_2503_18118_b200 import parallel
    w = CONFIGS[2]
    D = 400
    nl = [256, 512, 1024, 2048]
    arr = xl.Array.ula(2048, w.fc_hz)
    u = xl.Users.polar(w.r, w.az)
    pitch = 0.5 * 299792458.0 / w.fc_hz
    full = xl.saturation_sweep(arr, nl, w.K, D, list(w.snr_db), w.receivers,
                               pos=xl.gen_drops(u, w.K, D, seed=3))
    parts = [xl.saturation_sweep(arr, nl, w.K, D // 2, list(w.snr_db), w.receivers,
                                 pos=xl.gen_drops(u, w.K, D // 2, seed=3, first_drop=f)) for f in (0, D // 2)]
    v = sum(parallel.pack_sweep(p, D // 2, pitch) for p in parts)
    comb = parallel.unpack_sweep(v, full["ergodic"].shape, pitch)
    assert np.array_equal(comb["n_valid"], full["n_valid"])
    assert np.nanmax(np.abs(comb["ergodic"] - full["ergodic"])) <= 1e-10
    assert comb["sat"][2] == full["sat"][2]
    assert abs(comb["sat"][0] - full["sat"][0]) <= 1e-12 * abs(full["sat"][0])


@pytest.mark.slow
def test_sweep_full_cfg2_every_drop_vs_oracle(xl, orc):
    """The bench workload at full size with nothing sampled: all 10^4 cfg2 drops, all nine N
    (each N recomputed independently by the oracle, no nesting), three SNRs, CAP/ZF/MMSE:
    every per-drop rate within 1e-6 bits/s/Hz, every ergodic mean within 1e-6, the valid
    counts and M_sat identical (the oracle runs ~1 min on the GPU box's host cores)."""
    w = CONFIGS[2]
    ag = xl.Array.ula(w.n_y, w.fc_hz)
    ug = xl.Users.polar(w.r, w.az)
    res = xl.saturation_sweep(ag, w.n_list, w.K, w.n_drops, w.snr_db, w.receivers, users=ug, seed=w.seed,
                              per_drop=True)
    pos = xl.gen_drops(ug, w.K, w.n_drops, seed=w.seed).cpu().numpy()
    erg, nv, sat, pdo = orc.saturation_sweep(orc.array("ula", n_y=w.n_y, fc_hz=w.fc_hz), w.n_list, pos, w.snr_db,
                                             w.receivers, per_drop=True)
    pd = res["per_drop"].cpu().numpy()
    assert np.array_equal(np.isnan(pd), np.isnan(pdo))
    ok = ~np.isnan(pdo)
    assert np.max(np.abs(pd[ok] - pdo[ok])) <= 1e-6
    assert np.array_equal(res["n_valid"], nv)
    assert np.nanmax(np.abs(res["ergodic"] - erg)) <= 1e-6
    assert res["sat"][2] == sat[2]


def test_sweep_cfg2_closed_form_every_drop_vs_oracle(xl, orc):
    """The closed-form half of the bench step (a4: the modified-ZF Gram of Eqs. (4)/(6)/
    (22)/(23) for every N of the sweep) on all 10^4 cfg2 drops: per-drop rates within
    1e-6 bits/s/Hz, the same flagged (NaN) receivers -- far below saturation the
    closed-form Gram is indefinite (R10) -- identical valid counts, ergodic means within
    1e-6."""
    w = CONFIGS[2]
    ag = xl.Array.ula(w.n_y, w.fc_hz)
    ug = xl.Users.polar(w.r, w.az)
    pos_d = xl.gen_drops(ug, w.K, w.n_drops, seed=w.seed)
    res = xl.saturation_sweep(ag, w.n_list, w.K, w.n_drops, w.snr_db, w.receivers, pos=pos_d,
                              gram_kind=xl.GRAM_CLOSED_FORM, per_drop=True)
    erg, nv, _, pdo, ergv = orc.saturation_sweep(orc.array("ula", n_y=w.n_y, fc_hz=w.fc_hz), w.n_list,
                                                 pos_d.cpu().numpy(), w.snr_db, w.receivers, gram_kind=1,
                                                 per_drop=True, valid_mean=True)
    pd = res["per_drop"].cpu().numpy()
    assert np.array_equal(np.isnan(pd), np.isnan(pdo))
    assert np.isnan(pdo).any() and (~np.isnan(pdo)).any()
    ok = ~np.isnan(pdo)
    assert np.max(np.abs(pd[ok] - pdo[ok])) <= 1e-6
    assert np.array_equal(res["n_valid"], nv)
    assert np.array_equal(np.isnan(res["ergodic"]), np.isnan(erg))
    assert np.nanmax(np.abs(res["ergodic"] - erg)) <= 1e-6
    assert np.nanmax(np.abs(res["ergodic_valid"] - ergv)) <= 1e-6


@pytest.mark.parametrize("prec", ["fp32", "mat32"])
def test_gram_fp32_user_close_to_the_array(xl, orc, prec):
    """Users 0.3-0.6 m from a 100 GHz ULA (x well below the configs' 0.52 m minimum): the
    fp32 tensor-core generators' Taylor steps stay inside the 1e-4 tier where the phase
    curvature is largest."""
    K, N = 16, 8192
    rng = np.random.default_rng(5)
    p = np.zeros((2, K, 3))
    p[..., 0] = rng.uniform(0.3, 0.6, (2, K))
    p[..., 1] = rng.uniform(-5.0, 5.0, (2, K))
    pos = torch.tensor(p, device="cuda")
    a, ao = xl.Array.ula(N, 100e9), orc.array("ula", n_y=N, fc_hz=100e9)
    G = xl.gram_exact(a, pos, precision=xl.FP32, mode=xl.MATERIALIZED if prec == "mat32" else xl.FUSED)
    assert normalized_err(G.cpu().numpy(), orc.gram_exact(ao, p)) <= 1e-4


@pytest.mark.parametrize("K", [8, 100])
def test_empty_batches_every_entry_point(xl, K):
    """Zero drops through every per-drop entry point: empty outputs, no error, no launch
    touching memory (small and large K paths)."""
    a = xl.Array.ula(512, 28e9)
    pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, 0)
    assert pos.shape == (0, K, 3)
    G = xl.gram_exact(a, pos)
    assert G.shape == (0, K, K)
    if K <= 64:
        assert xl.gram_exact(a, pos, precision=xl.FP32, mode=xl.MATERIALIZED).shape == (0, K, K)
    Gt, fl = xl.gram_closed_form(a, pos)
    assert Gt.shape == (0, K, K) and fl.shape == (0,)
    allr = xl.RECV_CAP | xl.RECV_ZF | xl.RECV_MMSE | xl.RECV_MRC
    r, fl = xl.sum_rate(G, [0.0, 10.0], allr)
    assert r.shape == (0, 2, 4) and fl.shape == (0,)
    rs, bo, _, fa = xl.app_a_bounds(G, [0.0])
    assert rs.shape == (0, 2) and bo.shape == (0, 1, 3) and fa.shape == (0,)
    if K <= 64:
        rm, _ = xl.sum_rate_mismatched(G, Gt, [10.0])
        assert rm.shape == (0, 1)


@pytest.mark.parametrize("kind,n_y,n_z,K,D", [("ula", 256, 1, 4, 5000), ("ula", 1, 1, 3, 64), ("ula", 31, 1, 5, 64),
                                              ("ula", 999, 1, 2, 64), ("ula", 4096, 1, 4, 40), ("ula", 256, 1, 1, 64),
                                              ("upa", 37, 23, 4, 64), ("upa", 64, 64, 5, 16)])
def test_gram_warp_kernel(xl, orc, kind, n_y, n_z, K, D):
    """Kernel W (one warp per drop, small single-level arrays, K <= 5): the automatic choice at
    >= 4736 drops (cfg1 geometry) and forced by XLMIMO_OPT_GRAM_KERNEL = 5 on smaller batches,
    ragged N, N = 1, UPA; every entry vs the oracle at the fp64 tier, exactly Hermitian."""
    fc = 28e9 if kind == "ula" else 100e9
    ag, ao = _arr(xl, orc, kind, n_y, n_z, fc)
    ug, _ = _users(xl, orc, (5.0, 50.0) if kind == "ula" else (2.0, 20.0), (-60.0, 60.0),
                   (0.0, 0.0) if kind == "ula" else (-30.0, 30.0))
    pos = xl.gen_drops(ug, K, D, seed=21)
    with xl.option(xl.OPT_GRAM_KERNEL, 0 if D >= 4736 else 5):
        G = xl.gram_exact(ag, pos).cpu().numpy()
    idx = np.arange(D) if D <= 64 else np.r_[0:40, D - 40:D]
    Go = orc.gram_exact(ao, pos.cpu().numpy()[idx])
    assert normalized_err(G[idx], Go) <= 1e-9
    assert np.array_equal(G, np.conj(np.swapaxes(G, 1, 2)))
    assert np.all(np.imag(np.diagonal(G, axis1=1, axis2=2)) == 0)


@pytest.mark.parametrize("kind,n_y,n_z,K,D", [("ula", 100003, 1, 24, 600), ("upa", 40, 2500, 12, 600),
                                              ("upa", 48, 2083, 40, 300)])
def test_fused_fp32_long_chunks(xl, orc, kind, n_y, n_z, K, D):
    """The fused fp32 kernel at launch sizes that give it long work items (its adaptive chunk:
    the longest of 8K..64K elements leaving >= 4 waves, here 32K / 64K with a ragged last
    item), on 16- and 8-element tasks (UPA rows of 40 elements: TE = 8) -- every entry of
    sampled drops against the oracle at the fp32 tier (1e-4 normalised, R9)."""
    a, ao = _arr(xl, orc, kind, n_y, n_z, 100e9)
    u, _ = _users(xl, orc, (2.0, 20.0), (-60.0, 60.0), (-30.0, 30.0) if kind == "upa" else (0.0, 0.0))
    pos = xl.gen_drops(u, K, D, seed=17)
    G = xl.gram_exact(a, pos, precision=xl.FP32).cpu().numpy()
    pick = [0, D // 2, D - 1]
    Go = orc.gram_exact_blas(ao, pos.cpu().numpy()[pick])
    assert normalized_err(G[pick], Go) <= 1e-4
    for d in pick:
        assert np.array_equal(G[d], np.conj(G[d].T))


@pytest.mark.parametrize("K,N", [(24, 1501), (40, 2049), (64, 3001), (100, 1003), (120, 999), (128, 777)])
def test_mt2_ring_option_parity(xl, orc, K, N):
    """MT2's 3-deep mbarrier ring (XLMIMO_OPT_MT2_BUFFERS = 3; two buffers are the default since
    late round 2): full-length tiles where three planes fit, half-length ones above, against the
    oracle at the fp64 tier, on ragged N."""
    ag, ao = _arr(xl, orc, "ula", N, 1, 100e9)
    pos = xl.gen_drops(xl.Users.polar((1.0, 12.0), (-60.0, 60.0)), K, 3, seed=K)
    with xl.option(xl.OPT_MT2_BUFFERS, 3):
        G = xl.gram_exact(ag, pos).cpu().numpy()
    assert normalized_err(G, orc.gram_exact(ao, pos.cpu().numpy())) <= 1e-9
