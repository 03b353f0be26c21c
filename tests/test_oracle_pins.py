"""Pins of the CPU oracle to things other than itself ("Pins").

Each test names the passage it checks.  Independent references used here:
numpy's Philox bit generator, mpmath at 40 digits, numpy.linalg (LAPACK),
scipy's incomplete beta, hand 2x2 algebra, the paper's closed forms and the
worked examples in tests/golden/spec_paper_examples.json.
"""
import json
import math
import os

import mpmath as mp
import numpy as np
import pytest

from tests._util import normalized_err

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_paper_examples.json")))
C = 299792458.0


def fc_for(lam):
    return C / lam


# --------------------------------------------------------------------------- a1: RNG and drops
def test_philox_matches_numpy_bit_generator(orc):
    """R19: Philox4x64-10 (Salmon et al.) == numpy.random.Philox, whose first block is
    generated from counter+1 (numpy increments before generating)."""
    rng = np.random.default_rng(1234)
    for _ in range(20):
        ctr = rng.integers(0, 2 ** 63, size=4, dtype=np.uint64)
        ctr[0] = ctr[0] & np.uint64(0x7FFFFFFFFFFFFFF0)  # avoid carry out of word 0
        key = rng.integers(0, 2 ** 63, size=2, dtype=np.uint64)
        ref = np.random.Philox(counter=ctr, key=key).random_raw(4)
        nxt = ctr.copy()
        nxt[0] += np.uint64(1)
        assert np.array_equal(orc.philox4x64_10(nxt, key), ref)


def test_gen_drops_law_and_determinism(orc):
    """R3: r ~ U[r_min, r_max] from the array centre, az ~ U[az_min, az_max] from broadside."""
    u = orc.users(r=(3.0, 30.0), az=(-60.0, 60.0))
    p1 = orc.gen_drops(u, 8, 4000, seed=7)
    p2 = orc.gen_drops(u, 8, 4000, seed=7)
    assert np.array_equal(p1, p2)
    assert not np.array_equal(p1, orc.gen_drops(u, 8, 4000, seed=8))
    r = np.hypot(p1[..., 0], p1[..., 1])
    az = np.degrees(np.arctan2(p1[..., 1], p1[..., 0]))
    assert r.min() >= 3.0 - 1e-12 and r.max() <= 30.0 + 1e-12
    assert az.min() >= -60.0 - 1e-9 and az.max() <= 60.0 + 1e-9
    assert np.all(p1[..., 0] > 0) and np.all(p1[..., 2] == 0.0)
    n = r.size
    assert abs(r.mean() - 16.5) < 4 * (27.0 / math.sqrt(12)) / math.sqrt(n)
    assert abs(az.mean()) < 4 * (120.0 / math.sqrt(12)) / math.sqrt(n)
    # first_drop offset addresses the same stream (checkpoint / sharding property)
    assert np.array_equal(orc.gen_drops(u, 8, 100, seed=7, first_drop=1000), p1[1000:1100])


def test_gen_drops_upa_elevation_law(orc):
    """R3/R5 (UPA users of config 4): |p| = r ~ U[r_min, r_max], elevation asin(z/|p|) ~ U[el_min,
    el_max], azimuth atan2(y, x) ~ U[az_min, az_max] (x = r cos el cos az, y = r cos el sin az,
    z = r sin el), each independent.  Asymmetric ranges so a swapped sign, a swapped angle or a
    degree/radian slip moves a mean by many standard errors; a KS test for the uniform law."""
    from scipy import stats
    r_rng, az_rng, el_rng = (2.0, 20.0), (-20.0, 60.0), (-10.0, 40.0)
    p = orc.gen_drops(orc.users(r=r_rng, az=az_rng, el=el_rng), 32, 2000, seed=5)
    r = np.sqrt(np.sum(p * p, axis=-1)).ravel()
    el = np.degrees(np.arcsin(p[..., 2].ravel() / r))
    az = np.degrees(np.arctan2(p[..., 1], p[..., 0])).ravel()
    assert r.min() >= r_rng[0] * (1 - 1e-14) and r.max() <= r_rng[1] * (1 + 1e-14)
    assert el.min() >= el_rng[0] - 1e-9 and el.max() <= el_rng[1] + 1e-9
    assert az.min() >= az_rng[0] - 1e-9 and az.max() <= az_rng[1] + 1e-9
    n = r.size
    for v, (a, b) in ((r, r_rng), (el, el_rng), (az, az_rng)):
        se = (b - a) / math.sqrt(12) / math.sqrt(n)
        assert abs(v.mean() - 0.5 * (a + b)) < 4 * se
        assert stats.kstest(v, "uniform", args=(a, b - a)).pvalue > 1e-4
    # independence of the three draws (Philox words 0/1/2): correlations within 4 / sqrt(n)
    c = np.corrcoef(np.stack([r, el, az]))
    assert np.all(np.abs(c[np.triu_indices(3, 1)]) < 4 / math.sqrt(n))
    # the elevation plane: cos(el) scales the horizontal projection, x > 0 always (same side)
    assert np.all(p[..., 0] > 0)
    np.testing.assert_allclose(np.hypot(p[..., 0], p[..., 1]).ravel(), r * np.cos(np.radians(el)), rtol=1e-12)


# --------------------------------------------------------------------------- a2: geometry + channel
@pytest.mark.parametrize("ex", GOLD["element_y"])
def test_element_coordinates_spec_examples(orc, ex):
    arr = orc.array("ula", n_y=ex["M"], fc_hz=fc_for(ex["lambda"]))
    y, z = orc.element_pos(arr, ex["m"] - 1)
    assert y == pytest.approx(ex["y"], abs=1e-15) and z == 0.0


def test_element_coordinates_symmetric(orc):
    """SPEC.md:86 midpoint symmetry y(m) + y(M+1-m) = 0."""
    for M in (1, 2, 7, 256):
        arr = orc.array("ula", n_y=M)
        ys = [orc.element_pos(arr, m)[0] for m in range(M)]
        assert max(abs(a + b) for a, b in zip(ys, ys[::-1])) < 1e-15


@pytest.mark.parametrize("ex", GOLD["coef_magnitude"])
def test_coef_magnitude_spec_examples(orc, ex):
    arr = orc.array("ula", n_y=ex["M"], fc_hz=fc_for(ex["lambda"]))
    h = orc.channel_coef(arr, [ex["user"][0], ex["user"][1], 0.0], 0)
    assert abs(h) == pytest.approx(ex["abs_h"], rel=1e-14)


def _mp_coef(lam, beta0, ux, uy, uz, ey, ez, xeff):
    r = mp.sqrt(mp.mpf(ux) ** 2 + (mp.mpf(uy) - ey) ** 2 + (mp.mpf(uz) - ez) ** 2)
    return mp.sqrt(beta0) * mp.exp(-2j * mp.pi * r / lam) / r * mp.sqrt(xeff / r)


def _mp_gram(kind, n_y, n_z, fc, pos):
    """40-digit brute force of Eq. (3) and G = H^H H (P12)."""
    mp.mp.dps = 40
    lam = mp.mpf(C) / mp.mpf(fc)
    pitch = lam / 2
    K = pos.shape[0]
    els = []
    if kind == "ula":
        for m in range(n_y):
            els.append(((m + 1 - mp.mpf(n_y + 1) / 2) * pitch, mp.mpf(0)))
    else:
        for q in range(n_z):
            for p in range(n_y):
                els.append(((p + 1 - mp.mpf(n_y + 1) / 2) * pitch, (q + 1 - mp.mpf(n_z + 1) / 2) * pitch))
    H = []
    for i in range(K):
        ux, uy, uz = (mp.mpf(float(v)) for v in pos[i])
        xeff = mp.sqrt(ux ** 2 + uz ** 2) if kind == "ula" else abs(ux)
        H.append([_mp_coef(lam, 1, ux, uy, uz, ey, ez, xeff) for (ey, ez) in els])
    G = np.zeros((K, K), dtype=complex)
    for i in range(K):
        for j in range(K):
            s = mp.fsum(mp.conj(a) * b for a, b in zip(H[i], H[j]))
            G[i, j] = complex(s)
    return G, H


@pytest.mark.parametrize("kind,n_y,n_z,fc", [("ula", 64, 1, 100e9), ("ula", 33, 1, 28e9), ("upa", 6, 5, 100e9)])
def test_gram_exact_vs_mpmath(orc, kind, n_y, n_z, fc):
    """P12: oracle exact Gram (a3) equals a 40-digit brute force of Eq. (3) + H^H H
    within the fp64 phase-reduction floor (q ~ 1e4 => ~1e-12 rad)."""
    rng = np.random.default_rng(5)
    el = (-30.0, 30.0) if kind == "upa" else (0.0, 0.0)
    u = orc.users(r=(2.0, 20.0), az=(-70.0, 70.0), el=el)
    pos = orc.gen_drops(u, 4, 1, seed=int(rng.integers(1 << 30)))
    arr = orc.array(kind, n_y=n_y, n_z=n_z, fc_hz=fc)
    G = orc.gram_exact(arr, pos)[0]
    Gmp, Hmp = _mp_gram(kind, n_y, n_z, fc, pos[0])
    assert normalized_err(G, Gmp) < 2e-11
    # and the per-coefficient channel (a2)
    H = orc.channel_matrix(arr, pos[0])
    Href = np.array([[complex(v) for v in row] for row in Hmp]).T
    assert np.max(np.abs(H - Href) / np.abs(Href)) < 2e-11


def test_gram_invariants(orc):
    """P4: Hermitian, real positive diagonal, PSD, |rho_ij| <= 1."""
    u = orc.users(r=(2.0, 20.0), az=(-75.0, 75.0))
    pos = orc.gen_drops(u, 6, 5, seed=3)
    G = orc.gram_exact(orc.array("ula", n_y=512, fc_hz=100e9), pos)
    assert np.array_equal(G, np.conj(np.swapaxes(G, 1, 2)))
    d = np.real(np.diagonal(G, axis1=1, axis2=2))
    assert np.all(d > 0) and np.all(np.imag(np.diagonal(G, axis1=1, axis2=2)) == 0)
    for g in G:
        ev = np.linalg.eigvalsh(g)
        assert ev.min() >= -1e-9 * np.trace(g).real
    rho = np.abs(G) / np.sqrt(d[:, :, None] * d[:, None, :])
    assert rho.max() <= 1 + 1e-12


def test_single_element_rank_one(orc):
    """P14: N = 1 => G = h h^H (rank one) and ZF fails (flag bit 0) for K >= 2."""
    pos = orc.gen_drops(orc.users(), 3, 1, seed=1)
    G = orc.gram_exact(orc.array("ula", n_y=1), pos)
    h = orc.channel_matrix(orc.array("ula", n_y=1), pos[0])[0]
    assert np.allclose(G[0], np.outer(np.conj(h), h), rtol=1e-14, atol=0)
    rates, fl = orc.sum_rate(G, [10.0], orc.RECV_ZF | orc.RECV_MMSE)
    assert fl[0] & 1 and np.isnan(rates[0, 0, 0]) and np.isfinite(rates[0, 0, 1])


# --------------------------------------------------------------------------- Eq. (4)/(5)/(12): power
def test_diag_matches_eq4(orc):
    """P1: exact G_ii (Eq. 3 summed) vs the closed-form Eq. (4) midpoint-rule integral:
    <= 6e-6 relative for every N, <= 1e-7 once N >= 4096 and x >= 3 m."""
    cases = [(1.0, 0.0), (5.0, 2.0), (3.0, -10.0), (30.0, 0.0), (1.5, 7.0), (0.2, 0.1)]
    for fc in (28e9, 100e9, 140e9):
        for N in (16, 256, 4096, 65536):
            arr = orc.array("ula", n_y=N, fc_hz=fc)
            lam = orc.wavelength(arr)
            pos = np.array([[[x, y, 0.0] for (x, y) in cases]])
            G = orc.gram_exact(arr, pos)[0]
            for i, (x, y) in enumerate(cases):
                ref = orc.power_eq4(N, lam, 1.0, x, y)
                rel = abs(G[i, i].real - ref) / ref
                assert rel < 6e-6
                if N >= 4096 and x >= 3.0:
                    assert rel < 1e-7


@pytest.mark.parametrize("t", [0.5, 0.8, 0.9, 0.99])
@pytest.mark.parametrize("x", [1.0, 5.0, 10.0])
def test_eq4_over_eq5_is_t_at_eq12(orc, t, x):
    """P2: Eqs. (10)-(12): at y = 0 and real M = 4 x t/(lambda sqrt(1-t^2)), Eq.(4)/Eq.(5) == t."""
    lam = C / 100e9
    M = 4 * x * t / (lam * math.sqrt(1 - t * t))
    r = orc.power_eq4(M, lam, 1.0, x, 0.0) / orc.power_limit_eq5(lam, 1.0, x)
    assert r == pytest.approx(t, abs=2e-15)


def test_eq4_eq5_spec_examples(orc):
    for ex in GOLD["power_limit_eq5"]:
        assert orc.power_limit_eq5(ex["lambda"], ex["beta0"], ex["x"]) == pytest.approx(ex["value"], rel=1e-14)
    for ex in GOLD["eq4_threshold"]:
        r = orc.power_eq4(ex["M"], ex["lambda"], 1.0, ex["x"], ex["y"]) / orc.power_limit_eq5(ex["lambda"], 1.0, ex["x"])
        assert r == pytest.approx(ex["t"], abs=ex["ratio_tol"]) and r >= ex["t"]
    for ex in GOLD["eq12_threshold"]:
        M = 4 * ex["x"] * ex["t"] / (ex["lambda"] * math.sqrt(1 - ex["t"] ** 2))
        assert M == pytest.approx(ex["M_real"], abs=ex["tol"])
    # Eq. (4) -> Eq. (5) as M -> infinity and monotone in M
    lam = 0.003
    vals = [orc.power_eq4(M, lam, 1.0, 1.0, 0.3) for M in (10, 100, 1000, 10 ** 4, 10 ** 6, 10 ** 9)]
    assert all(b >= a for a, b in zip(vals, vals[1:]))
    assert vals[-1] == pytest.approx(orc.power_limit_eq5(lam, 1.0, 1.0), rel=1e-8)


# --------------------------------------------------------------------------- Eq. (6)/(8): correlation
def test_corr_eq6_vs_exact_spm_regime(orc):
    """P3 / R6: |rho_exact| and arg(rho_exact) (rho = h_i^H h_j/(|h_i||h_j|))
    agree with Eq. (6) where the stationary point u* lies well inside the array
    (|u*| <= N lambda/40) and ||x_i|-|x_j|| >= 10 lambda: <= 2.5 % / 0.02 rad at
    N = 16384, 100 GHz (1.73 % / 0.0125 rad)."""
    fc, N = 100e9, 16384
    lam = C / fc
    arr = orc.array("ula", n_y=N, fc_hz=fc)
    rng = np.random.default_rng(11)
    got = 0
    while got < 12:
        xi, xj = rng.uniform(1, 10, 2)
        yi, yj = rng.uniform(-7.5, 7.5, 2)
        if abs(xi - xj) < 10 * lam:
            continue
        ustar = yi - xi * (yj - yi) / (xj - xi)
        if abs(ustar) > N * lam / 40:
            continue
        got += 1
        pos = np.array([[[xi, yi, 0.0], [xj, yj, 0.0]]])
        G = orc.gram_exact(arr, pos)[0]
        rho = G[0, 1] / math.sqrt(G[0, 0].real * G[1, 1].real)
        ref = orc.corr_eq6(N, lam, xi, yi, xj, yj)
        assert abs(abs(rho) - abs(ref)) / abs(ref) < 0.025
        assert abs(np.angle(rho / ref)) < 0.02


def test_corr_exact_tends_to_eq8(orc):
    """P3: as N grows the exact correlation tends to the constant of Eq. (8)."""
    fc = 100e9
    lam = C / fc
    xi, yi, xj, yj = 1.0, 0.2, 2.0, 0.1
    lim = orc.corr_limit_eq8(lam, xi, yi, xj, yj)
    errs = []
    for N in (2 ** 14, 2 ** 16, 2 ** 18):
        G = orc.gram_exact(orc.array("ula", n_y=N, fc_hz=fc), np.array([[[xi, yi, 0.0], [xj, yj, 0.0]]]))[0]
        rho = G[0, 1] / math.sqrt(G[0, 0].real * G[1, 1].real)
        errs.append(abs(rho - lim) / abs(lim))
    assert errs[-1] < 2e-3 and errs[-1] < errs[0]
    # Eq. (6) itself tends to Eq. (8) as M -> infinity
    assert abs(orc.corr_eq6(1e12, lam, xi, yi, xj, yj) - lim) < 1e-8 * abs(lim)


def test_corr_spec_examples(orc):
    for ex in GOLD["corr_limit_eq8"]:
        r = orc.corr_limit_eq8(ex["lambda"], ex["ui"][0], ex["ui"][1], ex["uj"][0], ex["uj"][1])
        assert abs(r) == pytest.approx(ex["abs_rho"], rel=1e-13)
        # sgn(|x_i| - |x_j|) = sgn(-1) = -1: phase = -(2 pi d/lambda - pi/4) (SPEC.md:236 text garbled)
        d = 1.0
        ph = -(2 * math.pi * d / ex["lambda"] - math.pi / 4)
        assert abs(np.angle(r / abs(r) / complex(math.cos(ph), math.sin(ph)))) < 1e-9
    # equal radial distance => zero, sgn(0) = -1 (Eq. 7)
    assert abs(orc.corr_eq6(1000, 0.003, 2.0, 0.0, 2.0, 1.0)) == 0.0
    # swap i<->j conjugates (R6)
    a = orc.corr_eq6(5000, 0.003, 1.3, 0.2, 2.1, -0.4)
    b = orc.corr_eq6(5000, 0.003, 2.1, -0.4, 1.3, 0.2)
    assert abs(a - np.conj(b)) < 1e-9 * abs(a)


# --------------------------------------------------------------------------- a4: closed-form Gram
def test_closed_form_gram_structure(orc):
    """Eqs. (22)-(23): diag = Eq. (4); off-diag magnitude equals the
    simplified form 2 beta0 |dx| / (sqrt(lambda) d^{3/2} sqrt(x_i x_j)) (the Eq. 4 brackets
    cancel, R8) -- an algebraic identity independent of how the oracle writes Eq. (6)."""
    arr = orc.array("ula", n_y=4096, fc_hz=100e9)
    lam = orc.wavelength(arr)
    pos = orc.gen_drops(orc.users(r=(2.0, 20.0), az=(-75.0, 75.0)), 6, 3, seed=2)
    G, fl = orc.gram_closed_form(arr, pos)
    for d in range(3):
        assert np.array_equal(G[d], np.conj(G[d].T))
        for i in range(6):
            xi, yi = pos[d, i, 0], pos[d, i, 1]
            assert G[d, i, i].real == pytest.approx(orc.power_eq4(4096, lam, 1.0, xi, yi), rel=1e-15)
            for j in range(i + 1, 6):
                xj, yj = pos[d, j, 0], pos[d, j, 1]
                dx = abs(xi) - abs(xj)
                dd = math.hypot(dx, yi - yj)
                simp = 2 * abs(dx) / (math.sqrt(lam) * dd ** 1.5 * math.sqrt(xi * xj))
                assert abs(G[d, i, j]) == pytest.approx(simp, rel=1e-12)
                # phase: sgn(dx) (2 pi d/lambda - pi/4), Eq. (6)
                ph = (1 if dx > 0 else -1) * (2 * math.pi * dd / lam - math.pi / 4)
                assert abs(np.angle(G[d, i, j] / abs(G[d, i, j]) * complex(math.cos(ph), -math.sin(ph)))) < 1e-8


def test_closed_form_degenerate_and_k1(orc):
    arr = orc.array("ula", n_y=1024, fc_hz=100e9)
    lam = orc.wavelength(arr)
    pos = np.array([[[2.0, 0.0, 0.0], [2.0 + 0.5 * lam, 1.0, 0.0], [5.0, -1.0, 0.0]]])
    G, fl = orc.gram_closed_form(arr, pos)
    assert fl[0] & 8  # |dx| < lambda
    pos1 = np.array([[[3.0, 1.0, 0.0]]])
    G1, fl1 = orc.gram_closed_form(arr, pos1)
    assert fl1[0] == 0 and G1[0, 0, 0].real == orc.power_eq4(1024, lam, 1.0, 3.0, 1.0)
    # K=1 rate = log2(1 + rho Eq.4) (P5)
    r, _ = orc.sum_rate(G1, [10.0], orc.RECV_ZF)
    assert r[0, 0, 0] == pytest.approx(math.log2(1 + 10 * orc.power_eq4(1024, lam, 1.0, 3.0, 1.0)), rel=1e-14)


def test_closed_form_regime_cfg3(orc):
    """P15 (regime, not parity): at cfg3 geometry the closed form is within a few % of the exact
    Gram (median relative Frobenius ~0.6 %)."""
    arr = orc.array("ula", n_y=16384, fc_hz=100e9)
    pos = orc.gen_drops(orc.users(r=(2.0, 20.0), az=(-75.0, 75.0)), 16, 4, seed=0)
    Ge = orc.gram_exact(arr, pos)
    Gc, _ = orc.gram_closed_form(arr, pos)
    rel = [np.linalg.norm(Gc[d] - Ge[d]) / np.linalg.norm(Ge[d]) for d in range(4)]
    assert np.median(rel) < 0.03


# --------------------------------------------------------------------------- a5: receivers
def _first_principles_rates(H, rho):
    """Combiner SINRs from H itself (P7): MRC w=h_i; ZF W=(H^H H)^{-1} H^H;
    MMSE SINR_i = rho h_i^H (I + rho sum_{j!=i} h_j h_j^H)^{-1} h_i; CAP via LAPACK slogdet."""
    M, K = H.shape
    G = H.conj().T @ H
    cap = np.linalg.slogdet(np.eye(K) + rho * G)[1] / math.log(2)
    mrc = zf = mmse = 0.0
    W = np.linalg.inv(G) @ H.conj().T
    for i in range(K):
        w = H[:, i]
        sig = rho * abs(w.conj() @ H[:, i]) ** 2
        intf = rho * sum(abs(w.conj() @ H[:, j]) ** 2 for j in range(K) if j != i)
        mrc += math.log2(1 + sig / (intf + np.linalg.norm(w) ** 2))
        zf += math.log2(1 + rho / np.linalg.norm(W[i]) ** 2)
        R = np.eye(M) + rho * sum(np.outer(H[:, j], H[:, j].conj()) for j in range(K) if j != i)
        mmse += math.log2(1 + (rho * H[:, i].conj() @ np.linalg.solve(R, H[:, i])).real)
    return cap, zf, mmse, mrc


def test_receivers_vs_first_principles(orc):
    arr = orc.array("ula", n_y=48, fc_hz=28e9)
    pos = orc.gen_drops(orc.users(r=(3.0, 30.0)), 5, 3, seed=4)
    G = orc.gram_exact(arr, pos)
    allr = orc.RECV_CAP | orc.RECV_ZF | orc.RECV_MMSE | orc.RECV_MRC
    snr = [0.0, 10.0, 20.0]
    rates, fl = orc.sum_rate(G, snr, allr)
    assert np.all(fl == 0)
    for d in range(3):
        H = orc.channel_matrix(arr, pos[d])
        for s, sdb in enumerate(snr):
            ref = _first_principles_rates(H, 10 ** (sdb / 10))
            assert np.allclose(rates[d, s], ref, rtol=1e-10, atol=1e-10)


def test_receivers_k1_k2_and_diagonal(orc):
    """P5, P6: K=1 all receivers = log2(1+rho g); K=2 hand formulas; diagonal G => all equal."""
    rho = 10.0
    g = np.array([[[3.5 + 0j]]])
    r, _ = orc.sum_rate(g, [10.0], 15)
    assert np.allclose(r[0, 0], math.log2(1 + rho * 3.5), rtol=1e-15)
    a, c, b = 2.0, 3.0, 0.7 - 0.4j
    G2 = np.array([[[a, b], [np.conj(b), c]]])
    r, _ = orc.sum_rate(G2, [10.0], 15)
    det = (1 + rho * a) * (1 + rho * c) - rho ** 2 * abs(b) ** 2
    zf = math.log2(1 + rho * (a * c - abs(b) ** 2) / c) + math.log2(1 + rho * (a * c - abs(b) ** 2) / a)
    inv11 = (1 + rho * c) / det
    inv22 = (1 + rho * a) / det
    mmse = math.log2(1 / inv11) + math.log2(1 / inv22)
    mrc = math.log2(1 + rho * a * a / (a + rho * abs(b) ** 2)) + math.log2(1 + rho * c * c / (c + rho * abs(b) ** 2))
    assert np.allclose(r[0, 0], [math.log2(det), zf, mmse, mrc], rtol=1e-13)
    Gd = np.array([np.diag([1.0, 2.0, 0.5]).astype(complex)])
    r, _ = orc.sum_rate(Gd, [3.0], 15)
    assert np.ptp(r[0, 0]) < 1e-13


def test_receiver_ordering_and_flags(orc):
    """P7: CAP >= MMSE >= max(ZF, MRC); singular G => ZF NaN + flag bit 0."""
    arr = orc.array("ula", n_y=128, fc_hz=28e9)
    pos = orc.gen_drops(orc.users(r=(5.0, 50.0)), 4, 40, seed=9)
    G = orc.gram_exact(arr, pos)
    r, fl = orc.sum_rate(G, [0.0, 10.0, 30.0], 15)
    ok = np.all(np.isfinite(r), axis=(1, 2))
    rr = r[ok]
    assert np.all(rr[..., 0] >= rr[..., 2] - 1e-9)
    assert np.all(rr[..., 2] >= np.maximum(rr[..., 1], rr[..., 3]) - 1e-9)
    pos2 = np.array([[[3.0, 1.0, 0.0], [3.0, 1.0, 0.0]]])
    G2 = orc.gram_exact(arr, pos2)
    r2, fl2 = orc.sum_rate(G2, [10.0], orc.RECV_ZF | orc.RECV_CAP)
    assert fl2[0] & 1 and np.isnan(r2[0, 0, 1]) and np.isfinite(r2[0, 0, 0])
    gbad = np.array([[[np.nan, 0], [0, 1.0]]], dtype=complex)
    r3, fl3 = orc.sum_rate(gbad, [10.0], 15)
    assert fl3[0] & 16 and np.all(np.isnan(r3))


# --------------------------------------------------------------------------- a6: saturation
@pytest.mark.parametrize("ex", GOLD["multiuser_bounds"])
def test_multiuser_bounds_spec_examples(orc, ex):
    pos = np.array([[[u[0], u[1], 0.0] for u in ex["users"]]])
    up, dn = orc.saturation_coords(pos, ex["t"])
    assert up[0] == pytest.approx(ex["y_up"], abs=ex["tol"])
    assert dn[0] == pytest.approx(ex["y_down"], abs=ex["tol"])
    # translation equivariance y -> y + 5
    pos[..., 1] += 5.0
    up2, dn2 = orc.saturation_coords(pos, ex["t"])
    assert up2[0] - up[0] == pytest.approx(5.0, abs=1e-12) and dn2[0] - dn[0] == pytest.approx(5.0, abs=1e-12)


def _eq17_paper(x_min, x_max, y_min, y_max, t, K):
    """Eq. (17) with the undefined '(2N+1)' read as (2K+1) (R16) and
    B(x; a, b) the non-regularised incomplete beta (R17) = betainc * beta."""
    from scipy.special import beta, betainc
    s = t / math.sqrt(1 - t * t)
    L1 = x_min * s + y_min
    R1 = min(x_min * s + y_max, x_max * s + y_min)
    L2 = max(x_min * s + y_max, x_max * s + y_min)
    R2 = x_max * s + y_max
    a = (L2 - 2 * R1 + R2) / (2 * (R2 - R1))
    b = (R1 - L1) / (2 * (R2 - R1))
    xb = (R1 - L1) / (2 * (R2 - R1))
    B = betainc(1.5, K, xb) * beta(1.5, K)
    return (R2 - a ** K * (L2 - 2 * R1 + R2) / (2 * (K + 1)) - a ** K * (R1 - L1)
            - b ** K * (R1 - L1) / (2 * (K + 1) * (2 * K + 1))
            - math.sqrt(2) * K * math.sqrt((R1 - L1) * (R2 - R1)) * B)


@pytest.mark.parametrize("rect", [(1.0, 10.0, -7.5, 7.5), (1.0, 2.0, -7.5, 7.5)])
@pytest.mark.parametrize("K", [1, 2, 10, 100, 1000])
def test_appendix_b_quadrature_equals_eq17(orc, rect, K):
    """P9: the Appendix B pipeline (oracle quadrature of F_z^K) equals Eq. (17) with (2K+1)."""
    q = orc.ergodic_y_up_rect(*rect, 0.9, K)
    assert q == pytest.approx(_eq17_paper(*rect, 0.9, K), abs=1e-9)
    # Eq. (18): E[y_up] + E[y_down] = y_min + y_max
    assert q + orc.ergodic_y_down_rect(*rect, 0.9, K) == pytest.approx(rect[2] + rect[3], abs=1e-12)


def test_appendix_b_limits_and_paper_numbers(orc):
    """Eqs. (19)-(20): K -> inf gives the corner points; P10: the E2 setting saturates
    'around 10^4 antennas'; K_list monotone."""
    s = orc.slope(0.9)
    R2 = 10 * s + 7.5
    assert orc.ergodic_y_up_rect(1, 10, -7.5, 7.5, 0.9, 10 ** 4) == pytest.approx(R2, rel=0.01)
    vals = [orc.ergodic_y_up_rect(1, 10, -7.5, 7.5, 0.9, K) for K in (1, 2, 5, 10, 100, 1000)]
    assert all(b >= a for a, b in zip(vals, vals[1:])) and vals[-1] <= R2
    # K = 1: mean of z = s (x_min+x_max)/2 + (y_min+y_max)/2
    assert vals[0] == pytest.approx(s * 5.5, abs=1e-9)
    lam = C / 100e9
    e2 = GOLD["paper_settings"]["E2_capacity_vs_ant"]
    up = orc.ergodic_y_up_rect(*e2["x"], *e2["y"], 0.9, e2["K"])
    dn = orc.ergodic_y_down_rect(*e2["x"], *e2["y"], 0.9, e2["K"])
    M = math.ceil((up - dn) / (lam / 2))
    assert 0.5 * e2["M_sat_order"] < M < 2 * e2["M_sat_order"]
    # App. C envelope dominates the beta term
    from scipy.special import beta, betainc
    L1, R1, L2, R2b = orc.trapezoid_breakpoints(1, 10, -7.5, 7.5, 0.9)
    for K in (2, 10, 100, 1000):
        xb = (R1 - L1) / (2 * (R2b - R1))
        term = math.sqrt(2) * K * math.sqrt((R1 - L1) * (R2b - R1)) * betainc(1.5, K, xb) * beta(1.5, K)
        env = math.sqrt(2) * math.sqrt((R1 - L1) * (R2b - R1)) * math.gamma(1.5) * K ** -0.5
        assert term <= env * 1.05  # '~' asymptotic, Gamma(b)/Gamma(a+b) ~ b^-a


def test_hexagonal_packing_numbers():
    """P11: App. A arithmetic."""
    ex = GOLD["hexagonal_packing"][0]
    dens = 2 / (math.sqrt(3) * ex["d"] ** 2)
    assert dens == pytest.approx(ex["density"], abs=5e-4)
    assert round(ex["area_m2"] * dens) == ex["cap"]


def test_polar_saturation_quadrature_vs_monte_carlo(orc):
    """R15: the oracle's polar-law Appendix B quadrature agrees with the Monte Carlo mean of
    the per-drop Eqs. (13)-(16) (oracle drops) within 4 standard errors, cfg2 law."""
    u = orc.users(r=(3.0, 30.0), az=(-60.0, 60.0))
    pos = orc.gen_drops(u, 8, 20000, seed=123)
    up, dn = orc.saturation_coords(pos, 0.9)
    lam = C / 28e9
    Eup, Edn, M = orc.ergodic_saturation_polar(3.0, 30.0, -60.0, 60.0, 0.9, 8, lam / 2)
    assert abs(up.mean() - Eup) < 4 * up.std() / math.sqrt(up.size)
    assert abs(dn.mean() - Edn) < 4 * dn.std() / math.sqrt(dn.size)
    assert M == pytest.approx(20383, rel=0.01)


def test_capacity_saturates_in_n(orc):
    """P8 (north_star): per-drop capacity is non-decreasing in N for nested centred arrays and
    levels off at the analytic saturation point (cfg2 geometry; fewer drops)."""
    w_nl = [2 ** k for k in range(8, 17)]
    arr = orc.array("ula", n_y=65536, fc_hz=28e9)
    pos = orc.gen_drops(orc.users(r=(3.0, 30.0)), 8, 12, seed=0)
    erg, nv, sat, pd = orc.saturation_sweep(arr, w_nl, pos, [0.0, 10.0, 20.0], orc.RECV_CAP, per_drop=True)
    cap = pd[..., 0]                                 # (D, nN, S)
    assert np.all(np.diff(cap, axis=1) >= -1e-9)
    norm = erg[:, :, 0] / erg[-1:, :, 0]             # (nN, S)
    msat = 20383
    for n, N in enumerate(w_nl):
        if N >= msat:
            assert np.all(norm[n] >= 0.99)
        if N <= msat / 5:
            assert np.all(norm[n] <= 0.95)
    # faster convergence at higher SNR
    assert norm[4, 2] >= norm[4, 0]
    assert sat[2] == math.ceil((sat[0] - sat[1]) / (C / 28e9 / 2))


def test_sweep_statistics_with_invalid_drops(orc):
    """R10 / PAPER.md:177-178, 228: the sweep's reductions, pinned against numpy on its own
    per-drop table.  cfg1 geometry through the closed-form Gram (SURVEY.md:582 Q10: ~39 % of
    the drops have an indefinite G~ at N = 256, so their ZF rate is NaN):
      n_valid       = the count of non-NaN per-drop rates in each (N, SNR, receiver) column;
      ergodic       = the plain mean over ALL drops when the column has no NaN, else NaN
                      (an expectation over a subset of the drops is not the ergodic value);
      ergodic_valid = the mean over the non-NaN drops (conditional mean);
      sat[0], sat[1]= E[y_up], E[y_down]: means over drops of the per-drop Eqs. (13)-(16),
                      here re-derived geometrically -- y_up_i is the element coordinate seen
                      from user i at sin(angle) = t, (y_up_i - y_i)/hypot(x_i, y_up_i - y_i) = t;
      sat[2]        = ceil((E[y_up] - E[y_down]) / pitch)  (M_sat);
      sat[3]        = std(extent/pitch, ddof=1)/sqrt(D), extent = y_up - y_down per drop."""
    lam = C / 28e9
    pitch = lam / 2
    t = 0.9
    D = 300
    pos = orc.gen_drops(orc.users(r=(5.0, 50.0), az=(-60.0, 60.0)), 4, D, seed=3)
    nl = [64, 128, 256]
    rec = orc.RECV_CAP | orc.RECV_ZF | orc.RECV_MMSE
    arr = orc.array("ula", n_y=256, fc_hz=28e9)
    erg, nv, sat, pd, ergv = orc.saturation_sweep(arr, nl, pos, [0.0, 10.0], rec, gram_kind=1, t=t,
                                                  per_drop=True, valid_mean=True)
    assert pd.shape == (D, 3, 2, 3)
    ok = ~np.isnan(pd)
    np.testing.assert_array_equal(nv, ok.sum(axis=0))
    assert np.any(nv < D)                              # NaN drops are exercised (full columns below)
    with np.errstate(invalid="ignore"):
        np.testing.assert_allclose(ergv, np.nanmean(pd, axis=0), rtol=1e-13, atol=0)
    full = nv == D
    np.testing.assert_allclose(erg[full], pd.mean(axis=0)[full], rtol=1e-13, atol=0)
    assert np.all(np.isnan(erg[~full]))
    # the same per-drop table with the exact Gram has no NaN: ergodic == ergodic_valid == mean
    erg_x, nv_x, sat_x, pd_x, ergv_x = orc.saturation_sweep(arr, nl, pos[:40], [10.0], rec, t=t, per_drop=True,
                                                            valid_mean=True)
    assert np.all(nv_x == 40)
    np.testing.assert_allclose(erg_x, pd_x.mean(axis=0), rtol=1e-13)
    np.testing.assert_array_equal(erg_x, ergv_x)
    # saturation statistics from the geometry
    x = np.hypot(pos[..., 0], pos[..., 2])
    y = pos[..., 1]
    off = x * t / math.sqrt(1 - t * t)
    up_i, dn_i = y + off, y - off
    np.testing.assert_allclose((up_i - y) / np.hypot(x, up_i - y), t, rtol=1e-12)
    np.testing.assert_allclose((y - dn_i) / np.hypot(x, y - dn_i), t, rtol=1e-12)
    up, dn = up_i.max(axis=1), dn_i.min(axis=1)
    ext = (up - dn) / pitch
    assert sat[0] == pytest.approx(up.mean(), rel=1e-13)
    assert sat[1] == pytest.approx(dn.mean(), rel=1e-13)
    assert sat[2] == math.ceil((up.mean() - dn.mean()) / pitch)
    assert sat[3] == pytest.approx(np.std(ext, ddof=1) / math.sqrt(D), rel=1e-9)
    # sat is geometry only: the exact sweep on the first 40 drops gives their own M_sat
    assert sat_x[2] == math.ceil((up[:40].mean() - dn[:40].mean()) / pitch)


def test_upa_diagonal_solid_angle(orc):
    """P17 / R5: UPA diagonal = (4 beta0/lambda^2) * solid angle of the array rectangle."""
    fc = 100e9
    lam = C / fc
    for (ny, nz) in [(64, 64), (128, 32)]:
        arr = orc.array("upa", n_y=ny, n_z=nz, fc_hz=fc)
        pos = orc.gen_drops(orc.users(r=(2.0, 20.0), az=(-60, 60), el=(-30, 30)), 3, 1, seed=ny)
        G = orc.gram_exact(arr, pos)[0]
        for i in range(3):
            x, y, z = pos[0, i]
            Y, Z = ny * lam / 4, nz * lam / 4
            om = 0.0
            for sy, yc in ((1, Y), (-1, -Y)):
                for sz, zc in ((1, Z), (-1, -Z)):
                    u, v = yc - y, zc - z
                    om += sy * sz * math.atan(u * v / (x * math.sqrt(x * x + u * u + v * v)))
            assert G[i, i].real == pytest.approx(4 / lam ** 2 * om, rel=1e-5)


def test_upa_reduces_to_ula_and_rotates(orc):
    """R5 pins of the UPA off-diagonal (beyond the tiny-array mpmath check): a UPA with one
    row (n_z = 1) IS the centred ULA of PAPER.md:52 for users in the z = 0 plane (same
    element coordinates, x_eff = |x|); a single column (n_y = 1) is the same ULA along z,
    so users mirrored (y, z) -> (z, y) see the identical Gram; and the 180-degree rotation
    (y, z) -> (-y, -z) of the users about the array axis maps the centred grid onto itself,
    leaving G unchanged.  The ULA path is pinned independently (mpmath, Eq. (4))."""
    fc = 100e9
    pos = orc.gen_drops(orc.users(r=(2.0, 20.0), az=(-60, 60)), 5, 3, seed=31)   # z = 0
    G_upa = orc.gram_exact(orc.array("upa", n_y=300, n_z=1, fc_hz=fc), pos)
    G_ula = orc.gram_exact(orc.array("ula", n_y=300, fc_hz=fc), pos)
    assert normalized_err(G_upa, G_ula) < 1e-13
    pz = orc.gen_drops(orc.users(r=(2.0, 20.0), az=(-60, 60), el=(-30, 30)), 5, 3, seed=32)
    swapped = pz[..., [0, 2, 1]].copy()
    G_col = orc.gram_exact(orc.array("upa", n_y=1, n_z=257, fc_hz=fc), pz)
    G_row = orc.gram_exact(orc.array("upa", n_y=257, n_z=1, fc_hz=fc), swapped)
    # (the distance sums dy^2 + dz^2 in the other order: 1-ulp r, the fp64 phase floor)
    assert normalized_err(G_col, G_row) < 1e-11
    arr = orc.array("upa", n_y=20, n_z=13, fc_hz=fc)
    rot = pz.copy()
    rot[..., 1:] *= -1.0
    assert normalized_err(orc.gram_exact(arr, rot), orc.gram_exact(arr, pz)) < 1e-11


# --------------------------------------------------------------------------- NEXT-1 / NEXT-4
def _first_principles_mismatched(H, Gt, rho):
    """W = G~^{-1} H^H applied to the true H (numpy/LAPACK inverse): T = W H, noise W W^H / rho."""
    W = np.linalg.inv(Gt) @ H.conj().T
    T = W @ H
    c = 0.0
    for i in range(T.shape[0]):
        sig = abs(T[i, i]) ** 2
        intf = sum(abs(T[i, j]) ** 2 for j in range(T.shape[0]) if j != i)
        c += math.log2(1 + sig / (intf + np.linalg.norm(W[i]) ** 2 / rho))
    return c


def test_mismatched_rate_first_principles_and_zf_limit(orc):
    """NEXT-1 (R11): the modified-ZF effective rate equals the first-principles SINR of
    W = G~^{-1} H^H on H; with G~ = G it is exactly the ZF rate (A = I)."""
    arr = orc.array("ula", n_y=40, fc_hz=100e9)
    lam = orc.wavelength(arr)
    pos = orc.gen_drops_rect((1.0, 2.0), (-7.5, 7.5), 5, 3, seed=8)
    G = orc.gram_exact(arr, pos)
    Gt, _ = orc.gram_closed_form(arr, pos)
    snr = [0.0, 10.0, 30.0]
    r, fl = orc.sum_rate_mismatched(G, Gt, snr)
    for d in range(3):
        H = orc.channel_matrix(arr, pos[d])
        for s, sdb in enumerate(snr):
            assert r[d, s] == pytest.approx(_first_principles_mismatched(H, Gt[d], 10 ** (sdb / 10)), rel=1e-9)
    rz, _ = orc.sum_rate_mismatched(G, G, snr)
    zf, _ = orc.sum_rate(G, snr, orc.RECV_ZF)
    assert np.allclose(rz, zf[..., 0], rtol=1e-11)
    # singular model Gram -> NaN + flag bit 5
    Gs = Gt.copy()
    Gs[0] = 0.0
    rs, fls = orc.sum_rate_mismatched(G, Gs, snr)
    assert np.all(np.isnan(rs[0])) and fls[0] & 32 and np.all(np.isfinite(rs[1:]))


def test_modified_zf_worse_below_saturation_equal_after(orc):
    """PAPER.md:273-275 (E2 setting: K = 10, x ~ U(1,2), y ~ U[-7.5,7.5] m, 100 GHz, transmit
    SNR set for a 33 dB limit at (1.5 m, 0)): the modified ZF is worse than ZF well below the
    saturation point and reaches it beyond."""
    lam = C / 100e9
    rho_db = 10 * math.log10(10 ** 3.3 * lam * 1.5 / 4)  # P * 4 beta0/(lambda x) / sigma^2 = 33 dB at x = 1.5 (Eq. 5)
    pos = orc.gen_drops_rect((1.0, 2.0), (-7.5, 7.5), 10, 4, seed=2)
    out = {}
    for N in (256, 25000):
        arr = orc.array("ula", n_y=N, fc_hz=100e9)
        G = orc.gram_exact(arr, pos)
        Gt, _ = orc.gram_closed_form(arr, pos)
        zf, _ = orc.sum_rate(G, [rho_db], orc.RECV_ZF)
        mz, _ = orc.sum_rate_mismatched(G, Gt, [rho_db])
        out[N] = (zf[:, 0, 0], mz[:, 0])
    zf, mz = out[256]
    assert np.all(mz < zf)                                  # "worse performance ... at the beginning"
    zf, mz = out[25000]
    assert np.all(np.abs(mz - zf) / zf < 0.01)              # same capacity after the saturation point


def test_rect_drops_law(orc):
    pos = orc.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), 8, 5000, seed=4)
    assert pos[..., 0].min() >= 1.0 and pos[..., 0].max() <= 10.0 and np.all(pos[..., 2] == 0)
    assert abs(pos[..., 0].mean() - 5.5) < 4 * 9 / math.sqrt(12) / math.sqrt(pos[..., 0].size)
    assert abs(pos[..., 1].mean()) < 4 * 15 / math.sqrt(12) / math.sqrt(pos[..., 1].size)
    assert np.array_equal(orc.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), 8, 10, seed=4, first_drop=7), pos[7:17])


# --------------------------------------------------------------------------- NEXT-3: Appendix A
def _app_a_grams(orc):
    """Exact Grams of the paper's E1/E3 user field, 100 GHz, a few K and M."""
    out = []
    for K, M, seed in [(3, 512, 1), (8, 4096, 2), (16, 2048, 3), (5, 64, 4)]:
        pos = orc.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, 6, seed=seed)
        out.append(orc.gram_exact(orc.array("ula", n_y=M, fc_hz=100e9), pos))
    return out


def test_gram_exact_blas_equals_compensated_loops(orc):
    """The large-K oracle Gram (library matmul of the Eq. (3) H) is the same definition
    as the Neumaier loops."""
    a = orc.array("ula", n_y=700, fc_hz=100e9)
    pos = orc.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), 12, 3, seed=5)
    assert normalized_err(orc.gram_exact_blas(a, pos), orc.gram_exact(a, pos)) < 1e-14


def test_app_a_bounds_bracket_capacity(orc):
    """Hadamard U >= det(I + rho G) >= det(R) prod(1 + a_i) = L, for
    every drop and received SNR (the paper's range 0..30 dB and beyond)."""
    snr = [-10.0, 0.0, 10.0, 30.0, 60.0]
    for G in _app_a_grams(orc):
        rs, bo, _, fl = orc.bounds_app_a(G, snr)
        assert np.all(fl == 0)
        lu, cap, ll = bo[..., 0], bo[..., 1], bo[..., 2]
        assert np.all(lu >= cap - 1e-12) and np.all(cap >= ll - 1e-12)
        # log2 L - log2 U = log2 det R <= 0 (Hadamard on R)
        assert np.all(rs[:, 0] <= 1e-14)


def test_app_a_against_lapack_and_determinant_identity(orc):
    """Each output against numpy.linalg (LAPACK): log2 U from the diagonal, C by slogdet,
    log2 det R by slogdet of D^{-1/2} G D^{-1/2}, and the decomposition of PAPER.md:300-305,
    det(rho G) = det(P) det(R) with P = Diag(a_i)."""
    snr = [0.0, 20.0]
    for G in _app_a_grams(orc):
        rs, bo, _, _ = orc.bounds_app_a(G, snr)
        K = G.shape[1]
        for d in range(G.shape[0]):
            g = G[d]
            dg = np.real(np.diag(g))
            R = g / np.sqrt(np.outer(dg, dg))
            ldr = np.linalg.slogdet(R)[1] / math.log(2)
            assert abs(rs[d, 0] - ldr) < 1e-10 * max(1.0, abs(ldr))
            assert abs(rs[d, 1] + ldr / K) < 1e-10
            for s, sdb in enumerate(snr):
                rho = 10 ** (sdb / 10)
                cap = np.linalg.slogdet(np.eye(K) + rho * g)[1] / math.log(2)
                lu = np.sum(np.log2(1 + rho * dg))
                assert abs(bo[d, s, 0] - lu) < 1e-12 * lu
                assert abs(bo[d, s, 1] - cap) < 1e-10 * cap
                assert abs(bo[d, s, 2] - (ldr + lu)) < 1e-10 * lu
                ldp = np.linalg.slogdet(rho * g)[1] / math.log(2)
                assert abs(ldp - (np.sum(np.log2(rho * dg)) + rs[d, 0])) < 1e-9 * abs(ldp)


def test_app_a_two_users_and_subset_expansion(orc):
    """K = 2 by hand: det R = 1 - |r_12|^2, U = (1+a1)(1+a2), L = (1-|r|^2)(1+a1)(1+a2),
    C = 1 + a1 + a2 + a1 a2 (1 - |r|^2).  K = 3: det(I + P^1/2 R P^1/2) is the sum over
    subsets S of prod_{i in S} a_i det R_S (principal minors), so C >= L term by term."""
    a = orc.array("ula", n_y=300, fc_hz=100e9)
    pos = orc.gen_drops_rect((1.0, 3.0), (-1.0, 1.0), 2, 10, seed=11)
    G = orc.gram_exact(a, pos)
    rs, bo, _, _ = orc.bounds_app_a(G, [3.0])
    rho = 10 ** 0.3
    for d in range(10):
        a1, a2 = rho * G[d, 0, 0].real, rho * G[d, 1, 1].real
        r2 = abs(G[d, 0, 1]) ** 2 / (G[d, 0, 0].real * G[d, 1, 1].real)
        assert abs(2 ** rs[d, 0] - (1 - r2)) < 1e-12
        assert abs(2 ** bo[d, 0, 0] - (1 + a1) * (1 + a2)) < 1e-12 * (1 + a1) * (1 + a2)
        assert abs(2 ** bo[d, 0, 1] - (1 + a1 + a2 + a1 * a2 * (1 - r2))) < 1e-11 * (1 + a1) * (1 + a2)
        assert abs(2 ** bo[d, 0, 2] - (1 - r2) * (1 + a1) * (1 + a2)) < 1e-11 * (1 + a1) * (1 + a2)
    pos3 = orc.gen_drops_rect((1.0, 3.0), (-1.0, 1.0), 3, 5, seed=12)
    G3 = orc.gram_exact(a, pos3)
    _, bo3, _, _ = orc.bounds_app_a(G3, [0.0])
    import itertools
    for d in range(5):
        dg = G3[d].diagonal().real
        R = G3[d] / np.sqrt(np.outer(dg, dg))
        tot = 0.0
        for n in range(4):
            for S in itertools.combinations(range(3), n):
                minor = np.linalg.det(R[np.ix_(S, S)]).real if S else 1.0
                tot += np.prod(dg[list(S)]) * minor
        assert abs(2 ** bo3[d, 0, 1] - tot) < 1e-11 * tot


def test_app_a_eigenvalues_jacobi(orc):
    """-E_K[log2 lambda^R]: the Jacobi eigenvalues of R equal LAPACK's
    eigvalsh, sum to tr R = K, and their mean log2 is minus the gap (from Cholesky)."""
    for G in _app_a_grams(orc):
        rs, _, ev, _ = orc.bounds_app_a(G, [0.0], eig=True)
        dg = np.real(np.diagonal(G, axis1=1, axis2=2))
        R = G / np.sqrt(dg[:, :, None] * dg[:, None, :])
        K = G.shape[1]
        assert np.max(np.abs(ev - np.linalg.eigvalsh(R))) < 1e-12
        assert np.max(np.abs(ev.sum(1) - K)) < 1e-12 * K
        assert np.max(np.abs(-np.mean(np.log2(ev), axis=1) - rs[:, 1])) < 1e-12
        assert np.all(np.diff(ev, axis=1) >= 0)


def test_app_a_diagonal_gram_and_flags(orc):
    """Orthogonal users (diagonal G): R = I, det R = 1, gap 0, L = U = C.  A zero
    diagonal or non-finite entry gives NaN + flag; an indefinite G flags bit 0."""
    G = np.zeros((3, 4, 4), complex)
    G[0] = np.diag([1.0, 2.0, 3.0, 4.0])
    G[1] = np.diag([1.0, 0.0, 3.0, 4.0])
    G[2] = np.diag([1.0, 2.0, np.inf, 4.0])
    rs, bo, ev, fl = orc.bounds_app_a(G, [10.0], eig=True)
    assert rs[0, 0] == 0.0 and rs[0, 1] == 0.0 and np.allclose(ev[0], 1.0)
    assert abs(bo[0, 0, 0] - bo[0, 0, 1]) < 1e-13 and bo[0, 0, 2] == bo[0, 0, 0]
    assert fl[1] == 4 and np.all(np.isnan(bo[1])) and fl[2] == 16 and np.all(np.isnan(rs[2]))
    Gi = np.array([[[1.0, 2.0], [2.0, 1.0]]], complex)  # |r| = 2: not a correlation matrix
    rs, bo, _, fl = orc.bounds_app_a(Gi, [0.0])
    assert fl[0] & 1 and np.isnan(rs[0, 0]) and np.isnan(bo[0, 0, 2]) and np.isfinite(bo[0, 0, 0])


def test_app_a_paper_gap_k1000(orc):
    """PAPER.md:331-335 (Fig. K_vs_E): with the Sec. IV-C user field (x ~ U[1, 10] m,
    y ~ U[-7.5, 7.5] m, 100 GHz) the negative empirical expectation
    -E_K[log2 lambda^R] grows with K and reaches 0.064 at K = 1000.  Array: M = 35 000
    elements (the E1 ergodic saturation size; the paper does not state M).
    One drop at K = 1000 (the mean over 1000 eigenvalues is already self-averaging)."""
    a = orc.array("ula", n_y=35000, fc_hz=100e9)
    gaps = {}
    for K, D in [(10, 4), (100, 4), (1000, 1)]:
        pos = orc.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, D, seed=0)
        rs, _, _, fl = orc.bounds_app_a(orc.gram_exact_blas(a, pos), [0.0])
        assert np.all(fl == 0)
        gaps[K] = float(np.mean(rs[:, 1]))
    assert gaps[10] < gaps[100] < gaps[1000]
    assert abs(gaps[1000] - 0.064) < 1.0e-3, gaps
