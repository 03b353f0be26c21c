"""Full-size parity on every config, entry by entry (north_star: "match the CPU oracle
within the stated tolerances on every config").

Each config is run at its own array size and user count, in the launch configuration
bench.py times, and compared with the oracle on EVERY Gram entry of the drops checked:
  cfg4  UPA 256 x 256 (N = 65 536), K = 32, 16 drops: fused fp64 (DMMA), fused fp32
        (tcgen05), materialised complex64 H (TMA -> tcgen05);
  cfg5  ULA N = 2^20, K = 64, 4 drops: the same three paths, the oracle's Gram from its
        own Eq. (3) H and one library matmul (gram_exact_blas, pinned equal to the
        compensated loops in tests/test_oracle_pins.py);
and the fp32-tier per-drop rates (1e-3 bits/s/Hz against the oracle's fp64 rates)
through the tensor-core fp32 Grams on cfg3 (the sweep entry at fp32, 1000 drops, MMSE),
cfg4 (ZF + MMSE) and cfg5 (CAP + ZF + MMSE).
Tolerances: Gram |dG_ij|/sqrt(G_ii G_jj) <= 1e-9 (fp64) / 1e-4 (fp32) (R9); rates 1e-6
(fp64) / 1e-3 (fp32); flags identical.
"""
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


def _hermitian(G):
    assert np.array_equal(G, np.conj(np.swapaxes(G, 1, 2)))
    assert np.all(np.imag(np.diagonal(G, axis1=1, axis2=2)) == 0)


# --------------------------------------------------------------------------- cfg4
@pytest.fixture(scope="module")
def cfg4(xl, orc):
    w = CONFIGS[4]
    ag = xl.Array.upa(w.n_y, w.n_z, w.fc_hz)
    ao = orc.array("upa", n_y=w.n_y, n_z=w.n_z, fc_hz=w.fc_hz)
    pos = xl.gen_drops(xl.Users.polar(w.r, w.az, w.el), w.K, 16, seed=w.seed)
    Go = orc.gram_exact(ao, pos.cpu().numpy())
    return w, ag, pos, Go


@pytest.mark.parametrize("prec", ["fp64", "fp32", "mat32"])
def test_cfg4_full_size_every_entry(xl, cfg4, prec):
    w, ag, pos, Go = cfg4
    G = xl.gram_exact(ag, pos, precision=xl.FP64 if prec == "fp64" else xl.FP32,
                      mode=xl.MATERIALIZED if prec == "mat32" else xl.FUSED).cpu().numpy()
    assert G.shape == (16, 32, 32)
    assert normalized_err(G, Go) <= (1e-9 if prec == "fp64" else 1e-4)
    _hermitian(G)


@pytest.mark.parametrize("prec", ["fp64", "fp32", "mat32"])
def test_cfg4_rates_every_drop(xl, orc, cfg4, prec):
    """cfg4's receivers (ZF + MMSE at 10 dB) on the three Gram paths vs the oracle's fp64
    rates on its own Gram: 1e-6 bit (fp64) / 1e-3 bit (fp32 tier)."""
    w, ag, pos, Go = cfg4
    G = xl.gram_exact(ag, pos, precision=xl.FP64 if prec == "fp64" else xl.FP32,
                      mode=xl.MATERIALIZED if prec == "mat32" else xl.FUSED)
    r, fl = xl.sum_rate(G, w.snr_db, w.receivers)
    ro, flo = orc.sum_rate(Go, w.snr_db, w.receivers)
    assert np.array_equal(fl.cpu().numpy().astype(np.uint32), flo)
    assert np.max(np.abs(r.cpu().numpy() - ro)) <= (1e-6 if prec == "fp64" else 1e-3)


# --------------------------------------------------------------------------- cfg5
@pytest.fixture(scope="module")
def cfg5(xl, orc):
    w = CONFIGS[5]
    ag = xl.Array.ula(w.n_y, w.fc_hz)
    ao = orc.array("ula", n_y=w.n_y, fc_hz=w.fc_hz)
    pos = xl.gen_drops(xl.Users.polar(w.r, w.az), w.K, 4, seed=w.seed)
    Go = orc.gram_exact_blas(ao, pos.cpu().numpy())
    return w, ag, pos, Go


@pytest.mark.parametrize("prec", ["fp64", "fp32", "mat32"])
def test_cfg5_full_size_every_entry(xl, cfg5, prec):
    w, ag, pos, Go = cfg5
    G = xl.gram_exact(ag, pos, precision=xl.FP64 if prec == "fp64" else xl.FP32,
                      mode=xl.MATERIALIZED if prec == "mat32" else xl.FUSED).cpu().numpy()
    assert G.shape == (4, 64, 64)
    assert normalized_err(G, Go) <= (1e-9 if prec == "fp64" else 1e-4)
    _hermitian(G)


@pytest.mark.parametrize("prec", ["fp64", "fp32", "mat32"])
def test_cfg5_rates_every_drop(xl, orc, cfg5, prec):
    """cfg5's receivers (CAP + ZF + MMSE at 10 dB) through each Gram path vs the oracle."""
    w, ag, pos, Go = cfg5
    G = xl.gram_exact(ag, pos, precision=xl.FP64 if prec == "fp64" else xl.FP32,
                      mode=xl.MATERIALIZED if prec == "mat32" else xl.FUSED)
    r, fl = xl.sum_rate(G, w.snr_db, w.receivers)
    ro, flo = orc.sum_rate(Go, w.snr_db, w.receivers)
    assert np.array_equal(fl.cpu().numpy().astype(np.uint32), flo)
    assert np.max(np.abs(r.cpu().numpy() - ro)) <= (1e-6 if prec == "fp64" else 1e-3)


# --------------------------------------------------------------------------- cfg3 fp32 tier
def test_cfg3_fp32_sweep_rates_every_drop(xl, orc):
    """cfg3 ("MMSE ... exact fp64 and fp32 Gram") at its full array size, 1000 drops, through
    the sweep entry at fp32 (the fused TF32 tcgen05 Gram, one level): every per-drop MMSE rate
    within 1e-3 bit of the oracle's fp64 rate, ergodic mean within 1e-3, counts identical; and
    the fp64 sweep on the same drops within 1e-6."""
    w = CONFIGS[3]
    D = 1000
    ag = xl.Array.ula(w.n_y, w.fc_hz)
    pos = xl.gen_drops(xl.Users.polar(w.r, w.az), w.K, D, seed=w.seed)
    ao = orc.array("ula", n_y=w.n_y, fc_hz=w.fc_hz)
    erg, nv, sat, pdo = orc.saturation_sweep(ao, [w.n_y], pos.cpu().numpy(), w.snr_db, w.receivers, per_drop=True)
    for prec, tol in ((xl.FP32, 1e-3), (xl.FP64, 1e-6)):
        res = xl.saturation_sweep(ag, [w.n_y], w.K, D, w.snr_db, w.receivers, pos=pos, precision=prec,
                                  per_drop=True)
        pd = res["per_drop"].cpu().numpy()
        assert np.array_equal(np.isnan(pd), np.isnan(pdo))
        assert np.nanmax(np.abs(pd - pdo)) <= tol
        assert np.array_equal(res["n_valid"], nv)
        assert np.nanmax(np.abs(res["ergodic"] - erg)) <= tol
        assert res["sat"][2] == sat[2]


# --------------------------------------------------------------------------- a1 bit for bit
@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_draw_words_bit_exact_and_positions_within_2ulp(xl, orc, cfg):
    """R19: the Philox4x64-10 words behind every drop are bit-identical to the oracle's
    generator (itself pinned to numpy's Philox); r, az, el are then the same doubles on both
    sides (no FMA contraction), so positions (r cos el cos az, r cos el sin az, r sin el) differ
    only by libm vs CUDA sin/cos: <= 2 ulp per coordinate for planar users (el = 0, one trig
    factor), <= 3 ulp for the UPA's 3-D users (two trig factors, cfg4)."""
    w = CONFIGS[cfg]
    n = min(w.n_drops, 256)
    words = xl.draw_words(w.K, n, seed=w.seed).cpu().numpy()
    for d in range(n):
        for k in range(w.K):
            ref = orc.philox4x64_10(np.array([d, k, 0, 0], dtype=np.uint64), np.array([w.seed, 0], dtype=np.uint64))
            assert np.array_equal(words[d, k], ref), (d, k)
    pg = xl.gen_drops(xl.Users.polar(w.r, w.az, w.el), w.K, 2000, seed=w.seed).cpu().numpy()
    po = orc.gen_drops(orc.users(r=w.r, az=w.az, el=w.el), w.K, 2000, seed=w.seed)
    exact_zero = po == 0.0
    assert np.array_equal(pg[exact_zero], po[exact_zero])
    ulp = np.abs(pg - po)[~exact_zero] / np.spacing(np.abs(po[~exact_zero]))
    assert ulp.max() <= (3.0 if w.el != (0.0, 0.0) else 2.0), ulp.max()
    # first_drop addressing of the words (sharding / resume)
    tail = xl.draw_words(w.K, 10, seed=w.seed, first_drop=n - 10).cpu().numpy()
    assert np.array_equal(tail, words[n - 10:])
