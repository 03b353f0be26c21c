"""Parity in the launch configuration bench.py times (the full drop count of each bench
record, the same entry points and options), on sampled drops the oracle computes one by
one, plus properties that hold at any size.

  headline  cfg5, 1000 drops through xlmimo_saturation_sweep (exact fp64 and closed form,
            per-drop rates): 16 sampled drops (first, last, spread) vs the oracle's Gram
            (Eq. (3) H and one library matmul) and receivers at 1e-6 bit; every drop of the
            closed-form sweep vs the oracle's closed-form sweep (O(K^2) per drop); ergodic
            = mean of the per-drop rates, n_valid = non-NaN count.
  cfg5 fp32 / materialised, 1000 drops through gram_exact: the same 16 drops at 1e-4 (Gram)
            and 1e-3 bit (rates).
  cfg1 steady state, 10^6 drops (kernel W): 64 sampled drops at 1e-9; the closed-form
            Gram and flags of 4096 sampled drops.
  cfg3 10^5 drops and cfg4 10^4 drops, fp64 and fp32: 16 sampled drops each.
Tolerances as in test_fullsize_gpu.py (R9): Gram |dG_ij| / sqrt(G_ii G_jj) <= 1e-9 (fp64)
/ 1e-4 (fp32); rates 1e-6 / 1e-3 bits/s/Hz; flags identical.
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


def _sample(D, n, seed=0):
    rng = np.random.default_rng(seed)
    mid = rng.choice(np.arange(1, D - 1), size=n - 2, replace=False)
    return np.sort(np.r_[0, mid, D - 1])


def _arrays(xl, orc, w):
    if w.kind == "ula":
        return xl.Array.ula(w.n_y, w.fc_hz), orc.array("ula", n_y=w.n_y, fc_hz=w.fc_hz)
    return xl.Array.upa(w.n_y, w.n_z, w.fc_hz), orc.array("upa", n_y=w.n_y, n_z=w.n_z, fc_hz=w.fc_hz)


# --------------------------------------------------------------------------- cfg5 (headline)
@pytest.fixture(scope="module")
def cfg5(xl, orc):
    w = CONFIGS[5]
    D = w.n_drops
    ag, ao = _arrays(xl, orc, w)
    pos = xl.gen_drops(xl.Users.polar(w.r, w.az), w.K, D, seed=1000)  # the bench's first step
    S = _sample(D, 16)
    Go = orc.gram_exact_blas(ao, pos.cpu().numpy()[S])
    return w, ag, ao, pos, S, Go


def test_headline_sweep_sampled_drops(xl, orc, cfg5):
    w, ag, ao, pos, S, Go = cfg5
    D = pos.shape[0]
    res = xl.saturation_sweep(ag, [w.N], w.K, D, list(w.snr_db), w.receivers, pos=pos, t=w.t, per_drop=True)
    pd = res["per_drop"].cpu().numpy()  # [D, 1, n_snr, R]
    assert pd.shape == (D, 1, len(w.snr_db), xl.n_recv(w.receivers))
    ro, flo = orc.sum_rate(Go, w.snr_db, w.receivers)
    assert np.all(flo == 0)
    assert np.max(np.abs(pd[S, 0] - ro)) <= 1e-6
    # properties over all 1000 drops
    assert np.all(np.isfinite(pd))
    assert np.array_equal(np.asarray(res["n_valid"]).reshape(-1), np.full(pd.shape[2] * pd.shape[3], D))
    assert np.allclose(np.asarray(res["ergodic"]).reshape(-1), pd.mean(axis=0).reshape(-1), rtol=1e-12, atol=0)


def test_headline_closed_form_sweep_every_drop(xl, orc, cfg5):
    w, ag, ao, pos, S, Go = cfg5
    D = pos.shape[0]
    res = xl.saturation_sweep(ag, [w.N], w.K, D, list(w.snr_db), w.receivers, pos=pos, t=w.t, per_drop=True,
                              gram_kind=xl.GRAM_CLOSED_FORM)
    erg, nv, sat, pdo = orc.saturation_sweep(ao, [w.N], pos.cpu().numpy(), w.snr_db, w.receivers, gram_kind=1,
                                             t=w.t, per_drop=True)
    pd = res["per_drop"].cpu().numpy()
    assert np.array_equal(np.isnan(pd), np.isnan(pdo))
    assert np.nanmax(np.abs(pd - pdo)) <= 1e-6
    assert np.array_equal(np.asarray(res["n_valid"]), nv)
    assert res["sat"][2] == sat[2]


@pytest.mark.parametrize("mode", ["fp32", "mat32"])
def test_cfg5_fp32_paths_sampled_drops(xl, orc, cfg5, mode):
    w, ag, ao, pos, S, Go = cfg5
    G = xl.gram_exact(ag, pos, precision=xl.FP32, mode=xl.MATERIALIZED if mode == "mat32" else xl.FUSED)
    assert G.shape == (pos.shape[0], w.K, w.K)
    Gs = G.cpu().numpy()[S]
    assert normalized_err(Gs, Go) <= 1e-4
    r, fl = xl.sum_rate(G[torch.as_tensor(S, device=G.device)], list(w.snr_db), w.receivers)
    ro, flo = orc.sum_rate(Go, w.snr_db, w.receivers)
    assert np.array_equal(fl.cpu().numpy().astype(np.uint32), flo)
    assert np.max(np.abs(r.cpu().numpy() - ro)) <= 1e-3


# --------------------------------------------------------------------------- cfg1 steady state
def test_cfg1_steady_state_sampled_drops(xl, orc):
    w = CONFIGS[1]
    D = 10 ** 6
    ag, ao = _arrays(xl, orc, w)
    pos = xl.gen_drops(xl.Users.polar(w.r, w.az), w.K, D, seed=5000)
    G = xl.gram_exact(ag, pos)
    Gc, fl = xl.gram_closed_form(ag, pos)
    P = pos.cpu().numpy()
    S = _sample(D, 64, 1)
    assert normalized_err(G.cpu().numpy()[S], orc.gram_exact(ao, P[S])) <= 1e-9
    allr = xl.RECV_CAP | xl.RECV_ZF | xl.RECV_MMSE | xl.RECV_MRC
    r, rfl = xl.sum_rate(G[torch.as_tensor(S, device=G.device)], list(w.snr_db), allr)
    ro, rflo = orc.sum_rate(orc.gram_exact(ao, P[S]), w.snr_db, allr)
    assert np.array_equal(rfl.cpu().numpy().astype(np.uint32), rflo)
    assert np.max(np.abs(r.cpu().numpy() - ro)) <= 1e-6
    S2 = _sample(D, 4096, 2)
    Gco, flo = orc.gram_closed_form(ao, P[S2])
    assert np.array_equal(fl.cpu().numpy().astype(np.uint32)[S2], flo)
    assert normalized_err(Gc.cpu().numpy()[S2], Gco) <= 1e-9


# --------------------------------------------------------------------------- cfg3 / cfg4
@pytest.mark.parametrize("cfg,prec", [(3, "fp64"), (3, "fp32"), (4, "fp64"), (4, "fp32")])
def test_cfg3_cfg4_bench_size_sampled_drops(xl, orc, cfg, prec):
    w = CONFIGS[cfg]
    D = w.n_drops
    ag, ao = _arrays(xl, orc, w)
    pos = xl.gen_drops(xl.Users.polar(w.r, w.az, w.el), w.K, D, seed=7000)
    G = xl.gram_exact(ag, pos, precision=xl.FP64 if prec == "fp64" else xl.FP32)
    S = _sample(D, 16, cfg)
    Go = orc.gram_exact(ao, pos.cpu().numpy()[S])
    assert normalized_err(G.cpu().numpy()[S], Go) <= (1e-9 if prec == "fp64" else 1e-4)
    r, fl = xl.sum_rate(G[torch.as_tensor(S, device=G.device)], list(w.snr_db), w.receivers)
    ro, flo = orc.sum_rate(Go, w.snr_db, w.receivers)
    assert np.array_equal(fl.cpu().numpy().astype(np.uint32), flo)
    assert np.max(np.abs(r.cpu().numpy() - ro)) <= (1e-6 if prec == "fp64" else 1e-3)
