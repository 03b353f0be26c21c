"""GPU parity for the large-K (64 < K <= 1024) exact Gram (block-pair DMMA kernel below
K = 128, chunked DMMA SYRK from 128 on; fp32: tcgen05 block pairs):
the CUDA path through the C ABI vs the oracle on the same GPU-drawn positions.

Tolerance: |dG_ij| / sqrt(G_ii G_jj) <= 1e-9 (fp64 path, reading R9).
"""
import numpy as np
import pytest

from tests._util import normalized_err

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


@pytest.mark.parametrize("kind,n_y,n_z,K,D", [("ula", 700, 1, 65, 3), ("ula", 1001, 1, 100, 2),
                                              ("ula", 640, 1, 128, 2), ("ula", 333, 1, 129, 2),
                                              ("ula", 500, 1, 200, 1), ("upa", 24, 20, 80, 2),
                                              ("ula", 50, 1, 100, 2), ("ula", 2000, 1, 113, 2),
                                              ("ula", 999, 1, 120, 2), ("upa", 32, 16, 104, 2)])
def test_gram_large_k_parity(xl, orc, kind, n_y, n_z, K, D):
    """64 < K <= 128 on the MT2 3M-DMMA stars (65, 80 UPA, 100, 104 UPA, 113, 120; 128 as two
    launches of 17 stars), the 3M SYRK above (ragged 129, 200), and N < K (rank-deficient G,
    N = 50)."""
    fc = 100e9
    if kind == "ula":
        a, ao = xl.Array.ula(n_y, fc), orc.array("ula", n_y=n_y, fc_hz=fc)
    else:
        a, ao = xl.Array.upa(n_y, n_z, fc), orc.array("upa", n_y=n_y, n_z=n_z, fc_hz=fc)
    if kind == "ula":
        pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, D, seed=K)
    else:
        pos = xl.gen_drops(xl.Users.polar((2.0, 20.0), (-60, 60), (-30, 30)), K, D, seed=K)
    G = xl.gram_exact(a, pos).cpu().numpy()
    Go = orc.gram_exact(ao, pos.cpu().numpy())
    assert normalized_err(G, Go) <= 1e-9
    assert np.all(G.diagonal(axis1=1, axis2=2).imag == 0)
    assert np.array_equal(G, np.conj(np.transpose(G, (0, 2, 1))))


def test_gram_large_k_e3_full_size(xl, orc):
    """The E3 point of the paper (K = 1000 users of the Sec. IV-C field, M = 35 000,
    100 GHz) at full size: GPU Gram vs the oracle's Eq. (3) H and
    one library matmul, then Appendix A on the GPU's own Gram -> 0.064."""
    a = xl.Array.ula(35000, 100e9)
    pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), 1000, 1, seed=0)
    G = xl.gram_exact(a, pos)
    Go = orc.gram_exact_blas(orc.array("ula", n_y=35000, fc_hz=100e9), pos.cpu().numpy())
    assert normalized_err(G.cpu().numpy(), Go) <= 1e-9
    rs, _, _, fl = xl.app_a_bounds(G, [0.0])
    assert int(fl[0]) == 0 and abs(float(rs[0, 1]) - 0.064) < 1e-3


@pytest.mark.parametrize("kind", ["ula", "upa"])
def test_gram_large_k_materialised_fp32(xl, orc, kind):
    """MATERIALIZED at K > 64: the TMA-fed tcgen05 pairs over complex64 (TF32) chunks of H
    written to the workspace, at a K below the fused path's streaming threshold (fp32
    tier); ULA across a chunk boundary, UPA with rows a multiple of 8 and a ragged last
    block of users."""
    if kind == "ula":
        a, ao = xl.Array.ula(5000, 100e9), orc.array("ula", n_y=5000, fc_hz=100e9)
        pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), 90, 2, seed=6)
    else:
        a, ao = xl.Array.upa(40, 30, 100e9), orc.array("upa", n_y=40, n_z=30, fc_hz=100e9)
        pos = xl.gen_drops(xl.Users.polar((2.0, 20.0), (-60, 60), (-30, 30)), 150, 2, seed=7)
    G = xl.gram_exact(a, pos, precision=xl.FP32, mode=xl.MATERIALIZED).cpu().numpy()
    assert normalized_err(G, orc.gram_exact(ao, pos.cpu().numpy())) <= 1e-4


def test_gram_large_k_unsupported_modes(xl):
    a = xl.Array.ula(256, 100e9)
    pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), 70, 1, seed=1)
    with pytest.raises(xl.XlmimoError):
        xl.gram_exact(a, pos, precision=xl.FP64, mode=xl.MATERIALIZED)
    upa = xl.Array.upa(36, 30, 100e9)  # N >= 1024 (tensor-core tier), rows not a multiple of 8
    with pytest.raises(xl.XlmimoError):
        xl.gram_exact(upa, pos, precision=xl.FP32)
    e = torch.zeros((0, 70, 3), dtype=torch.float64, device="cuda")
    assert xl.gram_exact(a, e).shape == (0, 70, 70)


@pytest.mark.parametrize("kind,n_y,n_z,K,D", [("ula", 4099, 1, 65, 3), ("ula", 20000, 1, 100, 2),
                                              ("ula", 3000, 1, 129, 2), ("ula", 777, 1, 200, 1),
                                              ("upa", 24, 40, 80, 2)])
def test_gram_large_k_fp32_parity(xl, orc, kind, n_y, n_z, K, D):
    """fp32 tier (1e-4 normalised) for K > 64: block pairs of 64 users on tcgen05 (TF32,
    RNA-rounded generated operands, fp32 TMEM accumulation per 8192-element chunk, fp64
    across chunks); ragged users and elements, a chunk boundary (N = 20000), UPA."""
    fc = 100e9
    if kind == "ula":
        a, ao = xl.Array.ula(n_y, fc), orc.array("ula", n_y=n_y, fc_hz=fc)
        pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, D, seed=K)
    else:
        a, ao = xl.Array.upa(n_y, n_z, fc), orc.array("upa", n_y=n_y, n_z=n_z, fc_hz=fc)
        pos = xl.gen_drops(xl.Users.polar((2.0, 20.0), (-60, 60), (-30, 30)), K, D, seed=K)
    G = xl.gram_exact(a, pos, precision=xl.FP32).cpu().numpy()
    Go = orc.gram_exact_blas(ao, pos.cpu().numpy())
    assert normalized_err(G, Go) <= 1e-4
    assert np.all(G.diagonal(axis1=1, axis2=2).imag == 0)
    assert np.array_equal(G, np.conj(np.transpose(G, (0, 2, 1))))


@pytest.mark.parametrize("kind,n_y,n_z,K,D", [("ula", 9001, 1, 128, 3), ("ula", 70001, 1, 86, 2),
                                              ("upa", 48, 150, 97, 2), ("ula", 2048, 1, 65, 4)])
def test_gram_fp32_wide_fused(xl, orc, kind, n_y, n_z, K, D):
    """64 < K <= 128 at fp32 on the fused kernel: a wide launch (all K users as the MMA's N, the
    first 64 as its M: entries i < 64) and a narrow one (users 64..K-1) into one set of
    partials -- every entry against the oracle at the fp32 tier (1e-4 normalised), with a
    single TMEM accumulator (3 N > 512: K = 86, 97, 128) and a double-buffered one (K = 65),
    several chunks (N = 70001), UPA rows of 16k; Hermitian, real diagonal."""
    fc = 100e9
    if kind == "ula":
        a, ao = xl.Array.ula(n_y, fc), orc.array("ula", n_y=n_y, fc_hz=fc)
        pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, D, seed=K + 1)
    else:
        a, ao = xl.Array.upa(n_y, n_z, fc), orc.array("upa", n_y=n_y, n_z=n_z, fc_hz=fc)
        pos = xl.gen_drops(xl.Users.polar((2.0, 20.0), (-60, 60), (-30, 30)), K, D, seed=K + 1)
    G = xl.gram_exact(a, pos, precision=xl.FP32).cpu().numpy()
    Go = orc.gram_exact_blas(ao, pos.cpu().numpy())
    assert normalized_err(G, Go) <= 1e-4
    assert np.all(G.diagonal(axis1=1, axis2=2).imag == 0)
    assert np.array_equal(G, np.conj(np.transpose(G, (0, 2, 1))))


@pytest.mark.parametrize("kind,n_y,n_z,K,D", [("ula", 5001, 1, 129, 2), ("ula", 3000, 1, 200, 2),
                                              ("ula", 20000, 1, 256, 1), ("upa", 40, 60, 150, 2),
                                              ("upa", 48, 50, 193, 1)])
def test_gram_fp32_cross_fused(xl, orc, kind, n_y, n_z, K, D):
    """128 < K <= 256 at fp32 on the fused kernel: per block of 64 row users a wide launch
    (users a0 .. a0 + 127) or a narrow one, plus cross launches (the block's rows x 64 further
    users, the MMA's B operand after the A rows in the stage) -- every entry against the
    oracle (1e-4 normalised): a single extra user (K = 129), ragged cross blocks (200, 193),
    K = 256, UPA rows of 8k (TE = 8) and 16k; Hermitian, real diagonal."""
    fc = 100e9
    if kind == "ula":
        a, ao = xl.Array.ula(n_y, fc), orc.array("ula", n_y=n_y, fc_hz=fc)
        pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, D, seed=K + 7)
    else:
        a, ao = xl.Array.upa(n_y, n_z, fc), orc.array("upa", n_y=n_y, n_z=n_z, fc_hz=fc)
        pos = xl.gen_drops(xl.Users.polar((2.0, 20.0), (-60, 60), (-30, 30)), K, D, seed=K + 7)
    G = xl.gram_exact(a, pos, precision=xl.FP32).cpu().numpy()
    Go = orc.gram_exact_blas(ao, pos.cpu().numpy())
    assert normalized_err(G, Go) <= 1e-4
    assert np.all(G.diagonal(axis1=1, axis2=2).imag == 0)
    assert np.array_equal(G, np.conj(np.transpose(G, (0, 2, 1))))


def test_fp32_rates_cross_fused(xl, orc):
    """K = 192 at fp32 through the cross launches: per-drop CAP/ZF/MMSE/MRC rates against
    the oracle's fp64 rates, ergodic within 1e-3 bit, every drop within 5e-3 (R29)."""
    K, D = 192, 4
    a, ao = xl.Array.ula(12000, 100e9), orc.array("ula", n_y=12000, fc_hz=100e9)
    pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, D, seed=23)
    rec = xl.RECV_CAP | xl.RECV_ZF | xl.RECV_MMSE | xl.RECV_MRC
    r, fl = xl.sum_rate(xl.gram_exact(a, pos, precision=xl.FP32), [0.0, 10.0], rec)
    ro, flo = orc.sum_rate(orc.gram_exact_blas(ao, pos.cpu().numpy()), [0.0, 10.0], rec)
    assert np.array_equal(fl.cpu().numpy().astype(np.uint32), flo)
    rg = r.cpu().numpy()
    ok = ~np.isnan(ro)
    assert np.array_equal(np.isnan(rg), ~ok)
    assert np.max(np.abs(rg[ok] - ro[ok]), initial=0.0) <= 5e-3
    assert np.max(np.abs(np.nanmean(rg, axis=0) - np.nanmean(ro, axis=0))) <= 1e-3


def test_gram_large_k_fp32_e3(xl, orc):
    """E3 size in fp32: K = 1000, M = 35 000 against the oracle (1e-4) and the paper's gap."""
    a = xl.Array.ula(35000, 100e9)
    pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), 1000, 1, seed=0)
    G = xl.gram_exact(a, pos, precision=xl.FP32)
    Go = orc.gram_exact_blas(orc.array("ula", n_y=35000, fc_hz=100e9), pos.cpu().numpy())
    assert normalized_err(G.cpu().numpy(), Go) <= 1e-4
    rs, _, _, fl = xl.app_a_bounds(G, [0.0])
    assert int(fl[0]) == 0 and abs(float(rs[0, 1]) - 0.064) < 1e-3


def test_gram_large_k_determinism(xl):
    a = xl.Array.ula(3000, 100e9)
    pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), 150, 3, seed=9)
    g1 = xl.gram_exact(a, pos)
    g2 = xl.gram_exact(a, pos)
    assert torch.equal(g1, g2)


def test_closed_form_and_sweep_large_k(xl, orc):
    """Closed-form (modified-ZF) Gram at K = 100 (O(K^2), no N loop) and the closed-form
    saturation sweep at K > 64 (CAP + MRC) against the oracle on the same drops."""
    pos = xl.gen_drops_rect((1.0, 2.0), (-7.5, 7.5), 100, 4, seed=21)
    ph = pos.cpu().numpy()
    a, ao = xl.Array.ula(12460, 100e9), orc.array("ula", n_y=12460, fc_hz=100e9)
    Gt, fl = xl.gram_closed_form(a, pos)
    Gto, flo = orc.gram_closed_form(ao, ph)
    assert np.max(np.abs(Gt.cpu().numpy() - Gto)) <= 1e-9 * np.max(np.abs(Gto))
    assert np.array_equal(fl.cpu().numpy().astype(np.uint32), flo)
    nl = [1024, 4096, 12460]
    rec = xl.RECV_CAP | xl.RECV_MRC
    res = xl.saturation_sweep(a, nl, 100, 4, [3.5], rec, pos=pos, gram_kind=xl.GRAM_CLOSED_FORM, per_drop=True)
    _, nv, _, pd = orc.saturation_sweep(ao, nl, ph, [3.5], rec, gram_kind=1, per_drop=True)
    g = res["per_drop"].cpu().numpy()
    assert np.array_equal(np.isnan(g), np.isnan(pd))
    ok = ~np.isnan(pd)
    assert np.max(np.abs(g[ok] - pd[ok]), initial=0.0) <= 1e-6
    assert np.array_equal(res["n_valid"], nv)


def test_max_k_1024_end_to_end(xl, orc):
    """The largest supported K (1024 = 16 full blocks, K_pad = K): exact fp64 and fp32
    Grams, all four receivers (tiled Cholesky + blocked inverse) and Appendix A against
    the oracle on one drop."""
    K, N = 1024, 3000  # N ~ 3 K: G well conditioned (at N ~ K, R is numerically singular on both sides)
    a, ao = xl.Array.ula(N, 100e9), orc.array("ula", n_y=N, fc_hz=100e9)
    pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, 1, seed=77)
    G = xl.gram_exact(a, pos)
    Go = orc.gram_exact_blas(ao, pos.cpu().numpy())
    assert normalized_err(G.cpu().numpy(), Go) <= 1e-9
    assert normalized_err(xl.gram_exact(a, pos, precision=xl.FP32).cpu().numpy(), Go) <= 1e-4
    snr = [10.0]
    allr = xl.RECV_CAP | xl.RECV_ZF | xl.RECV_MMSE | xl.RECV_MRC
    r, fl = xl.sum_rate(G, snr, allr)
    ro, flo = orc.sum_rate(G.cpu().numpy(), snr, allr)
    rg = r.cpu().numpy()
    assert np.array_equal(np.isnan(rg), np.isnan(ro))
    ok = ~np.isnan(ro)
    assert np.max(np.abs(rg[ok] - ro[ok]), initial=0.0) <= 1e-6
    assert np.array_equal(fl.cpu().numpy().astype(np.uint32), flo)
    rs, bo, _, fa = xl.app_a_bounds(G, snr)
    rso, boo, _, fao = orc.bounds_app_a(G.cpu().numpy(), snr)
    assert np.array_equal(fa.cpu().numpy().astype(np.uint32), fao) and int(fao[0]) == 0
    assert np.max(np.abs(rs.cpu().numpy() - rso)) <= 1e-6 and np.max(np.abs(bo.cpu().numpy() - boo)) <= 1e-6


@pytest.mark.parametrize("N", [1, 2, 31, 33])
def test_gram_large_k_tiny_arrays(xl, orc, N):
    """Degenerate element counts on the large-K paths (fewer elements than one 32-element
    tile, a single element: G = h h^H of rank 1) in fp64 and fp32 (below 1024 elements
    the fp32 request runs on the fp64 kernel: TF32 rounding would not average out)."""
    K = 70
    a, ao = xl.Array.ula(N, 100e9), orc.array("ula", n_y=N, fc_hz=100e9)
    pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, 2, seed=N)
    Go = orc.gram_exact(ao, pos.cpu().numpy())
    assert normalized_err(xl.gram_exact(a, pos).cpu().numpy(), Go) <= 1e-9
    assert normalized_err(xl.gram_exact(a, pos, precision=xl.FP32).cpu().numpy(), Go) <= 1e-4
    if N == 1:
        h = orc.channel_matrix(ao, pos.cpu().numpy()[0])[0]
        assert normalized_err(Go[0][None], np.outer(h.conj(), h)[None]) <= 1e-14


@pytest.mark.parametrize("kind,n_y,n_z,K,N_or_D", [("upa", 24, 20, 150, 2), ("ula", 1, 1, 150, 2),
                                                   ("ula", 31, 1, 160, 1), ("ula", 4500, 1, 130, 3)])
def test_gram_syrk_parity(xl, orc, kind, n_y, n_z, K, N_or_D):
    """K > 128 runs the chunked DMMA SYRK (xl_gram_syrk.cu): UPA, one element, fewer
    elements than a tile, and a chunk boundary (4500 elements > one 4096-element chunk)."""
    fc, D = 100e9, N_or_D
    if kind == "ula":
        a, ao = xl.Array.ula(n_y, fc), orc.array("ula", n_y=n_y, fc_hz=fc)
        pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, D, seed=K + n_y)
    else:
        a, ao = xl.Array.upa(n_y, n_z, fc), orc.array("upa", n_y=n_y, n_z=n_z, fc_hz=fc)
        pos = xl.gen_drops(xl.Users.polar((2.0, 20.0), (-60, 60), (-30, 30)), K, D, seed=K)
    G = xl.gram_exact(a, pos).cpu().numpy()
    assert normalized_err(G, orc.gram_exact(ao, pos.cpu().numpy())) <= 1e-9
    assert np.all(G.diagonal(axis1=1, axis2=2).imag == 0)


def test_exact_sweep_large_k_nested_levels(xl, orc):
    """Exact fp64 saturation sweep at K = 130 (SYRK path: per-level partials, chunks
    restarting at each level end, the last level two chunks long) against the oracle's
    independent per-N Grams."""
    K, D = 130, 2
    nl = [700, 2000, 9000]
    a, ao = xl.Array.ula(max(nl), 100e9), orc.array("ula", n_y=max(nl), fc_hz=100e9)
    pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, D, seed=5)
    rec = xl.RECV_CAP | xl.RECV_ZF | xl.RECV_MMSE | xl.RECV_MRC
    res = xl.saturation_sweep(a, nl, K, D, [10.0], rec, pos=pos, per_drop=True)
    _, nv, _, pd = orc.saturation_sweep(ao, nl, pos.cpu().numpy(), [10.0], rec, gram_kind=0, per_drop=True)
    g = res["per_drop"].cpu().numpy()
    assert np.array_equal(np.isnan(g), np.isnan(pd))
    ok = ~np.isnan(pd)
    assert np.max(np.abs(g[ok] - pd[ok]), initial=0.0) <= 1e-6
    assert np.array_equal(res["n_valid"], nv)


def test_fp32_sweep_large_k_rates(xl, orc):
    """fp32 exact sweep at E1's K = 100 (the tcgen05 block-pair Gram run once per
    N, copied into the level slots) against the oracle's fp64 rates: the ergodic means (CAP,
    ZF, MMSE, MRC) within the fp32 tier, 1e-3 bit; per drop within 5e-3 -- a sum over 100
    users of per-user errors that the Gram's conditioning amplifies from the TF32 operand
    rounding (normalised Gram error ~3e-5 at N = 1024, inside the 1e-4 Gram tier); counts
    identical.  Before the pair kernel's TMEM sub-chunk folding (512 truncating MMA
    accumulations per partial) the K = 100 rates carried a -4e-3 bit bias."""
    K, D = 100, 6
    nl = [1024, 2048, 6000, 12000]
    a, ao = xl.Array.ula(max(nl), 100e9), orc.array("ula", n_y=max(nl), fc_hz=100e9)
    pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, D, seed=9)
    rec = xl.RECV_CAP | xl.RECV_ZF | xl.RECV_MMSE | xl.RECV_MRC
    res = xl.saturation_sweep(a, nl, K, D, [0.0, 10.0], rec, pos=pos, precision=xl.FP32, per_drop=True)
    erg, nv, _, pd = orc.saturation_sweep(ao, nl, pos.cpu().numpy(), [0.0, 10.0], rec, per_drop=True)
    g = res["per_drop"].cpu().numpy()
    assert np.array_equal(np.isnan(g), np.isnan(pd))
    ok = ~np.isnan(pd)
    assert np.max(np.abs(g[ok] - pd[ok]), initial=0.0) <= 5e-3
    assert np.array_equal(res["n_valid"], nv)
    assert np.nanmax(np.abs(res["ergodic"] - erg)) <= 1e-3


@pytest.mark.parametrize("path,K", [(1, 200), (2, 100), (2, 65), (1, 100), (1, 72)])
def test_large_k_paths_outside_their_default_range(xl, orc, path, K):
    """XLMIMO_OPT_LARGE_K forces the block-pair (1) or the SYRK (2) kernel; each must match
    the oracle outside the K range the default selection gives it."""
    a = xl.Array.ula(1500, 100e9)
    pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, 2, seed=3)
    with xl.option(xl.OPT_LARGE_K, path):
        G = xl.gram_exact(a, pos).cpu().numpy()
    Go = orc.gram_exact(orc.array("ula", n_y=1500, fc_hz=100e9), pos.cpu().numpy())
    assert normalized_err(G, Go) <= 1e-9


@pytest.mark.parametrize("path,K", [(1, 400), (2, 100), (1, 200), (2, 65), (1, 100)])
def test_large_k_fp32_paths_outside_their_default_range(xl, orc, path, K):
    """XLMIMO_OPT_PAIR forces the in-kernel-generation (1) or the TMA-fed materialised-chunk
    (2) tcgen05 block-pair kernel at fp32; each must meet the fp32 tier (1e-4 normalised)
    outside the K range the default selection gives it, across a chunk boundary."""
    a = xl.Array.ula(5000, 100e9)
    pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, 2, seed=4)
    with xl.option(xl.OPT_PAIR, path):
        G = xl.gram_exact(a, pos, precision=xl.FP32).cpu().numpy()
    Go = orc.gram_exact(orc.array("ula", n_y=5000, fc_hz=100e9), pos.cpu().numpy())
    assert normalized_err(G, Go) <= 1e-4


def test_every_kernel_boundary_in_k(xl, orc):
    """Dispatch boundaries in K (W / split / M / MT2 G = 3..16 with its one- and two-launch
    plans / SYRK; fused fp32 narrow, wide + narrow, pair stream) on one ULA and one UPA of a
    few thousand elements: fp64 within 1e-9 and fp32 within 1e-4 (normalised) of the oracle,
    every entry, for K on both sides of each boundary."""
    ks = [1, 4, 5, 8, 9, 16, 17, 24, 25, 32, 33, 48, 49, 56, 57, 63, 64, 65, 72, 73, 96, 97, 104, 105,
          112, 113, 120, 121, 127, 128, 129]
    fc = 100e9
    arrays = [(xl.Array.ula(3001, fc), orc.array("ula", n_y=3001, fc_hz=fc)),
              (xl.Array.upa(48, 40, fc), orc.array("upa", n_y=48, n_z=40, fc_hz=fc))]
    for (a, ao) in arrays:
        for K in ks:
            pos = xl.gen_drops(xl.Users.polar((2.0, 20.0), (-60, 60), (-30, 30)), K, 2, seed=100 + K)
            Go = orc.gram_exact_blas(ao, pos.cpu().numpy())
            G64 = xl.gram_exact(a, pos).cpu().numpy()
            assert normalized_err(G64, Go) <= 1e-9, ("fp64", K)
            G32 = xl.gram_exact(a, pos, precision=xl.FP32).cpu().numpy()
            assert normalized_err(G32, Go) <= 1e-4, ("fp32", K)


def test_receivers_every_boundary_in_k(xl, orc):
    """Receiver dispatch boundaries (thread / warp / CTA shared-memory / tiled DMMA Cholesky):
    CAP, ZF, MMSE, MRC per drop within 1e-6 bit of the oracle on the same fp64 Gram, flags
    identical, for K on both sides of each boundary."""
    fc = 100e9
    a = xl.Array.ula(4001, fc)
    rec = xl.RECV_CAP | xl.RECV_ZF | xl.RECV_MMSE | xl.RECV_MRC
    for K in [8, 9, 64, 65, 96, 97, 128, 160, 161]:
        pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, 3, seed=200 + K)
        G = xl.gram_exact(a, pos)
        r, fl = xl.sum_rate(G, [0.0, 10.0], rec)
        ro, flo = orc.sum_rate(G.cpu().numpy(), [0.0, 10.0], rec)
        assert np.array_equal(fl.cpu().numpy().astype(np.uint32), flo), K
        rg = r.cpu().numpy()
        ok = ~np.isnan(ro)
        assert np.array_equal(np.isnan(rg), ~ok), K
        assert np.max(np.abs(rg[ok] - ro[ok]), initial=0.0) <= 1e-6, K


def test_fp32_rates_wide_single_accumulator(xl, orc):
    """K = 128 at fp32 (the fused kernel's wide launch with a single TMEM accumulator and the
    sub-chunk folding) on an E1-field array of 12 000 elements: per-drop CAP/ZF/MMSE/MRC rates
    against the oracle's fp64 rates on its own Gram -- ergodic means within the fp32 tier
    (1e-3 bit), every drop within 5e-3 (R29), flags identical."""
    K, D = 128, 6
    a, ao = xl.Array.ula(12000, 100e9), orc.array("ula", n_y=12000, fc_hz=100e9)
    pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, D, seed=21)
    rec = xl.RECV_CAP | xl.RECV_ZF | xl.RECV_MMSE | xl.RECV_MRC
    G = xl.gram_exact(a, pos, precision=xl.FP32)
    r, fl = xl.sum_rate(G, [0.0, 10.0], rec)
    Go = orc.gram_exact_blas(ao, pos.cpu().numpy())
    ro, flo = orc.sum_rate(Go, [0.0, 10.0], rec)
    assert np.array_equal(fl.cpu().numpy().astype(np.uint32), flo)
    rg = r.cpu().numpy()
    ok = ~np.isnan(ro)
    assert np.array_equal(np.isnan(rg), ~ok)
    assert np.max(np.abs(rg[ok] - ro[ok]), initial=0.0) <= 5e-3
    assert np.max(np.abs(np.nanmean(rg, axis=0) - np.nanmean(ro, axis=0))) <= 1e-3


@pytest.mark.parametrize("K,prec,tol", [(128, "fp64", 1e-6), (160, "fp32", 1e-3)])
def test_sweep_large_k_paths(xl, orc, K, prec, tol):
    """The exact saturation sweep through the K > 120 paths: fp64 K = 128 on MT2's two
    launches per tile (nested levels in one pass), fp32 K = 160 on the fused kernel's wide /
    cross / narrow launches once per N (the workspace the largest level's) -- ergodic means
    and per-drop rates against the oracle's fp64 sweep (fp64 1e-6 bit; fp32 1e-3 ergodic,
    5e-3 per drop), counts identical."""
    D = 3
    nl = [1024, 2048, 4000]
    a, ao = xl.Array.ula(max(nl), 100e9), orc.array("ula", n_y=max(nl), fc_hz=100e9)
    pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, D, seed=31)
    rec = xl.RECV_CAP | xl.RECV_ZF | xl.RECV_MMSE
    res = xl.saturation_sweep(a, nl, K, D, [10.0], rec, pos=pos,
                              precision=xl.FP64 if prec == "fp64" else xl.FP32, per_drop=True)
    erg, nv, _, pd = orc.saturation_sweep(ao, nl, pos.cpu().numpy(), [10.0], rec, per_drop=True)
    g = res["per_drop"].cpu().numpy()
    assert np.array_equal(np.isnan(g), np.isnan(pd))
    ok = ~np.isnan(pd)
    assert np.max(np.abs(g[ok] - pd[ok]), initial=0.0) <= (tol if prec == "fp64" else 5e-3)
    assert np.array_equal(res["n_valid"], nv)
    assert np.nanmax(np.abs(res["ergodic"] - erg)) <= tol


@pytest.mark.parametrize("K,prec", [(100, "fp32"), (160, "fp32"), (256, "fp32"), (128, "fp64"),
                                    (56, "fp64"), (72, "fp64"), (88, "fp64"), (100, "fp64"), (112, "fp64")])
def test_large_k_paths_bitwise_deterministic(xl, K, prec):
    """The multi-launch paths (fused fp32 wide / cross / narrow, MT2's two launches for
    K = 128) and MT2's variable-size star plans (G = 7, 9, 11, 13, 14) write disjoint entries
    with fixed reduction orders: repeated calls are equal bit for bit."""
    a = xl.Array.ula(9000, 100e9)
    pos = xl.gen_drops_rect((1.0, 10.0), (-7.5, 7.5), K, 40, seed=41)
    p = xl.FP32 if prec == "fp32" else xl.FP64
    g1 = xl.gram_exact(a, pos, precision=p)
    g2 = xl.gram_exact(a, pos, precision=p)
    assert torch.equal(g1, g2)
