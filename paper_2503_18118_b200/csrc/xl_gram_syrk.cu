// xl_gram_syrk.cu -- exact fp64 Gram for large K (a2 + a3: Eq. (3), the
// inner products of H^H H PAPER.md:74, 240, 273) as a chunked Hermitian rank-k update:
//
//   for each chunk of CH elements (a level of the nested sweep never straddles a chunk):
//     h_chunk_f64_kernel : H[b][u][e] = h_u(element c0 + e), fp64 complex, users padded
//                          to K_pad = 32 nt with zero rows (B drops x K_pad x CH x 16 B,
//                          sized to stay L2-resident);
//     gram_syrk_kernel   : per (drop, 32 x 32 tile pair ti <= tj, element quarter) one
//                          warp accumulates C += H_ti H_tj^H on DMMA (xl_dmma_tile.cuh)
//                          into its partial tile;
//   gram_syrk_reduce_kernel : G(i, j) = conj(sum of the partials), prefix over levels,
//                          Hermitian mirror, Im diag = 0.
//
// Against the block-pair kernel (gram_blk_kernel, xl_gram.cu), which regenerates both
// 64-user blocks of every block pair (17x redundant generation at K = 1000), every
// coefficient is generated once per drop; the price is the chunk round trip through L2.
#include <cstring>
#include <type_traits>

#include "xl_common.cuh"
#include "xl_dmma_tile.cuh"

namespace {
using namespace xlt;

struct SyrkP {
  const double *pos;
  int K, Kp;
  int64_t n_y, n_z, N;  // N: last level end (parity of the ULA centred order)
  double inv_lambda, pitch, sqrt_beta0;
};

struct SyrkPlan {
  int Kp, nt, npairs, CH, nsub, B;
};

constexpr int kSyrkWarps = 8;
// Complex products in the 3M form on half tiles (column halves), as MT2: three DMMAs per
// fragment pair instead of four.  E3 field, ms (4M -> 3M): K = 160 89.8 -> 83.6, 256 59.1
// -> 54.7, 1000 82.6 -> 73.4 (tools/ab_syrk.py); row halves (2) 74.9 at K = 1000.  0: 4M.
#ifndef XL_SYRK_3M
#define XL_SYRK_3M 1
#endif

// Batch size B (drops), chunk CH = nsub x chs elements: the items of one SYRK launch
// (B x tile pairs x nsub, one warp each, 8 per SM) should fill whole waves of the
// 148 x 8 warp slots (a launch drains before the next chunk), items should be long
// against the C-tile round trip (~8 k-steps), and the H chunk (B x K_pad x CH x 16 B)
// should stay within 64 MB of L2.
SyrkPlan syrk_plan(int K, int64_t n_drops) {
  SyrkPlan p;
  p.Kp = (K + kTile - 1) / kTile * kTile;
  p.nt = p.Kp / kTile;
  p.npairs = p.nt * (p.nt + 1) / 2;
  const int64_t slots = 148 * kSyrkWarps;
  const int64_t cap = 64ll << 20;
  double best = -1.0;
  p.B = 1;
  p.nsub = 4;
  p.CH = 1024;
  const int64_t bmax = n_drops < 64 ? (n_drops < 1 ? 1 : n_drops) : 64;
  for (int64_t B = 1; B <= bmax; ++B)
    for (int nsub = 1; nsub <= 32; ++nsub)
      for (int chs = 128; chs <= 512; chs += 64) {
        const int64_t CH = (int64_t)nsub * chs;
        if (CH < 1024 || CH > 4096 || B * p.Kp * CH * (int64_t)sizeof(double2) > cap) continue;
        const int64_t items = B * p.npairs * nsub;
        const int64_t waves = (items + slots - 1) / slots;
        const double score = (double)items / (double)(waves * slots) * (chs / 4.0) / (chs / 4.0 + 8.0);
        if (score > best + 1e-9) {
          best = score;
          p.B = (int)B;
          p.nsub = nsub;
          p.CH = (int)CH;
        }
      }
  return p;
}

size_t al256(size_t x) { return (x + 255) / 256 * 256; }

template <int KIND>
__global__ void __launch_bounds__(256) h_chunk_f64_kernel(SyrkP P, int64_t drop0, int64_t c0, int64_t c1, int CH,
                                                          double2 *H) {
  const int64_t row = blockIdx.x;  // b * Kp + u
  const int b = (int)(row / P.Kp), u = (int)(row - (int64_t)b * P.Kp);
  const bool active = u < P.K;
  xl::UserC uc = {1.0, 0.0, 0.0, 0.0};
  if (active) uc = xl::make_user(P.pos + ((drop0 + b) * P.K + u) * 3, KIND, P.sqrt_beta0);
  const double c4 = 4.0 * P.inv_lambda;
  const bool n_odd = (P.N & 1) != 0;
  double2 *out = H + row * CH;
  const double ny0 = 0.5 * (double)(P.n_y - 1), nz0 = 0.5 * (double)(P.n_z - 1);
  for (int e = threadIdx.x; e < CH; e += blockDim.x) {
    const int64_t t = c0 + e;
    double hr = 0.0, hi = 0.0;
    if (active && t < c1) {
      double r2;
      if (KIND == XLMIMO_ULA) {
        const double dy = xl::ula_y_centred(t, n_odd, P.pitch) - uc.y;
        r2 = fma(dy, dy, uc.xz2);
      } else {  // N < 2^31 (checked on the host)
        const uint32_t tt = (uint32_t)t, ny = (uint32_t)P.n_y;
        const uint32_t q = tt / ny, pp = tt - q * ny;
        const double dy = ((double)pp - ny0) * P.pitch - uc.y;
        const double dz = ((double)q - nz0) * P.pitch - uc.z;
        r2 = fma(dz, dz, fma(dy, dy, uc.xz2));
      }
      xl::coef_fast(r2, uc.amp, c4, hr, hi);
    }
    out[e] = make_double2(hr, hi);
  }
}

__device__ __forceinline__ void pair_decode(int p, int nt, int &ti, int &tj) {
  int i = 0;
  while (p >= nt - i) {
    p -= nt - i;
    ++i;
  }
  ti = i;
  tj = i + p;
}

// item = ((b * nsub + sub) * npairs + pair): the warps of a CTA share sub and mostly ti,
// so their A rows coincide.  partial[b][lvl][sub][pair][32][32] (row-major) += H_ti H_tj^H
// over the chunk's elements [sub CH/nsub, (sub + 1) CH/nsub).
__global__ void __launch_bounds__(32 * kSyrkWarps, 1)
    gram_syrk_kernel(const double2 *__restrict__ H, int K, int Kp, int nt, int CH, int nsub, int npairs,
                     int64_t n_items, int lvl, int n_lvl, double2 *partial) {
  const int lane = threadIdx.x & 31;
  const int64_t item = (int64_t)blockIdx.x * kSyrkWarps + (threadIdx.x >> 5);
  if (item >= n_items) return;
  const int pair = (int)(item % npairs);
  const int64_t bs = item / npairs;
  const int sub = (int)(bs % nsub);
  const int64_t b = bs / nsub;
  int ti, tj;
  pair_decode(pair, nt, ti, tj);
  const int chs = CH / nsub;
  const double2 *A = H + ((size_t)b * Kp + (size_t)ti * kTile) * CH + (size_t)sub * chs;
  const double2 *Bm = H + ((size_t)b * Kp + (size_t)tj * kTile) * CH + (size_t)sub * chs;
  double2 *pt = partial + ((((size_t)b * n_lvl + lvl) * nsub + sub) * npairs + pair) * (kTile * kTile);
  // the last tile holds K - 32 (nt - 1) users: only its first v row/column fragments
  // are computed (8 v >= its users; the rest of the partial stays 0 and is never read)
  const int v = (K - (nt - 1) * kTile + 7) / 8;
  const bool lj = tj == nt - 1, li = ti == nt - 1;
  auto run = [&](auto mb, auto nb) {
    constexpr int MB = decltype(mb)::value, NB = decltype(nb)::value;
#if XL_SYRK_3M
    // 3M on half tiles (three accumulator sets of a 32 x 32 tile do not fit the registers),
    // added into the partial in memory
#if XL_SYRK_3M == 2  // halves along the rows
    constexpr int MBA = MB < 2 ? MB : 2, MBB = MB - MBA;
    ctile_mma3m_nt<MBA, NB, 0, 0, 8>(pt, kTile, A, CH, Bm, CH, chs / 4, lane);
    if constexpr (MBB > 0) ctile_mma3m_nt<MBB, NB, MBA, 0, 8>(pt, kTile, A, CH, Bm, CH, chs / 4, lane);
#else
    constexpr int NBA = NB < 2 ? NB : 2, NBB = NB - NBA;
    ctile_mma3m_nt<MB, NBA, 0, 0, 8>(pt, kTile, A, CH, Bm, CH, chs / 4, lane);
    if constexpr (NBB > 0) ctile_mma3m_nt<MB, NBB, 0, NBA, 8>(pt, kTile, A, CH, Bm, CH, chs / 4, lane);
#endif
#else
    CTile c;
    ctile_load<false, MB, NB>(c, pt, kTile, lane);
    ctile_mma<true, true, true, MB, NB, 8>(c, A, CH, Bm, CH, chs / 4, lane);  // long slices: prefetch 8 ahead
    ctile_store<false, MB, NB>(c, pt, kTile, lane);
#endif
  };
  using I1 = std::integral_constant<int, 1>;
  using I2 = std::integral_constant<int, 2>;
  using I3 = std::integral_constant<int, 3>;
  using I4 = std::integral_constant<int, 4>;
  if (!lj || v == 4) run(I4{}, I4{});
  else if (!li) {
    if (v == 1) run(I4{}, I1{});
    else if (v == 2) run(I4{}, I2{});
    else run(I4{}, I3{});
  } else {
    if (v == 1) run(I1{}, I1{});
    else if (v == 2) run(I2{}, I2{});
    else run(I3{}, I3{});
  }
}

// block (b, row i): threads over j >= i
__global__ void __launch_bounds__(256) gram_syrk_reduce_kernel(const double2 *__restrict__ partial, int K, int nt,
                                                               int nsub, int npairs, int n_lvl, double *out) {
  const int64_t b = blockIdx.x / K;
  const int i = (int)(blockIdx.x - b * K);
  const int ti = i / kTile, ri = i % kTile;
  for (int j = i + threadIdx.x; j < K; j += blockDim.x) {
    const int tj = j / kTile;
    const int pair = ti * nt - ti * (ti - 1) / 2 + (tj - ti);
    const int off = ri * kTile + (j % kTile);
    double re = 0.0, im = 0.0;
    for (int l = 0; l < n_lvl; ++l) {
      for (int sb = 0; sb < nsub; ++sb) {
        const double2 v = partial[((((size_t)b * n_lvl + l) * nsub + sb) * npairs + pair) * (kTile * kTile) + off];
        re += v.x;
        im += v.y;
      }
      // G(i, j) = sum conj(h_i) h_j = conj(C(i, j))
      double *g = out + ((size_t)b * n_lvl + l) * (size_t)K * K * 2;
      g[((size_t)i * K + j) * 2] = re;
      g[((size_t)i * K + j) * 2 + 1] = (i == j) ? 0.0 : -im;
      g[((size_t)j * K + i) * 2] = re;
      g[((size_t)j * K + i) * 2 + 1] = (i == j) ? 0.0 : im;
    }
  }
}

}  // namespace

namespace xlh {

size_t gram_syrk_ws_bytes(int K, int64_t n_drops, int n_lvl) {
  if (n_drops <= 0) return 0;
  const SyrkPlan p = syrk_plan(K, n_drops);
  return al256((size_t)p.B * p.Kp * p.CH * sizeof(double2)) +
         al256((size_t)p.B * n_lvl * p.nsub * p.npairs * kTile * kTile * sizeof(double2));
}

int launch_gram_syrk(const ArrayP &a, const double *pos, int K, int64_t n_drops, const int64_t *lvl_end, int n_lvl,
                     double *out, void *ws, size_t ws_bytes, cudaStream_t s) {
  if (n_drops == 0) return XLMIMO_OK;
  const size_t need = gram_syrk_ws_bytes(K, n_drops, n_lvl);
  if (ws_bytes < need || !ws) return set_error(XLMIMO_EWORKSPACE, "gram: workspace %zu < %zu bytes", ws_bytes, need);
  const SyrkPlan p = syrk_plan(K, n_drops);
  if (a.kind != XLMIMO_ULA && lvl_end[n_lvl - 1] >= ((int64_t)1 << 31))
    return set_error(XLMIMO_EUNSUPPORTED, "gram_exact: a UPA with K > 64 needs N < 2^31");
  SyrkP P;
  P.pos = pos;
  P.K = K;
  P.Kp = p.Kp;
  P.n_y = a.n_y;
  P.n_z = a.kind == XLMIMO_ULA ? 1 : a.n_z;
  P.N = lvl_end[n_lvl - 1];
  P.inv_lambda = 1.0 / a.lambda;
  P.pitch = a.pitch;
  P.sqrt_beta0 = a.sqrt_beta0;
  double2 *H = (double2 *)ws;
  double2 *partial = (double2 *)((char *)ws + al256((size_t)p.B * p.Kp * p.CH * sizeof(double2)));
  const size_t part_bytes = (size_t)p.B * n_lvl * p.nsub * p.npairs * kTile * kTile * sizeof(double2);
  for (int64_t d0 = 0; d0 < n_drops; d0 += p.B) {
    const int nb = (int)((n_drops - d0) < p.B ? (n_drops - d0) : p.B);
    P.pos = pos;
    if (cudaMemsetAsync(partial, 0, part_bytes, s) != cudaSuccess) return check_launch("gram_syrk memset");
    int64_t lv0 = 0;
    for (int l = 0; l < n_lvl; ++l) {
      const int64_t lv1 = lvl_end[l];
      for (int64_t c0 = lv0; c0 < lv1; c0 += p.CH) {
        const int64_t c1 = (lv1 - c0) < p.CH ? lv1 : c0 + p.CH;
        {
          KTimer tm(s, "gram_syrk_h_chunk_fp64");
          const unsigned grid = (unsigned)(nb * p.Kp);
          if (a.kind == XLMIMO_ULA)
            h_chunk_f64_kernel<XLMIMO_ULA><<<grid, 256, 0, s>>>(P, d0, c0, c1, p.CH, H);
          else
            h_chunk_f64_kernel<XLMIMO_UPA><<<grid, 256, 0, s>>>(P, d0, c0, c1, p.CH, H);
          tm.stop(s);
          count_launch();
        }
        {
          KTimer tm(s, "gram_syrk_dmma_fp64");
          const int64_t n_items = (int64_t)nb * p.nsub * p.npairs;
          gram_syrk_kernel<<<(unsigned)((n_items + kSyrkWarps - 1) / kSyrkWarps), 32 * kSyrkWarps, 0, s>>>(
              H, K, p.Kp, p.nt, p.CH, p.nsub, p.npairs, n_items, l, n_lvl, partial);
          tm.stop(s);
          count_launch();
        }
        const int rc = check_launch("gram_syrk kernels");
        if (rc) return rc;
      }
      lv0 = lv1;
    }
    KTimer tr(s, "gram_reduce");
    gram_syrk_reduce_kernel<<<(unsigned)(nb * K), 256, 0, s>>>(partial, K, p.nt, p.nsub, p.npairs, n_lvl,
                                                             out + (size_t)d0 * n_lvl * K * K * 2);
    tr.stop(s);
    count_launch();
    const int rc = check_launch("gram_syrk_reduce_kernel");
    if (rc) return rc;
  }
  return XLMIMO_OK;
}

}  // namespace xlh
