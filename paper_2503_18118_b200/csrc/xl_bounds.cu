// xl_bounds.cu -- NEXT-3: Appendix A per drop, the large-K
// (K > 64) log-determinant path shared with the receivers, and the eigenvalues of
// the correlation matrix R.
//
// Per drop, with a_i = rho G_ii (the diagonal of (P/sigma_n^2) H^H H):
//   log2 U = sum_i log2(1 + a_i)              Hadamard upper bound
//   R_ij   = G_ij / sqrt(G_ii G_jj)           correlation matrix
//   log2 L = log2 det R + log2 U              Schur-Horn lower bound
//   C      = log2 det(I + rho G)              the capacity they bracket (Eq. (9))
//   gap    = -log2 det(R) / K                 max normalised gap, Eq. (eq9)
// log2 det comes from a Cholesky factor (2 sum log2 L_kk); a pivot that is not > 0
// marks the matrix not positive definite (R10).
//
// Kernels
//  * bounds_warp_kernel (K <= 64): one warp per drop, the packed lower triangle in
//    shared memory, the same warp Cholesky as the receivers.
//  * chol_smem_kernel (64 < K <= 96): one CTA per matrix, packed lower triangle in
//    shared memory, unblocked right-looking Cholesky.
//  * chol_tiled_kernel (K > 96): one CTA per matrix in a global workspace slot, two
//    CTAs per SM, tiled Cholesky with 32 x 32 complex tiles on DMMA (panel groups of
//    4, inverted diagonal tiles).  O(K^3/6) complex MACs per matrix; with dinv the
//    blocked inverse L^{-1} (another K^3/6) on the same tile products.
//  * finish kernels: one CTA per drop; scan G (finite, positive diagonal), log2 U /
//    MRC from G, assemble outputs and flags.
//  * eig_jacobi_kernel (K <= 64): eigenvalues of R by the parallel (round-robin)
//    cyclic Jacobi method, one warp per drop, lane = one disjoint (p, q) pair per
//    round; each rotation first makes A_pq real by a phase on column/row q, then
//    zeroes it with the real plane rotation (t = sgn(theta)/(|theta| + sqrt(theta^2+1)),
//    theta = (a_qq - a_pp)/(2|a_pq|)).
#include <cstdio>
#include <cstring>

#include "xl_common.cuh"
#include "xl_dmma_tile.cuh"
#include "xl_linalg.cuh"

namespace {
using namespace xlt;

constexpr int kCtaThreads = 256;
constexpr double kNaN = __builtin_nan("");

struct BoundsParams {
  const double *gram;
  double *rstat;   // [D][2]
  double *bounds;  // [D][S][3]
  uint32_t *flags;
  int K;
  int64_t n_drops;
  int n_snr;
  double rho[xl::kMaxSnr];
};

// ------------------------------------------------------------------ K <= 64
template <int RPL>
__global__ void __launch_bounds__(256) bounds_warp_kernel(BoundsParams P) {
  extern __shared__ double2 smem[];
  const int K = P.K;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double2 *As = smem + (size_t)warp * (K * (K + 1) / 2);  // packed lower triangle (xl_linalg.cuh)
  const int64_t d = (int64_t)blockIdx.x * nw + warp;
  if (d >= P.n_drops) return;
  const double2 *G = reinterpret_cast<const double2 *>(P.gram) + (size_t)d * K * K;
  double *rs = P.rstat + 2 * d, *bo = P.bounds + (size_t)d * P.n_snr * 3;
  uint32_t fl = 0;

  bool fin = true, dpos = true;
  for (int e = lane; e < K * K; e += 32) fin &= isfinite(G[e].x) && isfinite(G[e].y);
  for (int i = lane; i < K; i += 32) dpos &= G[i * K + i].x > 0.0;
  fin = __all_sync(0xffffffffu, fin);
  dpos = __all_sync(0xffffffffu, dpos);
  if (!fin || !dpos) {
    if (lane < 2) rs[lane] = kNaN;
    for (int e = lane; e < 3 * P.n_snr; e += 32) bo[e] = kNaN;
    if (lane == 0 && P.flags) P.flags[d] = fin ? XLMIMO_FLAG_MRC_UNDEF : XLMIMO_FLAG_NONFINITE;
    return;
  }
  // R, packed lower: R_ij = conj(R_ji) = conj(G_ji) / sqrt(G_ii G_jj), unit diagonal
  for (int j = 0; j < K; ++j) {
    const int oj = xlk::poff(K, j);
    for (int i = j + lane; i < K; i += 32) {
      const double2 g = G[j * K + i];
      const double s = rsqrt(G[i * K + i].x) * rsqrt(G[j * K + j].x);
      As[oj + i - j] = (i == j) ? make_double2(1.0, 0.0) : make_double2(g.x * s, -g.y * s);
    }
  }
  __syncwarp();
  double ldr = kNaN;
  if (xlk::warp_cholesky_packed<RPL>(As, K, lane)) {
    double part = 0.0;
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int k = lane + 32 * r;
      if (k < K) part += 2.0 * log2(As[xlk::poff(K, k)].x);
    }
    ldr = xlk::warp_sum(part);
  } else {
    fl |= XLMIMO_FLAG_G_NOT_PD;
  }
  if (lane == 0) {
    rs[0] = ldr;
    rs[1] = -ldr / (double)K;
  }
  for (int s = 0; s < P.n_snr; ++s) {
    const double rho = P.rho[s];
    double lu = 0.0;
    for (int i = lane; i < K; i += 32) lu += log2(1.0 + rho * G[i * K + i].x);
    lu = xlk::warp_sum(lu);
    __syncwarp();
    for (int j = 0; j < K; ++j) {
      const int oj = xlk::poff(K, j);
      for (int i = j + lane; i < K; i += 32) {
        const double2 g = G[j * K + i];
        As[oj + i - j] = (i == j) ? make_double2(1.0 + rho * g.x, 0.0) : make_double2(rho * g.x, -rho * g.y);
      }
    }
    __syncwarp();
    double cap = kNaN;
    if (xlk::warp_cholesky_packed<RPL>(As, K, lane)) {
      double part = 0.0;
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        const int k = lane + 32 * r;
        if (k < K) part += 2.0 * log2(As[xlk::poff(K, k)].x);
      }
      cap = xlk::warp_sum(part);
    } else {
      fl |= XLMIMO_FLAG_A_NOT_PD;
    }
    if (lane == 0) {
      bo[3 * s + 0] = lu;
      bo[3 * s + 1] = cap;
      bo[3 * s + 2] = ldr + lu;
    }
  }
  if (lane == 0 && P.flags) P.flags[d] = fl;
}

// ------------------------------------------------------------------ K > 64: log-determinants
// Problem p = (drop d, matrix m): m = 0 .. n_mat-1.  first_is_r: m == 0 builds R (App. A);
// every other m builds alpha_m I + rho_m G (I + rho G for CAP/MMSE, G for ZF).
// log2det[p] = log2 det (NaN if not PD / not built); dinv[p][i] = [A^{-1}]_ii when
// requested (shared-memory kernel only).
struct CholParams {
  const double *gram;
  double2 *ws;       // tiled kernel: [n_slots][Kp][Kp]
  double *log2det;   // [n_prob]
  double *dinv;      // [n_prob][K] or null
  double2 *xscr;     // tiled + dinv: per slot [8 warps][Kp][32] column panels of L^{-1}
  double2 *dvs;      // tiled + dinv: per slot [nt][32][32] inverses of the diagonal tiles
  int K, Kp, nt;
  int64_t n_prob;
  int n_mat;         // matrices per drop
  int first_is_r;    // matrix 0 of each drop is R
  double rho[xl::kMaxSnr + 2];    // rho of matrix m (unused for R)
  double alpha[xl::kMaxSnr + 2];  // identity weight of matrix m
};

// value (i, j) of problem matrix (R or alpha I + rho G), i, j < K
__device__ __forceinline__ double2 chol_entry(const double2 *G, int K, int i, int j, bool is_r, double rho,
                                              double alpha, bool &good) {
  const double2 g = G[(size_t)i * K + j];
  good &= isfinite(g.x) && isfinite(g.y);
  if (is_r) {
    const double gi = G[(size_t)i * K + i].x, gj = G[(size_t)j * K + j].x;
    good &= gi > 0.0 && gj > 0.0;
    if (i == j) return make_double2(1.0, 0.0);
    const double s = rsqrt(gi) * rsqrt(gj);
    return make_double2(g.x * s, g.y * s);
  }
  return (i == j) ? make_double2(alpha + rho * g.x, 0.0) : make_double2(rho * g.x, rho * g.y);
}

// 64 < K <= kSmemMaxK: one CTA per matrix, the packed lower triangle resident in shared
// memory (column-major packed: column j holds rows j..K-1 at off(j) = jK - j(j-1)/2),
// unblocked right-looking Cholesky: per column j the pivot, the column scaled by
// 1/L_jj, and the rank-1 update of the trailing triangle with warps over columns and
// lanes over rows (contiguous, conflict-free).
// With dinv requested, [A^{-1}]_ii = ||L^{-1} e_i||^2 follows: warp per i, forward
// substitution L x = e_i with x_m held by lane m % 32 (register slot m / 32), the
// pivot element broadcast by shuffle, the column of L read from shared memory.
constexpr int kSmemK = 160;
// Largest K on the shared-memory kernel: the tiled DMMA kernel wins from K ~ 100 on
// (1000 CAP + ZF + MMSE receivers, ms smem / tiled: K = 72 1.09 / 1.57, 100 2.56 / 2.42,
// 128 6.43 / 2.43, 160 10.05 / 3.50; tools/ab_chol.py).
#ifndef XL_CHOL_SMEM_MAXK
#define XL_CHOL_SMEM_MAXK 96
#endif
constexpr int kSmemMaxK = XL_CHOL_SMEM_MAXK;
constexpr int kSmemRpl = (kSmemK + 31) / 32;

__global__ void __launch_bounds__(kCtaThreads) chol_smem_kernel(CholParams P) {
  extern __shared__ double2 Ls[];
  __shared__ double s_inv[kSmemK];  // 1 / L_jj
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = kCtaThreads / 32;
  const int K = P.K;
  auto off = [K](int j) { return j * K - j * (j - 1) / 2; };
  for (int64_t prob = blockIdx.x; prob < P.n_prob; prob += gridDim.x) {
    const int64_t d = prob / P.n_mat;
    const int m = (int)(prob - d * P.n_mat);
    const bool is_r = P.first_is_r && m == 0;
    const double2 *G = reinterpret_cast<const double2 *>(P.gram) + (size_t)d * K * K;
    bool good = true;
    // column j of the lower triangle = conj of row j of G (coalesced reads)
    for (int j = warp; j < K; j += NW)
      for (int i = j + lane; i < K; i += 32) {
        const double2 v = chol_entry(G, K, j, i, is_r, P.rho[m], P.alpha[m], good);
        Ls[off(j) + i - j] = make_double2(v.x, -v.y);
      }
    const int ok0 = __syncthreads_and(good ? 1 : 0);
    double ld = 0.0;
    bool ok = ok0 != 0;
    for (int j = 0; j < K && ok; ++j) {
      const int oj = off(j);
      const double piv = Ls[oj].x;  // every thread reads the same value: uniform branch
      if (!(piv > 0.0) || !isfinite(piv)) {
        ok = false;
        break;
      }
      const double ljj = sqrt(piv), inv = 1.0 / ljj;
      if (tid == 0) {
        ld += 2.0 * log2(ljj);
        s_inv[j] = inv;
      }
      __syncthreads();  // all pivot reads done before the column is rescaled
      for (int i = j + tid; i < K; i += kCtaThreads) {
        double2 v = Ls[oj + i - j];
        Ls[oj + i - j] = (i == j) ? make_double2(ljj, 0.0) : make_double2(v.x * inv, v.y * inv);
      }
      __syncthreads();
      // A_ic -= L_ij conj(L_cj), j < c <= i
      for (int c = j + 1 + warp; c < K; c += NW) {
        const double2 lc = Ls[oj + c - j];
        const int oc = off(c);
        for (int i = c + lane; i < K; i += 32) {
          const double2 li = Ls[oj + i - j];
          double2 a = Ls[oc + i - c];
          a.x -= li.x * lc.x + li.y * lc.y;
          a.y -= li.y * lc.x - li.x * lc.y;
          Ls[oc + i - c] = a;
        }
      }
      __syncthreads();
    }
    if (tid == 0) P.log2det[prob] = ok ? ld : kNaN;
    if (P.dinv) {
      double *dout = P.dinv + (size_t)prob * K;
      for (int i = warp; i < K; i += NW) {
        if (!ok) {
          if (lane == 0) dout[i] = kNaN;
          continue;
        }
        double xr[kSmemRpl], xi[kSmemRpl];
#pragma unroll
        for (int r = 0; r < kSmemRpl; ++r) {
          xr[r] = (lane + 32 * r == i) ? 1.0 : 0.0;
          xi[r] = 0.0;
        }
        double sum = 0.0;
        for (int k = i; k < K; ++k) {
          const int rk = k >> 5;
          double vr = 0.0, vi = 0.0;
#pragma unroll
          for (int r = 0; r < kSmemRpl; ++r)
            if (r == rk) {
              vr = xr[r];
              vi = xi[r];
            }
          vr = __shfl_sync(0xffffffffu, vr, k & 31) * s_inv[k];
          vi = __shfl_sync(0xffffffffu, vi, k & 31) * s_inv[k];
          sum += vr * vr + vi * vi;
          const int ok2 = off(k);
#pragma unroll
          for (int r = 0; r < kSmemRpl; ++r) {
            const int mm = lane + 32 * r;
            if (mm > k && mm < K) {
              const double2 l = Ls[ok2 + mm - k];  // L_mk
              xr[r] -= l.x * vr - l.y * vi;
              xi[r] -= l.x * vi + l.y * vr;
            }
          }
        }
        if (lane == 0) dout[i] = sum;
      }
    }
    __syncthreads();
  }
}

// K > kSmemMaxK: one CTA per matrix in a global workspace slot (K_pad = 32 nt, row-major,
// lower triangle used), tiled Cholesky with 32 x 32 complex tiles, panels in groups of
// kGrp = 8 (left-looking inside a group, right-looking between groups):
//  (0) the tiles of column k take the group's earlier panels: A_ik -= L_i,G' L_k,G'^H;
//  (1) warp 0 factors the diagonal tile in shared memory and inverts it (lane = column);
//  (2) panel X_ik = A_ik L_kk^{-H}, one tile product per warp;
//  (3) after the group, every trailing tile A_ij -= L_i,G L_j,G^H once (inner dimension
//      128), tiles flattened over the warps (no per-column barrier).
// Every tile product runs on the FP64 tensor path: per 4-wide k-step 4 x 4 fragment
// pairs x 4 real DMMA m8n8k4 (RR, II, IR, RI), the 64 accumulator registers of the
// complex tile resident, operand fragments read straight from the slot (L2, prefetched
// PFD k-steps ahead) with a one-step register double buffer.  DMMA and DFMA share
// the FP64 pipe at the same FMA rate; the tensor path needs one
// instruction per 256 FMAs and no shared-memory operand traffic.
#ifndef XB_GRP
#define XB_GRP 8  // measured K = 1000: 2 -> 20.3 ms, 4 -> 18.5, 8 / 12 / 16 -> 17.8
#endif
constexpr int kGrp = XB_GRP;     // panels per trailing update
constexpr int kLdY = kTile + 2;  // per-warp Y tile row stride (conflict-free B-fragment reads)
constexpr int kLdI = kTile + 4;  // L_kk^{-1} row stride (conflict-free B_NT fragment reads)
// Two CTAs of 4 warps per SM, each on its own matrix: one CTA's serial steps (diagonal
// factor, barriers) overlap the other's tensor work.
constexpr int kTiledThreads = 128;
constexpr int kTiledPerSm = 2;
constexpr size_t kTiledSmem = (size_t)(kTiledThreads / 32) * kTile * kLdY * sizeof(double2);

__global__ void __launch_bounds__(kTiledThreads, kTiledPerSm) chol_tiled_kernel(CholParams P) {
  extern __shared__ double2 tsm[];       // per-warp Y tiles [8][32][kLdY]
  __shared__ double2 T[kTile * kTile];   // diagonal tile, column-major T[c*32 + r]
  __shared__ double2 LI[kTile * kLdI];   // its inverse, row-major
  __shared__ int s_ok, s_next;
  __shared__ double s_ld;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = kTiledThreads / 32;
  const int K = P.K, Kp = P.Kp, nt = P.nt;
  double2 *A = P.ws + (size_t)blockIdx.x * Kp * Kp;
  double2 *W = tsm + warp * kTile * kLdY;
#ifdef XB_PROF
  long long pt[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tl = clock64();
#define XB_T(i)                      \
  if (tid == 0) {                    \
    const long long t_ = clock64();  \
    pt[i] += t_ - tl;                \
    tl = t_;                         \
  }
#else
#define XB_T(i)
#endif

  for (int64_t prob = blockIdx.x; prob < P.n_prob; prob += gridDim.x) {
    const int64_t d = prob / P.n_mat;
    const int m = (int)(prob - d * P.n_mat);
    const bool is_r = P.first_is_r && m == 0;
    const double2 *G = reinterpret_cast<const double2 *>(P.gram) + (size_t)d * K * K;
    bool good = true;
    // lower triangle of the problem matrix (identity padding), 8 row loads in flight per
    // lane; R scales by 1/sqrt(G_ii G_jj) from a table in the (idle) Y-tile memory
    double *sd = reinterpret_cast<double *>(tsm);
    if (is_r) {
      for (int j = tid; j < K; j += kTiledThreads) {
        const double g = G[(size_t)j * K + j].x;
        good &= g > 0.0;
        sd[j] = rsqrt(g);
      }
      __syncthreads();
    }
    const double rho = P.rho[m], alpha = P.alpha[m];
    for (int i = warp; i < Kp; i += NW) {
      const double si = (is_r && i < K) ? sd[i] : 0.0;
      for (int j0 = 0; j0 <= i; j0 += 256) {
        double2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int j = j0 + 32 * u + lane;
          v[u] = (i < K && j <= i) ? G[(size_t)i * K + j] : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int j = j0 + 32 * u + lane;
          if (j > i) continue;
          double2 w = v[u];
          if (i >= K) {
            w = make_double2(i == j ? 1.0 : 0.0, 0.0);
          } else {
            good &= isfinite(w.x) && isfinite(w.y);
            if (is_r) {
              const double sc = si * sd[j];
              w = (i == j) ? make_double2(1.0, 0.0) : make_double2(w.x * sc, w.y * sc);
            } else {
              w = (i == j) ? make_double2(alpha + rho * w.x, 0.0) : make_double2(rho * w.x, rho * w.y);
            }
          }
          A[(size_t)i * Kp + j] = w;
        }
      }
    }
    const int ok0 = __syncthreads_and(good ? 1 : 0);
    if (tid == 0) {
      s_ok = ok0;
      s_ld = 0.0;
      s_next = 0;
    }
    __syncthreads();
    XB_T(0)
    // s_ok is only read right after the barrier that follows its one writer (step 1),
    // so every warp sees the same value and leaves the loop together.
    // Panels in groups of kGrp: column k of a group first takes the updates of the
    // group's earlier panels (left-looking), is factored (1) and solved (2); the
    // trailing tiles then take the whole group at once (3), so each trailing tile is
    // read and written once per group, with an inner dimension of 32 kGrp.
    for (int g0 = 0; g0 < nt && ok0; g0 += kGrp) {
      const int g1 = min(g0 + kGrp, nt);
      for (int k = g0; k < g1; ++k) {
        const int k0 = k * kTile;
        if (k > g0) {  // tiles (i, k), i >= k: A_ik -= L_i,[g0,k) L_k,[g0,k)^H
          const int nkb = (k - g0) * (kTile / 4);
          for (int i = k + warp; i < nt; i += NW) {
            const int i0 = i * kTile;
            if (i + NW < nt) tile_prefetch_l2(A + (size_t)(i0 + NW * kTile) * Kp + k0, Kp, lane);
            CTile c;
            ctile_load<true>(c, A + (size_t)i0 * Kp + k0, Kp, lane);  // -A_ik += L L^H
            ctile_mma<true, true, true>(c, A + (size_t)i0 * Kp + g0 * kTile, Kp, A + (size_t)k0 * Kp + g0 * kTile,
                                        Kp, nkb, lane);
            ctile_store<true>(c, A + (size_t)i0 * Kp + k0, Kp, lane);
          }
          __syncthreads();
          XB_T(1)
        }
        if (warp == 0) {  // (1)
          {
            double2 v[kTile];  // all 32 loads in flight (the tile is in L2)
#pragma unroll
            for (int c = 0; c < kTile; ++c) v[c] = A[(size_t)(k0 + lane) * Kp + k0 + c];
#pragma unroll
            for (int c = 0; c < kTile; ++c) T[c * kTile + lane] = (lane >= c) ? v[c] : make_double2(0.0, 0.0);
          }
          const bool okf = xlk::warp_cholesky<1>(T, kTile, lane);
          if (okf && P.dinv)  // the inverse phase reads L_kk back from the slot
            for (int c = 0; c <= lane; ++c) A[(size_t)(k0 + lane) * Kp + k0 + c] = T[c * kTile + lane];
          if (okf) {  // L_kk^{-1} by lane = column c: x_r = (delta_rc - sum_{m<r} L_rm x_m) / L_rr
            double2 x[kTile];
#pragma unroll
            for (int r = 0; r < kTile; ++r) {
              double xr = (r == lane) ? 1.0 : 0.0, xi = 0.0;
#pragma unroll
              for (int mm = 0; mm < r; ++mm) {
                const double2 l = T[mm * kTile + r];  // L_r,mm
                xr -= l.x * x[mm].x - l.y * x[mm].y;
                xi -= l.x * x[mm].y + l.y * x[mm].x;
              }
              const double inv = 1.0 / T[r * kTile + r].x;
              x[r] = make_double2(xr * inv, xi * inv);
            }
            double2 *dv = P.dinv ? P.dvs + ((size_t)blockIdx.x * nt + k) * kTile * kTile : nullptr;
#pragma unroll
            for (int r = 0; r < kTile; ++r) {
              LI[r * kLdI + lane] = x[r];
              if (dv) dv[r * kTile + lane] = x[r];  // row r, col lane (the inverse phase's Dinv_k)
            }
          }
          const double dg = T[lane * kTile + lane].x;
          const double part = okf ? 2.0 * log2(dg) : 0.0;
          const double sum = xlk::warp_sum(part);
          if (lane == 0) {
            if (okf) s_ld += sum;
            else s_ok = 0;
          }
        }
        __syncthreads();
        XB_T(2)
        if (!s_ok) break;
        // (2) panel X_ik = A_ik L_kk^{-H}, tiles i > k over the warps (DMMA, L_kk^{-1} in LI)
        for (int i = k + 1 + warp; i < nt; i += NW) {
          const int i0 = i * kTile;
          CTile c;
          ctile_zero(c);
          ctile_mma<true, true, false>(c, A + (size_t)i0 * Kp + k0, Kp, LI, kLdI, kTile / 4, lane);
          ctile_store<false>(c, A + (size_t)i0 * Kp + k0, Kp, lane);
        }
        __syncthreads();
        XB_T(3)
      }
      if (!s_ok) break;
      // (3) tiles (i, j) = (g1+ii, g1+jj), jj <= ii, row by row (warps that run together
      // share L_i,G): A_ij -= L_i,G L_j,G^H over the group's columns G = [g0, g1)
      const int nrem = nt - g1;
      const int npair = nrem * (nrem + 1) / 2;
      const int nkb = (g1 - g0) * (kTile / 4);
      auto decode = [&](int p, int &i0, int &j0) {
        int ii = (int)((sqrtf(8.0f * (float)p + 1.0f) - 1.0f) * 0.5f);
        while ((ii + 1) * (ii + 2) / 2 <= p) ++ii;
        while (ii * (ii + 1) / 2 > p) --ii;
        i0 = (g1 + ii) * kTile;
        j0 = (g1 + p - ii * (ii + 1) / 2) * kTile;
      };
      for (int p = warp; p < npair; p += NW) {
        int i0, j0;
        decode(p, i0, j0);
        if (p + NW < npair) {
          int pi0, pj0;
          decode(p + NW, pi0, pj0);
          tile_prefetch_l2(A + (size_t)pi0 * Kp + pj0, Kp, lane);
        }
        CTile c;
        ctile_load<true>(c, A + (size_t)i0 * Kp + j0, Kp, lane);  // -A_ij += L L^H
        ctile_mma<true, true, true>(c, A + (size_t)i0 * Kp + g0 * kTile, Kp, A + (size_t)j0 * Kp + g0 * kTile, Kp,
                                    nkb, lane);
        ctile_store<true>(c, A + (size_t)i0 * Kp + j0, Kp, lane);
      }
      __syncthreads();
      XB_T(4)
    }
    if (tid == 0) P.log2det[prob] = s_ok ? s_ld : kNaN;
    if (P.dinv) {
      // ---- [A^{-1}]_cc = sum_i |X_ic|^2, X = L^{-1}, by blocked forward substitution:
      // (a) Dinv_i = L_ii^{-1} for every diagonal tile: written by the factorisation;
      // (b) column blocks j handed out largest first by a shared counter:
      //     X_jj = Dinv_j, X_ij = -Dinv_i sum_{k=j}^{i-1} L_ik X_kj (DMMA tiles), the panel
      //     X_{.j} kept in the warp's global scratch, column norms accumulated.
      double *dout = P.dinv + (size_t)prob * K;
      const bool fact = s_ok != 0;
      double2 *Dv = P.dvs + (size_t)blockIdx.x * nt * kTile * kTile;
      __syncthreads();
      XB_T(5)
      double2 *Xp = P.xscr + ((size_t)blockIdx.x * NW + warp) * Kp * kTile;  // [row - j0][32]
      for (;;) {
        int j = 0;
        if (lane == 0) j = atomicAdd(&s_next, 1);
        j = __shfl_sync(0xffffffffu, j, 0);
        if (j >= nt) break;
        const int j0 = j * kTile;
        if (!fact) {
          if (j0 + lane < K) dout[j0 + lane] = kNaN;
          continue;
        }
        // X_jj = Dinv_j; lane c: column c norm
        double nrm = 0.0;
        for (int r = 0; r < kTile; ++r) {
          const double2 v = Dv[((size_t)j * kTile + r) * kTile + lane];
          Xp[(size_t)r * kTile + lane] = v;
          nrm += v.x * v.x + v.y * v.y;
        }
        double part[4][2];
#pragma unroll
        for (int nb = 0; nb < 4; ++nb) part[nb][0] = part[nb][1] = 0.0;
        __syncwarp();
        for (int i = j + 1; i < nt; ++i) {
          const int i0 = i * kTile;
          CTile c;
          ctile_zero(c);
          // Y = sum_{k=j}^{i-1} L_ik X_kj: L_i,[j,i) is contiguous in the row, X_[j,i),j in the panel
          ctile_mma<false, false, true>(c, A + (size_t)i0 * Kp + j0, Kp, Xp, kTile, (i - j) * (kTile / 4), lane);
          ctile_store<false>(c, W, kLdY, lane);  // Y -> shared
          __syncwarp();
          ctile_zero(c);  // X_ij = -Dinv_i Y
          ctile_mma<false, false, false>(c, Dv + (size_t)i * kTile * kTile, kTile, W, kLdY, kTile / 4, lane);
          ctile_store<true>(c, Xp + (size_t)(i - j) * kTile * kTile, kTile, lane);
#pragma unroll
          for (int mb = 0; mb < 4; ++mb)
#pragma unroll
            for (int nb = 0; nb < 4; ++nb)
#pragma unroll
              for (int e = 0; e < 2; ++e)
                part[nb][e] += c.r[mb][nb][e] * c.r[mb][nb][e] + c.i[mb][nb][e] * c.i[mb][nb][e];
          __syncwarp();
        }
        // column c = 8 nb + 2 qc + e: add the 8 row groups (lanes 4 qr + qc), then X_jj's part
#pragma unroll
        for (int nb = 0; nb < 4; ++nb)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            double v = part[nb][e];
            v += __shfl_xor_sync(0xffffffffu, v, 4);
            v += __shfl_xor_sync(0xffffffffu, v, 8);
            v += __shfl_xor_sync(0xffffffffu, v, 16);
            part[nb][e] = v;
          }
        // lane c gathers its column from lane qc = (c / 2) % 4, slot (nb, e) = (c / 8, c % 2)
        double tot = 0.0;
#pragma unroll
        for (int nb = 0; nb < 4; ++nb)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const double v = __shfl_sync(0xffffffffu, part[nb][e], (lane >> 1) & 3);
            if ((lane >> 3) == nb && (lane & 1) == e) tot = v;
          }
        if (j0 + lane < K) dout[j0 + lane] = nrm + tot;
        __syncwarp();
      }
    }
    __syncthreads();
    XB_T(6)
  }
#ifdef XB_PROF
  if (blockIdx.x == 0 && tid == 0)
    printf("chol_tiled phases (Mcycles, CTA 0): init %.2f left %.2f diag %.2f panel %.2f trail %.2f dinv_a %.2f dinv_b %.2f\n",
           pt[0] * 1e-6, pt[1] * 1e-6, pt[2] * 1e-6, pt[3] * 1e-6, pt[4] * 1e-6, pt[5] * 1e-6, pt[6] * 1e-6);
#endif
#undef XB_T
}

// scan one drop's Gram: finite entries and positive diagonal (block-wide)
__device__ void scan_gram(const double2 *G, int K, bool &fin, bool &dpos) {
  bool f = true, p = true;
  for (int64_t e = threadIdx.x; e < (int64_t)K * K; e += blockDim.x) f &= isfinite(G[e].x) && isfinite(G[e].y);
  for (int i = threadIdx.x; i < K; i += blockDim.x) p &= G[(size_t)i * K + i].x > 0.0;
  fin = __syncthreads_and(f ? 1 : 0) != 0;
  dpos = __syncthreads_and(p ? 1 : 0) != 0;
}

__device__ double block_sum(double v, double *red) {
  v = xlk::warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < nw; ++w) s += red[w];  // fixed order
  return s;
}


// ------------------------------------------------------------------ eigenvalues of R (64 < K <= 1024)
// One CTA per matrix, R = D^{-1/2} G D^{-1/2} in a global slot (row-major, full Hermitian),
// reduced to a real symmetric tridiagonal by K - 2 Householder reflections (unblocked:
// for column k, v = x - alpha e1 with alpha = -e^{j arg x0} |x|, beta = 2 / v^H v, the
// trailing block B <- H B H = B - v w^H - w v^H with p = beta B v, w = p - (beta/2)(v^H p) v;
// the off-diagonal |alpha| -- a unitary diagonal similarity makes the complex tridiagonal
// real), then every eigenvalue by bisection on Sturm counts (thread t finds the t-th
// smallest, so the output is ascending).  Householder reduction is backward stable
// (eigenvalue errors ~ K eps ||R||); the oracle's serial cyclic Jacobi is the reference.
constexpr int kEigThreads = 1024;

__global__ void __launch_bounds__(kEigThreads, 1) eig_householder_kernel(const double *gram, int K, int64_t n_drops,
                                                                         double *eig, double2 *slots) {
  extern __shared__ double2 esm[];
  double2 *v = esm, *w = esm + K;                    // Householder vector, p / w
  double *dg = reinterpret_cast<double *>(w + K);    // tridiagonal diagonal
  double *oe = dg + K;                               // off-diagonal |alpha|
  __shared__ double red[kEigThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = kEigThreads / 32;
  double2 *A = slots + (size_t)blockIdx.x * K * K;
  for (int64_t d = blockIdx.x; d < n_drops; d += gridDim.x) {
    const double2 *G = reinterpret_cast<const double2 *>(gram) + (size_t)d * K * K;
    double *ev = eig + (size_t)d * K;
    bool ok = true;
    for (int i = tid; i < K; i += kEigThreads) ok &= G[(size_t)i * K + i].x > 0.0 && isfinite(G[(size_t)i * K + i].x);
    for (size_t e = tid; e < (size_t)K * K; e += kEigThreads) ok &= isfinite(G[e].x) && isfinite(G[e].y);
    if (!__syncthreads_and(ok ? 1 : 0)) {
      for (int i = tid; i < K; i += kEigThreads) ev[i] = kNaN;
      continue;
    }
    for (size_t e = tid; e < (size_t)K * K; e += kEigThreads) {
      const int r = (int)(e / K), c = (int)(e - (size_t)r * K);
      const double s = rsqrt(G[(size_t)r * K + r].x) * rsqrt(G[(size_t)c * K + c].x);
      const double2 g = G[e];
      A[e] = r == c ? make_double2(1.0, 0.0) : make_double2(g.x * s, g.y * s);
    }
    __syncthreads();
    for (int k = 0; k + 1 < K; ++k) {
      const int n = K - k - 1, o = k + 1;  // trailing block rows/cols o .. K-1
      double part = 0.0;
      for (int i = tid; i < n; i += kEigThreads) {
        const double2 x = A[(size_t)(o + i) * K + k];
        v[i] = x;
        part += x.x * x.x + x.y * x.y;
      }
      const double sigma = block_sum(part, red);  // ends with a barrier: v is visible
      const double2 x0 = v[0];
      const double a0 = sqrt(x0.x * x0.x + x0.y * x0.y), nx = sqrt(sigma);
      if (tid == 0) dg[k] = A[(size_t)k * K + k].x;
      if (sigma - a0 * a0 <= 1e-300 || n == 1) {  // column already reduced: no reflection
        if (tid == 0) oe[k] = a0;
        __syncthreads();
        continue;
      }
      const double2 ph = a0 > 0.0 ? make_double2(x0.x / a0, x0.y / a0) : make_double2(1.0, 0.0);
      const double2 alpha = make_double2(-ph.x * nx, -ph.y * nx);
      const double2 v0 = make_double2(x0.x - alpha.x, x0.y - alpha.y);
      const double vv = sigma - a0 * a0 + v0.x * v0.x + v0.y * v0.y;
      const double beta = 2.0 / vv;
      __syncthreads();
      if (tid == 0) {
        v[0] = v0;
        oe[k] = nx;
      }
      __syncthreads();
      // p = beta B v: a warp per row, lanes along the row (coalesced)
      double vpart = 0.0;
      for (int i = warp; i < n; i += NW) {
        const double2 *row = A + (size_t)(o + i) * K + o;
        double sr = 0.0, si = 0.0;
        for (int j = lane; j < n; j += 32) {
          const double2 b = row[j], vj = v[j];
          sr = fma(b.x, vj.x, fma(-b.y, vj.y, sr));
          si = fma(b.x, vj.y, fma(b.y, vj.x, si));
        }
        sr = xlk::warp_sum(sr) * beta;
        si = xlk::warp_sum(si) * beta;
        if (lane == 0) {
          w[i] = make_double2(sr, si);
          const double2 vi = v[i];
          vpart += vi.x * sr + vi.y * si;  // Re(conj(v_i) p_i)
        }
      }
      const double vhp = block_sum(vpart, red);
      const double kk = 0.5 * beta * vhp;
      for (int i = tid; i < n; i += kEigThreads) {
        const double2 p = w[i], vi = v[i];
        w[i] = make_double2(p.x - kk * vi.x, p.y - kk * vi.y);
      }
      __syncthreads();
      // B <- B - v w^H - w v^H
      for (int i = warp; i < n; i += NW) {
        double2 *row = A + (size_t)(o + i) * K + o;
        const double2 vi = v[i], wi = w[i];
        for (int j = lane; j < n; j += 32) {
          const double2 vj = v[j], wj = w[j];
          double2 b = row[j];
          // v_i conj(w_j) + w_i conj(v_j)
          b.x -= vi.x * wj.x + vi.y * wj.y + wi.x * vj.x + wi.y * vj.y;
          b.y -= vi.y * wj.x - vi.x * wj.y + wi.y * vj.x - wi.x * vj.y;
          row[j] = b;
        }
      }
      __syncthreads();
    }
    if (tid == 0) dg[K - 1] = A[(size_t)(K - 1) * K + (K - 1)].x;
    __syncthreads();
    // Gershgorin bounds, then bisection: thread t -> the t-th smallest eigenvalue
    double lo = INFINITY, hi = -INFINITY;
    for (int i = 0; i < K; ++i) {
      const double r = (i > 0 ? oe[i - 1] : 0.0) + (i + 1 < K ? oe[i] : 0.0);
      lo = fmin(lo, dg[i] - r);
      hi = fmax(hi, dg[i] + r);
    }
    for (int t = tid; t < K; t += kEigThreads) {
      double a = lo, b = hi;
      for (int it = 0; it < 200 && b - a > 1e-15 * fmax(1.0, fabs(a) + fabs(b)); ++it) {
        const double x = 0.5 * (a + b);
        int cnt = 0;
        double q = dg[0] - x;
        cnt += q < 0.0;
        for (int i = 1; i < K; ++i) {
          if (q == 0.0) q = 1e-300;
          q = dg[i] - x - oe[i - 1] * oe[i - 1] / q;
          cnt += q < 0.0;
        }
        if (cnt > t) b = x;  // at least t + 1 eigenvalues below x
        else a = x;
      }
      ev[t] = 0.5 * (a + b);
    }
    __syncthreads();
  }
}

// App. A outputs from the tiled log-dets (matrix 0 = R, 1 + s = I + rho_s G)
__global__ void __launch_bounds__(kCtaThreads) bounds_finish_kernel(BoundsParams P, const double *log2det) {
  __shared__ double red[kCtaThreads / 32];
  const int64_t d = blockIdx.x;
  const int K = P.K;
  const double2 *G = reinterpret_cast<const double2 *>(P.gram) + (size_t)d * K * K;
  double *rs = P.rstat + 2 * d, *bo = P.bounds + (size_t)d * P.n_snr * 3;
  bool fin, dpos;
  scan_gram(G, K, fin, dpos);
  if (!fin || !dpos) {
    if (threadIdx.x < 2) rs[threadIdx.x] = kNaN;
    for (int e = threadIdx.x; e < 3 * P.n_snr; e += blockDim.x) bo[e] = kNaN;
    if (threadIdx.x == 0 && P.flags) P.flags[d] = fin ? XLMIMO_FLAG_MRC_UNDEF : XLMIMO_FLAG_NONFINITE;
    return;
  }
  const double *ld = log2det + d * (1 + P.n_snr);
  uint32_t fl = 0;
  const double ldr = ld[0];
  if (isnan(ldr)) fl |= XLMIMO_FLAG_G_NOT_PD;
  for (int s = 0; s < P.n_snr; ++s) {
    double lu = 0.0;
    for (int i = threadIdx.x; i < K; i += blockDim.x) lu += log2(1.0 + P.rho[s] * G[(size_t)i * K + i].x);
    lu = block_sum(lu, red);
    const double cap = ld[1 + s];
    if (isnan(cap)) fl |= XLMIMO_FLAG_A_NOT_PD;
    if (threadIdx.x == 0) {
      bo[3 * s + 0] = lu;
      bo[3 * s + 1] = cap;
      bo[3 * s + 2] = ldr + lu;
    }
  }
  if (threadIdx.x == 0) {
    rs[0] = ldr;
    rs[1] = -ldr / (double)K;
    if (P.flags) P.flags[d] = fl;
  }
}

// Large-K receivers: CAP from the log-dets of I + rho G, MMSE from the diagonal of its
// inverse, ZF from the diagonal of G^{-1}, MRC straight from G; same
// output order and flag rules as the warp receivers (xl_rates.cu).
struct LargeRateParams {
  const double *gram;
  double *rates;
  uint32_t *flags;
  int K;
  int n_snr, n_recv;
  uint32_t receivers;
  int n_mat, mat_g;  // problems per drop; index of the G problem (ZF) or -1
  double rho[xl::kMaxSnr];
};

__global__ void __launch_bounds__(kCtaThreads) rates_large_finish_kernel(LargeRateParams P, const double *log2det,
                                                                         const double *dinv) {
  __shared__ double red[kCtaThreads / 32];
  const int64_t d = blockIdx.x;
  const int K = P.K;
  const double2 *G = reinterpret_cast<const double2 *>(P.gram) + (size_t)d * K * K;
  double *out = P.rates + (size_t)d * P.n_snr * P.n_recv;
  bool fin, dpos;
  scan_gram(G, K, fin, dpos);
  if (!fin) {
    for (int e = threadIdx.x; e < P.n_snr * P.n_recv; e += blockDim.x) out[e] = kNaN;
    if (threadIdx.x == 0 && P.flags) P.flags[d] |= XLMIMO_FLAG_NONFINITE;
    return;
  }
  uint32_t fl = 0;
  const bool mrc = (P.receivers & XLMIMO_RECV_MRC) != 0;
  if (mrc && !dpos) fl |= XLMIMO_FLAG_MRC_UNDEF;
  const int64_t pg = d * P.n_mat + P.mat_g;
  const bool zf_ok = P.mat_g >= 0 && !isnan(log2det[pg]);
  if (P.mat_g >= 0 && !zf_ok) fl |= XLMIMO_FLAG_G_NOT_PD;
  for (int s = 0; s < P.n_snr; ++s) {
    int r = 0;
    const double rho = P.rho[s];
    const int64_t pa = d * P.n_mat + s;
    const bool a_used = (P.receivers & (XLMIMO_RECV_CAP | XLMIMO_RECV_MMSE)) != 0;
    const bool a_ok = a_used && !isnan(log2det[pa]);
    if (a_used && !a_ok) fl |= XLMIMO_FLAG_A_NOT_PD;
    if (P.receivers & XLMIMO_RECV_CAP) {
      if (threadIdx.x == 0) out[s * P.n_recv + r] = a_ok ? log2det[pa] : kNaN;
      ++r;
    }
    if (P.receivers & XLMIMO_RECV_ZF) {  // SINR_i = rho / [G^{-1}]_ii
      double part = 0.0;
      if (zf_ok)
        for (int i = threadIdx.x; i < K; i += blockDim.x) part += log2(1.0 + rho / dinv[pg * K + i]);
      const double c = block_sum(part, red);
      if (threadIdx.x == 0) out[s * P.n_recv + r] = zf_ok ? c : kNaN;
      ++r;
    }
    if (P.receivers & XLMIMO_RECV_MMSE) {  // SINR_i = 1 / [(I + rho G)^{-1}]_ii - 1
      double part = 0.0;
      if (a_ok)
        for (int i = threadIdx.x; i < K; i += blockDim.x) part += log2(1.0 + (1.0 / dinv[pa * K + i] - 1.0));
      const double c = block_sum(part, red);
      if (threadIdx.x == 0) out[s * P.n_recv + r] = a_ok ? c : kNaN;
      ++r;
    }
    if (mrc) {
      double part = 0.0;
      for (int i = threadIdx.x; i < K; i += blockDim.x) {
        const double gii = G[(size_t)i * K + i].x;
        double intf = 0.0;
        for (int j = 0; j < K; ++j)
          if (j != i) {
            const double2 g = G[(size_t)i * K + j];
            intf += g.x * g.x + g.y * g.y;
          }
        part += log2(1.0 + rho * gii * gii / (gii + rho * intf));
      }
      const double c = block_sum(part, red);
      if (threadIdx.x == 0) out[s * P.n_recv + r] = dpos ? c : kNaN;
      ++r;
    }
  }
  if (threadIdx.x == 0 && P.flags) P.flags[d] |= fl;
}

// ------------------------------------------------------------------ eigenvalues of R (K <= 64)
__global__ void __launch_bounds__(128) eig_jacobi_kernel(const double *gram, int K, int64_t n_drops, double *eig) {
  extern __shared__ double2 smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int Kp = K + (K & 1), ld = Kp + 1, npair = Kp / 2;
  double2 *A = smem + (size_t)warp * Kp * ld;  // column-major A[c*ld + r]
  const int64_t d = (int64_t)blockIdx.x * nw + warp;
  if (d >= n_drops) return;
  const double2 *G = reinterpret_cast<const double2 *>(gram) + (size_t)d * K * K;
  double *ev = eig + (size_t)d * K;
  bool ok = true;
  for (int e = lane; e < K * K; e += 32) ok &= isfinite(G[e].x) && isfinite(G[e].y);
  for (int i = lane; i < K; i += 32) ok &= G[i * K + i].x > 0.0;
  if (!__all_sync(0xffffffffu, ok)) {
    for (int i = lane; i < K; i += 32) ev[i] = kNaN;
    return;
  }
  for (int e = lane; e < Kp * Kp; e += 32) {
    const int c = e / Kp, r = e - c * Kp;
    double2 v = make_double2(0.0, 0.0);
    if (r < K && c < K) {
      if (r == c) {
        v.x = 1.0;
      } else {
        const double2 g = G[r * K + c];
        const double s = rsqrt(G[r * K + r].x) * rsqrt(G[c * K + c].x);
        v = make_double2(g.x * s, g.y * s);
      }
    }
    A[c * ld + r] = v;
  }
  __syncwarp();
  for (int sweep = 0; sweep < 40; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int e = lane; e < Kp * Kp; e += 32) {
      const int c = e / Kp, r = e - c * Kp;
      const double2 v = A[c * ld + r];
      const double m = v.x * v.x + v.y * v.y;
      tot += m;
      if (r != c) off += m;
    }
    off = xlk::warp_sum(off);
    tot = xlk::warp_sum(tot);
    if (off <= 1e-30 * tot) break;
    for (int round = 0; round < Kp - 1; ++round) {
      // round-robin pairing: position 0 fixed, the others rotate
      int p = 0, q = 0;
      const bool act = lane < npair;
      if (act) {
        const int a = lane, b = Kp - 1 - lane;
        p = (a == 0) ? 0 : (a - 1 + round) % (Kp - 1) + 1;
        q = (b - 1 + round) % (Kp - 1) + 1;
      }
      double c = 1.0, s = 0.0, er = 1.0, ei = 0.0, t = 0.0, bmag = 0.0;
      if (act) {
        const double2 apq = A[q * ld + p];
        bmag = sqrt(apq.x * apq.x + apq.y * apq.y);
        if (bmag > 0.0) {
          er = apq.x / bmag;  // e^{-j phi} = conj(A_pq) / |A_pq|
          ei = -apq.y / bmag;
          const double theta = (A[q * ld + q].x - A[p * ld + p].x) / (2.0 * bmag);
          t = 1.0 / (fabs(theta) + sqrt(theta * theta + 1.0));
          if (theta < 0.0) t = -t;
          c = rsqrt(t * t + 1.0);
          s = t * c;
        }
      }
      const bool rot = act && bmag > 0.0;
      __syncwarp();
      // columns: col_p' = c col_p - s e col_q ; col_q' = s col_p + c e col_q   (e = e^{-j phi})
      if (rot) {
        double2 *cp = A + p * ld, *cq = A + q * ld;
        for (int r = 0; r < Kp; ++r) {
          const double2 xp = cp[r], xq0 = cq[r];
          const double2 xq = make_double2(xq0.x * er - xq0.y * ei, xq0.x * ei + xq0.y * er);
          cp[r] = make_double2(c * xp.x - s * xq.x, c * xp.y - s * xq.y);
          cq[r] = make_double2(s * xp.x + c * xq.x, s * xp.y + c * xq.y);
        }
      }
      __syncwarp();
      // rows: row_p' = c row_p - s conj(e) row_q ; row_q' = s row_p + c conj(e) row_q
      if (rot) {
        for (int cc = 0; cc < Kp; ++cc) {
          double2 *col = A + cc * ld;
          const double2 xp = col[p], xq0 = col[q];
          const double2 xq = make_double2(xq0.x * er + xq0.y * ei, -xq0.x * ei + xq0.y * er);
          col[p] = make_double2(c * xp.x - s * xq.x, c * xp.y - s * xq.y);
          col[q] = make_double2(s * xp.x + c * xq.x, s * xp.y + c * xq.y);
        }
      }
      __syncwarp();
      if (rot) {
        A[q * ld + p] = make_double2(0.0, 0.0);
        A[p * ld + q] = make_double2(0.0, 0.0);
        A[p * ld + p].y = 0.0;
        A[q * ld + q].y = 0.0;
      }
      __syncwarp();
    }
  }
  // ascending: rank of each of the first K diagonal entries (ties by index);
  // the padded index (odd K) holds an exact 0 that is never coupled and is skipped.
  for (int i = lane; i < K; i += 32) {
    const double v = A[i * ld + i].x;
    int rank = 0;
    for (int j = 0; j < K; ++j) {
      const double w = A[j * ld + j].x;
      rank += (w < v) || (w == v && j < i);
    }
    ev[rank] = v;
  }
}

int n_chol_slots(int64_t n_prob) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
    cudaGetLastError();  // a failed query (no device) must not leak into check_launch
  }
  return (int)(n_prob < sms ? n_prob : sms);
}
int n_tiled_slots(int64_t n_prob) {
  const int64_t n = (int64_t)kTiledPerSm * n_chol_slots(INT32_MAX);
  return (int)(n_prob < n ? n_prob : n);
}

size_t align256(size_t x) { return (x + 255) / 256 * 256; }

size_t chol_slot_bytes(int K, int64_t n_prob, bool with_dinv) {
  if (K <= kSmemMaxK) return 0;
  const int Kp = (K + kTile - 1) / kTile * kTile;
  const size_t slots = (size_t)n_tiled_slots(n_prob);
  size_t b = align256(slots * Kp * Kp * sizeof(double2));
  if (with_dinv) b += align256(slots * ((kTiledThreads / 32) * (size_t)Kp * kTile + (size_t)Kp * kTile) * sizeof(double2));
  return b;
}

int launch_chol(const double *gram, int K, int64_t n_drops, int n_mat, bool first_is_r, const double *rho,
                const double *alpha, double *log2det, double *dinv, void *ws, size_t ws_bytes, cudaStream_t s) {
  CholParams C;
  memset(&C, 0, sizeof(C));
  C.gram = gram;
  C.K = K;
  C.nt = (K + kTile - 1) / kTile;
  C.Kp = C.nt * kTile;
  C.n_prob = n_drops * n_mat;
  C.n_mat = n_mat;
  C.first_is_r = first_is_r ? 1 : 0;
  for (int m = 0; m < n_mat; ++m) {
    C.rho[m] = rho[m];
    C.alpha[m] = alpha[m];
  }
  C.log2det = log2det;
  C.dinv = dinv;
  C.ws = (double2 *)ws;
  xlh::KTimer tm(s, "chol_logdet");
  if (K <= kSmemMaxK) {
    const size_t smem = (size_t)K * (K + 1) / 2 * sizeof(double2);
    const int per_sm = (int)((220 * 1024) / (smem + kSmemK * sizeof(double)));
    const int64_t grid = (int64_t)n_chol_slots(C.n_prob) * (per_sm > 1 ? per_sm : 1);
    cudaFuncSetAttribute(chol_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    chol_smem_kernel<<<(unsigned)(grid < C.n_prob ? grid : C.n_prob), kCtaThreads, smem, s>>>(C);
  } else {
    const int slots = n_tiled_slots(C.n_prob);
    if (chol_slot_bytes(K, C.n_prob, dinv != nullptr) > ws_bytes)
      return xlh::set_error(XLMIMO_EWORKSPACE, "large-K Cholesky: workspace too small");
    if (dinv) {  // slot matrices, then the L^{-1} panels, then the diagonal-tile inverses
      C.xscr = (double2 *)((char *)ws + align256((size_t)slots * C.Kp * C.Kp * sizeof(double2)));
      C.dvs = C.xscr + (size_t)slots * (kTiledThreads / 32) * C.Kp * kTile;
    }
    cudaFuncSetAttribute(chol_tiled_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTiledSmem);
    chol_tiled_kernel<<<slots, kTiledThreads, kTiledSmem, s>>>(C);
  }
  tm.stop(s);
  xlh::count_launch();
  return xlh::check_launch("chol_logdet kernel");
}


}  // namespace

namespace xlh {

// Eigenvalue slots for 64 < K: one K x K complex matrix per resident CTA (one per SM).
int eig_ctas(int64_t n_drops) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return (int)(n_drops < sms ? n_drops : sms);
}
size_t eig_ws_bytes(int K, int64_t n_drops) {
  if (K <= xl::kMaxK || n_drops == 0) return 0;
  return align256((size_t)eig_ctas(n_drops) * K * K * sizeof(double2));
}

// Scratch for the large-K path: Cholesky slots + per-problem log-dets.
size_t large_k_ws_bytes(int K, int64_t n_drops, int n_mat, bool with_dinv) {
  if (K <= xl::kMaxK || n_drops == 0 || n_mat == 0) return 0;
  const size_t n_prob = (size_t)n_drops * n_mat;
  return chol_slot_bytes(K, (int64_t)n_prob, with_dinv) + align256(n_prob * sizeof(double)) +
         (with_dinv ? align256(n_prob * K * sizeof(double)) : 0);
}

int launch_bounds(const double *gram, int K, int64_t n_drops, const double *snr_db, int n_snr, double *rstat,
                  double *bounds, double *eig, uint32_t *flags, void *ws, size_t ws_bytes, cudaStream_t s) {
  if (n_drops == 0) return XLMIMO_OK;
  BoundsParams P;
  memset(&P, 0, sizeof(P));
  P.gram = gram;
  P.rstat = rstat;
  P.bounds = bounds;
  P.flags = flags;
  P.K = K;
  P.n_drops = n_drops;
  P.n_snr = n_snr;
  for (int i = 0; i < n_snr; ++i) P.rho[i] = pow(10.0, snr_db[i] / 10.0);
  int rc = XLMIMO_OK;
  if (K <= xl::kMaxK) {
    const size_t per_warp = (size_t)K * (K + 1) / 2 * sizeof(double2);
    int nw = (int)((96 * 1024) / per_warp);
    nw = nw > 8 ? 8 : (nw < 1 ? 1 : nw);
    const int64_t blocks = (n_drops + nw - 1) / nw;
    KTimer tm(s, "app_a_bounds");
    if (K <= 32) {
      cudaFuncSetAttribute(bounds_warp_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(per_warp * nw));
      bounds_warp_kernel<1><<<(unsigned)blocks, 32 * nw, per_warp * nw, s>>>(P);
    } else {
      cudaFuncSetAttribute(bounds_warp_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(per_warp * nw));
      bounds_warp_kernel<2><<<(unsigned)blocks, 32 * nw, per_warp * nw, s>>>(P);
    }
    tm.stop(s);
    count_launch();
    rc = check_launch("bounds_warp_kernel");
  } else {
    const int n_mat = 1 + n_snr;
    const int64_t n_prob = n_drops * n_mat;
    const size_t chol_b = chol_slot_bytes(K, n_prob, false);
    if (ws_bytes < large_k_ws_bytes(K, n_drops, n_mat, false) || !ws)
      return set_error(XLMIMO_EWORKSPACE, "app_a_bounds: workspace %zu < %zu", ws_bytes,
                       large_k_ws_bytes(K, n_drops, n_mat, false));
    double *log2det = (double *)((char *)ws + chol_b);
    double rho[xl::kMaxSnr + 1], alpha[xl::kMaxSnr + 1];
    rho[0] = 0.0;
    alpha[0] = 0.0;
    for (int i = 0; i < n_snr; ++i) {
      rho[1 + i] = P.rho[i];
      alpha[1 + i] = 1.0;
    }
    rc = launch_chol(gram, K, n_drops, n_mat, true, rho, alpha, log2det, nullptr, ws, chol_b, s);
    if (rc) return rc;
    KTimer tm(s, "app_a_finish");
    bounds_finish_kernel<<<(unsigned)n_drops, kCtaThreads, 0, s>>>(P, log2det);
    tm.stop(s);
    count_launch();
    rc = check_launch("bounds_finish_kernel");
  }
  if (rc || !eig) return rc;
  if (K > xl::kMaxK) {  // Householder tridiagonalisation + bisection, slots after the Cholesky scratch
    const size_t off = align256(large_k_ws_bytes(K, n_drops, 1 + n_snr, false));
    if (ws_bytes < off + eig_ws_bytes(K, n_drops) || !ws)
      return set_error(XLMIMO_EWORKSPACE, "app_a_bounds: eigenvalues need %zu workspace bytes",
                       off + eig_ws_bytes(K, n_drops));
    const size_t smem = (size_t)K * 2 * sizeof(double2) + (size_t)K * 2 * sizeof(double);
    KTimer tm(s, "eig_householder");
    cudaFuncSetAttribute(eig_householder_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    eig_householder_kernel<<<(unsigned)eig_ctas(n_drops), kEigThreads, smem, s>>>(gram, K, n_drops, eig,
                                                                               (double2 *)((char *)ws + off));
    tm.stop(s);
    count_launch();
    return check_launch("eig_householder_kernel");
  }
  const int Kp = K + (K & 1);
  const size_t per_warp = (size_t)Kp * (Kp + 1) * sizeof(double2);
  int nw = (int)((100 * 1024) / per_warp);
  nw = nw > 4 ? 4 : (nw < 1 ? 1 : nw);
  KTimer tm(s, "eig_jacobi");
  cudaFuncSetAttribute(eig_jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(per_warp * nw));
  eig_jacobi_kernel<<<(unsigned)((n_drops + nw - 1) / nw), 32 * nw, per_warp * nw, s>>>(gram, K, n_drops, eig);
  tm.stop(s);
  count_launch();
  return check_launch("eig_jacobi_kernel");
}

size_t sum_rate_large_ws_bytes(int K, int64_t n_drops, int n_snr, uint32_t receivers) {
  const int n_a = (receivers & (XLMIMO_RECV_CAP | XLMIMO_RECV_MMSE)) ? n_snr : 0;
  const int n_g = (receivers & XLMIMO_RECV_ZF) ? 1 : 0;
  return large_k_ws_bytes(K, n_drops, n_a + n_g, (receivers & (XLMIMO_RECV_ZF | XLMIMO_RECV_MMSE)) != 0);
}

// Problems per drop: I + rho_s G for every SNR (CAP and/or MMSE), then G (ZF).
int launch_sum_rate_large(const double *gram, int K, int64_t n_drops, const double *snr_db, int n_snr,
                          uint32_t receivers, double *rates, uint32_t *flags, void *ws, size_t ws_bytes,
                          cudaStream_t s) {
  if (n_drops == 0) return XLMIMO_OK;
  LargeRateParams P;
  memset(&P, 0, sizeof(P));
  P.gram = gram;
  P.rates = rates;
  P.flags = flags;
  P.K = K;
  P.n_snr = n_snr;
  P.receivers = receivers;
  P.n_recv = __builtin_popcount(receivers & 15u);
  for (int i = 0; i < n_snr; ++i) P.rho[i] = pow(10.0, snr_db[i] / 10.0);
  const int n_a = (receivers & (XLMIMO_RECV_CAP | XLMIMO_RECV_MMSE)) ? n_snr : 0;
  const int n_g = (receivers & XLMIMO_RECV_ZF) ? 1 : 0;
  const bool need_dinv = (receivers & (XLMIMO_RECV_ZF | XLMIMO_RECV_MMSE)) != 0;
  P.n_mat = n_a + n_g;
  P.mat_g = n_g ? n_a : -1;
  double *log2det = nullptr, *dinv = nullptr;
  if (P.n_mat) {
    const int64_t n_prob = n_drops * P.n_mat;
    const size_t need = sum_rate_large_ws_bytes(K, n_drops, n_snr, receivers);
    if (ws_bytes < need || !ws) return set_error(XLMIMO_EWORKSPACE, "sum_rate (K > 64): workspace %zu < %zu", ws_bytes, need);
    const size_t chol_b = chol_slot_bytes(K, n_prob, need_dinv);
    log2det = (double *)((char *)ws + chol_b);
    if (need_dinv) dinv = (double *)((char *)ws + chol_b + align256((size_t)n_prob * sizeof(double)));
    double rho[xl::kMaxSnr + 2], alpha[xl::kMaxSnr + 2];
    for (int i = 0; i < n_a; ++i) {
      rho[i] = P.rho[i];
      alpha[i] = 1.0;
    }
    if (n_g) {
      rho[n_a] = 1.0;
      alpha[n_a] = 0.0;
    }
    const int rc = launch_chol(gram, K, n_drops, P.n_mat, false, rho, alpha, log2det, dinv, ws, chol_b, s);
    if (rc) return rc;
  }
  KTimer tm(s, "sum_rate_large_finish");
  rates_large_finish_kernel<<<(unsigned)n_drops, kCtaThreads, 0, s>>>(P, log2det, dinv);
  tm.stop(s);
  count_launch();
  return check_launch("rates_large_finish_kernel");
}

}  // namespace xlh
