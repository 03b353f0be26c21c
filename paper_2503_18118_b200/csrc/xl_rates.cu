// xl_rates.cu -- a5: per-drop receivers on a K x K Gram (Eq. (9) PAPER.md:117-122,
// Eq. (21); SINR definitions, R12).
//
// One warp per Gram.  The factor lives in shared memory as a packed column-major
// lower triangle (K(K+1)/2 complex, xl_linalg.cuh) so lane = row accesses are
// conflict-free and up to 3 warps (K = 64) share 100 KB; lanes own rows for the
// Cholesky and for the in-place inverse X = L^{-1} whose column norms are the
// diagonal of the inverse.  For every SNR:
//   I + rho G = L L^H -> CAP = 2 sum log2 L_kk, [(I+rho G)^{-1}]_ii = sum_k |(L^{-1})_ki|^2;
//   G = L L^H once     -> [G^{-1}]_ii for ZF;  MRC straight from G.
// A pivot that is not > 0 (or not finite) marks the factorisation failed (R10).
#include <cstring>

#include "xl_common.cuh"
#include "xl_linalg.cuh"

namespace {

struct RateParams {
  const double *gram;
  double *rates;
  uint32_t *flags;
  int K;
  int64_t n_prob;
  int n_snr;
  uint32_t receivers;
  int n_recv;
  double rho[xl::kMaxSnr];
};

// Packed lower triangle per warp (K(K+1)/2 complex): column j of A = conj of row j of G
// (coalesced reads).  alpha I + rho G.
template <int RPL>
__device__ __forceinline__ void load_packed(double2 *Ls, const double2 *G, int K, int lane, double alpha,
                                            double rho) {
  for (int j = 0; j < K; ++j) {
    const int oj = xlk::poff(K, j);
    for (int i = j + lane; i < K; i += 32) {
      const double2 g = G[j * K + i];
      Ls[oj + i - j] = (i == j) ? make_double2(alpha + rho * g.x, 0.0) : make_double2(rho * g.x, -rho * g.y);
    }
  }
  __syncwarp();
}

template <int RPL>
__global__ void __launch_bounds__(256) rates_kernel(RateParams P) {
  extern __shared__ double2 smem[];
  const int K = P.K;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double2 *Ls = smem + (size_t)warp * (K * (K + 1) / 2);
  const int64_t prob = (int64_t)blockIdx.x * nw + warp;
  if (prob >= P.n_prob) return;
  const double2 *G = reinterpret_cast<const double2 *>(P.gram) + (size_t)prob * K * K;
  double *out = P.rates + (size_t)prob * P.n_snr * P.n_recv;
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  uint32_t fl = 0;

  // non-finite input -> all NaN (flag bit 4)
  bool fin = true;
  for (int e = lane; e < K * K; e += 32) fin &= isfinite(G[e].x) && isfinite(G[e].y);
  fin = __all_sync(0xffffffffu, fin);
  if (!fin) {
    for (int e = lane; e < P.n_snr * P.n_recv; e += 32) out[e] = nan;
    if (lane == 0 && P.flags) P.flags[prob] |= XLMIMO_FLAG_NONFINITE;
    return;
  }

  double zf_dinv[RPL];
  bool zf_ok = false;
  if (P.receivers & XLMIMO_RECV_ZF) {
    load_packed<RPL>(Ls, G, K, lane, 0.0, 1.0);
    zf_ok = xlk::warp_cholesky_packed<RPL>(Ls, K, lane);
    if (zf_ok) xlk::warp_inv_diag_packed<RPL>(Ls, K, lane, zf_dinv);
    else fl |= XLMIMO_FLAG_G_NOT_PD;
  }
  bool mrc_ok = true;
  for (int i = lane; i < K; i += 32) mrc_ok &= G[i * K + i].x > 0.0;
  mrc_ok = __all_sync(0xffffffffu, mrc_ok);
  if ((P.receivers & XLMIMO_RECV_MRC) && !mrc_ok) fl |= XLMIMO_FLAG_MRC_UNDEF;

  for (int s = 0; s < P.n_snr; ++s) {
    const double rho = P.rho[s];
    int r = 0;
    bool a_ok = false;
    double dinv[RPL];
    double cap_part = 0.0;
    if (P.receivers & (XLMIMO_RECV_CAP | XLMIMO_RECV_MMSE)) {
      __syncwarp();
      load_packed<RPL>(Ls, G, K, lane, 1.0, rho);
      a_ok = xlk::warp_cholesky_packed<RPL>(Ls, K, lane);
      if (!a_ok) fl |= XLMIMO_FLAG_A_NOT_PD;
      if (a_ok) {
#pragma unroll
        for (int rr = 0; rr < RPL; ++rr) {
          const int k = lane + 32 * rr;
          if (k < K) cap_part += 2.0 * log2(Ls[xlk::poff(K, k)].x);
        }
        if (P.receivers & XLMIMO_RECV_MMSE) xlk::warp_inv_diag_packed<RPL>(Ls, K, lane, dinv);
      }
    }
    if (P.receivers & XLMIMO_RECV_CAP) {
      const double c = xlk::warp_sum(cap_part);
      if (lane == 0) out[s * P.n_recv + r] = a_ok ? c : nan;
      ++r;
    }
    if (P.receivers & XLMIMO_RECV_ZF) {
      double part = 0.0;
#pragma unroll
      for (int rr = 0; rr < RPL; ++rr) {
        const int i = lane + 32 * rr;
        if (zf_ok && i < K) part += log2(1.0 + rho / zf_dinv[rr]);
      }
      const double c = xlk::warp_sum(part);
      if (lane == 0) out[s * P.n_recv + r] = zf_ok ? c : nan;
      ++r;
    }
    if (P.receivers & XLMIMO_RECV_MMSE) {
      double part = 0.0;
#pragma unroll
      for (int rr = 0; rr < RPL; ++rr) {
        const int i = lane + 32 * rr;
        if (a_ok && i < K) part += log2(1.0 + (1.0 / dinv[rr] - 1.0));
      }
      const double c = xlk::warp_sum(part);
      if (lane == 0) out[s * P.n_recv + r] = a_ok ? c : nan;
      ++r;
    }
    if (P.receivers & XLMIMO_RECV_MRC) {
      double part = 0.0;
#pragma unroll
      for (int rr = 0; rr < RPL; ++rr) {
        const int i = lane + 32 * rr;
        if (i < K) {
          const double gii = G[i * K + i].x;
          double intf = 0.0;
          for (int j = 0; j < K; ++j)
            if (j != i) {
              const double2 g = G[i * K + j];
              intf += g.x * g.x + g.y * g.y;
            }
          part += log2(1.0 + rho * gii * gii / (gii + rho * intf));
        }
      }
      const double c = xlk::warp_sum(part);
      if (lane == 0) out[s * P.n_recv + r] = mrc_ok ? c : nan;
      ++r;
    }
  }
  if (lane == 0 && P.flags) P.flags[prob] |= fl;
}

// ---------------------------------------------------------------------------
// Small K (<= 8): one thread per Gram, the factor in registers (fully unrolled, packed
// lower triangle: K(K+1)/2 complex entries, so K = 8 fits the register file instead of
// a 1 KB local-memory frame), G re-read from global/L1 whenever I + rho G is formed.
// Same definitions and failure rule as the warp kernel.
__host__ __device__ constexpr int tri(int i, int j) { return i * (i + 1) / 2 + j; }  // j <= i

template <int K>
__device__ __forceinline__ void load_a(const double2 *G, double rho, double diag, double (&ar)[K * (K + 1) / 2],
                                       double (&ai)[K * (K + 1) / 2]) {
  // lower triangle of diag*I + rho*G: A(i,j) = rho conj(G(j,i)) for i > j
#pragma unroll
  for (int j = 0; j < K; ++j)
#pragma unroll
    for (int i = j; i < K; ++i) {
      const double2 g = __ldg(G + j * K + i);
      ar[tri(i, j)] = (i == j ? diag : 0.0) + rho * g.x;
      ai[tri(i, j)] = -rho * g.y;
    }
}

// in-place lower Cholesky; linv = 1/L_jj
template <int K>
__device__ __forceinline__ bool chol_reg(double (&ar)[K * (K + 1) / 2], double (&ai)[K * (K + 1) / 2],
                                         double (&linv)[K]) {
#pragma unroll
  for (int j = 0; j < K; ++j) {
    double d = ar[tri(j, j)];
#pragma unroll
    for (int k = 0; k < j; ++k) d -= ar[tri(j, k)] * ar[tri(j, k)] + ai[tri(j, k)] * ai[tri(j, k)];
    if (!(d > 0.0) || !isfinite(d)) return false;
    const double ljj = sqrt(d), inv = 1.0 / ljj;
    ar[tri(j, j)] = ljj;
    ai[tri(j, j)] = 0.0;
    linv[j] = inv;
#pragma unroll
    for (int i = j + 1; i < K; ++i) {
      double sr = ar[tri(i, j)], si = ai[tri(i, j)];
#pragma unroll
      for (int k = 0; k < j; ++k) {  // - L_ik conj(L_jk)
        sr -= ar[tri(i, k)] * ar[tri(j, k)] + ai[tri(i, k)] * ai[tri(j, k)];
        si -= ai[tri(i, k)] * ar[tri(j, k)] - ar[tri(i, k)] * ai[tri(j, k)];
      }
      ar[tri(i, j)] = sr * inv;
      ai[tri(i, j)] = si * inv;
    }
  }
  return true;
}

template <int K>
__device__ __forceinline__ void inv_diag_reg(const double (&lr)[K * (K + 1) / 2], const double (&li)[K * (K + 1) / 2],
                                             const double (&linv)[K], double (&dinv)[K]) {
#pragma unroll
  for (int c = 0; c < K; ++c) {
    double xr[K], xi[K];
    xr[c] = linv[c];
    xi[c] = 0.0;
    double s = xr[c] * xr[c];
#pragma unroll
    for (int k = c + 1; k < K; ++k) {
      double tr = 0.0, ti = 0.0;
#pragma unroll
      for (int j = c; j < k; ++j) {
        tr += lr[tri(k, j)] * xr[j] - li[tri(k, j)] * xi[j];
        ti += lr[tri(k, j)] * xi[j] + li[tri(k, j)] * xr[j];
      }
      xr[k] = -tr * linv[k];
      xi[k] = -ti * linv[k];
      s += xr[k] * xr[k] + xi[k] * xi[k];
    }
    dinv[c] = s;
  }
}

template <int K>
__global__ void __launch_bounds__(128) rates_thread_kernel(RateParams P) {
  const int64_t prob = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (prob >= P.n_prob) return;
  const double2 *G = reinterpret_cast<const double2 *>(P.gram) + (size_t)prob * K * K;
  double *out = P.rates + (size_t)prob * P.n_snr * P.n_recv;
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  bool fin = true, mrc_ok = true;
#pragma unroll
  for (int j = 0; j < K; ++j)
#pragma unroll
    for (int i = j; i < K; ++i) {
      const double2 g = __ldg(G + j * K + i);
      fin &= isfinite(g.x) && isfinite(g.y);
      if (i == j) mrc_ok &= g.x > 0.0;
    }
  uint32_t fl = 0;
  if (!fin) {
    for (int e = 0; e < P.n_snr * P.n_recv; ++e) out[e] = nan;
    if (P.flags) P.flags[prob] |= XLMIMO_FLAG_NONFINITE;
    return;
  }
  double ar[K * (K + 1) / 2], ai[K * (K + 1) / 2], linv[K], zf_dinv[K];
  bool zf_ok = false;
  if (P.receivers & XLMIMO_RECV_ZF) {
    load_a<K>(G, 1.0, 0.0, ar, ai);
    zf_ok = chol_reg<K>(ar, ai, linv);
    if (zf_ok) inv_diag_reg<K>(ar, ai, linv, zf_dinv);
    else fl |= XLMIMO_FLAG_G_NOT_PD;
  }
  if ((P.receivers & XLMIMO_RECV_MRC) && !mrc_ok) fl |= XLMIMO_FLAG_MRC_UNDEF;
  for (int s = 0; s < P.n_snr; ++s) {
    const double rho = P.rho[s];
    int r = 0;
    bool a_ok = false;
    double cap = 0.0, mmse = 0.0;
    if (P.receivers & (XLMIMO_RECV_CAP | XLMIMO_RECV_MMSE)) {
      load_a<K>(G, rho, 1.0, ar, ai);
      a_ok = chol_reg<K>(ar, ai, linv);
      if (!a_ok) fl |= XLMIMO_FLAG_A_NOT_PD;
      if (a_ok) {
#pragma unroll
        for (int k = 0; k < K; ++k) cap += 2.0 * log2(ar[tri(k, k)]);
        if (P.receivers & XLMIMO_RECV_MMSE) {
          double dinv[K];
          inv_diag_reg<K>(ar, ai, linv, dinv);
#pragma unroll
          for (int i = 0; i < K; ++i) mmse += log2(1.0 + (1.0 / dinv[i] - 1.0));
        }
      }
    }
    if (P.receivers & XLMIMO_RECV_CAP) out[s * P.n_recv + r++] = a_ok ? cap : nan;
    if (P.receivers & XLMIMO_RECV_ZF) {
      double c = 0.0;
#pragma unroll
      for (int i = 0; i < K; ++i) c += log2(1.0 + rho / zf_dinv[i]);
      out[s * P.n_recv + r++] = zf_ok ? c : nan;
    }
    if (P.receivers & XLMIMO_RECV_MMSE) out[s * P.n_recv + r++] = a_ok ? mmse : nan;
    if (P.receivers & XLMIMO_RECV_MRC) {
      double c = 0.0;
#pragma unroll
      for (int i = 0; i < K; ++i) {
        double intf = 0.0;
        const double gii = __ldg(G + i * K + i).x;
#pragma unroll
        for (int j = 0; j < K; ++j)
          if (j != i) {
            const double2 g = __ldg(G + i * K + j);
            intf += g.x * g.x + g.y * g.y;
          }
        c += log2(1.0 + rho * gii * gii / (gii + rho * intf));
      }
      out[s * P.n_recv + r++] = mrc_ok ? c : nan;
    }
  }
  if (P.flags) P.flags[prob] |= fl;
}

// ---------------------------------------------------------------------------
// NEXT-1: modified-ZF effective rate.  Block per Gram pair, thread per row:
// in-place complex Gauss-Jordan with partial pivoting for B = G~^{-1} (pivot
// search by thread 0, first maximal |.|, as the oracle), A = B G, then per row
// SINR_i = |A_ii|^2 / (sum_{j!=i}|A_ij|^2 + Re[A B]_ii / rho); rates summed in
// row order by thread 0 (deterministic).
__global__ void __launch_bounds__(64) mismatched_kernel(const double *gram, const double *gram_model, int K,
                                                        int n_snr, RateParams P) {
  extern __shared__ double2 sm[];
  double2 *B = sm, *Gs = sm + K * K, *A = sm + 2 * K * K;
  __shared__ int singular;
  __shared__ int perm[xl::kMaxK];
  __shared__ double terms[xl::kMaxSnr][64];
  const int64_t prob = blockIdx.x;
  const int t = threadIdx.x;
  const double2 *Gm = reinterpret_cast<const double2 *>(gram_model) + (size_t)prob * K * K;
  const double2 *Gt = reinterpret_cast<const double2 *>(gram) + (size_t)prob * K * K;
  for (int e = t; e < K * K; e += blockDim.x) {
    B[e] = Gm[e];
    Gs[e] = Gt[e];
  }
  if (t == 0) singular = 0;
  __syncthreads();
  for (int k = 0; k < K; ++k) {
    if (t == 0) {
      int p = k;
      double best = -1.0;
      for (int i = k; i < K; ++i) {
        const double v = hypot(B[i * K + k].x, B[i * K + k].y);
        if (v > best) { best = v; p = i; }
      }
      if (!(best > 0.0)) singular = 1;
      perm[k] = p;
      if (p != k)
        for (int j = 0; j < K; ++j) {
          const double2 tmp = B[k * K + j];
          B[k * K + j] = B[p * K + j];
          B[p * K + j] = tmp;
        }
    }
    __syncthreads();
    if (singular) break;
    const double2 pv = B[k * K + k];
    const double den = pv.x * pv.x + pv.y * pv.y;
    const double ir = pv.x / den, ii = -pv.y / den;
    __syncthreads();
    for (int j = t; j < K; j += blockDim.x) {  // row k *= 1/pivot (B[k][k] := 1 first)
      const double2 a = (j == k) ? make_double2(1.0, 0.0) : B[k * K + j];
      B[k * K + j] = make_double2(a.x * ir - a.y * ii, a.x * ii + a.y * ir);
    }
    __syncthreads();
    if (t < K && t != k) {  // row t -= f * row k
      const double2 f = B[t * K + k];
      B[t * K + k] = make_double2(0.0, 0.0);
      for (int j = 0; j < K; ++j) {
        const double2 b = B[k * K + j];
        double2 a = B[t * K + j];
        a.x -= f.x * b.x - f.y * b.y;
        a.y -= f.x * b.y + f.y * b.x;
        B[t * K + j] = a;
      }
    }
    __syncthreads();
  }
  double *out = P.rates + (size_t)prob * n_snr;
  if (singular) {
    if (t < n_snr) out[t] = __longlong_as_double(0x7ff8000000000000LL);
    if (t == 0 && P.flags) P.flags[prob] |= XLMIMO_FLAG_MODEL_SINGULAR;
    return;
  }
  // undo the row swaps as column swaps (each thread its own row)
  if (t < K)
    for (int k = K - 1; k >= 0; --k) {
      const int p = perm[k];
      if (p != k) {
        const double2 tmp = B[t * K + k];
        B[t * K + k] = B[t * K + p];
        B[t * K + p] = tmp;
      }
    }
  __syncthreads();
  double sig = 0.0, intf = 0.0, noise = 0.0;
  if (t < K) {
    for (int j = 0; j < K; ++j) {  // A = B G, row t
      double sr = 0.0, si = 0.0;
      for (int k = 0; k < K; ++k) {
        const double2 b = B[t * K + k], g = Gs[k * K + j];
        sr += b.x * g.x - b.y * g.y;
        si += b.x * g.y + b.y * g.x;
      }
      A[t * K + j] = make_double2(sr, si);
      const double p = sr * sr + si * si;
      if (j == t) sig = p;
      else intf += p;
    }
    for (int k = 0; k < K; ++k) {  // Re [A B]_tt
      const double2 a = A[t * K + k], b = B[k * K + t];
      noise += a.x * b.x - a.y * b.y;
    }
    for (int s = 0; s < n_snr; ++s) terms[s][t] = log2(1.0 + sig / (intf + noise / P.rho[s]));
  }
  __syncthreads();
  if (t < n_snr) {
    double c = 0.0;
    for (int i = 0; i < K; ++i) c += terms[t][i];
    out[t] = c;
  }
}

template <int K>
void launch_rates_thread(const RateParams &P, cudaStream_t s) {
  rates_thread_kernel<K><<<(unsigned)((P.n_prob + 127) / 128), 128, 0, s>>>(P);
}

}  // namespace

namespace xlh {

int launch_sum_rate_mismatched(const double *gram, const double *gram_model, int K, int64_t n_prob,
                               const double *snr_db, int n_snr, double *rates, uint32_t *flags, cudaStream_t s) {
  if (n_prob == 0) return XLMIMO_OK;
  RateParams P;
  memset(&P, 0, sizeof(P));
  P.rates = rates;
  P.flags = flags;
  P.K = K;
  P.n_prob = n_prob;
  P.n_snr = n_snr;
  for (int i = 0; i < xl::kMaxSnr; ++i) P.rho[i] = i < n_snr ? pow(10.0, snr_db[i] / 10.0) : 0.0;
  const size_t smem = 3 * (size_t)K * K * sizeof(double2);
  cudaFuncSetAttribute(mismatched_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  KTimer tm(s, "sum_rate_mismatched");
  mismatched_kernel<<<(unsigned)n_prob, 64, smem, s>>>(gram, gram_model, K, n_snr, P);
  tm.stop(s);
  count_launch();
  return check_launch("mismatched_kernel");
}

int launch_sum_rate(const double *gram, int K, int64_t n_prob, const double *snr_db, int n_snr,
                    uint32_t receivers, double *rates, uint32_t *flags, cudaStream_t s) {
  if (n_prob == 0) return XLMIMO_OK;
  RateParams P;
  P.gram = gram;
  P.rates = rates;
  P.flags = flags;
  P.K = K;
  P.n_prob = n_prob;
  P.n_snr = n_snr;
  P.receivers = receivers;
  P.n_recv = __builtin_popcount(receivers & 15u);
  for (int i = 0; i < xl::kMaxSnr; ++i) P.rho[i] = i < n_snr ? pow(10.0, snr_db[i] / 10.0) : 0.0;
  const size_t per_warp = (size_t)K * (K + 1) / 2 * sizeof(double2);  // packed factor per warp
  int nw = (int)((100 * 1024) / per_warp);
  if (nw > 8) nw = 8;
  if (nw < 1) nw = 1;
  const size_t smem = per_warp * nw;
  const int64_t blocks = (n_prob + nw - 1) / nw;
  KTimer tm(s, "sum_rate");
  if (K <= 8) {
    switch (K) {
      case 1: launch_rates_thread<1>(P, s); break;
      case 2: launch_rates_thread<2>(P, s); break;
      case 3: launch_rates_thread<3>(P, s); break;
      case 4: launch_rates_thread<4>(P, s); break;
      case 5: launch_rates_thread<5>(P, s); break;
      case 6: launch_rates_thread<6>(P, s); break;
      case 7: launch_rates_thread<7>(P, s); break;
      default: launch_rates_thread<8>(P, s); break;
    }
  } else if (K <= 32) {
    cudaFuncSetAttribute(rates_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    rates_kernel<1><<<(unsigned)blocks, 32 * nw, smem, s>>>(P);
  } else {
    cudaFuncSetAttribute(rates_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    rates_kernel<2><<<(unsigned)blocks, 32 * nw, smem, s>>>(P);
  }
  tm.stop(s);
  count_launch();
  return check_launch("rates_kernel");
}

}  // namespace xlh
