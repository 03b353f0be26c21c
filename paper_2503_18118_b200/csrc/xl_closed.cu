// xl_closed.cu -- a4: closed-form ("modified ZF") Gram, Eqs. (4), (6), (7),
// (22), (23).  O(K^2) per drop, independent of N.
//
// Diagonal: G~_ii = (2 beta0/(lambda x_i)) B_i(M) with the Eq. (4) bracket
//   B_i = (M lambda - 4 y_i)/sqrt(16 x_i^2 + (M lambda - 4 y_i)^2)
//       + (M lambda + 4 y_i)/sqrt(16 x_i^2 + (M lambda + 4 y_i)^2).
// Off-diagonal: G~_ij = rho_ij sqrt(G~_ii G~_jj) with rho_ij of Eq. (6); the
// Eq. (4) brackets of rho_ij cancel against sqrt(G~_ii G~_jj) (R8), leaving
//   |G~_ij| = 2 beta0 |dx| / (sqrt(lambda) d^{3/2} sqrt(x_i x_j)),
//   arg G~_ij = sgn(dx) (2 pi frac(d/lambda) - pi/4),  sgn(0) = -1 (Eq. 7),
// dx = |x_i| - |x_j|, d = sqrt(dx^2 + (y_i - y_j)^2).  The oracle evaluates
// Eq. (6) term by term instead; parity checks the simplification.
#include "xl_common.cuh"

namespace {

constexpr int kMaxLvl = 32;
struct CfParams {
  const double *pos;
  double *out;
  uint32_t *flags;
  int K;
  int64_t n_drops;
  int n_lvl;
  double m_list[kMaxLvl];
  double lambda, beta0;
};

__device__ __forceinline__ void user_xy(const double *p, double &x, double &y) {
  x = sqrt(fma(p[0], p[0], p[2] * p[2]));  // distance to the array line (R21)
  y = p[1];
}

__global__ void __launch_bounds__(256) closed_form_kernel(CfParams P) {
  const int K = P.K;
  const int NP = K * (K + 1) / 2;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= P.n_drops * NP) return;
  const int64_t drop = idx / NP;
  const int p = (int)(idx - drop * NP);
  int i = 0, rem = p;
  while (rem >= K - i) { rem -= K - i; ++i; }
  const int j = i + rem;
  const double *pd = P.pos + drop * K * 3;
  double xi, yi;
  user_xy(pd + 3 * i, xi, yi);
  const double lam = P.lambda;
  if (i == j) {
    for (int l = 0; l < P.n_lvl; ++l) {
      const double ml = P.m_list[l] * lam;
      const double a = ml - 4.0 * yi, b = ml + 4.0 * yi, x16 = 16.0 * xi * xi;
      const double B = a / sqrt(fma(a, a, x16)) + b / sqrt(fma(b, b, x16));
      double *g = P.out + ((size_t)drop * P.n_lvl + l) * (size_t)K * K * 2;
      g[(i * K + i) * 2] = 2.0 * P.beta0 / (lam * xi) * B;
      g[(i * K + i) * 2 + 1] = 0.0;
    }
    return;
  }
  double xj, yj;
  user_xy(pd + 3 * j, xj, yj);
  const double dx = xi - xj, dy = yi - yj;
  const double d = sqrt(fma(dx, dx, dy * dy));
  const double mag = 2.0 * P.beta0 * fabs(dx) / (sqrt(lam) * d * sqrt(d) * sqrt(xi * xj));
  const double q = d / lam;
  const double sg = dx > 0.0 ? 1.0 : -1.0;
  const double ph = sg * (2.0 * 3.14159265358979323846 * (q - rint(q)) - 0.25 * 3.14159265358979323846);
  double s, c;
  sincos(ph, &s, &c);
  const double re = mag * c, im = mag * s;
  for (int l = 0; l < P.n_lvl; ++l) {
    double *g = P.out + ((size_t)drop * P.n_lvl + l) * (size_t)K * K * 2;
    g[(i * K + j) * 2] = re;
    g[(i * K + j) * 2 + 1] = im;
    g[(j * K + i) * 2] = re;
    g[(j * K + i) * 2 + 1] = -im;
  }
}

// flags[d] = DEGENERATE if some pair has ||x_i| - |x_j|| < lambda, else 0.
__global__ void __launch_bounds__(256) closed_form_flags_kernel(const double *pos, int K, int64_t n_drops,
                                                                double lambda, uint32_t *flags) {
  const int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= n_drops) return;
  const double *pd = pos + d * K * 3;
  uint32_t f = 0;
  for (int i = 0; i < K; ++i) {
    double xi, yi;
    user_xy(pd + 3 * i, xi, yi);
    for (int j = i + 1; j < K; ++j) {
      double xj, yj;
      user_xy(pd + 3 * j, xj, yj);
      if (fabs(xi - xj) < lambda) f = XLMIMO_FLAG_DEGENERATE;
    }
  }
  flags[d] = f;
}

}  // namespace

namespace xlh {

int launch_closed_form(const ArrayP &a, const double *pos, int K, int64_t n_drops, const int64_t *m_list,
                       int n_lvl, double *out, uint32_t *flags, cudaStream_t s) {
  if (n_lvl < 1 || n_lvl > kMaxLvl) return set_error(XLMIMO_EINVAL, "closed form: n_lvl out of range");
  if (n_drops == 0) return XLMIMO_OK;
  CfParams P;
  P.pos = pos;
  P.out = out;
  P.flags = flags;
  P.K = K;
  P.n_drops = n_drops;
  P.n_lvl = n_lvl;
  for (int l = 0; l < kMaxLvl; ++l) P.m_list[l] = l < n_lvl ? (double)m_list[l] : 0.0;
  P.lambda = a.lambda;
  P.beta0 = a.sqrt_beta0 * a.sqrt_beta0;
  const int64_t n = n_drops * (int64_t)K * (K + 1) / 2;
  KTimer tm(s, "closed_form");
  closed_form_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(P);
  tm.stop(s);
  count_launch();
  int rc = check_launch("closed_form_kernel");
  if (rc || !flags) return rc;
  KTimer tf(s, "closed_form_flags");
  closed_form_flags_kernel<<<(unsigned)((n_drops + 255) / 256), 256, 0, s>>>(pos, K, n_drops, a.lambda, flags);
  tf.stop(s);
  count_launch();
  return check_launch("closed_form_flags_kernel");
}

}  // namespace xlh
