// xl_sweep.cu -- a6: ergodic reductions of the saturation sweep.
//  * ergodic_reduce_kernel: mean over drops of each (N, SNR, receiver) column,
//    excluding NaN, with the valid count (R10); fixed-order block reduction.
//  * saturation_stats_kernel: per-drop Eqs. (13)-(16)
//      y_up = max_i (x_i t/sqrt(1-t^2) + y_i),  y_down = min_i (-x_i t/sqrt(1-t^2) + y_i),
//    their means over drops, M_sat = ceil((E[y_up] - E[y_down]) / pitch) (R15) and
//    the standard error of the per-drop extent / pitch.
#include "xl_common.cuh"

namespace {

constexpr int kRedThreads = 256;

__global__ void __launch_bounds__(kRedThreads) ergodic_reduce_kernel(const double *per_drop, int64_t n_drops,
                                                                     int n_out, double *mean, int64_t *count) {
  __shared__ double ss[kRedThreads];
  __shared__ long long sc[kRedThreads];
  const int col = blockIdx.x;
  double s = 0.0;
  long long c = 0;
  for (int64_t d = threadIdx.x; d < n_drops; d += kRedThreads) {
    const double v = per_drop[d * n_out + col];
    if (!isnan(v)) { s += v; ++c; }
  }
  ss[threadIdx.x] = s;
  sc[threadIdx.x] = c;
  __syncthreads();
  for (int o = kRedThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      ss[threadIdx.x] += ss[threadIdx.x + o];
      sc[threadIdx.x] += sc[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double nan = __longlong_as_double(0x7ff8000000000000LL);
    mean[col] = sc[0] ? ss[0] / (double)sc[0] : nan;
    count[col] = sc[0];
  }
}

__global__ void __launch_bounds__(kRedThreads) saturation_stats_kernel(const double *pos, int K, int64_t n_drops,
                                                                       double t, double pitch, double *sat) {
  __shared__ double s_up[kRedThreads], s_dn[kRedThreads], s_e[kRedThreads], s_e2[kRedThreads];
  const double sl = t / sqrt(1.0 - t * t);
  double su = 0.0, sd = 0.0, se = 0.0, se2 = 0.0;
  for (int64_t d = threadIdx.x; d < n_drops; d += kRedThreads) {
    double up = -INFINITY, dn = INFINITY;
    for (int i = 0; i < K; ++i) {
      const double *p = pos + (d * K + i) * 3;
      const double x = sqrt(fma(p[0], p[0], p[2] * p[2]));
      up = fmax(up, fma(x, sl, p[1]));    // Eqs. (13), (15)
      dn = fmin(dn, fma(-x, sl, p[1]));   // Eqs. (14), (16)
    }
    su += up;
    sd += dn;
    const double e = (up - dn) / pitch;
    se += e;
    se2 += e * e;
  }
  s_up[threadIdx.x] = su;
  s_dn[threadIdx.x] = sd;
  s_e[threadIdx.x] = se;
  s_e2[threadIdx.x] = se2;
  __syncthreads();
  for (int o = kRedThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      s_up[threadIdx.x] += s_up[threadIdx.x + o];
      s_dn[threadIdx.x] += s_dn[threadIdx.x + o];
      s_e[threadIdx.x] += s_e[threadIdx.x + o];
      s_e2[threadIdx.x] += s_e2[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double D = (double)n_drops;
    const double eu = s_up[0] / D, ed = s_dn[0] / D, me = s_e[0] / D;
    const double var = n_drops > 1 ? (s_e2[0] - D * me * me) / (D - 1.0) : 0.0;
    sat[0] = eu;
    sat[1] = ed;
    sat[2] = ceil((eu - ed) / pitch);
    sat[3] = sqrt(var > 0.0 ? var : 0.0) / sqrt(D);
  }
}

}  // namespace

namespace xlh {

int launch_ergodic_reduce(const double *per_drop, int64_t n_drops, int n_out, double *mean, int64_t *count,
                          cudaStream_t s) {
  if (n_out == 0) return XLMIMO_OK;
  KTimer tm(s, "ergodic_reduce");
  ergodic_reduce_kernel<<<n_out, kRedThreads, 0, s>>>(per_drop, n_drops, n_out, mean, count);
  tm.stop(s);
  count_launch();
  return check_launch("ergodic_reduce_kernel");
}

int launch_saturation_stats(const double *pos, int K, int64_t n_drops, double t, double pitch, double *sat,
                            cudaStream_t s) {
  KTimer tm(s, "saturation_stats");
  saturation_stats_kernel<<<1, kRedThreads, 0, s>>>(pos, K, n_drops, t, pitch, sat);
  tm.stop(s);
  count_launch();
  return check_launch("saturation_stats_kernel");
}

}  // namespace xlh
