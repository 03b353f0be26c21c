// xl_sweep.cu -- a6: ergodic reductions of the saturation sweep.
//  * ergodic_reduce_kernel: per (N, SNR, receiver) column, fixed-order block reduction
//    (R10): the valid (non-NaN) count, the mean over the valid drops (conditional mean)
//    and the ergodic mean over ALL drops -- defined only when every drop is valid, NaN
//    otherwise (an expectation over a subset of the drops is not the ergodic value).
//  * sat_partial_kernel + sat_final_kernel: per-drop Eqs. (13)-(16)
//      y_up = max_i (x_i t/sqrt(1-t^2) + y_i),  y_down = min_i (-x_i t/sqrt(1-t^2) + y_i),
//    their means over drops, M_sat = ceil((E[y_up] - E[y_down]) / pitch) (R15) and
//    the standard error of the per-drop extent / pitch.
#include "xl_common.cuh"

namespace {

constexpr int kRedThreads = 256;

__global__ void __launch_bounds__(kRedThreads) ergodic_reduce_kernel(const double *per_drop, int64_t n_drops,
                                                                     int n_out, double *mean, double *mean_valid,
                                                                     int64_t *count) {
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
    const double cond = sc[0] ? ss[0] / (double)sc[0] : nan;
    mean[col] = sc[0] == n_drops ? cond : nan;
    mean_valid[col] = cond;
    count[col] = sc[0];
  }
}

// Two stages, both deterministic: sat_partial_kernel -- a thread per drop (Eqs. (13)-(16)
// over its K users), fixed-order tree sums of (y_up, y_down, e, e^2) per block into
// part[block][4]; sat_final_kernel -- one warp adds the block partials in block order.
__global__ void __launch_bounds__(kRedThreads) sat_partial_kernel(const double *pos, int K, int64_t n_drops, double sl,
                                                                  double pitch, double *part) {
  __shared__ double sm[4][kRedThreads];
  const int64_t d = (int64_t)blockIdx.x * kRedThreads + threadIdx.x;
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  if (d < n_drops) {
    double up = -INFINITY, dn = INFINITY;
    for (int i = 0; i < K; ++i) {
      const double *p = pos + (d * K + i) * 3;
      const double x = sqrt(fma(p[0], p[0], p[2] * p[2]));
      up = fmax(up, fma(x, sl, p[1]));    // Eqs. (13), (15)
      dn = fmin(dn, fma(-x, sl, p[1]));   // Eqs. (14), (16)
    }
    const double e = (up - dn) / pitch;
    v[0] = up;
    v[1] = dn;
    v[2] = e;
    v[3] = e * e;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) sm[q][threadIdx.x] = v[q];
  __syncthreads();
  for (int o = kRedThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o)
#pragma unroll
      for (int q = 0; q < 4; ++q) sm[q][threadIdx.x] += sm[q][threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x < 4) part[blockIdx.x * 4 + threadIdx.x] = sm[threadIdx.x][0];
}

__global__ void sat_final_kernel(const double *part, int nb, int64_t n_drops, double pitch, double *sat) {
  if (threadIdx.x != 0) return;
  double t[4] = {0.0, 0.0, 0.0, 0.0};
  for (int b = 0; b < nb; ++b)
    for (int q = 0; q < 4; ++q) t[q] += part[b * 4 + q];
  const double D = (double)n_drops;
  const double eu = t[0] / D, ed = t[1] / D, me = t[2] / D;
  const double var = n_drops > 1 ? (t[3] - D * me * me) / (D - 1.0) : 0.0;
  sat[0] = eu;
  sat[1] = ed;
  sat[2] = ceil((eu - ed) / pitch);
  sat[3] = sqrt(var > 0.0 ? var : 0.0) / sqrt(D);
}

}  // namespace

namespace xlh {

int launch_ergodic_reduce(const double *per_drop, int64_t n_drops, int n_out, double *mean, double *mean_valid,
                          int64_t *count, cudaStream_t s) {
  if (n_out == 0) return XLMIMO_OK;
  KTimer tm(s, "ergodic_reduce");
  ergodic_reduce_kernel<<<n_out, kRedThreads, 0, s>>>(per_drop, n_drops, n_out, mean, mean_valid, count);
  tm.stop(s);
  count_launch();
  return check_launch("ergodic_reduce_kernel");
}

size_t saturation_stats_scratch(int64_t n_drops) {
  return (size_t)((n_drops + kRedThreads - 1) / kRedThreads) * 4 * sizeof(double);
}

int launch_saturation_stats(const double *pos, int K, int64_t n_drops, double t, double pitch, double *sat,
                            double *scratch, cudaStream_t s) {
  const int nb = (int)((n_drops + kRedThreads - 1) / kRedThreads);
  KTimer tm(s, "saturation_stats");
  sat_partial_kernel<<<nb, kRedThreads, 0, s>>>(pos, K, n_drops, t / sqrt(1.0 - t * t), pitch, scratch);
  sat_final_kernel<<<1, 32, 0, s>>>(scratch, nb, n_drops, pitch, sat);
  tm.stop(s);
  count_launch(2);
  return check_launch("saturation_stats kernels");
}

}  // namespace xlh
