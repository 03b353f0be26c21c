// xl_drops.cu -- a1: seeded user drops (R3, R5, R19).
#include "xl_common.cuh"

namespace {

__global__ void __launch_bounds__(256) gen_drops_kernel(xlmimo_users_t u, int K, int64_t n_total,
                                                        uint64_t seed, uint64_t first_drop, double *pos) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n_total) return;
  const int64_t d = idx / K;
  const int k = (int)(idx - d * K);
  const xl::u64x4 w = xl::philox4x64_10(first_drop + (uint64_t)d, (uint64_t)k, 0, 0, seed, 0);
  const double deg = 3.14159265358979323846 / 180.0;
  // explicit round-to-nearest multiply and add (no FMA contraction): r, az and el are then
  // the same doubles as any plain evaluation of the law (R3, R19), so positions differ only
  // by the sin/cos implementation (<= 2 ulp)
  const double r = __dadd_rn(u.r_min_m, __dmul_rn(u.r_max_m - u.r_min_m, xl::u01_53(w.v[0])));
  const double az = __dmul_rn(__dadd_rn(u.az_min_deg, __dmul_rn(u.az_max_deg - u.az_min_deg, xl::u01_53(w.v[1]))), deg);
  const double el = __dmul_rn(__dadd_rn(u.el_min_deg, __dmul_rn(u.el_max_deg - u.el_min_deg, xl::u01_53(w.v[2]))), deg);
  double sa, ca, se, ce;
  sincos(az, &sa, &ca);
  sincos(el, &se, &ce);
  double *p = pos + idx * 3;
  p[0] = __dmul_rn(__dmul_rn(r, ce), ca);
  p[1] = __dmul_rn(__dmul_rn(r, ce), sa);
  p[2] = __dmul_rn(r, se);
}

// NEXT-4: the paper's rectangle user field x ~ U[x0, x1], y ~ U[y0, y1].
__global__ void __launch_bounds__(256) gen_drops_rect_kernel(double x0, double x1, double y0, double y1, int K,
                                                             int64_t n_total, uint64_t seed, uint64_t first_drop,
                                                             double *pos) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n_total) return;
  const int64_t d = idx / K;
  const int k = (int)(idx - d * K);
  const xl::u64x4 w = xl::philox4x64_10(first_drop + (uint64_t)d, (uint64_t)k, 0, 0, seed, 0);
  double *p = pos + idx * 3;
  p[0] = __dadd_rn(x0, __dmul_rn(x1 - x0, xl::u01_53(w.v[0])));  // no FMA contraction (as gen_drops_kernel)
  p[1] = __dadd_rn(y0, __dmul_rn(y1 - y0, xl::u01_53(w.v[1])));
  p[2] = 0.0;
}

// The raw counter-based words behind both drop laws (R19), for a bit-exact audit.
__global__ void __launch_bounds__(256) draw_words_kernel(int K, int64_t n_total, uint64_t seed, uint64_t first_drop,
                                                         uint64_t *words) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n_total) return;
  const int64_t d = idx / K;
  const int k = (int)(idx - d * K);
  const xl::u64x4 w = xl::philox4x64_10(first_drop + (uint64_t)d, (uint64_t)k, 0, 0, seed, 0);
#pragma unroll
  for (int q = 0; q < 4; ++q) words[idx * 4 + q] = w.v[q];
}

}  // namespace

namespace xlh {

int launch_draw_words(int K, int64_t n_drops, uint64_t seed, uint64_t first_drop, uint64_t *words, cudaStream_t s) {
  const int64_t n = n_drops * (int64_t)K;
  if (n == 0) return XLMIMO_OK;
  KTimer tm(s, "draw_words");
  draw_words_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(K, n, seed, first_drop, words);
  tm.stop(s);
  count_launch();
  return check_launch("draw_words_kernel");
}

int launch_gen_drops_rect(double x0, double x1, double y0, double y1, int K, int64_t n_drops, uint64_t seed,
                          uint64_t first_drop, double *pos, cudaStream_t s) {
  const int64_t n = n_drops * (int64_t)K;
  if (n == 0) return XLMIMO_OK;
  KTimer tm(s, "gen_drops_rect");
  gen_drops_rect_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(x0, x1, y0, y1, K, n, seed, first_drop, pos);
  tm.stop(s);
  count_launch();
  return check_launch("gen_drops_rect_kernel");
}

int launch_gen_drops(const xlmimo_users_t &u, int K, int64_t n_drops, uint64_t seed, uint64_t first_drop,
                     double *pos, cudaStream_t s) {
  const int64_t n = n_drops * (int64_t)K;
  if (n == 0) return XLMIMO_OK;
  const int64_t blocks = (n + 255) / 256;
  KTimer tm(s, "gen_drops");
  gen_drops_kernel<<<(unsigned)blocks, 256, 0, s>>>(u, K, n, seed, first_drop, pos);
  tm.stop(s);
  count_launch();
  return check_launch("gen_drops_kernel");
}

}  // namespace xlh
