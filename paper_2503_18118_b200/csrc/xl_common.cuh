// xl_common.cuh -- device helpers shared by the xlmimo kernels (sm_100a).
//
// Product code: shares nothing with oracle/.  See include/xlmimo.h for the ABI
// and DESIGN.md for the kernel designs and the readings R1..R23.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/xlmimo.h"

namespace xl {

constexpr double kC = 299792458.0;  // m/s, exact (R2)
constexpr int kMaxK = 64;           // fused paths: K <= 64
constexpr int kMaxKLarge = 1024;    // large-K paths (tiled Cholesky, block-pair Gram)
constexpr int kMaxSnr = 16;

// ---------------------------------------------------------------------------
// Philox4x64-10 (Salmon et al., SC'11), device implementation (R19).
// ---------------------------------------------------------------------------
struct u64x4 { uint64_t v[4]; };

__device__ __forceinline__ u64x4 philox4x64_10(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3,
                                               uint64_t k0, uint64_t k1) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ULL, M1 = 0xCA5A826395121157ULL;
  const uint64_t W0 = 0x9E3779B97F4A7C15ULL, W1 = 0xBB67AE8584CAA73BULL;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t hi0 = __umul64hi(M0, c0), lo0 = M0 * c0;
    const uint64_t hi1 = __umul64hi(M1, c2), lo1 = M1 * c2;
    const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += W0; k1 += W1;
  }
  u64x4 o; o.v[0] = c0; o.v[1] = c1; o.v[2] = c2; o.v[3] = c3;
  return o;
}

__device__ __forceinline__ double u01_53(uint64_t w) { return (double)(w >> 11) * 0x1.0p-53; }

// ---------------------------------------------------------------------------
// Per-user constants of Eq. (3) for the fused generator.
//   ULA: r^2 = xz2 + (y_user - y_m)^2 with xz2 = x^2 + z^2 (R21), amplitude
//        sqrt(beta0) sqrt(x_eff) r^{-3/2} with x_eff = sqrt(xz2).
//   UPA: r^2 = x^2 + (y - y_p)^2 + (z - z_q)^2, x_eff = |x| (R5).
// ---------------------------------------------------------------------------
struct UserC {
  double xz2;   // ULA: x^2+z^2 ; UPA: x^2
  double y, z;  // user y (and z for UPA)
  double amp;   // sqrt(beta0) * sqrt(x_eff)
};

__device__ __forceinline__ UserC make_user(const double *p, int kind, double sqrt_beta0) {
  UserC u;
  const double x = p[0], y = p[1], z = p[2];
  if (kind == XLMIMO_ULA) {
    u.xz2 = fma(x, x, z * z);
    u.z = 0.0;
    u.amp = sqrt_beta0 * sqrt(sqrt(u.xz2));
  } else {
    u.xz2 = x * x;
    u.z = z;
    u.amp = sqrt_beta0 * sqrt(fabs(x));
  }
  u.y = y;
  return u;
}

// 1/sqrt(x) for positive normal x: MUFU.RSQ64H (no special-case branches with
// .ftz; it reads only the high word of x, so its error reaches ~1e-6 relative)
// + one third-order Householder step y (1 + e/2 + 3e^2/8), e = 1 - x y^2:
// error O(e^3) -> ~1 ulp.  (A plain Newton step leaves 1.5 e^2 ~ 4e-13, which
// moves the phase 2 pi r/lambda by ~1e-8 rad at r/lambda ~ 5e3: measured parity
// failure, so the cubic term is required.)  5 FP64 instructions.
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x * y, y, 1.0);
  const double p = fma(e, 0.375, 0.5);
  return fma(y * e, p, y);
}

// Near-minimax polynomials (Chebyshev-node Lawson fits in 50-digit arithmetic) in u = g^2
// for g in [-1/2, 1/2]: sin(pi/2 g) = g * S(u), cos(pi/2 g) = C(u).
//   XL_SINCOS_DEG 5: |err| <= 1.9e-15 (sin) / 5.6e-14 (cos), 11 FP64 instructions;
//   XL_SINCOS_DEG 4: |err| <= 1.7e-12 (sin) / 4.7e-11 (cos), 9 FP64 instructions.
// Either bound keeps a Gram entry within 2 max|err| sqrt(G_ii G_jj) of the exact one
// (Cauchy-Schwarz over the coefficient errors), under the fp64 tier's 1e-9 (R9).
#ifndef XL_SINCOS_DEG
#define XL_SINCOS_DEG 4
#endif
#if XL_SINCOS_DEG == 5
__constant__ double kSinPoly[6] = {1.5707963267948898981, -0.64596409750431005807, 0.079692626155777645619,
                                   -0.0046817525918122076931, 0.0001604292666631208935,
                                   -3.5563888496214387972e-6};
__constant__ double kCosPoly[6] = {0.99999999999994445739, -1.23370055012016865, 0.25366950715400581474,
                                   -0.020863468005621057384, 0.00091916175238771112641,
                                   -0.000024850988050231297507};
#elif XL_SINCOS_DEG == 4
__constant__ double kSinPoly[5] = {1.570796326757624, -0.6459640945217848, 0.0796925593294654,
                                   -0.004681141492935389, 0.00015798452268659335};
__constant__ double kCosPoly[5] = {0.9999999999529987, -1.2337005406691752, 0.25366920425732364,
                                   -0.020860073028414316, 0.000903634758823505};
#else
#error "XL_SINCOS_DEG must be 4 or 5"
#endif

// 1/sqrt(x) to ~3e-13 relative (MUFU seed + one Newton step, 4 FP64 instructions):
// enough for the amplitude r^{-3/2}, not for the phase (see rsqrt_nr).
__device__ __forceinline__ double rsqrt_newton(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x * y, y, 1.0);
  return fma(0.5 * y, e, y);
}

// h = amp * r^{-3/2} * e^{-j 2 pi r/lambda}  (Eq. 3), fp64, the fused generator's
// coefficient.  Phase: q4 = 4 r/lambda (quarter cycles), k = rint(q4) (FRND),
// quadrant = k mod 4 (F2I, XU pipe), g = q4 - k in [-1/2, 1/2] exactly, angle =
// (pi/2)(k + g): the fp64 range reduction of the north_star.  1/r to ~1 ulp
// (Householder), r^{-3/2} to ~3e-13 (Newton), sin / cos as above: 29 (degree 5) or 27
// (degree 4) FP64-pipe instructions + 2 MUFU + 1 F2I per coefficient, no branches.
// c4 = 4 / lambda.
__device__ __forceinline__ void coef_fast(double r2, double amp, double c4, double &re, double &im) {
  const double ir = rsqrt_nr(r2);
  const double r = r2 * ir;
  const double q4 = r * c4;
  const double k = rint(q4);       // FRND.F64
  const int qd = (int)k;           // F2I on the XU pipe (q4 < 2^31)
  const double g = q4 - k;         // exact, |g| <= 1/2
  const double u = g * g;
  double ps = kSinPoly[XL_SINCOS_DEG];
#pragma unroll
  for (int j = XL_SINCOS_DEG - 1; j >= 0; --j) ps = fma(ps, u, kSinPoly[j]);
  const double sn = ps * g;
  double pc = kCosPoly[XL_SINCOS_DEG];
#pragma unroll
  for (int j = XL_SINCOS_DEG - 1; j >= 0; --j) pc = fma(pc, u, kCosPoly[j]);
  const double cs = pc;
  const double a = amp * ir * rsqrt_newton(r);  // r^{-3/2}, ~3e-13 relative
  // quadrant q: (cos, sin) of (pi/2)(q + g) = q0 (cs, sn), q1 (-sn, cs), q2 (-cs, -sn), q3 (sn, -cs);
  // h = a (cos - j sin)  =>  re = a*c, im = a*(-s)
  const int q = qd & 3;
  const bool sw = q & 1;
  double c = sw ? sn : cs;
  double s = sw ? cs : sn;
  const int negc = ((q + 1) >> 1) & 1;  // q = 1, 2
  const int negs = (q >> 1) ^ 1;        // -s: flip unless q = 2, 3
  c = __hiloint2double(__double2hiint(c) ^ (negc << 31), __double2loint(c));
  s = __hiloint2double(__double2hiint(s) ^ (negs << 31), __double2loint(s));
  re = a * c;
  im = a * s;
}

// fp32 phasor and amplitude from fp64 distance / phase reduction (XLMIMO_FP32, K3):
// f = frac(r / lambda) in [-1/2, 1/2] reduced in fp64 (R13), then MUFU sin/cos of
// 2 pi f in fp32 (no quadrant split: MUFU takes the whole [-pi, pi] range).
__device__ __forceinline__ void coef_from_r2_f32(double r2, double amp, double inv_lambda, float &re,
                                                 float &im) {
  const double ir = rsqrt_nr(r2);
  const double r = r2 * ir;
  const double q = r * inv_lambda;
  const float f = (float)(q - rint(q));
  float s, c;
  __sincosf(6.28318530717958647692f * f, &s, &c);
  const float rf = (float)r;
  const float a = (float)amp * rsqrtf(rf) / rf;
  re = a * c;
  im = -a * s;
}

// Element coordinate of the "centred order" index t used by every exact-Gram
// kernel (ULA): for N even, t -> pair p = t>>1 at y = +-(p + 1/2) pitch; for N
// odd, t = 0 is the centre and t >= 1 -> +-(((t-1)>>1) + 1) pitch.  The first
// N' indices of this order are exactly the centred N'-element array of the same
// parity, which makes nested N a prefix (R18, saturation sweep).
__device__ __forceinline__ double ula_y_centred(int64_t t, bool n_odd, double pitch) {
  if (n_odd) {
    if (t == 0) return 0.0;
    const int64_t p = (t - 1) >> 1;
    const double y = (double)(p + 1) * pitch;
    return (t & 1) ? y : -y;
  }
  const int64_t p = t >> 1;
  const double y = ((double)p + 0.5) * pitch;
  return (t & 1) ? -y : y;
}
// the same for 0 <= t < 2^31 in 32-bit integer arithmetic
__device__ __forceinline__ double ula_y_centred(int t, bool n_odd, double pitch) {
  if (n_odd) {
    if (t == 0) return 0.0;
    const double y = (double)(((t - 1) >> 1) + 1) * pitch;
    return (t & 1) ? y : -y;
  }
  const double y = ((double)(t >> 1) + 0.5) * pitch;
  return (t & 1) ? -y : y;
}

}  // namespace xl

// ---------------------------------------------------------------------------
// Host-side internal interface between the ABI layer and the kernel files.
// ---------------------------------------------------------------------------
namespace xlh {

struct ArrayP {
  int kind;
  int64_t n_y, n_z;
  double lambda, pitch, sqrt_beta0;
};

void count_launch(uint64_t n = 1);

// Event bracket for the profiling hooks (no-op unless xlmimo_timing_enable(1)).
struct KTimer {
  void *rec = nullptr;
  KTimer(cudaStream_t s, const char *name);
  void stop(cudaStream_t s);
};
int set_error(int code, const char *fmt, ...);
int check_launch(const char *what);

// xl_drops.cu
int launch_gen_drops(const xlmimo_users_t &u, int K, int64_t n_drops, uint64_t seed, uint64_t first_drop,
                     double *pos, cudaStream_t s);

int launch_gen_drops_rect(double x0, double x1, double y0, double y1, int K, int64_t n_drops, uint64_t seed,
                          uint64_t first_drop, double *pos, cudaStream_t s);
// xl_rates.cu : NEXT-1 modified-ZF effective rate, rates [n_prob][n_snr]
int launch_sum_rate_mismatched(const double *gram, const double *gram_model, int K, int64_t n_prob,
                               const double *snr_db, int n_snr, double *rates, uint32_t *flags, cudaStream_t s);

// xl_gram.cu
// Exact Gram over element indices [0, N) in the "centred order", with snapshots
// at the level ends lvl_end[0..n_lvl-1] (ascending, last = N).  Output:
// out[drop][lvl][K][K][2] full Hermitian.  Scratch: gram_ws_bytes().
size_t gram_ws_bytes(const ArrayP &a, int K, int64_t n_drops, int n_lvl, int precision, int mode);
int launch_gram_exact(const ArrayP &a, const double *pos, int K, int64_t n_drops, const int64_t *lvl_end,
                      int n_lvl, int precision, int mode, double *out, void *ws, size_t ws_bytes,
                      cudaStream_t s);

// xl_gram_syrk.cu : large-K fp64 Gram as a chunked DMMA Hermitian rank-k update
size_t gram_syrk_ws_bytes(int K, int64_t n_drops, int n_lvl);
int launch_gram_syrk(const ArrayP &a, const double *pos, int K, int64_t n_drops, const int64_t *lvl_end, int n_lvl,
                     double *out, void *ws, size_t ws_bytes, cudaStream_t s);

// xl_stream_tc.cu : tcgen05 TF32 streaming Gram over a materialised batch
bool stream_tc_supported(int K, int64_t N);
int stream_tc_chunks(int64_t N);
int fused_tc_chunks(int64_t N, int64_t n_drops);
int stream_tc_parts(int K);
bool fused_tc_supported(const ArrayP &a, int K);
bool fused_tc_wide_supported(const ArrayP &a, int K);
int fused_tc_launches(int K);
#ifndef XL_FUSED_TC_MAXK
#define XL_FUSED_TC_MAXK 256  // tools/ab_cross.py: the fused launches win or tie up to 256
#endif
constexpr int kFusedTcMaxK = XL_FUSED_TC_MAXK;  // fp32 fused (generated fp16 operands) up to this K
bool fused_tc_supported_geometry(const ArrayP &a);
int launch_fused_tc(const ArrayP &a, const double *pos, int K, int64_t n_drops, int64_t N, double *ws,
                    cudaStream_t s);
int launch_stream_tc(const float *H, int K, int64_t N, int64_t drop0, int nb, double *ws, cudaStream_t s);
int launch_fused_tc_pair(const ArrayP &a, const double *pos, int K, int64_t n_drops, int64_t N, double *ws,
                         cudaStream_t s);
int fused_tc_pair_chunks(int64_t N);
bool materialise_tc_supported(const ArrayP &a);
int launch_h_materialise_tc(const ArrayP &a, const double *pos, int K, int64_t N, int64_t n_pad, int64_t drop0,
                            int nb, float *H, cudaStream_t s, int Kr = 0, int64_t t_first = 0, int l2_keep = 0);
size_t stream_pair_h_bytes(int K, int64_t n_drops, int64_t N);
int launch_stream_tc_pair(const ArrayP &a, const double *pos, int K, int64_t n_drops, int64_t N, double *ws,
                          float *H, cudaStream_t s);

// xl_closed.cu : out[drop][lvl][K][K][2] for M = n_list[lvl]
int launch_closed_form(const ArrayP &a, const double *pos, int K, int64_t n_drops, const int64_t *m_list,
                       int n_lvl, double *out, uint32_t *flags, cudaStream_t s);

// xl_rates.cu : problems = n_prob Grams [n_prob][K][K][2]; flags per problem
int launch_sum_rate(const double *gram, int K, int64_t n_prob, const double *snr_db, int n_snr,
                    uint32_t receivers, double *rates, uint32_t *flags, cudaStream_t s);

// xl_bounds.cu : Appendix A (NEXT-3) and the large-K (K > 64) receivers
size_t eig_ws_bytes(int K, int64_t n_drops);
size_t large_k_ws_bytes(int K, int64_t n_drops, int n_mat, bool with_dinv);
size_t sum_rate_large_ws_bytes(int K, int64_t n_drops, int n_snr, uint32_t receivers);
int launch_bounds(const double *gram, int K, int64_t n_drops, const double *snr_db, int n_snr, double *rstat,
                  double *bounds, double *eig, uint32_t *flags, void *ws, size_t ws_bytes, cudaStream_t s);
int launch_sum_rate_large(const double *gram, int K, int64_t n_drops, const double *snr_db, int n_snr,
                          uint32_t receivers, double *rates, uint32_t *flags, void *ws, size_t ws_bytes,
                          cudaStream_t s);

// xl_sweep.cu reductions
int64_t option(int id);
int launch_draw_words(int K, int64_t n_drops, uint64_t seed, uint64_t first_drop, uint64_t *words, cudaStream_t s);  // xlmimo_set_option value (0 = automatic)
int launch_ergodic_reduce(const double *per_drop, int64_t n_drops, int n_out, double *mean, double *mean_valid,
                          int64_t *count, cudaStream_t s);
size_t saturation_stats_scratch(int64_t n_drops);
int launch_saturation_stats(const double *pos, int K, int64_t n_drops, double t, double pitch, double *sat,
                            double *scratch, cudaStream_t s);

}  // namespace xlh
