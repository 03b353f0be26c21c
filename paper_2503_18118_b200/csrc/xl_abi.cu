// xl_abi.cu -- the extern "C" boundary of libxlmimo.so (include/xlmimo.h):
// argument validation, workspace carving, and the launch sequence of each
// entry point on the caller's stream.  No arithmetic of the method lives here.
#include <atomic>
#include <cmath>
#include <map>
#include <mutex>
#include <string>
#include <vector>
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include <nvtx3/nvToolsExt.h>

#include "xl_common.cuh"

namespace {

thread_local char g_err[512] = "";

// NVTX range around each compute entry point (header-only NVTX v3: a no-op unless a
// tool such as ncu / nsys injects itself), so profiles show the ABI call structure.
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
std::atomic<uint64_t> g_launches{0};
std::atomic<int64_t> g_opts[XLMIMO_OPT_COUNT];

bool bad_array(const xlmimo_array_t *a) {
  if (!a) return true;
  if (a->kind != XLMIMO_ULA && a->kind != XLMIMO_UPA) return true;
  if (!(a->fc_hz > 0.0) || !(a->spacing_wl > 0.0) || !(a->beta0 > 0.0)) return true;
  if (!std::isfinite(a->fc_hz) || !std::isfinite(a->spacing_wl) || !std::isfinite(a->beta0)) return true;
  if (a->n_y < 1) return true;
  if (a->kind == XLMIMO_UPA && a->n_z < 1) return true;
  return false;
}

bool bad_users(const xlmimo_users_t *u) {
  if (!u) return true;
  if (!(u->r_min_m > 0.0) || !(u->r_min_m <= u->r_max_m) || !std::isfinite(u->r_max_m)) return true;
  if (!(u->az_min_deg <= u->az_max_deg) || !(fabs(u->az_min_deg) < 90.0) || !(fabs(u->az_max_deg) < 90.0)) return true;
  if (!(u->el_min_deg <= u->el_max_deg) || !(fabs(u->el_min_deg) < 90.0) || !(fabs(u->el_max_deg) < 90.0)) return true;
  return false;
}

xlh::ArrayP to_params(const xlmimo_array_t *a) {
  xlh::ArrayP p;
  p.kind = a->kind;
  p.n_y = a->n_y;
  p.n_z = a->kind == XLMIMO_ULA ? 1 : a->n_z;
  p.lambda = xl::kC / a->fc_hz;
  p.pitch = a->spacing_wl * p.lambda;
  p.sqrt_beta0 = sqrt(a->beta0);
  return p;
}

int n_recv_of(uint32_t r) { return __builtin_popcount(r & 15u); }

size_t align256(size_t x) { return (x + 255) / 256 * 256; }

struct Carve {
  char *base;
  size_t off = 0;
  explicit Carve(void *b) : base((char *)b) {}
  void *take(size_t bytes) {
    void *p = base ? base + off : nullptr;
    off += align256(bytes);
    return p;
  }
};

// Layout of the saturation-sweep workspace (shared by the size query and the call).
// fp32 exact sweeps for K > 64 run the tcgen05 block-pair Gram once per N (its kernels have
// no nested levels): Gram of the n-th centred array into `g1`, copied into level n of `grams`.
bool sweep_per_level(int K, int gram_kind, int precision) {
  return K > xl::kMaxK && gram_kind == XLMIMO_GRAM_EXACT && precision == XLMIMO_FP32;
}

struct SweepWs {
  double *pos, *grams, *g1, *rates, *erg, *ergv, *sat, *satp;
  int64_t *nval;
  uint32_t *flags;
  void *gws, *rws;
  size_t gws_bytes, rws_bytes;
  size_t total;
};

SweepWs sweep_layout(void *ws, const xlh::ArrayP &ap, const int64_t *n_list, int n_n, int K, int64_t D, int n_snr,
                     uint32_t receivers, int gram_kind, int precision) {
  Carve c(ws);
  SweepWs w;
  const int R = n_recv_of(receivers);
  w.pos = (double *)c.take((size_t)D * K * 3 * sizeof(double));
  w.grams = (double *)c.take((size_t)D * n_n * K * K * 2 * sizeof(double));
  const bool per_level = sweep_per_level(K, gram_kind, precision) && n_n > 1;
  w.g1 = (double *)c.take(per_level ? (size_t)D * K * K * 2 * sizeof(double) : 0);
  w.rates = (double *)c.take((size_t)D * n_n * n_snr * R * sizeof(double));
  w.flags = (uint32_t *)c.take((size_t)D * n_n * sizeof(uint32_t));
  w.erg = (double *)c.take((size_t)n_n * n_snr * R * sizeof(double));
  w.ergv = (double *)c.take((size_t)n_n * n_snr * R * sizeof(double));
  w.nval = (int64_t *)c.take((size_t)n_n * n_snr * R * sizeof(int64_t));
  w.sat = (double *)c.take(4 * sizeof(double));
  w.satp = (double *)c.take(xlh::saturation_stats_scratch(D));
  w.gws_bytes = 0;
  if (gram_kind == XLMIMO_GRAM_EXACT) {
    xlh::ArrayP big = ap;
    big.n_y = n_list[n_n - 1];
    if (sweep_per_level(K, gram_kind, precision)) {  // the largest single-level workspace
      for (int l = 0; l < n_n; ++l) {
        big.n_y = n_list[l];
        const size_t b = xlh::gram_ws_bytes(big, K, D, 1, precision, XLMIMO_FUSED);
        if (b > w.gws_bytes) w.gws_bytes = b;
      }
    } else {
      w.gws_bytes = xlh::gram_ws_bytes(big, K, D, n_n, precision, XLMIMO_FUSED);
    }
  }
  w.gws = c.take(w.gws_bytes);
  // K > 64: receivers through the large-K path (CAP by Cholesky slots, MRC)
  w.rws_bytes = K > xl::kMaxK ? xlh::sum_rate_large_ws_bytes(K, D * n_n, n_snr, receivers) : 0;
  w.rws = c.take(w.rws_bytes);
  w.total = c.off;
  return w;
}

int validate_sweep(const xlmimo_array_t *array, const int64_t *n_list, int n_n, int K, int64_t n_drops,
                   const double *snr_db, int n_snr, uint32_t receivers, int gram_kind, int precision, double t) {
  if (bad_array(array)) return xlh::set_error(XLMIMO_EINVAL, "sweep: invalid array");
  if (array->kind != XLMIMO_ULA) return xlh::set_error(XLMIMO_EUNSUPPORTED, "sweep: ULA only");
  if (!n_list || n_n < 1 || n_n > 32) return xlh::set_error(XLMIMO_EINVAL, "sweep: n_list empty or > 32 entries");
  for (int i = 0; i < n_n; ++i) {
    if (n_list[i] < 1) return xlh::set_error(XLMIMO_EINVAL, "sweep: n_list[%d] < 1", i);
    if (i && n_list[i] <= n_list[i - 1]) return xlh::set_error(XLMIMO_EINVAL, "sweep: n_list not ascending");
    if ((n_list[i] & 1) != (n_list[0] & 1)) return xlh::set_error(XLMIMO_EINVAL, "sweep: n_list mixed parity");
  }
  if (K < 1 || K > xl::kMaxKLarge)
    return xlh::set_error(K < 1 ? XLMIMO_EINVAL : XLMIMO_EUNSUPPORTED, "sweep: K=%d", K);
  if (n_drops < 1) return xlh::set_error(XLMIMO_EINVAL, "sweep: n_drops < 1");
  if (!snr_db || n_snr < 1 || n_snr > xl::kMaxSnr) return xlh::set_error(XLMIMO_EINVAL, "sweep: n_snr out of [1,16]");
  if ((receivers & 15u) == 0 || (receivers & ~15u)) return xlh::set_error(XLMIMO_EINVAL, "sweep: receivers");
  if (gram_kind != XLMIMO_GRAM_EXACT && gram_kind != XLMIMO_GRAM_CLOSED_FORM)
    return xlh::set_error(XLMIMO_EINVAL, "sweep: gram_kind");
  if (gram_kind == XLMIMO_GRAM_CLOSED_FORM && array->spacing_wl != 0.5)
    return xlh::set_error(XLMIMO_EUNSUPPORTED, "sweep: the closed form assumes lambda/2 spacing (PAPER.md:52)");
  if (precision != XLMIMO_FP64 && precision != XLMIMO_FP32) return xlh::set_error(XLMIMO_EINVAL, "sweep: precision");
  if (!(t > 0.0 && t < 1.0)) return xlh::set_error(XLMIMO_EINVAL, "sweep: t not in (0,1)");
  return XLMIMO_OK;
}

int run_sweep(const xlmimo_array_t *array, const int64_t *n_list, int32_t n_n, const xlmimo_users_t *users,
              const double *pos, const double *pos_host, int32_t K, int64_t n_drops, uint64_t seed,
              const double *snr_db, int32_t n_snr, uint32_t receivers, int32_t gram_kind, int32_t precision,
              double t, double *ergodic, int64_t *n_valid, double *ergodic_valid, double *sat, double *per_drop,
              void *ws, size_t ws_bytes, cudaStream_t s) {
  const xlh::ArrayP ap = to_params(array);
  SweepWs w = sweep_layout(ws, ap, n_list, n_n, K, n_drops, n_snr, receivers, gram_kind, precision);
  if (!ws || ws_bytes < w.total)
    return xlh::set_error(XLMIMO_EWORKSPACE, "sweep: workspace %zu < %zu bytes", ws_bytes, w.total);
  int rc;
  const double *P = pos;
  if (pos_host) {
    if (cudaMemcpyAsync(w.pos, pos_host, (size_t)n_drops * K * 3 * sizeof(double), cudaMemcpyHostToDevice, s) !=
        cudaSuccess)
      return xlh::check_launch("sweep: H2D positions");
    P = w.pos;
  } else if (!P) {
    if ((rc = xlh::launch_gen_drops(*users, K, n_drops, seed, 0, w.pos, s))) return rc;
    P = w.pos;
  }
  if (gram_kind == XLMIMO_GRAM_EXACT && sweep_per_level(K, gram_kind, precision)) {
    xlh::ArrayP al = ap;
    const size_t gb = (size_t)K * K * 2 * sizeof(double);
    rc = XLMIMO_OK;
    for (int l = 0; l < n_n && !rc; ++l) {
      al.n_y = n_list[l];
      double *dst = n_n > 1 ? w.g1 : w.grams;
      rc = xlh::launch_gram_exact(al, P, K, n_drops, &n_list[l], 1, precision, XLMIMO_FUSED, dst, w.gws, w.gws_bytes,
                                  s);
      if (!rc && n_n > 1 &&
          cudaMemcpy2DAsync((char *)w.grams + l * gb, n_n * gb, w.g1, gb, gb, (size_t)n_drops,
                            cudaMemcpyDeviceToDevice, s) != cudaSuccess)
        rc = xlh::check_launch("sweep: level copy");
    }
  } else if (gram_kind == XLMIMO_GRAM_EXACT) {
    xlh::ArrayP big = ap;
    big.n_y = n_list[n_n - 1];
    rc = xlh::launch_gram_exact(big, P, K, n_drops, n_list, n_n, precision, XLMIMO_FUSED, w.grams, w.gws,
                                w.gws_bytes, s);
  } else {
    rc = xlh::launch_closed_form(ap, P, K, n_drops, n_list, n_n, w.grams, nullptr, s);
  }
  if (rc) return rc;
  double *rates = per_drop ? per_drop : w.rates;
  if (cudaMemsetAsync(w.flags, 0, (size_t)n_drops * n_n * sizeof(uint32_t), s) != cudaSuccess)
    return xlh::check_launch("sweep: memset flags");
  if (K > xl::kMaxK)
    rc = xlh::launch_sum_rate_large(w.grams, K, n_drops * n_n, snr_db, n_snr, receivers, rates, w.flags, w.rws,
                                    w.rws_bytes, s);
  else
    rc = xlh::launch_sum_rate(w.grams, K, n_drops * n_n, snr_db, n_snr, receivers, rates, w.flags, s);
  if (rc) return rc;
  const int n_out = n_n * n_snr * n_recv_of(receivers);
  if ((rc = xlh::launch_ergodic_reduce(rates, n_drops, n_out, w.erg, w.ergv, w.nval, s))) return rc;
  if ((rc = xlh::launch_saturation_stats(P, K, n_drops, t, ap.pitch, w.sat, w.satp, s))) return rc;
  if (cudaMemcpyAsync(ergodic, w.erg, (size_t)n_out * sizeof(double), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      (ergodic_valid && cudaMemcpyAsync(ergodic_valid, w.ergv, (size_t)n_out * sizeof(double),
                                        cudaMemcpyDeviceToHost, s) != cudaSuccess) ||
      cudaMemcpyAsync(n_valid, w.nval, (size_t)n_out * sizeof(int64_t), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaMemcpyAsync(sat, w.sat, 4 * sizeof(double), cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return xlh::check_launch("sweep: D2H results");
  if (cudaStreamSynchronize(s) != cudaSuccess) return xlh::check_launch("sweep: synchronize");
  return XLMIMO_OK;
}

}  // namespace

namespace {
struct TimingRec {
  std::string name;
  cudaEvent_t a, b;
};
std::mutex g_tmu;
std::atomic<bool> g_timing{false};
std::vector<TimingRec *> g_trecs;

void timing_clear() {
  for (TimingRec *r : g_trecs) {
    cudaEventDestroy(r->a);
    cudaEventDestroy(r->b);
    delete r;
  }
  g_trecs.clear();
}
}  // namespace

namespace xlh {

void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

KTimer::KTimer(cudaStream_t s, const char *name) {
  if (!g_timing.load(std::memory_order_relaxed)) return;
  TimingRec *r = new TimingRec{name, nullptr, nullptr};
  cudaEventCreate(&r->a);
  cudaEventCreate(&r->b);
  cudaEventRecord(r->a, s);
  rec = r;
}

void KTimer::stop(cudaStream_t s) {
  if (!rec) return;
  TimingRec *r = (TimingRec *)rec;
  cudaEventRecord(r->b, s);
  std::lock_guard<std::mutex> lk(g_tmu);
  g_trecs.push_back(r);
  rec = nullptr;
}

int set_error(int code, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_launch(const char *what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(XLMIMO_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return XLMIMO_OK;
}

}  // namespace xlh

extern "C" {

const char *xlmimo_last_error(void) { return g_err; }

uint64_t xlmimo_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int xlmimo_timing_enable(int32_t on) {
  std::lock_guard<std::mutex> lk(g_tmu);
  if (on) timing_clear();
  g_timing.store(on != 0);
  return XLMIMO_OK;
}

int xlmimo_timing_read(int32_t max_entries, char *names, int64_t *counts, double *total_ms) {
  std::lock_guard<std::mutex> lk(g_tmu);
  std::map<std::string, std::pair<int64_t, double>> agg;
  for (TimingRec *r : g_trecs) {
    if (cudaEventSynchronize(r->b) != cudaSuccess) return xlh::check_launch("timing_read");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r->a, r->b);
    auto &e = agg[r->name];
    e.first += 1;
    e.second += ms;
  }
  int n = 0;
  for (auto &kv : agg) {
    if (n >= max_entries) break;
    if (names) {
      strncpy(names + 64 * n, kv.first.c_str(), 63);
      names[64 * n + 63] = 0;
    }
    if (counts) counts[n] = kv.second.first;
    if (total_ms) total_ms[n] = kv.second.second;
    ++n;
  }
  return n;
}

int xlmimo_gen_drops(const xlmimo_users_t *users, int32_t K, int64_t n_drops, uint64_t seed, uint64_t first_drop,
                     double *pos, void *stream) {
  NvtxRange nvtx_range("xlmimo_gen_drops");
  g_err[0] = 0;
  if (bad_users(users)) return xlh::set_error(XLMIMO_EINVAL, "gen_drops: invalid user law");
  if (K < 1 || n_drops < 0 || (!pos && n_drops > 0))
    return xlh::set_error(XLMIMO_EINVAL, "gen_drops: K=%d n_drops=%lld pos=%p", K, (long long)n_drops, (void *)pos);
  return xlh::launch_gen_drops(*users, K, n_drops, seed, first_drop, pos, (cudaStream_t)stream);
}

size_t xlmimo_gram_exact_workspace(const xlmimo_array_t *array, int32_t K, int64_t n_drops, int32_t precision,
                                   int32_t mode) {
  if (bad_array(array) || K < 1 || K > xl::kMaxKLarge || n_drops < 0) return 0;
  if (K > xl::kMaxK && mode == XLMIMO_MATERIALIZED && precision != XLMIMO_FP32) return 0;  // unsupported
  return xlh::gram_ws_bytes(to_params(array), K, n_drops, 1, precision, mode);
}

int xlmimo_gram_exact(const xlmimo_array_t *array, const double *pos, int32_t K, int64_t n_drops,
                      int32_t precision, int32_t mode, double *gram, void *ws, size_t ws_bytes, void *stream) {
  NvtxRange nvtx_range("xlmimo_gram_exact");
  g_err[0] = 0;
  if (bad_array(array)) return xlh::set_error(XLMIMO_EINVAL, "gram_exact: invalid array");
  if (K < 1 || n_drops < 0) return xlh::set_error(XLMIMO_EINVAL, "gram_exact: K=%d n_drops=%lld", K, (long long)n_drops);
  if (K > xl::kMaxKLarge) return xlh::set_error(XLMIMO_EUNSUPPORTED, "gram_exact: K=%d > %d", K, xl::kMaxKLarge);
  if (precision != XLMIMO_FP64 && precision != XLMIMO_FP32) return xlh::set_error(XLMIMO_EINVAL, "gram_exact: precision");
  if (mode != XLMIMO_FUSED && mode != XLMIMO_MATERIALIZED) return xlh::set_error(XLMIMO_EINVAL, "gram_exact: mode");
  if (n_drops > 0 && (!pos || !gram)) return xlh::set_error(XLMIMO_EINVAL, "gram_exact: null pointer");
  const xlh::ArrayP ap = to_params(array);
  const int64_t N = ap.kind == XLMIMO_ULA ? ap.n_y : ap.n_y * ap.n_z;
  return xlh::launch_gram_exact(ap, pos, K, n_drops, &N, 1, precision, mode, gram, ws, ws_bytes,
                                (cudaStream_t)stream);
}

int xlmimo_gram_closed_form(const xlmimo_array_t *array, const double *pos, int32_t K, int64_t n_drops,
                            double *gram, uint32_t *flags, void *stream) {
  NvtxRange nvtx_range("xlmimo_gram_closed_form");
  g_err[0] = 0;
  if (bad_array(array)) return xlh::set_error(XLMIMO_EINVAL, "closed_form: invalid array");
  if (array->kind != XLMIMO_ULA) return xlh::set_error(XLMIMO_EUNSUPPORTED, "closed_form: ULA only (PAPER.md:40)");
  if (array->spacing_wl != 0.5)
    return xlh::set_error(XLMIMO_EUNSUPPORTED, "closed_form: Eqs. (4)/(6) assume lambda/2 spacing (PAPER.md:52)");
  if (K < 1 || n_drops < 0) return xlh::set_error(XLMIMO_EINVAL, "closed_form: K=%d", K);
  if (n_drops > 0 && (!pos || !gram)) return xlh::set_error(XLMIMO_EINVAL, "closed_form: null pointer");
  const xlh::ArrayP ap = to_params(array);
  const int64_t M = ap.n_y;
  return xlh::launch_closed_form(ap, pos, K, n_drops, &M, 1, gram, flags, (cudaStream_t)stream);
}

size_t xlmimo_sum_rate_workspace(int32_t K, int64_t n_drops, int32_t n_snr, uint32_t receivers) {
  if (K < 1 || K > xl::kMaxKLarge || n_drops < 0 || n_snr < 1 || n_snr > xl::kMaxSnr) return 0;
  if (K <= xl::kMaxK) return 0;
  return xlh::sum_rate_large_ws_bytes(K, n_drops, n_snr, receivers);
}

int xlmimo_sum_rate_ws(const double *gram, int32_t K, int64_t n_drops, const double *snr_db, int32_t n_snr,
                       uint32_t receivers, double *rates, uint32_t *flags, void *ws, size_t ws_bytes, void *stream) {
  NvtxRange nvtx_range("xlmimo_sum_rate_ws");
  g_err[0] = 0;
  if (K < 1 || n_drops < 0) return xlh::set_error(XLMIMO_EINVAL, "sum_rate: K=%d", K);
  if (K > xl::kMaxKLarge) return xlh::set_error(XLMIMO_EUNSUPPORTED, "sum_rate: K=%d > %d", K, xl::kMaxKLarge);
  if (!snr_db || n_snr < 1 || n_snr > xl::kMaxSnr) return xlh::set_error(XLMIMO_EINVAL, "sum_rate: n_snr out of [1,16]");
  if ((receivers & 15u) == 0 || (receivers & ~15u)) return xlh::set_error(XLMIMO_EINVAL, "sum_rate: receivers");
  if (n_drops > 0 && (!gram || !rates)) return xlh::set_error(XLMIMO_EINVAL, "sum_rate: null pointer");
  if (K > xl::kMaxK) {
    return xlh::launch_sum_rate_large(gram, K, n_drops, snr_db, n_snr, receivers, rates, flags, ws, ws_bytes,
                                      (cudaStream_t)stream);
  }
  return xlh::launch_sum_rate(gram, K, n_drops, snr_db, n_snr, receivers, rates, flags, (cudaStream_t)stream);
}

int xlmimo_sum_rate(const double *gram, int32_t K, int64_t n_drops, const double *snr_db, int32_t n_snr,
                    uint32_t receivers, double *rates, uint32_t *flags, void *stream) {
  return xlmimo_sum_rate_ws(gram, K, n_drops, snr_db, n_snr, receivers, rates, flags, nullptr, 0, stream);
}

size_t xlmimo_app_a_bounds_workspace(int32_t K, int64_t n_drops, int32_t n_snr, int32_t with_eig) {
  if (K < 1 || K > xl::kMaxKLarge || n_drops < 0 || n_snr < 1 || n_snr > xl::kMaxSnr) return 0;
  const size_t b = xlh::large_k_ws_bytes(K, n_drops, 1 + n_snr, false);
  if (!with_eig || K <= xl::kMaxK) return b;
  return (b + 255) / 256 * 256 + xlh::eig_ws_bytes(K, n_drops);
}

int xlmimo_app_a_bounds(const double *gram, int32_t K, int64_t n_drops, const double *snr_db, int32_t n_snr,
                        double *rstat, double *bounds, double *eig, uint32_t *flags, void *ws, size_t ws_bytes,
                        void *stream) {
  NvtxRange nvtx_range("xlmimo_app_a_bounds");
  g_err[0] = 0;
  if (K < 1 || n_drops < 0) return xlh::set_error(XLMIMO_EINVAL, "app_a_bounds: K=%d", K);
  if (K > xl::kMaxKLarge) return xlh::set_error(XLMIMO_EUNSUPPORTED, "app_a_bounds: K=%d > %d", K, xl::kMaxKLarge);
  if (!snr_db || n_snr < 1 || n_snr > xl::kMaxSnr)
    return xlh::set_error(XLMIMO_EINVAL, "app_a_bounds: n_snr out of [1,16]");
  if (n_drops > 0 && (!gram || !rstat || !bounds)) return xlh::set_error(XLMIMO_EINVAL, "app_a_bounds: null pointer");
  return xlh::launch_bounds(gram, K, n_drops, snr_db, n_snr, rstat, bounds, eig, flags, ws, ws_bytes,
                            (cudaStream_t)stream);
}

int xlmimo_sum_rate_mismatched(const double *gram, const double *gram_model, int32_t K, int64_t n_drops,
                               const double *snr_db, int32_t n_snr, double *rates, uint32_t *flags, void *stream) {
  NvtxRange nvtx_range("xlmimo_sum_rate_mismatched");
  g_err[0] = 0;
  if (K < 1 || n_drops < 0) return xlh::set_error(XLMIMO_EINVAL, "sum_rate_mismatched: K=%d", K);
  if (K > xl::kMaxK) return xlh::set_error(XLMIMO_EUNSUPPORTED, "sum_rate_mismatched: K=%d > %d", K, xl::kMaxK);
  if (!snr_db || n_snr < 1 || n_snr > xl::kMaxSnr)
    return xlh::set_error(XLMIMO_EINVAL, "sum_rate_mismatched: n_snr out of [1,16]");
  if (n_drops > 0 && (!gram || !gram_model || !rates))
    return xlh::set_error(XLMIMO_EINVAL, "sum_rate_mismatched: null pointer");
  return xlh::launch_sum_rate_mismatched(gram, gram_model, K, n_drops, snr_db, n_snr, rates, flags,
                                         (cudaStream_t)stream);
}

int xlmimo_gen_drops_rect(double x_min, double x_max, double y_min, double y_max, int32_t K, int64_t n_drops,
                          uint64_t seed, uint64_t first_drop, double *pos, void *stream) {
  NvtxRange nvtx_range("xlmimo_gen_drops_rect");
  g_err[0] = 0;
  if (!(x_min > 0.0) || !(x_min <= x_max) || !(y_min <= y_max) || !std::isfinite(x_max) || !std::isfinite(y_min) ||
      !std::isfinite(y_max))
    return xlh::set_error(XLMIMO_EINVAL, "gen_drops_rect: invalid rectangle");
  if (K < 1 || n_drops < 0 || (!pos && n_drops > 0)) return xlh::set_error(XLMIMO_EINVAL, "gen_drops_rect: K/n/pos");
  return xlh::launch_gen_drops_rect(x_min, x_max, y_min, y_max, K, n_drops, seed, first_drop, pos,
                                    (cudaStream_t)stream);
}

static const double kSnrProbe = 0.0;  // validate_sweep wants a non-null SNR list; the query has none

size_t xlmimo_saturation_sweep_workspace(const xlmimo_array_t *array, const int64_t *n_list, int32_t n_n, int32_t K,
                                         int64_t n_drops, int32_t n_snr, uint32_t receivers, int32_t gram_kind,
                                         int32_t precision) {
  char saved[sizeof(g_err)];  // a size query reports a bad argument as 0 bytes; the thread's last error stays
  memcpy(saved, g_err, sizeof(g_err));
  const int bad = validate_sweep(array, n_list, n_n, K, n_drops, &kSnrProbe, n_snr, receivers, gram_kind, precision,
                                 0.5);
  memcpy(g_err, saved, sizeof(g_err));
  if (bad) return 0;
  return sweep_layout(nullptr, to_params(array), n_list, n_n, K, n_drops, n_snr, receivers, gram_kind, precision)
      .total;
}

int xlmimo_saturation_sweep(const xlmimo_array_t *array, const int64_t *n_list, int32_t n_n,
                            const xlmimo_users_t *users, const double *pos, int32_t K, int64_t n_drops, uint64_t seed,
                            const double *snr_db, int32_t n_snr, uint32_t receivers, int32_t gram_kind,
                            int32_t precision, double t, double *ergodic, int64_t *n_valid, double *ergodic_valid,
                            double *sat, double *per_drop, void *ws, size_t ws_bytes, void *stream) {
  NvtxRange nvtx_range("xlmimo_saturation_sweep");
  g_err[0] = 0;
  int rc = validate_sweep(array, n_list, n_n, K, n_drops, snr_db, n_snr, receivers, gram_kind, precision, t);
  if (rc) return rc;
  if (!pos && bad_users(users)) return xlh::set_error(XLMIMO_EINVAL, "sweep: no positions and invalid user law");
  if (!ergodic || !n_valid || !sat) return xlh::set_error(XLMIMO_EINVAL, "sweep: null output");
  return run_sweep(array, n_list, n_n, users, pos, nullptr, K, n_drops, seed, snr_db, n_snr, receivers, gram_kind,
                   precision, t, ergodic, n_valid, ergodic_valid, sat, per_drop, ws, ws_bytes, (cudaStream_t)stream);
}

int xlmimo_saturation_sweep_host(const xlmimo_array_t *array, const int64_t *n_list, int32_t n_n,
                                 const double *pos_host, int32_t K, int64_t n_drops, const double *snr_db,
                                 int32_t n_snr, uint32_t receivers, int32_t gram_kind, int32_t precision, double t,
                                 double *ergodic, int64_t *n_valid, double *ergodic_valid, double *sat, void *ws,
                                 size_t ws_bytes, void *stream) {
  NvtxRange nvtx_range("xlmimo_saturation_sweep_host");
  g_err[0] = 0;
  int rc = validate_sweep(array, n_list, n_n, K, n_drops, snr_db, n_snr, receivers, gram_kind, precision, t);
  if (rc) return rc;
  if (!pos_host || !ergodic || !n_valid || !sat) return xlh::set_error(XLMIMO_EINVAL, "sweep_host: null pointer");
  return run_sweep(array, n_list, n_n, nullptr, nullptr, pos_host, K, n_drops, 0, snr_db, n_snr, receivers, gram_kind,
                   precision, t, ergodic, n_valid, ergodic_valid, sat, nullptr, ws, ws_bytes, (cudaStream_t)stream);
}

int xlmimo_draw_words(int32_t K, int64_t n_drops, uint64_t seed, uint64_t first_drop, uint64_t *words,
                      void *stream) {
  NvtxRange nvtx_range("xlmimo_draw_words");
  g_err[0] = 0;
  if (K < 1 || n_drops < 0 || (!words && n_drops > 0)) return xlh::set_error(XLMIMO_EINVAL, "draw_words: K/n/words");
  return xlh::launch_draw_words(K, n_drops, seed, first_drop, words, (cudaStream_t)stream);
}

int xlmimo_set_option(int32_t option, int64_t value) {
  g_err[0] = 0;
  if (option < 0 || option >= XLMIMO_OPT_COUNT) return xlh::set_error(XLMIMO_EINVAL, "set_option: %d", option);
  g_opts[option].store(value);
  return XLMIMO_OK;
}

int64_t xlmimo_get_option(int32_t option) {
  return (option < 0 || option >= XLMIMO_OPT_COUNT) ? 0 : g_opts[option].load();
}

}  // extern "C"

namespace xlh {
int64_t option(int id) { return xlmimo_get_option(id); }
}  // namespace xlh
