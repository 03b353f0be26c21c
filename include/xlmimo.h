/*
 * xlmimo.h -- C ABI of the B200 (sm_100a) Monte Carlo engine for near-field
 * XL-MIMO uplink sum capacity (Cui, Park, Alouini, arXiv 2503.18118).
 *
 * Citations "PAPER.md:L" are line numbers of the paper's LaTeX source;
 * "SPEC.md:L" of the CPU-program specification written from it; "R#" are the
 * readings of ambiguous passages listed in DESIGN.md.
 *
 * Conventions for every entry point
 *  - Return 0 (XLMIMO_OK) or a negative xlmimo_status_t; never abort, never throw.
 *    The message of the last failure on the calling thread is xlmimo_last_error().
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Device work is enqueued on it asynchronously; functions returning HOST
 *    outputs synchronise that stream before returning.
 *  - "dev" pointers are CUDA device pointers, "host" pointers host memory; all
 *    are owned by the caller (the library allocates no persistent memory and
 *    keeps no state between calls).  Scratch comes from a caller workspace of
 *    the size the matching *_workspace() query returns.
 *  - Units are SI (m, Hz); SNRs are in dB.  rho = 10^(snr/10) is
 *    the transmit SNR P / sigma_n^2 of Eq. (1)/(9) (R4).
 *  - Complex matrices are interleaved (re, im) fp64, row-major, [.][K][K][2].
 *  - Results are deterministic: fixed reduction orders, no floating-point atomics.
 */
#ifndef XLMIMO_H
#define XLMIMO_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define XLMIMO_API __attribute__((visibility("default")))
#else
#define XLMIMO_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    XLMIMO_OK = 0,
    XLMIMO_EINVAL = -1,        /* bad argument (null pointer, K<1, N<1, fc<=0, |az|>=90, t not in (0,1), ...) */
    XLMIMO_EUNSUPPORTED = -2,  /* valid but not provided (closed form for a UPA; K beyond a path's limit) */
    XLMIMO_EWORKSPACE = -3,    /* workspace smaller than the matching *_workspace() query */
    XLMIMO_ECUDA = -4          /* CUDA launch / runtime error (text in xlmimo_last_error) */
} xlmimo_status_t;

/* Array kinds.  ULA: PAPER.md:40,52 -- M elements on the y-axis, centred at the
 * origin, pitch spacing_wl*lambda (lambda/2 in the paper); element m (1-based) at
 * y_m = (m - (M+1)/2) * pitch (R1).  UPA: n_y x n_z grid in the y-z
 * plane, centred, same pitch on both axes (R5: outside the paper). */
enum { XLMIMO_ULA = 0, XLMIMO_UPA = 1 };
enum { XLMIMO_FP64 = 0, XLMIMO_FP32 = 1 };              /* arithmetic of the exact Gram */
enum { XLMIMO_FUSED = 0, XLMIMO_MATERIALIZED = 1 };     /* H generated on the fly vs streamed from HBM */
enum { XLMIMO_GRAM_EXACT = 0, XLMIMO_GRAM_CLOSED_FORM = 1 };
/* Receiver bitmask; rates are written in this order for the bits that are set. */
enum { XLMIMO_RECV_CAP = 1, XLMIMO_RECV_ZF = 2, XLMIMO_RECV_MMSE = 4, XLMIMO_RECV_MRC = 8 };
/* Per-drop flag bits (OR-ed).  A flagged drop never aborts the batch (R10, R22). */
enum {
    XLMIMO_FLAG_G_NOT_PD = 1,      /* Cholesky of G failed -> ZF rate NaN */
    XLMIMO_FLAG_A_NOT_PD = 2,      /* Cholesky of I + rho G failed (some SNR) -> CAP, MMSE NaN */
    XLMIMO_FLAG_MRC_UNDEF = 4,     /* some G_ii <= 0 -> MRC NaN */
    XLMIMO_FLAG_DEGENERATE = 8,    /* closed form: some pair with ||x_i|-|x_j|| < lambda */
    XLMIMO_FLAG_NONFINITE = 16     /* non-finite Gram entry -> every rate NaN */
};

typedef struct {
    int32_t kind;        /* XLMIMO_ULA or XLMIMO_UPA */
    int64_t n_y, n_z;    /* ULA: n_y = N (= the paper's M), n_z = 1.  UPA: N = n_y * n_z */
    double fc_hz;        /* carrier; lambda = 299792458 / fc_hz (c exact, R2) */
    double spacing_wl;   /* element pitch in wavelengths (0.5) */
    double beta0;        /* sqrt(beta0) gain of Eq. (3) (1) */
} xlmimo_array_t;

typedef struct {
    double r_min_m, r_max_m;        /* range from the array centre, r ~ U[r_min, r_max] (R3) */
    double az_min_deg, az_max_deg;  /* azimuth from broadside (+x), |az| < 90 (same side) */
    double el_min_deg, el_max_deg;  /* elevation (UPA users, R5); 0, 0 for planar users */
} xlmimo_users_t;

/* ------------------------------------------------------------------------- a1
 * Seeded user drops (the Monte Carlo draws implied by the ergodic analysis,
 * PAPER.md:177-178, 228).  Counter-based Philox4x64-10 (R19): key = (seed, 0),
 * counter = (first_drop + d, k, 0, 0); words 0/1/2 -> r, az, el as 53-bit
 * uniforms.  pos (dev, [n_drops][K][3] fp64, metres) = (r cos el cos az,
 * r cos el sin az, r sin el).  Any partition of the drop range by first_drop
 * reproduces the same drops (sharding / resume).
 * EINVAL: users/pos NULL, K < 1, n_drops < 0, r_min <= 0, r_min > r_max, |az| >= 90, |el| >= 90. */
XLMIMO_API int xlmimo_gen_drops(const xlmimo_users_t *users, int32_t K, int64_t n_drops, uint64_t seed,
                     uint64_t first_drop, double *pos, void *stream);

/* The raw draws behind xlmimo_gen_drops / xlmimo_gen_drops_rect (R19): words (dev
 * [n_drops][K][4] uint64) = Philox4x64-10 with key (seed, 0) at counter
 * (first_drop + d, k, 0, 0).  Exposed so the draws can be audited bit for bit against
 * any other implementation of the generator.  EINVAL: K < 1, n_drops < 0, words NULL. */
XLMIMO_API int xlmimo_draw_words(int32_t K, int64_t n_drops, uint64_t seed, uint64_t first_drop, uint64_t *words,
                                 void *stream);

/* ------------------------------------------------------------------------- a2+a3
 * Exact Gram G = H^H H of the PNUSW channel, Eq. (3):
 *   h_i(m) = sqrt(beta0) e^{-j 2 pi r_im / lambda} / r_im * sqrt(x_i / r_im),
 * x_i the user's distance to the array line (ULA, R21) or plane (UPA, R5), and
 *   G(i,j) = sum_m conj(h_i(m)) h_j(m)  (R6),
 * the inner products the paper names as the dominant cost.
 * The phase is reduced in fp64 as 2 pi frac(r/lambda) (R13).
 *   precision XLMIMO_FP64: fp64 everywhere.  XLMIMO_FP32: fp64 distance and
 *     phase reduction, fp32 phasor and in-tile accumulation, fp64 across tiles.
 *   mode XLMIMO_FUSED: H is never materialised.  XLMIMO_MATERIALIZED: H is
 *     written to the workspace as complex64 (TF32-rounded) and streamed back by TMA
 *     (fp32 only; for K > 64 as L2-sized chunks of scaled fp16 pairs, below).
 * pos (dev [n_drops][K][3]); gram (dev [n_drops][K][K][2]) full Hermitian with
 * Im G(i,i) = 0.  K <= 1024 -- 64 < K <= 1024 are the NEXT-3/E1-E3 user counts,
 * fp64 on DMMA in the 3M complex form, fused up to K = 128
 * (blocks of 8 users dealt to warps as stars; 120 < K <= 128 in two launches) and above
 * it as a chunked Hermitian rank-k update (H formed in the workspace a chunk of
 * elements at a time, <= 64 MB so it stays in L2, never whole); fp32 on tcgen05 (a UPA
 * needing rows that are a multiple of 8, one level): fused up to K = 256 with the
 * operands generated in-kernel as fp16 with a per-drop power-of-two scale (11
 * significant bits, as TF32; K > 64 as launches per block of 64 row users over at most
 * 128 column users each), and, from K = 257 on or in MATERIALIZED mode,
 * read by TMA from chunks of H written to the workspace as scaled fp16 pairs (<= 112 MB
 * per unit of drops x 4096-element chunks, so the reads hit L2).  Below 1024 elements
 * an fp32 request with K > 64 runs the fp64 kernels (the operand rounding would not
 * average out).
 * ws may be NULL iff the query returns 0.
 * EINVAL: bad array/arguments; EUNSUPPORTED: K > 1024, fp32 with K > 64 on an
 * unsupported UPA or with nested levels, or FP64 + MATERIALIZED; EWORKSPACE: ws_bytes
 * too small. */
XLMIMO_API size_t xlmimo_gram_exact_workspace(const xlmimo_array_t *array, int32_t K, int64_t n_drops,
                                   int32_t precision, int32_t mode);
XLMIMO_API int xlmimo_gram_exact(const xlmimo_array_t *array, const double *pos, int32_t K, int64_t n_drops,
                      int32_t precision, int32_t mode, double *gram, void *ws, size_t ws_bytes,
                      void *stream);

/* ------------------------------------------------------------------------- a4
 * Closed-form ("modified ZF") Gram, Eqs. (22)-(23):
 *   G~(i,i) = P_i/P by Eq. (4) with M = n_y,
 *   G~(i,j) = rho_ij sqrt(P_i P_j)/P with rho_ij of Eq. (6) and
 *   sgn of Eq. (7) (sgn(0) = -1).  With the finite-M P_i the Eq. (4) brackets
 *   cancel (R8): G~(i,j) = 2 beta0 |dx| / (sqrt(lambda) d^{3/2} sqrt(x_i x_j))
 *   * exp(j sgn(dx) (2 pi frac(d/lambda) - pi/4)),  dx = |x_i| - |x_j|.
 * O(K^2) per drop, independent of N.  gram as for xlmimo_gram_exact.
 * flags (dev [n_drops] or NULL): set (not OR-ed) to XLMIMO_FLAG_DEGENERATE or 0.
 * EUNSUPPORTED for a UPA (the paper is ULA-only) and for spacing_wl != 0.5:
 * Eq. (4)'s aperture M lambda and element density 2/lambda are the paper's lambda/2 array
 * (PAPER.md:52), so another pitch would silently disagree with the exact Gram. */
XLMIMO_API int xlmimo_gram_closed_form(const xlmimo_array_t *array, const double *pos, int32_t K, int64_t n_drops,
                            double *gram, uint32_t *flags, void *stream);

/* ------------------------------------------------------------------------- a5
 * Per-drop receivers on a Gram (exact or closed form), for each SNR:
 *   CAP  = log2 det(I + rho G), Eq. (9), = 2 sum log2 L_kk, L L^H = I + rho G;
 *   ZF   SINR_i = rho / [G^{-1}]_ii        (Eq. (21));
 *   MMSE SINR_i = 1/[(I + rho G)^{-1}]_ii - 1;
 *   MRC  SINR_i = rho g_ii^2 / (g_ii + rho sum_{j!=i} |g_ij|^2);
 *   rate = sum_i log2(1 + SINR_i) bits/s/Hz.
 * gram (dev [n_drops][K][K][2]); snr_db (host [n_snr], n_snr <= 16);
 * rates (dev [n_drops][n_snr][popcount(receivers)]); flags (dev [n_drops] or NULL):
 * OR-ed with the XLMIMO_FLAG_* bits (so a closed-form DEGENERATE bit survives).
 * A failed Cholesky gives NaN for the receivers it feeds (R10).  K <= 64 (no
 * workspace); for 64 < K <= 1024 use xlmimo_sum_rate_ws. */
XLMIMO_API int xlmimo_sum_rate(const double *gram, int32_t K, int64_t n_drops, const double *snr_db, int32_t n_snr,
                    uint32_t receivers, double *rates, uint32_t *flags, void *stream);

/* The same receivers with a caller workspace, for K up to 1024.  For K > 64 the
 * Cholesky factors of I + rho G (CAP, MMSE) and of G (ZF) are formed one CTA per
 * matrix -- resident in shared memory for K <= 96, tiled (32 x 32 complex) in the
 * workspace above -- and the ZF/MMSE diagonals of the inverse follow from X = L^{-1}
 * (in place for K <= 96; blocked forward substitution, diagonal-tile inverses and
 * per-warp column panels in the workspace above); MRC comes straight from G.  The
 * workspace query returns 0 when none is needed (K <= 64); ws may then be NULL.
 * EWORKSPACE: ws_bytes below the query. */
XLMIMO_API size_t xlmimo_sum_rate_workspace(int32_t K, int64_t n_drops, int32_t n_snr, uint32_t receivers);
XLMIMO_API int xlmimo_sum_rate_ws(const double *gram, int32_t K, int64_t n_drops, const double *snr_db,
                                  int32_t n_snr, uint32_t receivers, double *rates, uint32_t *flags, void *ws,
                                  size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------------- NEXT-3
 * Appendix A per drop: with a_i = rho G_ii (the diagonal of
 * (P/sigma_n^2) H^H H) and R_ij = G_ij / sqrt(G_ii G_jj),
 *   rstat  (dev [n_drops][2])        = { log2 det R, gap = -log2 det(R) / K }  -- the
 *            maximised normalised gap (U - L)/U of Eq. (eq9), = -E_K[log2 lambda^R]
 *            (PAPER.md:318-327);
 *   bounds (dev [n_drops][n_snr][3]) = { log2 U, log2 det(I + rho G), log2 L } with
 *            U = prod(1 + a_i) (Hadamard) and L = det(R) U
 *            (Schur-Horn), so log2 U >= C >= log2 L;
 *   eig    (dev [n_drops][K] or NULL) = eigenvalues of R ascending, whose mean log2 is
 *            -gap: parallel cyclic Jacobi for K <= 64; for K > 64 Householder reduction to
 *            a real tridiagonal and bisection on Sturm counts (Fig. K_vs_E's spectrum at
 *            K = 1000);
 *   flags  (dev [n_drops] or NULL, SET): G_NOT_PD (R not PD: log2 det R, gap, log2 L
 *            NaN), A_NOT_PD (I + rho G not PD for some SNR: that C NaN), MRC_UNDEF
 *            (some G_ii <= 0: R undefined, all NaN), NONFINITE (all NaN).
 * gram dev [n_drops][K][K][2]; snr_db host [n_snr] (<= 16).  K <= 1024; K > 64 needs
 * the workspace of the query (tiled Cholesky slots, plus with_eig != 0 one K x K complex
 * slot per resident CTA for the eigenvalues), K <= 64 none.
 * EUNSUPPORTED: K > 1024.  EWORKSPACE: ws_bytes below the query. */
XLMIMO_API size_t xlmimo_app_a_bounds_workspace(int32_t K, int64_t n_drops, int32_t n_snr, int32_t with_eig);
XLMIMO_API int xlmimo_app_a_bounds(const double *gram, int32_t K, int64_t n_drops, const double *snr_db,
                                   int32_t n_snr, double *rstat, double *bounds, double *eig, uint32_t *flags,
                                   void *ws, size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------------- a1..a6
 * Capacity-vs-N saturation sweep.  ULA only.  For every N in
 * n_list (host, ascending, all of one parity so the centred arrays nest, R18) and
 * the SAME drops (pos if non-NULL, else drawn from users/seed like xlmimo_gen_drops
 * with first_drop = 0): the Gram (exact, fused, computed in one pass over the
 * largest array as nested shells; or closed form per N), the receivers, and (R10)
 *   ergodic  (host [n_n][n_snr][n_recv]) = the ergodic mean over ALL n_drops drops
 *             -- NaN for a column in which any drop's rate is
 *            NaN (a failed Cholesky, e.g. an indefinite closed-form Gram: a mean over
 *            the surviving drops would be biased, so it is never reported as ergodic),
 *   n_valid  (host, same shape)          = number of drops whose rate is not NaN,
 *   ergodic_valid (host, same shape, or NULL) = mean over those n_valid drops only
 *            (a conditional mean; NaN if n_valid = 0; = ergodic when n_valid = n_drops),
 *   sat      (host [4]) = { E[y_up], E[y_down], M_sat, stderr(M_sat) } with the
 *            per-drop Eqs. (13)-(16) at threshold t (0.9,
 *            PAPER.md:228) and M_sat = ceil((E[y_up]-E[y_down]) / pitch) (R15),
 *   per_drop (dev [n_drops][n_n][n_snr][n_recv] or NULL).
 * array->n_y is ignored (the grid is n_list).  Synchronises `stream` before return.
 * K <= 1024 -- the paper's K = 100 curves.  For K > 64 an fp32 exact sweep
 * runs the tcgen05 Gram once per N (those launches have no nested levels): the same
 * Grams, O(sum N) instead of O(max N) work.
 * EINVAL also for n_list not ascending / mixed parity, t not in (0,1). */
XLMIMO_API size_t xlmimo_saturation_sweep_workspace(const xlmimo_array_t *array, const int64_t *n_list, int32_t n_n,
                                         int32_t K, int64_t n_drops, int32_t n_snr, uint32_t receivers,
                                         int32_t gram_kind, int32_t precision);
XLMIMO_API int xlmimo_saturation_sweep(const xlmimo_array_t *array, const int64_t *n_list, int32_t n_n,
                            const xlmimo_users_t *users, const double *pos, int32_t K, int64_t n_drops,
                            uint64_t seed, const double *snr_db, int32_t n_snr, uint32_t receivers,
                            int32_t gram_kind, int32_t precision, double t,
                            double *ergodic, int64_t *n_valid, double *ergodic_valid, double *sat,
                            double *per_drop, void *ws, size_t ws_bytes, void *stream);

/* Same as xlmimo_saturation_sweep with HOST positions (pos_host [n_drops][K][3],
 * pinned for full speed): copies them in, runs the sweep, returns host results.
 * This is the end-to-end entry the bench's "e2e" figure times. */
XLMIMO_API int xlmimo_saturation_sweep_host(const xlmimo_array_t *array, const int64_t *n_list, int32_t n_n,
                                 const double *pos_host, int32_t K, int64_t n_drops,
                                 const double *snr_db, int32_t n_snr, uint32_t receivers, int32_t gram_kind,
                                 int32_t precision, double t, double *ergodic, int64_t *n_valid,
                                 double *ergodic_valid, double *sat, void *ws, size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------------- NEXT-1
 * Effective ("mismatched") rate of the paper's modified ZF:
 * the ZF equalizer of Eq. (21) built from the closed-form Gram G~,
 * W = G~^{-1} H^H, applied to the TRUE channel y = H x + n (Eq. (1)).  With
 * A = G~^{-1} G and noise covariance G~^{-1} G G~^{-1} / rho (G~ Hermitian):
 *   SINR_i = |A_ii|^2 / (sum_{j!=i} |A_ij|^2 + [G~^{-1} G G~^{-1}]_ii / rho),
 *   rate = sum_i log2(1 + SINR_i)   (reading R11; "worse ... at the beginning").
 * gram (true G) and gram_model (G~): dev [n_drops][K][K][2]; snr_db host [n_snr] (<= 16);
 * rates dev [n_drops][n_snr]; flags dev [n_drops] or NULL, OR-ed with
 * XLMIMO_FLAG_MODEL_SINGULAR when G~ has an exactly zero pivot (rates NaN).  G~ is
 * inverted by complex Gauss-Jordan with partial pivoting.  K <= 64. */
enum { XLMIMO_FLAG_MODEL_SINGULAR = 32 };
XLMIMO_API int xlmimo_sum_rate_mismatched(const double *gram, const double *gram_model, int32_t K, int64_t n_drops,
                                          const double *snr_db, int32_t n_snr, double *rates, uint32_t *flags,
                                          void *stream);

/* ------------------------------------------------------------------------- NEXT-4
 * Seeded drops from the paper's own user field: x ~ U[x_min,
 * x_max] (0 < x_min <= x_max), y ~ U[y_min, y_max], z = 0 -- the rectangle on the right
 * of the array behind Eq. (17) and Figs. norm_cap / Capacity_vs_number_of_ant.  Same
 * Philox stream as xlmimo_gen_drops (word 0 -> x, word 1 -> y).  pos dev [n_drops][K][3].
 * EINVAL: K < 1, n_drops < 0, x_min <= 0, x_min > x_max, y_min > y_max, pos NULL. */
XLMIMO_API int xlmimo_gen_drops_rect(double x_min, double x_max, double y_min, double y_max, int32_t K,
                                     int64_t n_drops, uint64_t seed, uint64_t first_drop, double *pos, void *stream);

/* ------------------------------------------------------------------------- path options
 * Kernel-path overrides for A/B tests and tuning.  Process-global, 0 = automatic (the
 * measured default) for every option; they select WHICH kernel runs, never what is
 * computed: every choice meets the same parity tier.  Not for concurrent use with
 * running entry points.  The library reads no environment variables.
 *   XLMIMO_OPT_LARGE_K      fp64 Gram for 64 < K: 1 block pairs, 2 chunked SYRK
 *   XLMIMO_OPT_PAIR         fp32 Gram for 64 < K: 1 TF32 block pairs generated in-kernel, 2 TMA-fed
 *                           fp16 chunks (default: the fused fp16 kernel up to K = 256, chunks above)
 *   XLMIMO_OPT_GRAM_KERNEL  fused Gram, K <= 64: 1 split (K in {4,8}, ULA, fp64), 2 DMMA (K <= 16,
 *                           fp64), 3 CUDA-core register/tile kernels, 4 64-bit-index DMMA (K > 16)
 *   XLMIMO_OPT_SPLIT_NT     split kernel block variant: 64, 128, 192 (128 x 3/SM) or 256
 *   XLMIMO_OPT_DMMA_VARIANT DMMA kernel block shape 0..3 (xl_gram.cu, mma_variant)
 *   XLMIMO_OPT_MT2_BUFFERS  DMMA K = 17..128 tile buffers: 2 (default) or 3 (the ring of full-length tiles where it
 *                           fits, of half-length ones otherwise for K > 64)
 *   XLMIMO_OPT_STREAM       materialised fp32 stream: 1 CUDA cores instead of tcgen05
 * Returns XLMIMO_OK, or EINVAL for an unknown option (value not range-checked: an
 * out-of-range value means automatic). */
enum {
    XLMIMO_OPT_LARGE_K = 0, XLMIMO_OPT_PAIR = 1, XLMIMO_OPT_GRAM_KERNEL = 2, XLMIMO_OPT_SPLIT_NT = 3,
    XLMIMO_OPT_DMMA_VARIANT = 4, XLMIMO_OPT_MT2_BUFFERS = 5, XLMIMO_OPT_STREAM = 6, XLMIMO_OPT_COUNT = 7
};
XLMIMO_API int xlmimo_set_option(int32_t option, int64_t value);
XLMIMO_API int64_t xlmimo_get_option(int32_t option);

/* Thread-local text of the last non-zero return on this thread ("" if none). */
XLMIMO_API const char *xlmimo_last_error(void);

/* Number of xlmimo kernels launched by this process since load (for the bench's
 * gpu_launches count; monotone, never reset). */
XLMIMO_API uint64_t xlmimo_launch_count(void);

/* Profiling hooks (bench.py's roofline figure).  xlmimo_timing_enable(1) clears the
 * record and starts bracketing every kernel launch with CUDA events on the stream it is
 * launched on; xlmimo_timing_enable(0) stops.  xlmimo_timing_read() synchronises the
 * recorded events and writes, per kernel name (at most max_entries; names as
 * [max_entries][64] NUL-terminated), the launch count and the summed device time in
 * ms; it returns the number of entries (< 0 on CUDA error). */
XLMIMO_API int xlmimo_timing_enable(int32_t on);
XLMIMO_API int xlmimo_timing_read(int32_t max_entries, char *names, int64_t *counts, double *total_ms);

#ifdef __cplusplus
}
#endif
#endif /* XLMIMO_H */
