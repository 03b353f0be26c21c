/*
 * xlmimo_oracle.c -- plain, slow, obviously-correct fp64 CPU ORACLE.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2503_18118_b200/, include/xlmimo.h) never links,
 * imports or executes anything in oracle/, and this file shares no code,
 * header, table or constant generator with it.
 *
 * Every function follows the paper (PAPER.md = arXiv 2503.18118 LaTeX source,
 * cited by line) in its own order and notation, with plain loops, fp64,
 * std C99 complex arithmetic written out by hand, and Neumaier-compensated
 * sums where a long sum is formed.  Readings of ambiguous passages are the
 * ones listed in DESIGN.md section "Readings" (R1..R23, = SURVEY.md 8(c) Q1..Q23).
 *
 * Pins (tests/test_oracle_pins.py) tie each function to something other than
 * itself: numpy's Philox bit generator, mpmath 40-digit brute force, the
 * paper's closed forms Eq. (4)/(5)/(6)/(8)/(12)/(17), LAPACK (numpy.linalg)
 * det/inv on small K, hand 2x2 formulas, and invariants.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Speed of light, exact by SI definition (R2). */
#define OR_C_LIGHT 299792458.0
#define OR_PI 3.14159265358979323846

/* Own copies of the parameter records (deliberately NOT the product header). */
typedef struct {
    int32_t kind;       /* 0 = ULA on the y-axis; 1 = UPA in the y-z plane (R5) */
    int64_t n_y, n_z;   /* ULA: n_y = M, n_z = 1 */
    double fc_hz;       /* carrier; lambda = c / fc */
    double spacing_wl;  /* element pitch in wavelengths; 0.5 */
    double beta0;       /* sqrt(beta0) gain constant; 1 */
} or_array_t;

typedef struct {
    double r_min_m, r_max_m;       /* range from array centre, uniform in r (R3) */
    double az_min_deg, az_max_deg; /* azimuth from broadside (+x), uniform (R3) */
    double el_min_deg, el_max_deg; /* elevation, uniform (R5); 0,0 for planar users */
} or_users_t;

/* ------------------------------------------------------------------------ */
/* Philox4x64-10 counter-based generator (Salmon et al., SC'11), written     */
/* from its published definition.  R19: key = (seed, 0); counter =           */
/* (drop, user, 0, 0); pinned against numpy.random.Philox in the tests.     */
/* ------------------------------------------------------------------------ */
static void or_mulhilo64(uint64_t a, uint64_t b, uint64_t *hi, uint64_t *lo)
{
    unsigned __int128 p = (unsigned __int128)a * (unsigned __int128)b;
    *hi = (uint64_t)(p >> 64);
    *lo = (uint64_t)p;
}

void or_philox4x64_10(const uint64_t ctr_in[4], const uint64_t key_in[2], uint64_t out[4])
{
    const uint64_t M0 = 0xD2E7470EE14C6C93ULL, M1 = 0xCA5A826395121157ULL;
    const uint64_t W0 = 0x9E3779B97F4A7C15ULL, W1 = 0xBB67AE8584CAA73BULL;
    uint64_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint64_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        uint64_t hi0, lo0, hi1, lo1;
        or_mulhilo64(M0, c0, &hi0, &lo0);
        or_mulhilo64(M1, c2, &hi1, &lo1);
        uint64_t n0 = hi1 ^ c1 ^ k0;
        uint64_t n1 = lo1;
        uint64_t n2 = hi0 ^ c3 ^ k1;
        uint64_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += W0; k1 += W1;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* 53-bit uniform in [0,1) from a 64-bit word (R19). */
static double or_u01(uint64_t w) { return (double)(w >> 11) * (1.0 / 9007199254740992.0); }

/* a1: user positions of each drop (R3, R5, R19).  pos[d][k][3] = (x, y, z) m. */
void or_gen_drops(const or_users_t *u, int32_t K, int64_t n_drops, uint64_t seed,
                  uint64_t first_drop, double *pos)
{
    const double deg = OR_PI / 180.0;
    for (int64_t d = 0; d < n_drops; ++d) {
        for (int32_t k = 0; k < K; ++k) {
            uint64_t ctr[4] = {first_drop + (uint64_t)d, (uint64_t)k, 0, 0};
            uint64_t key[2] = {seed, 0};
            uint64_t w[4];
            or_philox4x64_10(ctr, key, w);
            double r = u->r_min_m + (u->r_max_m - u->r_min_m) * or_u01(w[0]);
            double az = (u->az_min_deg + (u->az_max_deg - u->az_min_deg) * or_u01(w[1])) * deg;
            double el = (u->el_min_deg + (u->el_max_deg - u->el_min_deg) * or_u01(w[2])) * deg;
            double *p = pos + ((size_t)d * K + k) * 3;
            p[0] = r * cos(el) * cos(az);
            p[1] = r * cos(el) * sin(az);
            p[2] = r * sin(el);
        }
    }
}

/* The paper's own user field: x ~ U[x_min, x_max],
 * y ~ U[y_min, y_max] (a rectangle on the right of the y-axis), z = 0.  Same
 * Philox stream as or_gen_drops: word 0 -> x, word 1 -> y. */
void or_gen_drops_rect(double x_min, double x_max, double y_min, double y_max, int32_t K, int64_t n_drops,
                       uint64_t seed, uint64_t first_drop, double *pos)
{
    for (int64_t d = 0; d < n_drops; ++d)
        for (int32_t k = 0; k < K; ++k) {
            uint64_t ctr[4] = {first_drop + (uint64_t)d, (uint64_t)k, 0, 0};
            uint64_t key[2] = {seed, 0};
            uint64_t w[4];
            or_philox4x64_10(ctr, key, w);
            double *p = pos + ((size_t)d * K + k) * 3;
            p[0] = x_min + (x_max - x_min) * or_u01(w[0]);
            p[1] = y_min + (y_max - y_min) * or_u01(w[1]);
            p[2] = 0.0;
        }
}

/* ------------------------------------------------------------------------ */
/* Geometry (R1, R5).                                                        */
/* ------------------------------------------------------------------------ */
double or_wavelength(const or_array_t *a) { return OR_C_LIGHT / a->fc_hz; }

int64_t or_num_elements(const or_array_t *a) { return a->kind == 0 ? a->n_y : a->n_y * a->n_z; }

/* Element m (0-based, natural order).  ULA: y_m = (m - (M+1)/2) * pitch for the
 * 1-based m of SPEC.md:59 (R1), on the y-axis, centred at the origin
 * (PAPER.md:52).  UPA: m = q*n_y + p -> (0, y_p, z_q), both axes centred (R5). */
void or_element_pos(const or_array_t *a, int64_t m, double *ey, double *ez)
{
    const double pitch = a->spacing_wl * or_wavelength(a);
    if (a->kind == 0) {
        *ey = ((double)(m + 1) - 0.5 * (double)(a->n_y + 1)) * pitch;
        *ez = 0.0;
    } else {
        int64_t p = m % a->n_y, q = m / a->n_y;
        *ey = ((double)(p + 1) - 0.5 * (double)(a->n_y + 1)) * pitch;
        *ez = ((double)(q + 1) - 0.5 * (double)(a->n_z + 1)) * pitch;
    }
}

/* The "x_i" of Eq. (3): distance from the user to the array line (ULA, by the
 * rotational symmetry of PAPER.md:52, R21) or to the array plane (UPA, R5). */
static double or_user_x(const or_array_t *a, const double *p)
{
    return a->kind == 0 ? sqrt(p[0] * p[0] + p[2] * p[2]) : fabs(p[0]);
}

/* a2: Eq. (3) PNUSW coefficient
 *   h_i(m) = sqrt(beta0) e^{-j 2 pi r/lambda} / r * sqrt(x_i / r).
 * The phase is reduced in fp64 as 2 pi frac(r/lambda) (R13). */
void or_channel_coef(const or_array_t *a, const double *p, int64_t m, double *re, double *im)
{
    double ey, ez;
    or_element_pos(a, m, &ey, &ez);
    const double lambda = or_wavelength(a);
    const double dx = p[0], dy = p[1] - ey, dz = p[2] - ez;
    const double r = sqrt(dx * dx + dy * dy + dz * dz);
    const double xi = or_user_x(a, p);
    const double amp = sqrt(a->beta0) / r * sqrt(xi / r);
    const double q = r / lambda;
    const double f = q - nearbyint(q);
    const double phase = 2.0 * OR_PI * f;
    *re = amp * cos(phase);
    *im = -amp * sin(phase);
}

/* H as [K][M][2] for one drop (small cases only). */
void or_channel_matrix(const or_array_t *a, const double *pos, int32_t K, double *H)
{
    const int64_t M = or_num_elements(a);
    for (int32_t i = 0; i < K; ++i)
        for (int64_t m = 0; m < M; ++m)
            or_channel_coef(a, pos + 3 * i, m, &H[((size_t)i * M + m) * 2], &H[((size_t)i * M + m) * 2 + 1]);
}

/* Neumaier (improved Kahan-Babuska) compensated accumulation. */
typedef struct { double s, c; } or_nsum;
static void or_nadd(or_nsum *a, double x)
{
    double t = a->s + x;
    if (fabs(a->s) >= fabs(x)) a->c += (a->s - t) + x;
    else a->c += (x - t) + a->s;
    a->s = t;
}

/* a3: exact Gram G = H^H H:
 *   G(i,j) = sum_m conj(h_i(m)) h_j(m)  for i <= j,  G(j,i) = conj G(i,j),
 *   Im G(i,i) = 0  (R6, R20).   gram[d][i][j][2], full Hermitian, row-major. */
static void or_gram_exact_one(const or_array_t *a, const double *pos, int32_t K, double *g)
{
    const int64_t M = or_num_elements(a);
    const int np = K * (K + 1) / 2;
    or_nsum *acc = (or_nsum *)calloc((size_t)np * 2, sizeof(or_nsum));
    double *h = (double *)malloc(sizeof(double) * 2 * K);
    for (int64_t m = 0; m < M; ++m) {
        for (int32_t i = 0; i < K; ++i) or_channel_coef(a, pos + 3 * i, m, &h[2 * i], &h[2 * i + 1]);
        int idx = 0;
        for (int32_t i = 0; i < K; ++i)
            for (int32_t j = i; j < K; ++j, ++idx) {
                /* conj(a) * b = (ar - j ai)(br + j bi) = (ar br + ai bi) + j (ar bi - ai br) */
                const double ar = h[2 * i], ai = h[2 * i + 1], br = h[2 * j], bi = h[2 * j + 1];
                or_nadd(&acc[2 * idx], ar * br);
                or_nadd(&acc[2 * idx], ai * bi);
                or_nadd(&acc[2 * idx + 1], ar * bi);
                or_nadd(&acc[2 * idx + 1], -ai * br);
            }
    }
    int idx = 0;
    for (int32_t i = 0; i < K; ++i)
        for (int32_t j = i; j < K; ++j, ++idx) {
            double re = acc[2 * idx].s + acc[2 * idx].c;
            double im = acc[2 * idx + 1].s + acc[2 * idx + 1].c;
            if (i == j) im = 0.0;
            g[((size_t)i * K + j) * 2] = re;
            g[((size_t)i * K + j) * 2 + 1] = im;
            g[((size_t)j * K + i) * 2] = re;
            g[((size_t)j * K + i) * 2 + 1] = -im;
        }
    free(h);
    free(acc);
}

static int or_threads(int32_t nthreads)
{
#ifdef _OPENMP
    return nthreads > 0 ? nthreads : omp_get_max_threads();
#else
    (void)nthreads;
    return 1;
#endif
}

void or_gram_exact(const or_array_t *a, const double *pos, int32_t K, int64_t n_drops, double *gram,
                   int32_t nthreads)
{
    int nt = or_threads(nthreads);
    (void)nt;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
    for (int64_t d = 0; d < n_drops; ++d)
        or_gram_exact_one(a, pos + (size_t)d * K * 3, K, gram + (size_t)d * K * K * 2);
}

/* ------------------------------------------------------------------------ */
/* a4: closed-form ("modified ZF") Gram, Eqs. (4), (6), (7), (22), (23).     */
/* ------------------------------------------------------------------------ */

/* The bracket of Eq. (4), evaluated as written (R23). */
static double or_eq4_bracket(double M, double lambda, double x, double y)
{
    double ml = M * lambda;
    return (-4.0 * y + ml) / sqrt(16.0 * x * x + (ml - 4.0 * y) * (ml - 4.0 * y)) +
           (4.0 * y + ml) / sqrt(16.0 * x * x + (ml + 4.0 * y) * (ml + 4.0 * y));
}

/* Eq. (4): P_i / P = (2 beta0 / (lambda x_i)) * bracket. */
double or_power_eq4(double M, double lambda, double beta0, double x, double y)
{
    return 2.0 * beta0 / (lambda * x) * or_eq4_bracket(M, lambda, x, y);
}

/* Eq. (5): P_i^lim / P = 4 beta0 / (lambda x_i). */
double or_power_limit_eq5(double lambda, double beta0, double x) { return 4.0 * beta0 / (lambda * x); }

/* Eq. (7): sgn(x) = -1 if x <= 0, +1 if x > 0 (R7). */
static double or_sgn_eq7(double x) { return x > 0.0 ? 1.0 : -1.0; }

/* Eq. (6): SPM correlation rho_ij, written term by term. */
void or_corr_eq6(double M, double lambda, double xi, double yi, double xj, double yj, double *re, double *im)
{
    const double dx = fabs(xi) - fabs(xj);
    const double dy = yi - yj;
    const double d2 = dx * dx + dy * dy;
    double mag = sqrt(lambda) * fabs(dx) / pow(d2, 0.75);
    mag *= pow(or_eq4_bracket(M, lambda, xi, yi), -0.5);
    mag *= pow(or_eq4_bracket(M, lambda, xj, yj), -0.5);
    /* phase sgn(dx) * (2 pi d / lambda - pi/4), with 2 pi d/lambda reduced as 2 pi frac(d/lambda) (R13) */
    const double q = sqrt(d2) / lambda;
    const double ph = or_sgn_eq7(dx) * (2.0 * OR_PI * (q - nearbyint(q)) - OR_PI / 4.0);
    *re = mag * cos(ph);
    *im = mag * sin(ph);
}

/* Eq. (8): M -> infinity limit of rho_ij (pin only). */
void or_corr_limit_eq8(double lambda, double xi, double yi, double xj, double yj, double *re, double *im)
{
    const double dx = fabs(xi) - fabs(xj);
    const double d = sqrt(dx * dx + (yi - yj) * (yi - yj));
    const double cosg = fabs(dx) / d;
    const double mag = sqrt(lambda) * cosg / (2.0 * sqrt(d));
    const double q = d / lambda;
    const double ph = or_sgn_eq7(dx) * (2.0 * OR_PI * (q - nearbyint(q)) - OR_PI / 4.0);
    *re = mag * cos(ph);
    *im = mag * sin(ph);
}

/* Eq. (22)/(23): G~(i,i) = P_i/P by Eq. (4);
 * G~(i,j) = rho_ij sqrt(P_i P_j)/P by Eq. (6) with the finite-M P_i (R8).
 * flags bit 3 if some pair has ||x_i|-|x_j|| < lambda (R7). ULA only. */
void or_gram_closed_form(const or_array_t *a, const double *pos, int32_t K, int64_t n_drops, double *gram,
                         uint32_t *flags)
{
    const double lambda = or_wavelength(a);
    const double M = (double)a->n_y;
    for (int64_t d = 0; d < n_drops; ++d) {
        const double *p = pos + (size_t)d * K * 3;
        double *g = gram + (size_t)d * K * K * 2;
        uint32_t fl = 0;
        for (int32_t i = 0; i < K; ++i) {
            const double xi = or_user_x(a, p + 3 * i), yi = p[3 * i + 1];
            const double Pi = or_power_eq4(M, lambda, a->beta0, xi, yi);
            g[((size_t)i * K + i) * 2] = Pi;
            g[((size_t)i * K + i) * 2 + 1] = 0.0;
            for (int32_t j = i + 1; j < K; ++j) {
                const double xj = or_user_x(a, p + 3 * j), yj = p[3 * j + 1];
                const double Pj = or_power_eq4(M, lambda, a->beta0, xj, yj);
                double rr, ri;
                or_corr_eq6(M, lambda, xi, yi, xj, yj, &rr, &ri);
                const double s = sqrt(Pi * Pj);
                g[((size_t)i * K + j) * 2] = rr * s;
                g[((size_t)i * K + j) * 2 + 1] = ri * s;
                g[((size_t)j * K + i) * 2] = rr * s;
                g[((size_t)j * K + i) * 2 + 1] = -ri * s;
                if (fabs(fabs(xi) - fabs(xj)) < lambda) fl |= 8u;
            }
        }
        if (flags) flags[d] = fl;
    }
}

/* ------------------------------------------------------------------------ */
/* a5: per-drop receivers (Eq. (9); Eq. (21);  */
/* SINRs SPEC.md:303-329, R12).  Complex Cholesky written by hand.           */
/* ------------------------------------------------------------------------ */

/* Lower Cholesky of Hermitian A (K x K, [K][K][2]) into L; returns 0 on success,
 * -1 if a pivot is not > 0 (A not positive definite, R10). */
static int or_cholesky(const double *A, int K, double *L)
{
    memset(L, 0, sizeof(double) * 2 * K * K);
    for (int j = 0; j < K; ++j) {
        double d = A[(j * K + j) * 2];
        for (int k = 0; k < j; ++k) d -= L[(j * K + k) * 2] * L[(j * K + k) * 2] + L[(j * K + k) * 2 + 1] * L[(j * K + k) * 2 + 1];
        if (!(d > 0.0)) return -1;
        const double ljj = sqrt(d);
        L[(j * K + j) * 2] = ljj;
        for (int i = j + 1; i < K; ++i) {
            /* L_ij = (A_ij - sum_k L_ik conj(L_jk)) / L_jj */
            double sr = A[(i * K + j) * 2], si = A[(i * K + j) * 2 + 1];
            for (int k = 0; k < j; ++k) {
                const double ar = L[(i * K + k) * 2], ai = L[(i * K + k) * 2 + 1];
                const double br = L[(j * K + k) * 2], bi = L[(j * K + k) * 2 + 1];
                sr -= ar * br + ai * bi;
                si -= ai * br - ar * bi;
            }
            L[(i * K + j) * 2] = sr / ljj;
            L[(i * K + j) * 2 + 1] = si / ljj;
        }
    }
    return 0;
}

/* diag(A^{-1})_i = sum_k |(L^{-1})_{k i}|^2 with A = L L^H (forward substitution). */
static void or_inv_diag(const double *L, int K, double *dinv, double *x /* scratch 2K */)
{
    for (int i = 0; i < K; ++i) {
        double s = 0.0;
        for (int k = 0; k < K; ++k) { x[2 * k] = 0.0; x[2 * k + 1] = 0.0; }
        for (int k = i; k < K; ++k) {
            /* solve L x = e_i: x_k = (delta_ki - sum_{j<k} L_kj x_j) / L_kk */
            double rr = (k == i) ? 1.0 : 0.0, ri = 0.0;
            for (int j = i; j < k; ++j) {
                const double lr = L[(k * K + j) * 2], li = L[(k * K + j) * 2 + 1];
                rr -= lr * x[2 * j] - li * x[2 * j + 1];
                ri -= lr * x[2 * j + 1] + li * x[2 * j];
            }
            const double lkk = L[(k * K + k) * 2];
            x[2 * k] = rr / lkk;
            x[2 * k + 1] = ri / lkk;
            s += x[2 * k] * x[2 * k] + x[2 * k + 1] * x[2 * k + 1];
        }
        dinv[i] = s;
    }
}

/* receivers bitmask: 1 = CAP (Eq. 9), 2 = ZF, 4 = MMSE, 8 = MRC; rates[d][s][r] for the
 * set bits in that order.  flags: bit0 chol(G) failed (ZF NaN); bit1 chol(I+rho G) failed
 * (CAP, MMSE NaN); bit2 MRC undefined (g_ii <= 0); bit4 non-finite input (all NaN). */
void or_sum_rate(const double *gram, int32_t K, int64_t n_drops, const double *snr_db, int32_t n_snr,
                 uint32_t receivers, double *rates, uint32_t *flags)
{
    int n_recv = 0;
    for (int b = 0; b < 4; ++b) n_recv += (receivers >> b) & 1u;
    const double nan = NAN;
    double *A = (double *)malloc(sizeof(double) * 2 * K * K);
    double *L = (double *)malloc(sizeof(double) * 2 * K * K);
    double *dinv = (double *)malloc(sizeof(double) * K);
    double *x = (double *)malloc(sizeof(double) * 2 * K);
    for (int64_t d = 0; d < n_drops; ++d) {
        const double *G = gram + (size_t)d * K * K * 2;
        double *out = rates + (size_t)d * n_snr * n_recv;
        uint32_t fl = flags ? (flags[d] & 8u) : 0u; /* keep the closed-form bit if present */
        int finite = 1;
        for (int e = 0; e < 2 * K * K; ++e) finite &= isfinite(G[e]) ? 1 : 0;
        if (!finite) {
            fl |= 16u;
            for (int e = 0; e < n_snr * n_recv; ++e) out[e] = nan;
            if (flags) flags[d] = fl;
            continue;
        }
        /* ZF: SINR_i = rho / [G^{-1}]_ii, G^{-1} diag from chol(G). */
        int zf_ok = 0;
        if (receivers & 2u) {
            zf_ok = or_cholesky(G, K, L) == 0;
            if (zf_ok) or_inv_diag(L, K, dinv, x);
            else fl |= 1u;
        }
        double *zf_dinv = (double *)malloc(sizeof(double) * K);
        memcpy(zf_dinv, dinv, sizeof(double) * K);
        int mrc_ok = 1;
        for (int i = 0; i < K; ++i) mrc_ok &= G[(i * K + i) * 2] > 0.0;
        if ((receivers & 8u) && !mrc_ok) fl |= 4u;
        for (int s = 0; s < n_snr; ++s) {
            const double rho = pow(10.0, snr_db[s] / 10.0);
            int r = 0;
            int a_ok = 0;
            if (receivers & 5u) {
                for (int i = 0; i < K; ++i)
                    for (int j = 0; j < K; ++j) {
                        A[(i * K + j) * 2] = (i == j ? 1.0 : 0.0) + rho * G[(i * K + j) * 2];
                        A[(i * K + j) * 2 + 1] = rho * G[(i * K + j) * 2 + 1];
                    }
                a_ok = or_cholesky(A, K, L) == 0;
                if (!a_ok) fl |= 2u;
            }
            if (receivers & 1u) { /* CAP = log2 det(I + rho G) = 2 sum log2 L_kk (Eq. 9) */
                double c = 0.0;
                for (int k = 0; k < K; ++k) c += 2.0 * log2(L[(k * K + k) * 2]);
                out[s * n_recv + r++] = a_ok ? c : nan;
            }
            if (receivers & 2u) {
                double c = 0.0;
                for (int i = 0; i < K; ++i) c += log2(1.0 + rho / zf_dinv[i]);
                out[s * n_recv + r++] = zf_ok ? c : nan;
            }
            if (receivers & 4u) { /* MMSE: SINR_i = 1/[(I + rho G)^{-1}]_ii - 1 */
                double c = 0.0;
                if (a_ok) {
                    or_inv_diag(L, K, dinv, x);
                    for (int i = 0; i < K; ++i) c += log2(1.0 + (1.0 / dinv[i] - 1.0));
                }
                out[s * n_recv + r++] = a_ok ? c : nan;
            }
            if (receivers & 8u) { /* MRC: rho g_ii^2 / (g_ii + rho sum_{j!=i} |g_ij|^2) */
                double c = 0.0;
                for (int i = 0; i < K; ++i) {
                    const double gii = G[(i * K + i) * 2];
                    double intf = 0.0;
                    for (int j = 0; j < K; ++j)
                        if (j != i) intf += G[(i * K + j) * 2] * G[(i * K + j) * 2] + G[(i * K + j) * 2 + 1] * G[(i * K + j) * 2 + 1];
                    c += log2(1.0 + rho * gii * gii / (gii + rho * intf));
                }
                out[s * n_recv + r++] = mrc_ok ? c : nan;
            }
        }
        free(zf_dinv);
        if (flags) flags[d] = fl;
    }
    free(A); free(L); free(dinv); free(x);
}

/* ------------------------------------------------------------------------ */
/* NEXT-1: effective rate of the "modified ZF": the ZF      */
/* equalizer of Eq. (21) built from the closed-form Gram G~,   */
/* W = G~^{-1} H^H, applied to the true channel y = H x + n (Eq. 1):          */
/*   W y = A x + W n,  A = G~^{-1} G,  cov(W n) = sigma^2 G~^{-1} G G~^{-1},  */
/*   SINR_i = |A_ii|^2 / (sum_{j!=i} |A_ij|^2 + [G~^{-1} G G~^{-1}]_ii / rho). */
/* "worse performance ... at the beginning" is this rate below */
/* saturation (reading R11).                                                  */
/* ------------------------------------------------------------------------ */

/* In-place complex Gauss-Jordan inverse with partial pivoting (plain loops).
 * Returns 0, or -1 if a pivot is exactly zero (singular). */
static int or_cinv(double *M, int K)
{
    int *perm = (int *)malloc(sizeof(int) * K);
    for (int k = 0; k < K; ++k) {
        int p = k;
        double best = -1.0;
        for (int i = k; i < K; ++i) {
            const double v = hypot(M[(i * K + k) * 2], M[(i * K + k) * 2 + 1]);
            if (v > best) { best = v; p = i; }
        }
        perm[k] = p;
        if (!(best > 0.0)) { free(perm); return -1; }
        if (p != k)
            for (int j = 0; j < K; ++j)
                for (int c = 0; c < 2; ++c) {
                    const double t = M[(k * K + j) * 2 + c];
                    M[(k * K + j) * 2 + c] = M[(p * K + j) * 2 + c];
                    M[(p * K + j) * 2 + c] = t;
                }
        /* 1 / pivot */
        const double pr = M[(k * K + k) * 2], pi = M[(k * K + k) * 2 + 1];
        const double den = pr * pr + pi * pi;
        const double ir = pr / den, ii = -pi / den;
        M[(k * K + k) * 2] = 1.0;
        M[(k * K + k) * 2 + 1] = 0.0;
        for (int j = 0; j < K; ++j) { /* row k *= 1/pivot */
            const double ar = M[(k * K + j) * 2], ai = M[(k * K + j) * 2 + 1];
            M[(k * K + j) * 2] = ar * ir - ai * ii;
            M[(k * K + j) * 2 + 1] = ar * ii + ai * ir;
        }
        for (int i = 0; i < K; ++i) {
            if (i == k) continue;
            const double fr = M[(i * K + k) * 2], fi = M[(i * K + k) * 2 + 1];
            M[(i * K + k) * 2] = 0.0;
            M[(i * K + k) * 2 + 1] = 0.0;
            for (int j = 0; j < K; ++j) { /* row i -= f * row k */
                const double br = M[(k * K + j) * 2], bi = M[(k * K + j) * 2 + 1];
                M[(i * K + j) * 2] -= fr * br - fi * bi;
                M[(i * K + j) * 2 + 1] -= fr * bi + fi * br;
            }
        }
    }
    for (int k = K - 1; k >= 0; --k) /* undo the row swaps as column swaps */
        if (perm[k] != k)
            for (int i = 0; i < K; ++i)
                for (int c = 0; c < 2; ++c) {
                    const double t = M[(i * K + k) * 2 + c];
                    M[(i * K + k) * 2 + c] = M[(i * K + perm[k]) * 2 + c];
                    M[(i * K + perm[k]) * 2 + c] = t;
                }
    free(perm);
    return 0;
}

/* rates[d][s] (bits/s/Hz); flags bit 5 (32) when G~ is singular (rates NaN). */
void or_sum_rate_mismatched(const double *gram, const double *gram_model, int32_t K, int64_t n_drops,
                            const double *snr_db, int32_t n_snr, double *rates, uint32_t *flags)
{
    double *B = (double *)malloc(sizeof(double) * 2 * K * K);
    double *A = (double *)malloc(sizeof(double) * 2 * K * K);
    for (int64_t d = 0; d < n_drops; ++d) {
        const double *G = gram + (size_t)d * K * K * 2;
        memcpy(B, gram_model + (size_t)d * K * K * 2, sizeof(double) * 2 * K * K);
        if (or_cinv(B, K) != 0) {
            for (int s = 0; s < n_snr; ++s) rates[d * n_snr + s] = NAN;
            if (flags) flags[d] |= 32u;
            continue;
        }
        for (int i = 0; i < K; ++i) /* A = B G */
            for (int j = 0; j < K; ++j) {
                double sr = 0.0, si = 0.0;
                for (int k = 0; k < K; ++k) {
                    const double br = B[(i * K + k) * 2], bi = B[(i * K + k) * 2 + 1];
                    const double gr = G[(k * K + j) * 2], gi = G[(k * K + j) * 2 + 1];
                    sr += br * gr - bi * gi;
                    si += br * gi + bi * gr;
                }
                A[(i * K + j) * 2] = sr;
                A[(i * K + j) * 2 + 1] = si;
            }
        for (int s = 0; s < n_snr; ++s) {
            const double rho = pow(10.0, snr_db[s] / 10.0);
            double c = 0.0;
            for (int i = 0; i < K; ++i) {
                double sig = 0.0, intf = 0.0, noise = 0.0;
                for (int j = 0; j < K; ++j) {
                    const double p = A[(i * K + j) * 2] * A[(i * K + j) * 2] + A[(i * K + j) * 2 + 1] * A[(i * K + j) * 2 + 1];
                    if (j == i) sig = p; else intf += p;
                }
                for (int k = 0; k < K; ++k) { /* [A B]_ii = sum_k A_ik B_ki, real for Hermitian PSD G */
                    noise += A[(i * K + k) * 2] * B[(k * K + i) * 2] - A[(i * K + k) * 2 + 1] * B[(k * K + i) * 2 + 1];
                }
                c += log2(1.0 + sig / (intf + noise / rho));
            }
            rates[d * n_snr + s] = c;
        }
    }
    free(A); free(B);
}

/* ------------------------------------------------------------------------ */
/* a6: saturation coordinates (Eqs. 13-16) and the sweep.  */
/* ------------------------------------------------------------------------ */

/* Per drop: y_up = max_i (x_i t/sqrt(1-t^2) + y_i), y_down = min_i (-x_i t/sqrt(1-t^2) + y_i). */
void or_saturation_coords(const double *pos, int32_t K, int64_t n_drops, double t, double *y_up, double *y_down)
{
    const double s = t / sqrt(1.0 - t * t);
    for (int64_t d = 0; d < n_drops; ++d) {
        double up = -INFINITY, dn = INFINITY;
        for (int32_t i = 0; i < K; ++i) {
            const double *p = pos + ((size_t)d * K + i) * 3;
            const double x = sqrt(p[0] * p[0] + p[2] * p[2]);
            const double u = x * s + p[1];   /* Eq. (13) */
            const double w = -x * s + p[1];  /* Eq. (14) */
            if (u > up) up = u;              /* Eq. (15) */
            if (w < dn) dn = w;              /* Eq. (16) */
        }
        y_up[d] = up;
        y_down[d] = dn;
    }
}

/* Saturation sweep (ULA): for every N in n_list, independently (no nesting,
 * R18), the Gram of the same drops, the receivers, and per (N, SNR, receiver)
 * column (R10): n_valid = the number of drops whose rate is not NaN;
 * ergodic = the mean over ALL drops (the expectation of PAPER.md:177-178, 228),
 * which exists only when every drop is valid, else NaN; ergodic_valid (optional)
 * = the mean over the valid drops only (a conditional mean, NaN if none).
 * sat = {E[y_up], E[y_down], M_sat, stderr(M_sat)} with
 * M_sat = ceil((E[y_up] - E[y_down]) / pitch) and
 * stderr = sample std (ddof 1) of the per-drop extent (y_up - y_down)/pitch over sqrt(D).
 * gram_kind: 0 exact, 1 closed form.  per_drop (optional) [D][n_n][n_snr][n_recv]. */
void or_saturation_sweep(const or_array_t *a_in, const int64_t *n_list, int32_t n_n, const double *pos,
                         int32_t K, int64_t n_drops, const double *snr_db, int32_t n_snr, uint32_t receivers,
                         int32_t gram_kind, double t, double *ergodic, int64_t *n_valid, double *ergodic_valid,
                         double *sat, double *per_drop, int32_t nthreads)
{
    int n_recv = 0;
    for (int b = 0; b < 4; ++b) n_recv += (receivers >> b) & 1u;
    const size_t per = (size_t)n_snr * n_recv;
    double *g = (double *)malloc(sizeof(double) * 2 * K * K * (size_t)n_drops);
    double *rt = (double *)malloc(sizeof(double) * per * (size_t)n_drops);
    uint32_t *fl = (uint32_t *)calloc((size_t)n_drops, sizeof(uint32_t));
    for (int32_t n = 0; n < n_n; ++n) {
        or_array_t a = *a_in;
        a.n_y = n_list[n];
        a.n_z = 1;
        if (gram_kind == 0) or_gram_exact(&a, pos, K, n_drops, g, nthreads);
        else or_gram_closed_form(&a, pos, K, n_drops, g, fl);
        or_sum_rate(g, K, n_drops, snr_db, n_snr, receivers, rt, fl);
        for (size_t e = 0; e < per; ++e) {
            or_nsum acc = {0.0, 0.0};
            int64_t cnt = 0;
            for (int64_t d = 0; d < n_drops; ++d) {
                const double v = rt[(size_t)d * per + e];
                if (per_drop) per_drop[((size_t)d * n_n + n) * per + e] = v;
                if (!isnan(v)) { or_nadd(&acc, v); ++cnt; }
            }
            const double cond = cnt ? (acc.s + acc.c) / (double)cnt : NAN;
            ergodic[(size_t)n * per + e] = cnt == n_drops ? cond : NAN;
            if (ergodic_valid) ergodic_valid[(size_t)n * per + e] = cond;
            n_valid[(size_t)n * per + e] = cnt;
        }
    }
    double *up = (double *)malloc(sizeof(double) * (size_t)n_drops);
    double *dn = (double *)malloc(sizeof(double) * (size_t)n_drops);
    or_saturation_coords(pos, K, n_drops, t, up, dn);
    const double pitch = a_in->spacing_wl * or_wavelength(a_in);
    or_nsum su = {0, 0}, sd = {0, 0}, se = {0, 0}, se2 = {0, 0};
    for (int64_t d = 0; d < n_drops; ++d) {
        or_nadd(&su, up[d]);
        or_nadd(&sd, dn[d]);
        const double e = (up[d] - dn[d]) / pitch;
        or_nadd(&se, e);
        or_nadd(&se2, e * e);
    }
    const double D = (double)n_drops;
    const double Eu = (su.s + su.c) / D, Ed = (sd.s + sd.c) / D;
    const double me = (se.s + se.c) / D;
    const double var = n_drops > 1 ? ((se2.s + se2.c) - D * me * me) / (D - 1.0) : 0.0;
    sat[0] = Eu;
    sat[1] = Ed;
    sat[2] = ceil((Eu - Ed) / pitch);
    sat[3] = sqrt(var > 0 ? var : 0.0) / sqrt(D);
    free(up); free(dn); free(g); free(rt); free(fl);
}

/* ------------------------------------------------------------------------ */
/* NEXT-3: Appendix A, per drop, in the paper's order.    */
/*   a_i  = rho G_ii, the diagonal of (P/sigma_n^2) H^H H;    */
/*   U    = prod_i (1 + a_i), Hadamard's upper bound;    */
/*   R_ij = G_ij / (||h_i|| ||h_j||), the correlation matrix; */
/*   L    = det(R) prod_i (1 + a_i), the Schur-Horn lower bound; */
/*   C    = log2 det(I + rho G), the capacity they bracket (Eq. 9);          */
/*   gap  = -log2 det(R) / sum_i log2(1 + 1) = -(1/K) log2 det R, the        */
/*          maximised normalised gap of Eq. (eq9), whose   */
/*          last line is -E_K[log2 lambda^R] (same number; pinned by the     */
/*          eigenvalues below).                                             */
/*   rstat[d][2]     = { log2 det R, gap }                                  */
/*   bounds[d][s][3] = { log2 U, C, log2 L } for rho = 10^(snr_db[s]/10)     */
/*   eig[d][K] (optional) = eigenvalues of R ascending, by cyclic Jacobi.    */
/* flags: bit0 R (= G scaled) not PD -> log2 det R, gap, log2 L NaN; bit1    */
/* I + rho G not PD -> C NaN; bit2 some G_ii <= 0 -> everything NaN (R is    */
/* undefined); bit4 non-finite G -> everything NaN.                          */
/* ------------------------------------------------------------------------ */

/* Eigenvalues of a Hermitian K x K matrix A ([K][K][2], destroyed) by the cyclic
 * Jacobi method: for each (p < q) with A_pq != 0, make A_pq real by the phase
 * rotation S = diag(.., e^{-j phi} at q, ..), then zero it with the real plane
 * rotation of Numerical Recipes 11.1 (theta = (a_qq - a_pp) / (2|a_pq|),
 * t = sgn(theta) / (|theta| + sqrt(theta^2 + 1))).  Sweeps until the off-diagonal
 * mass is below 1e-30 of the total.  ev ascending. */
static void or_jacobi_eig(double *A, int K, double *ev)
{
#define OR_A(i, j) (A + ((size_t)(i) * K + (j)) * 2)
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0, tot = 0.0;
        for (int i = 0; i < K; ++i)
            for (int j = 0; j < K; ++j) {
                const double m = OR_A(i, j)[0] * OR_A(i, j)[0] + OR_A(i, j)[1] * OR_A(i, j)[1];
                tot += m;
                if (i != j) off += m;
            }
        if (off <= 1e-30 * tot) break;
        for (int p = 0; p < K - 1; ++p)
            for (int q = p + 1; q < K; ++q) {
                const double br = OR_A(p, q)[0], bi = OR_A(p, q)[1];
                const double b = sqrt(br * br + bi * bi);
                if (b == 0.0) continue;
                /* phase: column q times e^{-j phi}, row q times e^{+j phi}, phi = arg A_pq */
                const double cr = br / b, ci = -bi / b; /* e^{-j phi} */
                for (int r = 0; r < K; ++r) {
                    double *x = OR_A(r, q); /* x *= e^{-j phi} */
                    const double xr = x[0] * cr - x[1] * ci, xi = x[0] * ci + x[1] * cr;
                    x[0] = xr; x[1] = xi;
                }
                for (int r = 0; r < K; ++r) {
                    double *x = OR_A(q, r); /* x *= e^{+j phi} */
                    const double xr = x[0] * cr + x[1] * ci, xi = -x[0] * ci + x[1] * cr;
                    x[0] = xr; x[1] = xi;
                }
                /* now A_pq = b (real); the real rotation */
                const double app = OR_A(p, p)[0], aqq = OR_A(q, q)[0];
                const double theta = (aqq - app) / (2.0 * b);
                double t = 1.0 / (fabs(theta) + sqrt(theta * theta + 1.0));
                if (theta < 0.0) t = -t;
                const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
                for (int r = 0; r < K; ++r) {
                    if (r == p || r == q) continue;
                    double *xp = OR_A(r, p), *xq = OR_A(r, q);
                    const double pr = c * xp[0] - s * xq[0], pi = c * xp[1] - s * xq[1];
                    const double qr = s * xp[0] + c * xq[0], qi = s * xp[1] + c * xq[1];
                    xp[0] = pr; xp[1] = pi; xq[0] = qr; xq[1] = qi;
                    OR_A(p, r)[0] = pr; OR_A(p, r)[1] = -pi; /* Hermitian mirror */
                    OR_A(q, r)[0] = qr; OR_A(q, r)[1] = -qi;
                }
                OR_A(p, p)[0] = app - t * b; OR_A(p, p)[1] = 0.0;
                OR_A(q, q)[0] = aqq + t * b; OR_A(q, q)[1] = 0.0;
                OR_A(p, q)[0] = OR_A(p, q)[1] = 0.0;
                OR_A(q, p)[0] = OR_A(q, p)[1] = 0.0;
            }
    }
    for (int i = 0; i < K; ++i) ev[i] = OR_A(i, i)[0];
    for (int i = 1; i < K; ++i) { /* insertion sort, ascending */
        const double v = ev[i];
        int j = i - 1;
        while (j >= 0 && ev[j] > v) { ev[j + 1] = ev[j]; --j; }
        ev[j + 1] = v;
    }
#undef OR_A
}

void or_bounds_app_a(const double *gram, int32_t K, int64_t n_drops, const double *snr_db, int32_t n_snr,
                     double *rstat, double *bounds, double *eig, uint32_t *flags, int32_t nthreads)
{
    int nt = or_threads(nthreads);
    (void)nt;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
    for (int64_t d = 0; d < n_drops; ++d) {
        const double *G = gram + (size_t)d * K * K * 2;
        double *rs = rstat + (size_t)d * 2, *bo = bounds + (size_t)d * n_snr * 3;
        double *ev = eig ? eig + (size_t)d * K : NULL;
        uint32_t fl = 0;
        int finite = 1, diag_ok = 1;
        for (int e = 0; e < 2 * K * K; ++e) finite &= isfinite(G[e]) ? 1 : 0;
        for (int i = 0; i < K && finite; ++i) diag_ok &= G[(i * K + i) * 2] > 0.0;
        if (!finite || !diag_ok) {
            fl |= finite ? 4u : 16u;
            rs[0] = rs[1] = NAN;
            for (int e = 0; e < 3 * n_snr; ++e) bo[e] = NAN;
            if (ev) for (int i = 0; i < K; ++i) ev[i] = NAN;
            if (flags) flags[d] = fl;
            continue;
        }
        double *R = (double *)malloc(sizeof(double) * 2 * K * K);
        double *Lf = (double *)malloc(sizeof(double) * 2 * K * K);
        double *A = (double *)malloc(sizeof(double) * 2 * K * K);
        /* R_ij = G_ij / sqrt(G_ii G_jj); ||h_i||^2 = G_ii */
        for (int i = 0; i < K; ++i)
            for (int j = 0; j < K; ++j) {
                const double s = sqrt(G[(i * K + i) * 2] * G[(j * K + j) * 2]);
                R[(i * K + j) * 2] = (i == j) ? 1.0 : G[(i * K + j) * 2] / s;
                R[(i * K + j) * 2 + 1] = (i == j) ? 0.0 : G[(i * K + j) * 2 + 1] / s;
            }
        double ldr = NAN;
        if (or_cholesky(R, K, Lf) == 0) {
            ldr = 0.0; /* log2 det R = 2 sum log2 L_kk */
            for (int k = 0; k < K; ++k) ldr += 2.0 * log2(Lf[(k * K + k) * 2]);
        } else {
            fl |= 1u;
        }
        rs[0] = ldr;
        rs[1] = -ldr / (double)K; /* -log2 det R / sum_i log2(1 + 1)  (Eq. eq9) */
        for (int s = 0; s < n_snr; ++s) {
            const double rho = pow(10.0, snr_db[s] / 10.0);
            double lu = 0.0;
            for (int i = 0; i < K; ++i) lu += log2(1.0 + rho * G[(i * K + i) * 2]); /* log2 U */
            for (int i = 0; i < K; ++i)
                for (int j = 0; j < K; ++j) {
                    A[(i * K + j) * 2] = (i == j ? 1.0 : 0.0) + rho * G[(i * K + j) * 2];
                    A[(i * K + j) * 2 + 1] = rho * G[(i * K + j) * 2 + 1];
                }
            double cap = NAN;
            if (or_cholesky(A, K, Lf) == 0) {
                cap = 0.0;
                for (int k = 0; k < K; ++k) cap += 2.0 * log2(Lf[(k * K + k) * 2]);
            } else {
                fl |= 2u;
            }
            bo[3 * s + 0] = lu;
            bo[3 * s + 1] = cap;
            bo[3 * s + 2] = ldr + lu; /* log2 L = log2 det R + log2 U */
        }
        if (ev) or_jacobi_eig(R, K, ev); /* R is not needed after this */
        free(R);
        free(Lf);
        free(A);
        if (flags) flags[d] = fl;
    }
}
