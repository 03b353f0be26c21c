// xl_dmma_tile.cuh -- complex 32 x 32 tile products on the FP64 tensor path (DMMA
// m8n8k4), shared by the tiled Cholesky / blocked inverse (xl_bounds.cu) and the
// large-K SYRK Gram (xl_gram_syrk.cu).
//
// A complex tile is held as DMMA accumulator fragments (64 registers per lane); a
// k-step of 4 columns is 4 x 4 fragment pairs x 4 real DMMAs (RR, II, IR, RI).
// Operand fragments are read straight from global memory (L2) with a one-step register
// double buffer and an L2 prefetch PFD k-steps ahead.  DMMA and DFMA share the
// FP64 pipe at the same FMA rate; the tensor path needs one
// instruction per 256 FMAs and no shared-memory operand traffic.
#pragma once
#include <cstddef>
#include <cuda_runtime.h>

namespace xlt {

constexpr int kTile = 32;

__device__ __forceinline__ void dmma_f64(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}
__device__ __forceinline__ double negd(double x) {  // sign flip on the integer pipe
  return __hiloint2double(__double2hiint(x) ^ (int)0x80000000, __double2loint(x));
}

// complex 32 x 32 tile in DMMA accumulator fragments: [mb][nb] covers rows 8 mb + lane/4,
// columns 8 nb + 2 (lane % 4) + {0, 1}
struct CTile {
  double r[4][4][2], i[4][4][2];
};
__device__ __forceinline__ void ctile_zero(CTile &c) {
#pragma unroll
  for (int mb = 0; mb < 4; ++mb)
#pragma unroll
    for (int nb = 0; nb < 4; ++nb)
#pragma unroll
      for (int e = 0; e < 2; ++e) c.r[mb][nb][e] = c.i[mb][nb][e] = 0.0;
}
// one k-step (4 columns of A / rows of B): a[mb] = A(8 mb + lane/4, 4 kb + lane%4),
// b[nb] = B(4 kb + lane%4, 8 nb + lane/4);  C += A B, or C += A conj(B) with CONJ_B:
// Re += ar br -+ ai bi, Im += ai br +- ar bi (one sign flip per fragment of A)
template <bool CONJ_B, int MB = 4, int NB = 4>
__device__ __forceinline__ void ctile_step(CTile &c, const double2 (&a)[4], const double2 (&b)[4]) {
  // the two DMMAs into one accumulator are 2 MB NB instructions apart; only the first
  // MB row / NB column fragments (trimmed tiles at the ragged edge of K)
#pragma unroll
  for (int mb = 0; mb < MB; ++mb)
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
      dmma_f64(c.r[mb][nb], a[mb].x, b[nb].x);
      dmma_f64(c.i[mb][nb], a[mb].y, b[nb].x);
    }
#pragma unroll
  for (int mb = 0; mb < MB; ++mb) {
    const double n = CONJ_B ? negd(a[mb].x) : negd(a[mb].y);
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
      dmma_f64(c.r[mb][nb], CONJ_B ? a[mb].y : n, b[nb].y);
      dmma_f64(c.i[mb][nb], CONJ_B ? n : a[mb].x, b[nb].y);
    }
  }
}
template <bool B_NT, int MB = 4, int NB = 4>
__device__ __forceinline__ void frag_load(double2 (&a)[4], double2 (&b)[4], const double2 *__restrict__ Am, size_t lda,
                                          const double2 *__restrict__ Bm, size_t ldb, int kb, int lane) {
  const int qr = lane >> 2, qc = lane & 3;
#pragma unroll
  for (int mb = 0; mb < MB; ++mb) a[mb] = Am[(size_t)(8 * mb + qr) * lda + 4 * kb + qc];
#pragma unroll
  for (int nb = 0; nb < NB; ++nb)
    b[nb] = B_NT ? Bm[(size_t)(8 * nb + qr) * ldb + 4 * kb + qc] : Bm[(size_t)(4 * kb + qc) * ldb + 8 * nb + qr];
}
template <bool B_NT>
__device__ __forceinline__ void frag_prefetch_l2(const double2 *Am, size_t lda, const double2 *Bm, size_t ldb, int q,
                                                 int lane) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(Am + (size_t)lane * lda + 4 * q));
  const double2 *pb = B_NT ? Bm + (size_t)lane * ldb + 4 * q : Bm + (size_t)(4 * q + (lane >> 2)) * ldb + 8 * (lane & 3);
  asm volatile("prefetch.global.L2 [%0];" ::"l"(pb));
}
// C += A (32 x 4 nkb, row-major, stride lda) * B (4 nkb x 32), B row-major (ldb) or, with
// B_NT, B(k, n) = Bt(n, k) from a row-major Bt (stride ldb) (conjugated with CONJ_B).  The
// fragments of k-step kb + 1 are loaded while kb's 64 DMMAs run, and (PF, operands in
// global memory) the lines of k-step kb + PFD are pulled into L2 meanwhile.  PFD = 4
// measured best for the Cholesky (K = 1000 receivers 31.4 / 32.4 / 35.7 ms at 4 / 8 / 16);
// the SYRK's long slices pass 8 (737 vs 740 ms at E3).  A template parameter, so every
// instantiation has one definition across translation units.
template <bool B_NT, bool CONJ_B, bool PF, int MB = 4, int NB = 4, int PFD = 4>
__device__ __forceinline__ void ctile_mma(CTile &c, const double2 *__restrict__ Am, size_t lda,
                                          const double2 *__restrict__ Bm, size_t ldb, int nkb, int lane) {
  if (PF)
    for (int q = 0; q < PFD && q < nkb; q += 2) frag_prefetch_l2<B_NT>(Am, lda, Bm, ldb, q, lane);
  double2 a[4], b[4];
  frag_load<B_NT, MB, NB>(a, b, Am, lda, Bm, ldb, 0, lane);
#pragma unroll 1
  for (int kb = 0; kb < nkb; ++kb) {
    if (PF && !(kb & 1) && kb + PFD < nkb) frag_prefetch_l2<B_NT>(Am, lda, Bm, ldb, kb + PFD, lane);
    double2 an[4], bn[4];
    frag_load<B_NT, MB, NB>(an, bn, Am, lda, Bm, ldb, kb + 1 < nkb ? kb + 1 : kb, lane);
    ctile_step<CONJ_B, MB, NB>(c, a, b);
#pragma unroll
    for (int q = 0; q < MB; ++q) a[q] = an[q];
#pragma unroll
    for (int q = 0; q < NB; ++q) b[q] = bn[q];
  }
}
// dst (MB 8 x NB 8 fragments from fragment (MB0, NB0), in memory) += A conj(Bt)^T, 3M form:
// P1 = Ar Br^T, P2 = Ai Bi^T, P3 = (Ar + Ai)(Br - Bi)^T accumulated over the k-steps, then
// Re C += P1 + P2, Im C += P3 - P1 + P2 (three DMMAs per fragment pair instead of four; the
// operand sums are one DADD per fragment).  B is row-major Bt (B_NT), conjugated.
template <int MB, int NB, int MB0, int NB0, int PFD>
__device__ __forceinline__ void ctile_mma3m_nt(double2 *dst, size_t ld, const double2 *__restrict__ Am, size_t lda,
                                               const double2 *__restrict__ Bm, size_t ldb, int nkb, int lane) {
  const int qr = lane >> 2, qc = lane & 3;
  double p1[MB][NB][2], p2[MB][NB][2], p3[MB][NB][2];
#pragma unroll
  for (int mb = 0; mb < MB; ++mb)
#pragma unroll
    for (int nb = 0; nb < NB; ++nb)
#pragma unroll
      for (int e = 0; e < 2; ++e) p1[mb][nb][e] = p2[mb][nb][e] = p3[mb][nb][e] = 0.0;
  for (int q = 0; q < PFD && q < nkb; q += 2) frag_prefetch_l2<true>(Am, lda, Bm, ldb, q, lane);
  auto load = [&](double2 (&a)[MB], double2 (&b)[NB], int kb) {
#pragma unroll
    for (int mb = 0; mb < MB; ++mb) a[mb] = Am[(size_t)(8 * (MB0 + mb) + qr) * lda + 4 * kb + qc];
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) b[nb] = Bm[(size_t)(8 * (NB0 + nb) + qr) * ldb + 4 * kb + qc];
  };
  double2 a[MB], b[NB];
  load(a, b, 0);
#pragma unroll 1
  for (int kb = 0; kb < nkb; ++kb) {
    if (!(kb & 1) && kb + PFD < nkb) frag_prefetch_l2<true>(Am, lda, Bm, ldb, kb + PFD, lane);
    double2 an[MB], bn[NB];
    load(an, bn, kb + 1 < nkb ? kb + 1 : kb);
    double bd[NB];
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) bd[nb] = b[nb].x - b[nb].y;
#pragma unroll
    for (int mb = 0; mb < MB; ++mb) {
      const double as = a[mb].x + a[mb].y;
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) {
        dmma_f64(p1[mb][nb], a[mb].x, b[nb].x);
        dmma_f64(p2[mb][nb], a[mb].y, b[nb].y);
        dmma_f64(p3[mb][nb], as, bd[nb]);
      }
    }
#pragma unroll
    for (int q = 0; q < MB; ++q) a[q] = an[q];
#pragma unroll
    for (int q = 0; q < NB; ++q) b[q] = bn[q];
  }
#pragma unroll
  for (int mb = 0; mb < MB; ++mb)
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
      double2 *q = dst + (size_t)(8 * (MB0 + mb) + qr) * ld + 8 * (NB0 + nb) + 2 * qc;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double2 v = q[e];
        q[e] = make_double2(v.x + (p1[mb][nb][e] + p2[mb][nb][e]), v.y + ((p3[mb][nb][e] - p1[mb][nb][e]) + p2[mb][nb][e]));
      }
    }
}

// pull a 32 x 32 complex tile (32 rows of 512 B) into L2 ahead of its use
__device__ __forceinline__ void tile_prefetch_l2(const double2 *src, size_t ld, int lane) {
  const char *p = reinterpret_cast<const char *>(src + (size_t)lane * ld);
#pragma unroll
  for (int q = 0; q < 4; ++q) asm volatile("prefetch.global.L2 [%0];" ::"l"(p + 128 * q));
}
template <bool NEG, int MB = 4, int NB = 4>
__device__ __forceinline__ void ctile_load(CTile &c, const double2 *src, size_t ld, int lane) {
  const int qr = lane >> 2, qc = lane & 3;
#pragma unroll
  for (int mb = 0; mb < MB; ++mb)
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
      const double2 *p = src + (size_t)(8 * mb + qr) * ld + 8 * nb + 2 * qc;
      const double2 v0 = p[0], v1 = p[1];
      c.r[mb][nb][0] = NEG ? -v0.x : v0.x;
      c.i[mb][nb][0] = NEG ? -v0.y : v0.y;
      c.r[mb][nb][1] = NEG ? -v1.x : v1.x;
      c.i[mb][nb][1] = NEG ? -v1.y : v1.y;
    }
}
template <bool NEG, int MB = 4, int NB = 4>
__device__ __forceinline__ void ctile_store(const CTile &c, double2 *dst, size_t ld, int lane) {
  const int qr = lane >> 2, qc = lane & 3;
#pragma unroll
  for (int mb = 0; mb < MB; ++mb)
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
      double2 *p = dst + (size_t)(8 * mb + qr) * ld + 8 * nb + 2 * qc;
#pragma unroll
      for (int e = 0; e < 2; ++e)
        p[e] = NEG ? make_double2(-c.r[mb][nb][e], -c.i[mb][nb][e]) : make_double2(c.r[mb][nb][e], c.i[mb][nb][e]);
    }
}

}  // namespace xlt
