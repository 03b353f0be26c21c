// xl_gram.cu -- a2+a3: exact Gram G = H^H H of the PNUSW channel (Eq. 3),
// generated on the fly (fused; never materialised), fp64 or fp32 phasors.
//
// PAPER.md:240 names "the inner product calculation for elements in H^H H" as
// the dominant cost; these kernels are that step.  Design (K2/K3):
//  * grid = n_drops x n_split blocks; a block owns one drop and a contiguous
//    range of element indices in the "centred order" (xl::ula_y_centred), so the
//    N' < N arrays of a saturation sweep are prefixes (R18);
//  * segment ends (level boundaries of the sweep, or N) emit a block-reduced
//    partial upper triangle to the workspace -- deterministic, no atomics;
//  * gram_reduce_kernel sums partials in fixed (level, split) order into the
//    full Hermitian K x K per (drop, level), Im diag = 0 (R20).
//  Small K (<= 8): every thread owns all K(K+1)/2 accumulators in registers and
//  generates the K coefficients of its element (kernel A).  Larger K (<= 64):
//  tiles of 32 elements are generated into shared memory as interleaved complex,
//  then each thread accumulates one 4x4 register block of the upper triangle
//  over a subset of the tile's elements (kernel B).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "xl_common.cuh"

namespace {

constexpr int kMaxLvl = 32;

struct GramParams {
  const double *pos;
  double *ws;          // partials [drop][split][lvl][NP][2]
  int K;
  int kind;
  int64_t n_y, n_z;
  int64_t N;           // total elements (last level end)
  int64_t chunk;       // elements per split
  int n_split;
  int n_lvl;
  int64_t lvl_end[kMaxLvl];
  double inv_lambda, pitch, sqrt_beta0;
  const float *hmat;   // materialised H (FROM_H kernels): [drop - h_drop0][K][2][N]
  int64_t h_drop0;     // first drop of the current batch (materialised mode; 0 otherwise)
};

struct ElemPos {
  double y, z;
};

__device__ __forceinline__ ElemPos element_pos(const GramParams &P, int64_t t) {
  ElemPos e;
  if (P.kind == XLMIMO_ULA) {
    e.y = xl::ula_y_centred(t, (P.N & 1) != 0, P.pitch);
    e.z = 0.0;
  } else {
    int64_t q, p;
    if (P.N < ((int64_t)1 << 31)) {  // 32-bit division (no 64-bit division subroutine)
      const uint32_t tt = (uint32_t)t, ny = (uint32_t)P.n_y;
      const uint32_t q32 = tt / ny;
      q = q32;
      p = tt - q32 * ny;
    } else {
      q = t / P.n_y;
      p = t - q * P.n_y;
    }
    e.y = ((double)p - 0.5 * (double)(P.n_y - 1)) * P.pitch;
    e.z = ((double)q - 0.5 * (double)(P.n_z - 1)) * P.pitch;
  }
  return e;
}

__device__ __forceinline__ double dist2(const xl::UserC &u, const ElemPos &e, int kind) {
  const double dy = e.y - u.y;
  double r2 = fma(dy, dy, u.xz2);
  if (kind != XLMIMO_ULA) {
    const double dz = e.z - u.z;
    r2 = fma(dz, dz, r2);
  }
  return r2;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// K4a: write H as planar complex64 [drop - h_drop0][K][2][N] (re plane, im plane,
// N contiguous) for a batch of drops, in the centred element order.  fp64 distance
// and phase reduction, fp32 phasor (XLMIMO_FP32).  Thread per element, coalesced
// stores along N.  Optionally rounds to TF32 (round-to-nearest-away) for the
// tensor-core stream (V8: hardware truncation would bias the diagonal by -7e-4).
// Layouts: planar  H[d][k][c][N]                    (CUDA-core stream)
//          tiled32 H[d][N32/32][k][c][32], N32 = n_pad (tcgen05 stream: one TMA box =
//                  2K rows x 128 B contiguous; padded elements are written as 0).
// grid = (ceil(n_pad / 256), n_batch): one drop per blockIdx.y, users staged in smem.
__global__ void __launch_bounds__(256) h_materialise_kernel(GramParams P, float *H, int64_t n_pad, int tiled,
                                                            int tf32) {
  __shared__ xl::UserC su[xl::kMaxK];
  const int bd = blockIdx.y;
  const int64_t drop = P.h_drop0 + bd;
  const int K = P.K;
  if (threadIdx.x < K) su[threadIdx.x] = xl::make_user(P.pos + (drop * K + threadIdx.x) * 3, P.kind, P.sqrt_beta0);
  __syncthreads();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_pad) return;
  const bool valid = t < P.N;
  const ElemPos ep = element_pos(P, valid ? t : 0);
  float *Hd = H + (size_t)bd * K * 2 * n_pad;
  for (int k = 0; k < K; ++k) {
    const xl::UserC u = su[k];
    float fr = 0.f, fi = 0.f;
    if (valid) xl::coef_from_r2_f32(dist2(u, ep, P.kind), u.amp, P.inv_lambda, fr, fi);
    if (tf32) {
      uint32_t a, b;
      asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(a) : "f"(fr));
      asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(b) : "f"(fi));
      fr = __uint_as_float(a);
      fi = __uint_as_float(b);
    }
    size_t o_re, o_im;
    if (tiled) {
      const size_t tile = (size_t)(t >> 5);
      o_re = ((tile * K + k) * 2) * 32 + (t & 31);
      o_im = o_re + 32;
    } else {
      o_re = ((size_t)k * 2) * n_pad + t;
      o_im = o_re + n_pad;
    }
    __stcs(Hd + o_re, fr);
    __stcs(Hd + o_im, fi);
  }
}

// ------------------------------------------------------------------ kernel A
template <int KT, int NT, bool FP32>
__global__ void __launch_bounds__(NT, 1) gram_small_kernel(GramParams P) {
  constexpr int NP = KT * (KT + 1) / 2;
  constexpr int NV = 2 * NP;
  constexpr int NW = NT / 32;
  __shared__ xl::UserC su[KT];
  __shared__ double red[NW][NV];

  const int64_t bdrop = blockIdx.x / P.n_split;
  const int split = blockIdx.x - (int)(bdrop * P.n_split);
  const int64_t drop = P.h_drop0 + bdrop;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < KT) su[tid] = xl::make_user(P.pos + (drop * KT + tid) * 3, P.kind, P.sqrt_beta0);
  __syncthreads();

  const int64_t s0 = (int64_t)split * P.chunk;
  const int64_t s1 = min(P.N, s0 + P.chunk);
  int64_t lv0 = 0;
  for (int l = 0; l < P.n_lvl; ++l) {
    const int64_t lv1 = P.lvl_end[l];
    const int64_t a = max(lv0, s0), b = min(lv1, s1);
    lv0 = lv1;
    double acc[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[v] = 0.0;
    for (int64_t t = a + tid; t < b; t += NT) {
      const ElemPos e = element_pos(P, t);
      double hr[KT], hi[KT];
#pragma unroll
      for (int i = 0; i < KT; ++i) {
        const xl::UserC u = su[i];
        const double r2 = dist2(u, e, P.kind);
        if (FP32) {
          float fr, fi;
          xl::coef_from_r2_f32(r2, u.amp, P.inv_lambda, fr, fi);
          hr[i] = fr; hi[i] = fi;
        } else {
          xl::coef_fast(r2, u.amp, 4.0 * P.inv_lambda, hr[i], hi[i]);
        }
      }
      int v = 0;
#pragma unroll
      for (int i = 0; i < KT; ++i) {
#pragma unroll
        for (int j = i; j < KT; ++j) {
          if (i == j) {
            acc[v] = fma(hr[i], hr[i], fma(hi[i], hi[i], acc[v]));
          } else {
            // conj(h_i) h_j = (ar br + ai bi) + j (ar bi - ai br)
            acc[v] = fma(hr[i], hr[j], fma(hi[i], hi[j], acc[v]));
            acc[v + 1] = fma(hr[i], hi[j], fma(-hi[i], hr[j], acc[v + 1]));
          }
          v += 2;
        }
      }
    }
    // block reduction, fixed order
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const double s = warp_sum(acc[v]);
      if (lane == 0) red[warp][v] = s;
    }
    __syncthreads();
    double *out = P.ws + (((size_t)drop * P.n_split + split) * P.n_lvl + l) * NV;
    for (int v = tid; v < NV; v += NT) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) s += red[w][v];
      out[v] = s;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ kernel A2
// K = 2*KH (KH in {2, 4}), ULA.  Two threads (lanes 2s, 2s+1) share each element:
// thread h generates users [h*KH, (h+1)*KH) (no duplicated generation), the two
// exchange their coefficients with one shuffle per value, and each accumulates
// its own-half triangle plus half of the cross block, so the K(K+1)/2 complex
// accumulators are split evenly and the register budget allows 2 blocks/SM.
// Cross block split: thread h sees theirs'[b] = partner.mine[(b + h) % KH] and
// takes the pairs (a, (a + d) % KH) for even d -- thread 0 covers the even
// diagonals of the cross block, thread 1 (whose view is rotated by one) the odd
// ones; split_map() inverts this for the output.
template <int KH>
__device__ __forceinline__ void split_map(int i, int j, int &parity, int &slot, bool &conj) {
  constexpr int NOWN = KH * (KH + 1) / 2, ND = KH / 2;
  if (j < KH) {
    parity = 0; slot = i * KH - i * (i - 1) / 2 + (j - i); conj = false;
  } else if (i >= KH) {
    const int a = i - KH, b = j - KH;
    parity = 1; slot = a * KH - a * (a - 1) / 2 + (b - a); conj = false;
  } else {
    const int a0 = i, b0 = j - KH;
    const int d = ((b0 - a0) % KH + KH) % KH;
    if ((d & 1) == 0) {
      parity = 0; slot = NOWN + a0 * ND + d / 2; conj = false;
    } else {
      const int d1 = ((a0 - b0 - 1) % KH + KH) % KH;
      parity = 1; slot = NOWN + b0 * ND + d1 / 2; conj = true;
    }
  }
}

template <int KH, int NT, int MINB, int UNR = 1>
__global__ void __launch_bounds__(NT, MINB) gram_split_kernel(GramParams P) {
  constexpr int K = 2 * KH;
  constexpr int NOWN = KH * (KH + 1) / 2;
  constexpr int ND = KH / 2;
  constexpr int NS = NOWN + KH * ND;  // complex accumulators per thread
  constexpr int NV = 2 * NS;
  constexpr int NW = NT / 32;
  constexpr int NSLOT = NT / 2;
  __shared__ double4 su[K];  // (xz2, y, amp, -)
  __shared__ double red[NW][2][NV];

  const int64_t bdrop = blockIdx.x / P.n_split;
  const int split = blockIdx.x - (int)(bdrop * P.n_split);
  const int64_t drop = P.h_drop0 + bdrop;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int h = tid & 1, eslot = tid >> 1;
  if (tid < K) {
    const xl::UserC u = xl::make_user(P.pos + (drop * K + tid) * 3, XLMIMO_ULA, P.sqrt_beta0);
    su[tid] = make_double4(u.xz2, u.y, u.amp, 0.0);
  }
  __syncthreads();
  const double c4 = 4.0 * P.inv_lambda;
  const bool n_odd = (P.N & 1) != 0;

  const int64_t s0 = (int64_t)split * P.chunk;
  const int64_t s1 = min(P.N, s0 + P.chunk);
  int64_t lv0 = 0;
  for (int l = 0; l < P.n_lvl; ++l) {
    const int64_t lv1 = P.lvl_end[l];
    const int64_t a = max(lv0, s0), b = min(lv1, s1);
    lv0 = lv1;
    double acc[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[v] = 0.0;
    // Even N: the centred order puts index t at y = +-(t/2 + 1/2) pitch with the sign set
    // by t's parity, which is fixed per thread (NSLOT is even), so y is one FMA of an
    // exactly incremented pair index: fma(p, +-pitch, +-pitch/2) == ((p + 1/2) pitch)
    // rounded once, bitwise what ula_y_centred gives.
    const int64_t ta = a + eslot;
    const double sgn = (ta & 1) ? -1.0 : 1.0;
    const double sp = sgn * P.pitch, sh = 0.5 * sgn * P.pitch;
    double pd = (double)(ta >> 1);
    for (int64_t t0 = a; t0 < b; t0 += NSLOT * UNR, pd += (double)(NSLOT * UNR / 2)) {  // warp-uniform trips
      double mr[UNR][KH], mi[UNR][KH];
      if (!n_odd && t0 + NSLOT * UNR <= b) {  // full iteration: no masking (uniform branch)
#pragma unroll
        for (int w = 0; w < UNR; ++w) {
          const double ey = fma(pd + (double)(w * NSLOT / 2), sp, sh);
#pragma unroll
          for (int q = 0; q < KH; ++q) {
            const double4 u = su[h * KH + q];
            const double dy = ey - u.y;
            xl::coef_fast(fma(dy, dy, u.x), u.z, c4, mr[w][q], mi[w][q]);
          }
        }
      } else {
#pragma unroll
        for (int w = 0; w < UNR; ++w) {
          const int64_t t = t0 + w * NSLOT + eslot;
          const bool valid = t < b;
          const double ey = xl::ula_y_centred(valid ? t : a, n_odd, P.pitch);
#pragma unroll
          for (int q = 0; q < KH; ++q) {
            const double4 u = su[h * KH + q];
            const double dy = ey - u.y;
            xl::coef_fast(fma(dy, dy, u.x), valid ? u.z : 0.0, c4, mr[w][q], mi[w][q]);
          }
        }
      }
#pragma unroll
      for (int w = 0; w < UNR; ++w) {
        double tr[KH], ti[KH];
#pragma unroll
        for (int q = 0; q < KH; ++q) {
          const double sr = h ? mr[w][q] : mr[w][(q + 1) % KH];
          const double si = h ? mi[w][q] : mi[w][(q + 1) % KH];
          tr[q] = __shfl_xor_sync(0xffffffffu, sr, 1);
          ti[q] = __shfl_xor_sync(0xffffffffu, si, 1);
        }
        int v = 0;
#pragma unroll
        for (int p = 0; p < KH; ++p) {
#pragma unroll
          for (int q = p; q < KH; ++q) {
            if (p == q) {
              acc[v] = fma(mr[w][p], mr[w][p], fma(mi[w][p], mi[w][p], acc[v]));
            } else {
              acc[v] = fma(mr[w][p], mr[w][q], fma(mi[w][p], mi[w][q], acc[v]));
              acc[v + 1] = fma(mr[w][p], mi[w][q], fma(-mi[w][p], mr[w][q], acc[v + 1]));
            }
            v += 2;
          }
        }
#pragma unroll
        for (int p = 0; p < KH; ++p) {
#pragma unroll
          for (int dd = 0; dd < ND; ++dd) {
            const int q = (p + 2 * dd) % KH;
            acc[v] = fma(mr[w][p], tr[q], fma(mi[w][p], ti[q], acc[v]));
            acc[v + 1] = fma(mr[w][p], ti[q], fma(-mi[w][p], tr[q], acc[v + 1]));
            v += 2;
          }
        }
      }
    }
    // reduce lanes of equal parity inside the warp, then the NW warps in fixed order through
    // shared memory: one partial per (drop, split, level) -- the per-warp partials of round 1
    // were 2.9x the algorithmic output bytes (ncu: 152 MB written per cfg2 launch).
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      double x = acc[v];
#pragma unroll
      for (int o = 2; o < 32; o <<= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (lane < 2) red[warp][lane][v] = x;
    }
    __syncthreads();
    constexpr int NP = K * (K + 1) / 2;
    double *out = P.ws + (((size_t)drop * P.n_split + split) * P.n_lvl + l) * (2 * NP);
    for (int p = tid; p < NP; p += NT) {
      int i = 0, rem = p;
      while (rem >= K - i) { rem -= K - i; ++i; }
      const int j = i + rem;
      int par, slot;
      bool cj;
      split_map<KH>(i, j, par, slot, cj);
      double re = 0.0, im = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        re += red[w][par][2 * slot];
        im += red[w][par][2 * slot + 1];
      }
      out[2 * p] = re;
      out[2 * p + 1] = (i == j) ? 0.0 : (cj ? -im : im);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ kernel W
// Small arrays (N <= kWarpMaxN, one level, K <= 6, fp64): one WARP per drop, lane l takes
// elements l, l + 32, ... (natural order), generates the drop's K coefficients per element
// (coef_fast) and keeps the K(K+1)/2 complex sums in registers; the warp then reduces them
// with a transpose-reduce (offsets 16..1, each lane keeping half of its values and
// receiving the other half: 31 shuffled doubles for 32 slots instead of 5 x the slot
// count), after which lane l holds slot l, and writes the Hermitian Gram directly -- no
// partials, no block barriers, no second kernel.  cfg1's steady state (10^6 drops of
// K = 4, N = 256) was 8.7 ms on the split kernel: one block per drop, per-warp partials
// and a separate reduce for 8 elements per thread.
constexpr int kWarpMaxN = 4096;
constexpr int64_t kWarpMinDrops = 148 * 32;  // >= 4 warps per SM sub-partition, else the split path
constexpr int kWarpBlock = 256;  // 8 drops per block

template <int K, int KIND>
__global__ void __launch_bounds__(kWarpBlock) gram_warp_kernel(GramParams P, int64_t n_drops, double *out) {
  constexpr int NP = K * (K + 1) / 2;
  static_assert(2 * NP <= 32, "gram_warp_kernel: K(K+1) <= 32");
  const int lane = threadIdx.x & 31;
  const int64_t drop = (int64_t)blockIdx.x * (kWarpBlock / 32) + (threadIdx.x >> 5);
  if (drop >= n_drops) return;  // whole warp
  // lane k forms user k (its amplitude takes two fp64 square roots: once per user, not once
  // per user and lane), then every lane takes the K users by shuffle
  double uy[K], uz[K], ux2[K], ua[K];
  xl::UserC mine{1.0, 0.0, 0.0, 0.0};
  if (lane < K) mine = xl::make_user(P.pos + (drop * K + lane) * 3, KIND, P.sqrt_beta0);
#pragma unroll
  for (int k = 0; k < K; ++k) {
    ux2[k] = __shfl_sync(0xffffffffu, mine.xz2, k);
    uy[k] = __shfl_sync(0xffffffffu, mine.y, k);
    uz[k] = __shfl_sync(0xffffffffu, mine.z, k);
    ua[k] = __shfl_sync(0xffffffffu, mine.amp, k);
  }
  double v[32];
#pragma unroll
  for (int q = 0; q < 32; ++q) v[q] = 0.0;
  const double c4 = 4.0 * P.inv_lambda;
  const int N = (int)P.N;
  const double y0 = -0.5 * (double)(KIND == XLMIMO_ULA ? P.N - 1 : P.n_y - 1) * P.pitch;
  const double z0 = -0.5 * (double)(P.n_z - 1) * P.pitch;
  for (int m = lane; m < N; m += 32) {
    double ey, ez = 0.0;
    if (KIND == XLMIMO_ULA) {
      ey = fma((double)m, P.pitch, y0);
    } else {
      const int q = m / (int)P.n_y, pp = m - q * (int)P.n_y;
      ey = fma((double)pp, P.pitch, y0);
      ez = fma((double)q, P.pitch, z0);
    }
    double hr[K], hi[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const double dy = ey - uy[k];
      double r2 = fma(dy, dy, ux2[k]);
      if (KIND != XLMIMO_ULA) {
        const double dz = ez - uz[k];
        r2 = fma(dz, dz, r2);
      }
      xl::coef_fast(r2, ua[k], c4, hr[k], hi[k]);
    }
    int q = 0;
#pragma unroll
    for (int i = 0; i < K; ++i)
#pragma unroll
      for (int j = i; j < K; ++j, ++q) {  // conj(h_i) h_j
        if (i == j) {
          v[2 * q] = fma(hr[i], hr[i], fma(hi[i], hi[i], v[2 * q]));
        } else {
          v[2 * q] = fma(hr[i], hr[j], fma(hi[i], hi[j], v[2 * q]));
          v[2 * q + 1] = fma(hr[i], hi[j], fma(-hi[i], hr[j], v[2 * q + 1]));
        }
      }
  }
  // transpose-reduce: after offset o the lane keeps slots [0, o) (lane bit clear) or [o, 2o)
  // (bit set), renumbered to [0, o); the final slot index is the lane index.
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < o; ++i) {
      if (i >= 2 * NP && i + o >= 2 * NP) continue;  // both halves are padding: stays 0
      const double send = up ? v[i] : v[i + o];
      const double keep = up ? v[i + o] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  if (lane < 2 * NP) {
    const int p = lane >> 1, part = lane & 1;
    int i = 0, rem = p;
    while (rem >= K - i) { rem -= K - i; ++i; }
    const int j = i + rem;
    double *g = out + (size_t)drop * K * K * 2;
    const double x = (part && i == j) ? 0.0 : v[0];
    g[(i * K + j) * 2 + part] = x;
    g[(j * K + i) * 2 + part] = part ? -x : x;
  }
}

template <int KIND>
void launch_warp_k(const GramParams &P, int K, int64_t n_drops, double *out, cudaStream_t s) {
  const unsigned blocks = (unsigned)((n_drops + kWarpBlock / 32 - 1) / (kWarpBlock / 32));
  switch (K) {
    case 1: gram_warp_kernel<1, KIND><<<blocks, kWarpBlock, 0, s>>>(P, n_drops, out); break;
    case 2: gram_warp_kernel<2, KIND><<<blocks, kWarpBlock, 0, s>>>(P, n_drops, out); break;
    case 3: gram_warp_kernel<3, KIND><<<blocks, kWarpBlock, 0, s>>>(P, n_drops, out); break;
    case 4: gram_warp_kernel<4, KIND><<<blocks, kWarpBlock, 0, s>>>(P, n_drops, out); break;
    case 5: gram_warp_kernel<5, KIND><<<blocks, kWarpBlock, 0, s>>>(P, n_drops, out); break;
    default: break;
  }
}

// ------------------------------------------------------------------ kernel M
// FP64 tensor-core (DMMA, mma.sync.m8n8k4.f64) Gram, warp-independent, K <= 8G.
// A warp covers 4 elements x 8 users per step: lane l computes the coefficient of
// user l/4 (+ 8g for group g) at element l%4 -- exactly the m8n8k4 A-fragment
// (row = user, k = element) and, for the same register, the B-fragment
// (k = element, col = user).  Per step and group pair (g1 <= g2):
//   diagonal (g, g):  RR += re^T re,  II += im^T im,  RI += re^T im:
//                     Re G = RR + II,  Im G(i,j) = RI(i,j) - RI(j,i);
//   cross (g1 < g2):  P1 += re1^T re2,  P2 += im1^T im2,  P3 += (re1 + im1)^T (re2 - im2):
//                     Re G = P1 + P2,  Im G = P1 - P2 - P3  (the 3M form of kernel MT2).  DMMA shares the FP64 pipe with DFMA on B200
// (tools/pipes.cu) and computes the redundant lower halves, but leaves each
// lane with one short coefficient chain and a handful of accumulator registers,
// so occupancy (latency hiding) is high and no shuffles are needed.
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int G>
struct MmaCfg {
  static constexpr int NDIAG = G;                 // RR, II, RI
  static constexpr int NCROSS = G * (G - 1) / 2;  // P1, P2, P3 (3M form, see kernel MT2)
  static constexpr int NMMA = 3 * NDIAG + 3 * NCROSS;
};

template <int G, int NT, int MINB, int KIND>
__global__ void __launch_bounds__(NT, MINB) gram_mma_kernel(GramParams P) {
  using Cfg = MmaCfg<G>;
  constexpr int NW = NT / 32;
  constexpr int NMMA = Cfg::NMMA;
  __shared__ double4 su[8 * G];            // (xz2, y, z, amp) per user
  __shared__ double cs[NW][NMMA][8][8];    // per-warp fragment staging at level ends

  const int64_t bdrop = blockIdx.x / P.n_split;
  const int split = blockIdx.x - (int)(bdrop * P.n_split);
  const int64_t drop = P.h_drop0 + bdrop;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int K = P.K;
  for (int u = tid; u < 8 * G; u += NT) {
    if (u < K) {
      const xl::UserC uc = xl::make_user(P.pos + (drop * K + u) * 3, KIND, P.sqrt_beta0);
      su[u] = make_double4(uc.xz2, uc.y, uc.z, uc.amp);
    } else {
      su[u] = make_double4(1.0, 0.0, 0.0, 0.0);  // padded user: zero amplitude
    }
  }
  __syncthreads();
  const double c4 = 4.0 * P.inv_lambda;
  const int ue = lane & 3, uu = lane >> 2;

  const int64_t s0 = (int64_t)split * P.chunk;
  const int64_t s1 = min(P.N, s0 + P.chunk);
  int64_t lv0 = 0;
  for (int l = 0; l < P.n_lvl; ++l) {
    const int64_t lv1 = P.lvl_end[l];
    const int64_t a = max(lv0, s0), b = min(lv1, s1);
    lv0 = lv1;
    double acc[NMMA][2];
#pragma unroll
    for (int m = 0; m < NMMA; ++m) acc[m][0] = acc[m][1] = 0.0;
    for (int64_t t0 = a + 4 * warp; t0 < b; t0 += 4 * NW) {  // warp-uniform trip count
      const int64_t t = t0 + ue;
      const bool valid = t < b;
      ElemPos ep = element_pos(P, valid ? t : a);
      double hr[G], hi[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const double4 u = su[uu + 8 * g];
        const double dy = ep.y - u.y;
        double r2 = fma(dy, dy, u.x);
        if (KIND != XLMIMO_ULA) {
          const double dz = ep.z - u.z;
          r2 = fma(dz, dz, r2);
        }
        xl::coef_fast(r2, valid ? u.w : 0.0, c4, hr[g], hi[g]);
      }
      int m = 0;
#pragma unroll
      for (int g1 = 0; g1 < G; ++g1) {
        dmma(acc[m++], hr[g1], hr[g1]);
        dmma(acc[m++], hi[g1], hi[g1]);
        dmma(acc[m++], hr[g1], hi[g1]);
        const double sg = hr[g1] + hi[g1];
#pragma unroll
        for (int g2 = g1 + 1; g2 < G; ++g2) {
          dmma(acc[m++], hr[g1], hr[g2]);
          dmma(acc[m++], hi[g1], hi[g2]);
          dmma(acc[m++], sg, hr[g2] - hi[g2]);
        }
      }
    }
    // stage the fragments (row = lane/4, cols 2(lane%4) + {0,1}) and assemble this
    // warp's partial upper triangle in the standard layout -- no block barrier.
#pragma unroll
    for (int mm = 0; mm < NMMA; ++mm) {
      cs[warp][mm][uu][2 * ue] = acc[mm][0];
      cs[warp][mm][uu][2 * ue + 1] = acc[mm][1];
    }
    __syncwarp();
    const int NP = K * (K + 1) / 2;
    double *out = P.ws + ((((size_t)drop * P.n_split + split) * P.n_lvl + l) * NW + warp) * (size_t)(2 * NP);
    for (int p = lane; p < NP; p += 32) {
      int i = 0, rem = p;
      while (rem >= K - i) { rem -= K - i; ++i; }
      const int j = i + rem;
      const int g1 = i >> 3, g2 = j >> 3, ii = i & 7, jj = j & 7;
      // job index of the (g1, g2) block: 3 slots per block, row-major over g1 <= g2
      const int base = 3 * (g1 * G - g1 * (g1 - 1) / 2);
      double re, im;
      if (g1 == g2) {
        re = cs[warp][base][ii][jj] + cs[warp][base + 1][ii][jj];
        im = cs[warp][base + 2][ii][jj] - cs[warp][base + 2][jj][ii];
      } else {
        const int c = base + 3 * (g2 - g1);
        const double p1 = cs[warp][c][ii][jj], p2 = cs[warp][c + 1][ii][jj];
        re = p1 + p2;
        im = p1 - p2 - cs[warp][c + 2][ii][jj];
      }
      out[2 * p] = re;
      out[2 * p + 1] = (i == j) ? 0.0 : im;
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------ kernel MT
// DMMA Gram for K = 17..64 (G = 3..8 user groups of 8), shared generation.
// Per tile of 4*S elements all threads generate the 8G x 4S coefficients into
// shared memory already in m8n8k4 fragment order (frag[s][g][lane], lane =
// 4*(user%8) + element%4, re and im planes), then each warp runs the DMMAs of its
// share of the group pairs (g1 <= g2): 3 per diagonal pair (RR, II, RI), 4 per
// cross pair (RR, II, RI, IR), loading 4 fragments (one LDS.64 per lane each) per
// pair.  At the level end the warps stage their fragments and the block writes
// one partial in the standard layout.
constexpr int kMtMaxPairs = 8;  // group pairs per warp (G = 8: 36 pairs over 8 warps)
struct MtPlan {
  int npairs[16];
  int g1[16][kMtMaxPairs], g2[16][kMtMaxPairs];
};

// jobs per G: G <= 4 splits cross pairs into two half-jobs (see make_mt_plan)
__host__ __device__ constexpr int mt_jobs(int G) { return G <= 4 ? G + G * (G - 1) : G * (G + 1) / 2; }
__host__ __device__ constexpr int mt_maxp(int G, int NW) { return (mt_jobs(G) + NW - 1) / NW + 1; }

template <int G, int S, int NW>
__global__ void __launch_bounds__(32 * NW, 1) gram_mma_tiled_kernel(GramParams P, MtPlan plan) {
  constexpr int NT = 32 * NW, NPAIR = G * (G + 1) / 2;
  constexpr bool HALVE = G <= 4;
  extern __shared__ __align__(16) double dsm[];
  double *fre = dsm;                  // 2 buffers x {re [S][G][32], im [S][G][32]}
  double *stage = dsm;                // [NPAIR][4][8][8] at level ends (aliases the tiles)
  __shared__ double4 su[8 * G];

  const int64_t bdrop = blockIdx.x / P.n_split;
  const int split = blockIdx.x - (int)(bdrop * P.n_split);
  const int64_t drop = P.h_drop0 + bdrop;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int K = P.K;
  for (int u = tid; u < 8 * G; u += NT) {
    if (u < K) {
      const xl::UserC uc = xl::make_user(P.pos + (drop * K + u) * 3, P.kind, P.sqrt_beta0);
      su[u] = make_double4(uc.xz2, uc.y, uc.z, uc.amp);
    } else {
      su[u] = make_double4(1.0, 0.0, 0.0, 0.0);
    }
  }
  constexpr int MAXP = mt_maxp(G, NW);  // bound used by make_mt_plan
  const int np = plan.npairs[warp];
  int pg1[MAXP], pg2[MAXP];
#pragma unroll
  for (int k = 0; k < MAXP; ++k) {
    pg1[k] = plan.g1[warp][k];
    pg2[k] = plan.g2[warp][k];
  }
  __syncthreads();
  const double c4 = 4.0 * P.inv_lambda;
  const int ulocal = lane >> 2, elocal = lane & 3;

  const int64_t s0 = (int64_t)split * P.chunk;
  const int64_t s1 = min(P.N, s0 + P.chunk);
  int64_t lv0 = 0;
  for (int l = 0; l < P.n_lvl; ++l) {
    const int64_t lv1 = P.lvl_end[l];
    const int64_t a = max(lv0, s0), b = min(lv1, s1);
    lv0 = lv1;
    double acc[MAXP][4][2];
#pragma unroll
    for (int k = 0; k < MAXP; ++k)
#pragma unroll
      for (int m = 0; m < 4; ++m) acc[k][m][0] = acc[k][m][1] = 0.0;
    // double-buffered tiles: generation of tile i+1 and the DMMAs of tile i run between
    // the same pair of barriers (one __syncthreads per tile)
    auto generate = [&](int64_t t0, int buf) {
      double *gre = fre + buf * (2 * S * G * 32), *gim = gre + S * G * 32;
      for (int c = tid; c < S * G * 32; c += NT) {
        const int s = c / (G * 32), rem = c - s * (G * 32), g = rem >> 5, ln = rem & 31;
        const int64_t t = t0 + 4 * s + (ln & 3);
        const int u = (ln >> 2) + 8 * g;
        const bool valid = t < b;
        const ElemPos ep = element_pos(P, valid ? t : a);
        const double4 uc = su[u];
        const double dy = ep.y - uc.y;
        double r2 = fma(dy, dy, uc.x);
        if (P.kind != XLMIMO_ULA) {
          const double dz = ep.z - uc.z;
          r2 = fma(dz, dz, r2);
        }
        double hr, hi;
        xl::coef_fast(r2, valid ? uc.w : 0.0, c4, hr, hi);
        gre[c] = hr;
        gim[c] = hi;
      }
    };
    if (a < b) generate(a, 0);
    __syncthreads();
    int buf = 0;
    for (int64_t t0 = a; t0 < b; t0 += 4 * S, buf ^= 1) {
      if (t0 + 4 * S < b) generate(t0 + 4 * S, buf ^ 1);
      const double *fre_c = fre + buf * (2 * S * G * 32);
      const double *fim_c = fre_c + S * G * 32;
      for (int s = 0; s < S; ++s) {
#pragma unroll
        for (int k = 0; k < MAXP; ++k) {
          if (k < np) {
            // part: 0 all, 1 RR+II, 2 RI+IR (compile-time 0 unless HALVE)
            const int g1 = pg1[k], g2 = pg2[k] & 255, part = HALVE ? (pg2[k] >> 8) : 0;
            const double ar = fre_c[(s * G + g1) * 32 + lane], ai = fim_c[(s * G + g1) * 32 + lane];
            const double br = fre_c[(s * G + g2) * 32 + lane], bi = fim_c[(s * G + g2) * 32 + lane];
            if (part != 2) {
              dmma(acc[k][0], ar, br);
              dmma(acc[k][1], ai, bi);
            }
            if (part != 1) {
              dmma(acc[k][2], ar, bi);
              if (g1 != g2) dmma(acc[k][3], ai, br);
            }
          }
        }
      }
      __syncthreads();
    }
    // stage fragments: pair index p(g1,g2) in row-major (g1 <= g2) order
#pragma unroll
    for (int k = 0; k < MAXP; ++k) {
      if (k < np) {
        const int g1 = pg1[k], g2 = pg2[k] & 255, part = HALVE ? (pg2[k] >> 8) : 0;
        const int p = g1 * G - g1 * (g1 - 1) / 2 + (g2 - g1);
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          if ((m < 2 && part == 2) || (m >= 2 && part == 1)) continue;  // the other half-job's slots
          stage[((p * 4 + m) * 8 + ulocal) * 8 + 2 * elocal] = acc[k][m][0];
          stage[((p * 4 + m) * 8 + ulocal) * 8 + 2 * elocal + 1] = acc[k][m][1];
        }
      }
    }
    __syncthreads();
    const int NP = K * (K + 1) / 2;
    double *out = P.ws + (((size_t)drop * P.n_split + split) * P.n_lvl + l) * (size_t)(2 * NP);
    for (int q = tid; q < NP; q += NT) {
      int i = 0, rem = q;
      while (rem >= K - i) { rem -= K - i; ++i; }
      const int j = i + rem;
      const int g1 = i >> 3, g2 = j >> 3, ii = i & 7, jj = j & 7;
      const int p = g1 * G - g1 * (g1 - 1) / 2 + (g2 - g1);
      const double *st = stage + (size_t)p * 4 * 64;
      const double re = st[0 * 64 + ii * 8 + jj] + st[1 * 64 + ii * 8 + jj];
      const double im = (g1 == g2) ? st[2 * 64 + ii * 8 + jj] - st[2 * 64 + jj * 8 + ii]
                                   : st[2 * 64 + ii * 8 + jj] - st[3 * 64 + ii * 8 + jj];
      out[2 * q] = re;
      out[2 * q + 1] = (i == j) ? 0.0 : im;
    }
    __syncthreads();
    (void)NPAIR;
  }
}

// Balanced assignment of the G(G+1)/2 group pairs (row-major) to 8 warps by DMMA count.
MtPlan make_mt_plan(int G, int nw) {
  MtPlan pl;
  memset(&pl, 0, sizeof(pl));
  const int maxp = mt_maxp(G, nw);
  // longest-processing-time greedy over jobs: diagonal pairs (3 DMMAs) and cross pairs
  // (4 DMMAs, or for G <= 4 -- fewer pairs than warps can balance -- two half-jobs
  // RR+II / RI+IR of 2 DMMAs each, encoded as g2 | part << 8).
  int load[16] = {0};
  const bool halve = G <= 4;
  auto place = [&](int g1, int g2code, int cost) {
    int w = -1;
    for (int c = 0; c < nw; ++c)
      if (pl.npairs[c] < maxp && (w < 0 || load[c] < load[w])) w = c;
    pl.g1[w][pl.npairs[w]] = g1;
    pl.g2[w][pl.npairs[w]] = g2code;
    ++pl.npairs[w];
    load[w] += cost;
  };
  if (halve)  // costliest first: diagonal (3) before the half-jobs (2)
    for (int g = 0; g < G; ++g) place(g, g, 3);
  for (int g1 = 0; g1 < G; ++g1)
    for (int g2 = g1 + 1; g2 < G; ++g2) {
      if (halve) {
        place(g1, g2 | (1 << 8), 2);
        place(g1, g2 | (2 << 8), 2);
      } else {
        place(g1, g2, 4);
      }
    }
  if (!halve)
    for (int g = 0; g < G; ++g) place(g, g, 3);
  return pl;
}

constexpr int kMtS = 8;  // 4-element steps per tile (32 elements)

template <int G>
size_t mt_smem_bytes() {
  const size_t tiles = 4 * (size_t)kMtS * G * 32 * sizeof(double);  // double-buffered re/im tiles
  const size_t stage = (size_t)(G * (G + 1) / 2) * 4 * 64 * sizeof(double);
  return tiles > stage ? tiles : stage;
}

// 16 warps for G >= 5 (more latency hiding, half the accumulators per warp), 8 below
template <int G>
void launch_mt(const GramParams &P, int64_t n_blocks, cudaStream_t s) {
  constexpr int NW = 16;
  static const MtPlan plan = make_mt_plan(G, NW);
  const size_t smem = mt_smem_bytes<G>();
  cudaFuncSetAttribute(gram_mma_tiled_kernel<G, kMtS, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  gram_mma_tiled_kernel<G, kMtS, NW><<<(unsigned)n_blocks, 32 * NW, smem, s>>>(P, plan);
}

// ------------------------------------------------------------------ kernel MT2
// DMMA Gram for K = 17..64 (the default for fp64 K > 16), three real DMMAs per
// complex 8 x 8 block.  With A, B the re / im fragment planes of 8 users each (one
// m8n8k4 fragment per 8 users and 4 elements), the block of plane groups (c, p) is
//   G(c, p) = sum conj(h_c) h_p:  Re = P1 + P2,  Im = P1 - P2 - P3,
//   P1 = A_c A_p^T,  P2 = B_c B_p^T,  P3 = (A_c + B_c)(A_p - B_p)^T
// (the 3M form of the complex product: one DMMA fewer than RR, II, RI, IR, for two
// fp64 adds on fragments -- its cancellation in Im costs ~eps sqrt(G_ii G_jj), i.e.
// nothing against the normalised 1e-9 tier, R9).  The G(G+1)/2 blocks g1 <= g2 are
// dealt to warps as STARS: a warp owns JPW blocks that share one centre group c
// (c, p_1..p_JPW), so A_c, B_c and A_c + B_c are loaded / formed once per step; a star
// decomposition exists when the blocks can be oriented so that every group's count of
// blocks it centres (its own diagonal block included) is a multiple of JPW -- a
// tournament score condition (Landau), found by a small search on the host
// (star_plan).  Warps are (star, step group sg): the stars over the steps s == sg mod
// SG of each tile; the SG partial accumulators meet in shared memory at level ends.
// NW = stars * SG is a multiple of 4 (same DMMA load per SM sub-partition) except
// G = 6, 7 (14 warps).  Tiles of 4S elements are generated (one 32-lane fragment row =
// 4 elements x 8 users per warp-iteration) into a double buffer or a 3-deep mbarrier
// ring; the tile length splits the S*G generated rows evenly over the warps.
// Measured (cfg5, K = 64, 1000 drops): 4 DMMAs per block 782 ms -> see DESIGN.md 6.1.
template <int G>
struct Mt2Cfg;
template <> struct Mt2Cfg<3> { static constexpr int JPW = 2, SG = 4, S = 8; };   // 3 stars, NW 12
template <> struct Mt2Cfg<4> { static constexpr int JPW = 2, SG = 4, S = 10; };  // 5 stars, NW 20
template <> struct Mt2Cfg<5> { static constexpr int JPW = 3, SG = 4, S = 8; };   // 5 stars, NW 20
template <> struct Mt2Cfg<6> { static constexpr int JPW = 3, SG = 2, S = 8; };   // 7 stars, NW 14
#ifndef XL_MT2_VARX
#define XL_MT2_VARX 1
#endif
#if XL_MT2_VARX
// 8 stars of 4 or 3 (centred counts 3,3,3,4,4,4,7) x 2 step groups = 16 warps instead of 7 x 2
// (sub-partition loads 14 each instead of 16/16/12/12; K = 56: 19.8 -> 18.4 ms)
template <> struct Mt2Cfg<7> {
  static constexpr int JPW = 4, SG = 2, S = 8, NSTAR = 8;
  static constexpr int cent[7] = {3, 3, 3, 4, 4, 4, 7};
};
#else
template <> struct Mt2Cfg<7> { static constexpr int JPW = 4, SG = 2, S = 8; };   // 7 stars, NW 14
#endif
template <> struct Mt2Cfg<8> { static constexpr int JPW = 3, SG = 1, S = 9; };   // 12 stars, NW 12, 12 rows/warp
// 64 < K <= 128 (the paper's K = 100 of E1/E2 and Fig. K_vs_E): one star per
// warp.  Uniform plans of a regular or near-regular tournament leave the warp count off a
// multiple of 4 for most G (the SM sub-partitions then carry unequal shares), so G = 9, 10, 12,
// 13, 14 (and 7, 16) use variable-size plans (star_plan_var); G = 11 and 15 stay uniform.
#ifndef XL_MT2_VAR9
#define XL_MT2_VAR9 1
#endif
#if XL_MT2_VAR9
// 12 stars of 4 or 3 (centred counts 4 x 6, 7 x 3) instead of 9 stars of 5 (SM sub-partition
// loads 12/11/11/11 blocks instead of 15/10/10/10; K = 72: 34.8 -> 29.2 ms)
template <> struct Mt2Cfg<9> {
  static constexpr int JPW = 4, SG = 1, S = 4, NSTAR = 12;
  static constexpr int cent[9] = {4, 4, 4, 4, 4, 4, 7, 7, 7};
};
#else
template <> struct Mt2Cfg<9> { static constexpr int JPW = 5, SG = 1, S = 4; };   // 9 stars
#endif
#if XL_MT2_VARX
// 16 stars of 4 or 3 (centred counts 4 x 4, 6 x 3, 7 x 3): loads 14/14/14/13 instead of 15/15/15/10
// (E1 field, K = 80, 1000 drops: 37.0 -> 36.0 ms)
template <> struct Mt2Cfg<10> {
  static constexpr int JPW = 4, SG = 1, S = 4, NSTAR = 16;
  static constexpr int cent[10] = {4, 4, 4, 4, 6, 6, 6, 7, 7, 7};
};
#else
template <> struct Mt2Cfg<10> { static constexpr int JPW = 5, SG = 1, S = 4; };  // 11 stars
#endif
#if XL_MT2_VARX
// 12 stars of 6 or 5 (centred counts 5 x 5, 6 x 5, 11; loads 17/17/16/16 instead of 18/18/18/12)
// on 48-element tiles, so that the 132 generated rows split evenly (11 per warp): K = 88
// 40.4 -> 37.7 ms (on 32-element tiles, 8 rows for 11 warps and none for the 12th: +3.8 %)
template <> struct Mt2Cfg<11> {
  static constexpr int JPW = 6, SG = 1, S = 6, NSTAR = 12;
  static constexpr int cent[11] = {5, 5, 5, 5, 5, 6, 6, 6, 6, 6, 11};
};
#else
template <> struct Mt2Cfg<11> { static constexpr int JPW = 6, SG = 1, S = 4; };  // 11 stars
#endif
#ifndef XL_MT2_VAR12
#define XL_MT2_VAR12 1
#endif
#if XL_MT2_VAR12
// 16 stars of 5 or 4 (centred counts 5 x 8, 9, 9, 10, 10) instead of 13 stars of 6 (loads
// 20/20/19/19 instead of 24/18/18/18; K = 96: 51.3 -> 44.8 ms)
template <> struct Mt2Cfg<12> {
  static constexpr int JPW = 5, SG = 1, S = 4, NSTAR = 16;
  static constexpr int cent[12] = {5, 5, 5, 5, 5, 5, 5, 5, 9, 9, 10, 10};
};
#else
template <> struct Mt2Cfg<12> { static constexpr int JPW = 6, SG = 1, S = 4; };  // 13 stars
#endif
#ifndef XL_MT2_VAR13
#define XL_MT2_VAR13 1
#endif
#if XL_MT2_VAR13
// G = 13 (K = 97..104, E1's K = 100): 13 stars of 7 put 4 warps on one SM sub-partition and 3
// on the others (the CTA runs at the busiest one's pace: 13/16); 16 stars of 6 or 5 blocks
// (centred counts 5,5,5,6,...,6,11,11,12: a Landau score sequence) dealt so that each
// sub-partition holds 22-23 blocks
// (E1 field, K = 100, 1000 drops: 60.9 -> 58.3 ms; 20 stars of 5 or 4 at 96 registers: 64.2 ms)
template <> struct Mt2Cfg<13> {
  static constexpr int JPW = 6, SG = 1, S = 4, NSTAR = 16;
  static constexpr int cent[13] = {5, 5, 5, 6, 6, 6, 6, 6, 6, 6, 11, 11, 12};
};
#else
template <> struct Mt2Cfg<13> { static constexpr int JPW = 7, SG = 1, S = 4; };  // 13 stars
#endif
#if XL_MT2_VARX
// 16 stars of 7 or 6 (centred counts 6 x 5, 7 x 7, 13, 13): loads 27/26/26/26 instead of 28/28/28/21
// (K = 112: 63.8 -> 60.1 ms; 20 stars of 6 or 5 spill at 96 registers: 72.5 ms)
template <> struct Mt2Cfg<14> {
  static constexpr int JPW = 7, SG = 1, S = 4, NSTAR = 16;
  static constexpr int cent[14] = {6, 6, 6, 6, 6, 7, 7, 7, 7, 7, 7, 7, 13, 13};
};
#else
template <> struct Mt2Cfg<14> { static constexpr int JPW = 7, SG = 1, S = 4; };  // 15 stars
#endif
template <> struct Mt2Cfg<15> { static constexpr int JPW = 6, SG = 1, S = 4; };  // 20 stars
// 120 < K <= 128: 34 stars of 4 dealt to two launches of 17 warps (a single launch of 17
// stars of 8 spills its accumulators); each launch generates all 16 groups
#if XL_MT2_VARX
// variable-size: 32 stars of 5 or 4 (every group centres 8 or 9 blocks), 16 per launch: loads
// 18 / 16 blocks per sub-partition in the two launches instead of 20 and 20
template <> struct Mt2Cfg<16> {
  static constexpr int JPW = 5, SG = 1, S = 4, NL = 2, NSTAR = 32;
  static constexpr int cent[16] = {8, 8, 8, 8, 8, 8, 8, 8, 9, 9, 9, 9, 9, 9, 9, 9};
};
#else
template <> struct Mt2Cfg<16> { static constexpr int JPW = 4, SG = 1, S = 4, NL = 2; };
#endif
template <int G, typename = void>
struct Mt2Launches { static constexpr int value = 1; };
template <int G>
struct Mt2Launches<G, decltype((void)Mt2Cfg<G>::NL, void())> { static constexpr int value = Mt2Cfg<G>::NL; };
// variable-size stars (JPW or JPW - 1 blocks): Mt2Cfg<G>::NSTAR stars with centred counts cent[]
template <int G, typename = void>
struct Mt2Var { static constexpr int value = 0; };
template <int G>
struct Mt2Var<G, decltype((void)Mt2Cfg<G>::NSTAR, void())> { static constexpr int value = Mt2Cfg<G>::NSTAR; };

// Tile planes: re, im and re - im, the 3M partner operand (A_p - B_p), formed once per
// coefficient by the generator instead of once per star and step by the consumers (the
// DADDs waited on the busy FP64 pipe: cfg5 196.6 -> 189.2 ms per 296 drops, cfg4 -1.9 %,
// K = 72 / 100 / 120 -3.8 / -2.3 / -0.4 %, bit-identical).  XL_MT2_DPLANE=0: two planes.
#ifndef XL_MT2_DPLANE
#define XL_MT2_DPLANE 1
#endif
constexpr int kMt2Planes = XL_MT2_DPLANE ? 3 : 2;
template <int G, int SM, int NBUF>  // SM: tile-length multiplier of Mt2Cfg<G>::S; NBUF tile buffers
struct Mt2 {
  static constexpr int J = G * (G + 1) / 2, JPW = Mt2Cfg<G>::JPW, SG = Mt2Cfg<G>::SG, S = SM * Mt2Cfg<G>::S;
  static constexpr int NL = Mt2Launches<G>::value;  // launches sharing the stars
  static constexpr int VAR = Mt2Var<G>::value;  // 0, or the star count of a variable-size plan
  static constexpr int JG = VAR ? VAR / NL : J / (JPW * NL), NW = JG * SG, NT = 32 * NW;  // stars per launch
  static constexpr int PLANE = S * G * 32;  // doubles in one (re or im) tile plane set
  static constexpr int ROWS = S * G;        // 32-lane fragment rows per tile
  static_assert((VAR ? VAR % NL == 0 : J % (JPW * NL) == 0) && S % SG == 0, "Mt2Cfg");
  static constexpr int NPL = kMt2Planes;  // re, im (, re - im: the 3M partner operand)
  static constexpr size_t tiles_bytes = (size_t)NPL * NBUF * PLANE * sizeof(double);  // NBUF buffers x planes
  static constexpr size_t stage_bytes = (size_t)JG * JPW * 3 * SG * 64 * sizeof(double);
  static constexpr size_t smem = tiles_bytes > stage_bytes ? tiles_bytes : stage_bytes;
  static constexpr bool fits = smem <= 220 * 1024;
};
// Mt2<G, SM, NBUF>::fits without instantiating Mt2 (launch-time shape choices)
template <int G, int SM, int NBUF>
constexpr bool mt2_fits() {
  constexpr int J = G * (G + 1) / 2, JPW = Mt2Cfg<G>::JPW, SG = Mt2Cfg<G>::SG, S = SM * Mt2Cfg<G>::S;
  constexpr int JG = Mt2Var<G>::value ? Mt2Var<G>::value / Mt2Launches<G>::value : J / (JPW * Mt2Launches<G>::value);
  constexpr size_t tiles = (size_t)kMt2Planes * NBUF * S * G * 32 * sizeof(double);
  constexpr size_t stage = (size_t)JG * JPW * 3 * SG * 64 * sizeof(double);
  return (tiles > stage ? tiles : stage) <= 220 * 1024;
}

// Star plan of the MT2 kernel: star s (warp's job group) = centre cen[s] and partners
// par[s][k]; blk[g1 * 16 + g2] (g1 <= g2) = 2 * (job s * JPW + k) + (1 if the star holds
// the block as (g2, g1), i.e. transposed).
constexpr int kMt2MaxG = 16;
struct StarPlan {
  int8_t cen[40];
  int8_t nj[40];  // blocks of star s (JPW, or JPW - 1 in a variable-size plan)
  int8_t par[40][8];
  int16_t blk[kMt2MaxG * kMt2MaxG];
};

struct FastDiv {  // q = (umulhi(m, t) + t) >> sh == t / d for 0 <= t < 2^31
  uint32_t m;
  int sh;
};

FastDiv make_fastdiv(uint32_t d) {
  int l = 0;
  while ((1ull << l) < d) ++l;
  FastDiv f;
  f.m = (uint32_t)((((1ull << l) - d) << 32) / d + 1);
  f.sh = l;
  return f;
}

template <int KIND>
__device__ __forceinline__ ElemPos element_pos32(const GramParams &P, int t, FastDiv fd, bool n_odd) {
  ElemPos e;
  if (KIND == XLMIMO_ULA) {
    e.y = xl::ula_y_centred(t, n_odd, P.pitch);
    e.z = 0.0;
  } else {
    const uint32_t tt = (uint32_t)t;
    const uint32_t q = (__umulhi(fd.m, tt) + tt) >> fd.sh;
    const uint32_t p = tt - q * (uint32_t)P.n_y;
    e.y = ((double)p - 0.5 * (double)(P.n_y - 1)) * P.pitch;
    e.z = ((double)q - 0.5 * (double)(P.n_z - 1)) * P.pitch;
  }
  return e;
}

__device__ __forceinline__ uint32_t mt_smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
// bounded parity wait (a broken protocol traps instead of hanging the GPU)
__device__ __forceinline__ void mt_wait(uint64_t *bar, uint32_t parity) {
  const uint32_t a = mt_smem_u32(bar);
  for (uint32_t it = 0; it < (1u << 28); ++it) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
    if (done) return;
  }
  __trap();
}
__device__ __forceinline__ void mt_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mt_smem_u32(bar)) : "memory");
}

// NBUF = 2: one __syncthreads per tile (generation of tile i+1 and the DMMAs of
// tile i between the same pair of barriers).  NBUF = 3: a ring with per-buffer
// full/empty mbarriers (every thread arrives), so warps drift up to a tile apart
// instead of draining the FP64 pipe at every tile boundary.
template <int G, int SM, int NBUF, int KIND>
__global__ void __launch_bounds__(Mt2<G, SM, NBUF>::NT, 1) gram_mt2_kernel(GramParams P, FastDiv fd,
                                                                         const __grid_constant__ StarPlan plan,
                                                                         int star0) {
  using C = Mt2<G, SM, NBUF>;
  constexpr int JPW = C::JPW, SG = C::SG, S = C::S, NW = C::NW, NT = C::NT, JG = C::JG;
  constexpr int PLANE = C::PLANE, ROWS = C::ROWS;
  extern __shared__ __align__(16) double dsm[];  // tiles [NBUF][re|im][S][G][32]; stage at level ends
  __shared__ double4 su[8 * G];
  __shared__ __align__(8) uint64_t mb_full[NBUF], mb_empty[NBUF];

  const int64_t bdrop = blockIdx.x / P.n_split;
  const int split = blockIdx.x - (int)(bdrop * P.n_split);
  const int64_t drop = P.h_drop0 + bdrop;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int K = P.K;
  for (int u = tid; u < 8 * G; u += NT) {
    if (u < K) {
      const xl::UserC uc = xl::make_user(P.pos + (drop * K + u) * 3, KIND, P.sqrt_beta0);
      su[u] = make_double4(uc.xz2, uc.y, uc.z, uc.amp);
    } else {
      su[u] = make_double4(1.0, 0.0, 0.0, 0.0);  // padded user: zero amplitude
    }
  }
  if (NBUF > 2 && tid == 0) {
    for (int i = 0; i < NBUF; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mt_smem_u32(&mb_full[i])), "r"(NT));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mt_smem_u32(&mb_empty[i])), "r"(NT));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const int jg = warp % JG, sg = warp / JG;
  const int coff = plan.cen[star0 + jg] * 32 + lane;  // the star's centre fragment
  const int nj = C::VAR ? (int)plan.nj[star0 + jg] : JPW;  // blocks of this warp's star
  int poff[JPW];                                      // its partners' fragments
#pragma unroll
  for (int k = 0; k < JPW; ++k) poff[k] = plan.par[star0 + jg][k] * 32 + lane;
  __syncthreads();
  const double c4 = 4.0 * P.inv_lambda;
  const bool n_odd = (P.N & 1) != 0;

  const int s0 = (int)min((int64_t)split * P.chunk, P.N);
  const int s1 = (int)min(P.N, (int64_t)s0 + P.chunk);
  int lv0 = 0;
  uint32_t T = 0;  // tiles issued so far (ring position, uniform)
  for (int l = 0; l < P.n_lvl; ++l) {
    const int lv1 = (int)P.lvl_end[l];
    const int a = max(lv0, s0), b = min(lv1, s1);
    lv0 = lv1;
    double acc[JPW][3][2];
#pragma unroll
    for (int k = 0; k < JPW; ++k)
#pragma unroll
      for (int m = 0; m < 3; ++m) acc[k][m][0] = acc[k][m][1] = 0.0;
    // warp w generates the consecutive rows [w R, (w+1) R) (row = s * G + g, g fastest),
    // so runs of up to G rows share one element step s and decode its coordinates once
    // (a UPA decode costs 4 FP64 ops, a ULA one 2: otherwise repeated for every group)
    // ROWS % NW != 0 (G = 6, 13): the first ROWS % NW warps take one row more -- spread over the
    // SM sub-partitions when that count is a multiple of 4 -- instead of R each and the tail warps
    // none (XL_MT2_ROWS_CEIL: the old split)
    constexpr int R = (ROWS + NW - 1) / NW, RLO = ROWS / NW, REX = ROWS % NW;
#ifdef XL_MT2_ROWS_CEIL
    const int rs = warp * R, rc = ROWS - rs < R ? ROWS - rs : R;
#else
    const int rs = warp * RLO + (warp < REX ? warp : REX), rc = RLO + (warp < REX ? 1 : 0);
#endif
    auto generate = [&](int t0, int buf) {
      double *gre = dsm + buf * (C::NPL * PLANE), *gim = gre + PLANE;
      int s_cur = -1;
      bool valid = false;
      ElemPos ep;
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const int row = rs + i;
        if (ROWS % NW == 0 || i < rc) {
          const int s = row / G, g = row - s * G;
          if (s != s_cur) {  // warp-uniform
            s_cur = s;
            const int t = t0 + 4 * s + (lane & 3);
            valid = t < b;
            ep = element_pos32<KIND>(P, valid ? t : a, fd, n_odd);
          }
          const double4 uc = su[8 * g + (lane >> 2)];
          const double dy = ep.y - uc.y;
          double r2 = fma(dy, dy, uc.x);
          if (KIND != XLMIMO_ULA) {
            const double dz = ep.z - uc.z;
            r2 = fma(dz, dz, r2);
          }
          double hr, hi;
#ifdef XL_EXP_MT2_NOGEN  // tuning experiment: the DMMA-side rate (results invalid)
          hr = r2 * 1e-9; hi = uc.w;
#else
          xl::coef_fast(r2, valid ? uc.w : 0.0, c4, hr, hi);
#endif
          gre[row * 32 + lane] = hr;
          gim[row * 32 + lane] = hi;
          if constexpr (C::NPL == 3) gim[PLANE + row * 32 + lane] = hr - hi;
        }
      }
    };
    auto consume = [&](int buf) {
      const double *cre = dsm + buf * (C::NPL * PLANE) + sg * (G * 32), *cim = cre + PLANE;
#pragma unroll
      for (int si = 0; si < S / SG; ++si) {
        const int so = si * SG * G * 32;
        const double ar = cre[so + coff], ai = cim[so + coff];
        const double as = ar + ai;
#pragma unroll
        for (int k = 0; k < JPW; ++k) {
          if (C::VAR && k >= nj) continue;  // a star of JPW - 1 blocks (warp-uniform)
          const double br = cre[so + poff[k]], bi = cim[so + poff[k]];
          const double bd = C::NPL == 3 ? cim[PLANE + so + poff[k]] : br - bi;
          dmma(acc[k][0], ar, br);  // P1
          dmma(acc[k][1], ai, bi);  // P2
          dmma(acc[k][2], as, bd);  // P3
        }
      }
    };
    if (NBUF == 2) {
      if (a < b) generate(a, 0);
      __syncthreads();
      int buf = 0;
      for (int t0 = a; t0 < b; t0 += 4 * S, buf ^= 1) {
        if (t0 + 4 * S < b) generate(t0 + 4 * S, buf ^ 1);
        consume(buf);
        __syncthreads();
      }
    } else {
      const int n = b > a ? (b - a + 4 * S - 1) / (4 * S) : 0;
      auto produce = [&](int i) {
        const uint32_t tt = T + i;
        const int bb = (int)(tt % NBUF);
        if (tt >= NBUF) mt_wait(&mb_empty[bb], (tt / NBUF - 1) & 1);  // tile tt - NBUF consumed
        generate(a + i * 4 * S, bb);
        mt_arrive(&mb_full[bb]);
      };
#pragma unroll
      for (int i = 0; i < NBUF - 1; ++i)
        if (i < n) produce(i);
      for (int i = 0; i < n; ++i) {
        if (i + NBUF - 1 < n) produce(i + NBUF - 1);
        const uint32_t tt = T + i;
        const int bb = (int)(tt % NBUF);
        mt_wait(&mb_full[bb], (tt / NBUF) & 1);
        consume(bb);
        mt_arrive(&mb_empty[bb]);
      }
      T += n;
      __syncthreads();  // every warp's DMMAs done before the stage aliases the tiles
    }
    // stage [q][m][sg][8][8] (C fragment: row lane/4, cols 2(lane%4) + {0,1})
#pragma unroll
    for (int k = 0; k < JPW; ++k) {
      const int q = jg * JPW + k;
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        double *st = dsm + ((q * 3 + m) * SG + sg) * 64 + (lane >> 2) * 8 + 2 * (lane & 3);
        st[0] = acc[k][m][0];
        st[1] = acc[k][m][1];
      }
    }
    __syncthreads();
    const int NP = K * (K + 1) / 2;
    double *out = P.ws + (((size_t)drop * P.n_split + split) * P.n_lvl + l) * (size_t)(2 * NP);
    for (int p = tid; p < NP; p += NT) {
      int i = 0, rem = p;
      while (rem >= K - i) { rem -= K - i; ++i; }
      const int j = i + rem;
      const int bq = plan.blk[(i >> 3) * kMt2MaxG + (j >> 3)];
      const int q = (bq >> 1) - star0 * JPW;  // this launch's job holding the block
      if (C::NL > 1 && (q < 0 || q >= JG * JPW)) continue;  // another launch's block
      const bool tr = bq & 1;  // block held as (g2, g1): read (j, i) and conjugate
      const int e = tr ? (j & 7) * 8 + (i & 7) : (i & 7) * 8 + (j & 7);
      const double *st = dsm + (size_t)q * 3 * SG * 64 + e;
      double p1 = 0.0, p2 = 0.0, p3 = 0.0;
#pragma unroll
      for (int g = 0; g < SG; ++g) {
        p1 += st[(0 * SG + g) * 64];
        p2 += st[(1 * SG + g) * 64];
        p3 += st[(2 * SG + g) * 64];
      }
      const double im = p1 - p2 - p3;
      out[2 * p] = p1 + p2;
      out[2 * p + 1] = (i == j) ? 0.0 : (tr ? -im : im);
    }
    __syncthreads();
  }
}

// Star decomposition of the G(G+1)/2 plane blocks into stars of JPW blocks sharing a centre
// (see kernel MT2): orient every pair {a, b} (a < b) towards one centre so that each group's
// centred-block count (+1 for its own diagonal block) is a multiple of JPW, by depth-first
// search over the pairs; then cut each group's list (diagonal first) into stars.
bool star_plan(int G, int JPW, StarPlan &pl) {
  int pa[kMt2MaxG * (kMt2MaxG - 1) / 2], pb[kMt2MaxG * (kMt2MaxG - 1) / 2], n = 0;
  for (int a = 0; a < G; ++a)
    for (int b = a + 1; b < G; ++b) { pa[n] = a; pb[n] = b; ++n; }
  int out[kMt2MaxG] = {0}, left[kMt2MaxG], to[kMt2MaxG * (kMt2MaxG - 1) / 2];
  for (int v = 0; v < G; ++v) left[v] = G - 1;
  auto can = [&](int v) {  // some multiple of JPW is still reachable for v
    for (int d = out[v]; d <= out[v] + left[v]; ++d)
      if ((d + 1) % JPW == 0) return true;
    return false;
  };
  std::vector<int> st;  // DFS over pairs: choice 0 = a centres, 1 = b centres
  int k = 0, choice = 0;
  while (k < n) {
    bool placed = false;
    for (; choice < 2; ++choice) {
      const int c = choice ? pb[k] : pa[k];
      ++out[c]; --left[pa[k]]; --left[pb[k]];
      if (can(pa[k]) && can(pb[k])) { to[k] = choice; st.push_back(choice); ++k; choice = 0; placed = true; break; }
      --out[c]; ++left[pa[k]]; ++left[pb[k]];
    }
    if (placed) continue;
    if (st.empty()) return false;  // no decomposition
    --k;
    choice = st.back();
    st.pop_back();
    const int c = choice ? pb[k] : pa[k];
    --out[c]; ++left[pa[k]]; ++left[pb[k]];
    ++choice;
  }
  for (int v = 0; v < G; ++v)
    if ((out[v] + 1) % JPW) return false;
  int ns = 0;
  for (int v = 0; v < G; ++v) {
    int list[kMt2MaxG], m = 0;
    list[m++] = v;
    for (int e = 0; e < n; ++e)
      if ((to[e] ? pb[e] : pa[e]) == v) list[m++] = to[e] ? pa[e] : pb[e];
    for (int q = 0; q < m; q += JPW, ++ns) {
      pl.cen[ns] = (int8_t)v;
      pl.nj[ns] = (int8_t)JPW;
      for (int t = 0; t < JPW; ++t) {
        const int p = list[q + t];
        pl.par[ns][t] = (int8_t)p;
        const int job = ns * JPW + t;
        if (v <= p) pl.blk[v * kMt2MaxG + p] = (int16_t)(2 * job);
        else pl.blk[p * kMt2MaxG + v] = (int16_t)(2 * job + 1);
      }
    }
  }
  return ns * JPW == G * (G + 1) / 2;
}

// Variable-size stars: orient the pairs so that group v centres exactly cent[v] blocks (its
// diagonal included; cent - 1 must be a tournament score sequence, Landau), by the same
// depth-first search with exact targets; cut each group's list into ceil(cent / JPW) stars
// of JPW or JPW - 1 blocks; order the stars by size (largest first) so that warp w = star w
// on sub-partition w % 4 gets an even share of blocks.  Jobs keep the slot stride JPW.
bool star_plan_var(int G, int JPW, int NSTAR, const int *cent, StarPlan &pl) {
  int pa[kMt2MaxG * (kMt2MaxG - 1) / 2], pb[kMt2MaxG * (kMt2MaxG - 1) / 2], n = 0;
  for (int a = 0; a < G; ++a)
    for (int b = a + 1; b < G; ++b) { pa[n] = a; pb[n] = b; ++n; }
  int out[kMt2MaxG] = {0}, left[kMt2MaxG], to[kMt2MaxG * (kMt2MaxG - 1) / 2];
  for (int v = 0; v < G; ++v) left[v] = G - 1;
  auto can = [&](int v) { return out[v] <= cent[v] - 1 && out[v] + left[v] >= cent[v] - 1; };
  std::vector<int> st;
  int k = 0, choice = 0;
  while (k < n) {
    bool placed = false;
    for (; choice < 2; ++choice) {
      const int c = choice ? pb[k] : pa[k];
      ++out[c]; --left[pa[k]]; --left[pb[k]];
      if (can(pa[k]) && can(pb[k])) { to[k] = choice; st.push_back(choice); ++k; choice = 0; placed = true; break; }
      --out[c]; ++left[pa[k]]; ++left[pb[k]];
    }
    if (placed) continue;
    if (st.empty()) return false;
    --k;
    choice = st.back();
    st.pop_back();
    const int c = choice ? pb[k] : pa[k];
    --out[c]; ++left[pa[k]]; ++left[pb[k]];
    ++choice;
  }
  int scen[40], snj[40], spar[40][8], ns = 0;
  for (int v = 0; v < G; ++v) {
    if (out[v] + 1 != cent[v]) return false;
    int list[kMt2MaxG], m = 0;
    list[m++] = v;
    for (int e = 0; e < n; ++e)
      if ((to[e] ? pb[e] : pa[e]) == v) list[m++] = to[e] ? pa[e] : pb[e];
    const int parts = (m + JPW - 1) / JPW, big = m - parts * (JPW - 1);  // parts of JPW, the rest JPW - 1
    if (big < 0 || ns + parts > 40) return false;
    for (int q = 0, i = 0; q < parts; ++q, ++ns) {
      const int sz = q < big ? JPW : JPW - 1;
      scen[ns] = v;
      snj[ns] = sz;
      for (int t = 0; t < JPW; ++t) spar[ns][t] = t < sz ? list[i + t] : v;
      i += sz;
    }
  }
  if (ns != NSTAR) return false;
  int ord[40];
  for (int i = 0; i < ns; ++i) ord[i] = i;
  std::stable_sort(ord, ord + ns, [&](int x, int y) { return snj[x] > snj[y]; });
  int total = 0;
  for (int w = 0; w < ns; ++w) {
    const int o = ord[w];
    pl.cen[w] = (int8_t)scen[o];
    pl.nj[w] = (int8_t)snj[o];
    for (int t = 0; t < JPW; ++t) {
      const int p = spar[o][t];
      pl.par[w][t] = (int8_t)p;
      if (t >= snj[o]) continue;
      const int v = scen[o], job = w * JPW + t;
      if (v <= p) pl.blk[v * kMt2MaxG + p] = (int16_t)(2 * job);
      else pl.blk[p * kMt2MaxG + v] = (int16_t)(2 * job + 1);
      ++total;
    }
  }
  return total == G * (G + 1) / 2;
}

template <int G, int SM, int NBUF, int KIND>
int launch_mt2_k(const GramParams &P, int64_t n_blocks, cudaStream_t s) {
  using C = Mt2<G, SM, NBUF>;
  static_assert(C::fits, "Mt2 shared memory");
  static StarPlan plan;
  static const bool ok = [] {
    if constexpr (C::VAR) return star_plan_var(G, C::JPW, C::VAR, Mt2Cfg<G>::cent, plan);
    else return star_plan(G, C::JPW, plan);
  }();
  if (!ok) return xlh::set_error(XLMIMO_EUNSUPPORTED, "mt2: no star decomposition for G=%d, JPW=%d", G, C::JPW);
  const FastDiv fd = make_fastdiv((uint32_t)P.n_y);
  cudaFuncSetAttribute(gram_mt2_kernel<G, SM, NBUF, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem);
  for (int l = 0; l < C::NL; ++l)  // each launch its share of the stars, disjoint entries of the partials
    gram_mt2_kernel<G, SM, NBUF, KIND><<<(unsigned)n_blocks, C::NT, C::smem, s>>>(P, fd, plan, l * C::JG);
  if (C::NL > 1) xlh::count_launch(C::NL - 1);  // the caller counts one
  return XLMIMO_OK;
}

// Tiles of 2*Mt2Cfg<G>::S steps in two buffers (one barrier per tile) for every G.  The 3-deep
// mbarrier ring (full-length tiles where three planes fit, half-length ones for K > 64
// otherwise) is kept as the XLMIMO_OPT_MT2_BUFFERS = 3 option: late round 2 it was slower or
// equal at every K on the E1 field (tools/ab_mt2buf.py, 1000 drops: K = 40 11.05 -> 10.74 ms,
// 48 15.85 -> 15.53, 72 29.23 -> 28.25, 80 35.92 -> 34.22, 100 58.8 -> 54.4, 120 64.5 -> 62.4).
template <int G>
int launch_mt2(const GramParams &P, int64_t n_blocks, cudaStream_t s) {
  const int env = (int)xlh::option(XLMIMO_OPT_MT2_BUFFERS);
  const bool ula = P.kind == XLMIMO_ULA;
  if constexpr (mt2_fits<G, 2, 2>()) {
    if (env != 3 || (G <= 8 && !mt2_fits<G, 2, 3>()))
      return ula ? launch_mt2_k<G, 2, 2, XLMIMO_ULA>(P, n_blocks, s) : launch_mt2_k<G, 2, 2, XLMIMO_UPA>(P, n_blocks, s);
  }
  if constexpr (mt2_fits<G, 2, 3>())
    return ula ? launch_mt2_k<G, 2, 3, XLMIMO_ULA>(P, n_blocks, s) : launch_mt2_k<G, 2, 3, XLMIMO_UPA>(P, n_blocks, s);
  else
    return ula ? launch_mt2_k<G, 1, 3, XLMIMO_ULA>(P, n_blocks, s) : launch_mt2_k<G, 1, 3, XLMIMO_UPA>(P, n_blocks, s);
}

// ------------------------------------------------------------------ kernel BLK
// DMMA Gram for 64 < K <= 1024 (NEXT-3 / E1-E3 user counts).  Users in blocks of 64
// (8 fragment planes).  A CTA owns (drop, block pair bi <= bj, element split) and
// computes the 64 x 64 block G[bi][bj] as 64 jobs (ga, gb) of four DMMAs (RR, II,
// RI, IR) per 4-element step, exactly the MT2 arithmetic.  For bi < bj both blocks'
// coefficients are generated per tile (16 planes: A = bi, B = bj); for bi == bj the 8
// planes serve as both operands and the lower-half jobs are computed but not written
// (the diagonal blocks are nb of the nb(nb+1)/2 pairs).  A warp owns one ga and four
// gb: one A fragment load per step feeds four jobs; jobs on padded planes and
// lower-half diagonal jobs skip their DMMAs.  Tiles of 32
// elements are generated into a 3-deep mbarrier ring (as MT2, NBUF = 3).  Level ends
// stage the 64 jobs' accumulators in shared memory and write the block's entries of
// the packed upper triangle [K(K+1)/2] of this (drop, split, level) partial.
constexpr int kBlkU = 64, kBlkG = 8, kBlkNW = 16, kBlkNT = 32 * kBlkNW, kBlkS = 8, kBlkNBUF = 3;
constexpr int kBlkPlane = kBlkS * 2 * kBlkG * 32;  // doubles per (re|im) tile plane set, 16 planes
constexpr size_t kBlkTiles = 2ull * kBlkNBUF * kBlkPlane * sizeof(double);
constexpr size_t kBlkStage = 64ull * 4 * 64 * sizeof(double);
constexpr size_t kBlkSmem = kBlkTiles > kBlkStage ? kBlkTiles : kBlkStage;
static_assert(kBlkSmem <= 220 * 1024, "BLK shared memory");

template <int KIND>
__global__ void __launch_bounds__(kBlkNT, 1) gram_blk_kernel(GramParams P, FastDiv fd, int n_pairs, int nb) {
  extern __shared__ __align__(16) double dsm[];  // tiles [NBUF][re|im][S][16][32]; stage at level ends
  __shared__ double4 su[2 * kBlkU];
  __shared__ __align__(8) uint64_t mb_full[kBlkNBUF], mb_empty[kBlkNBUF];
  constexpr int S = kBlkS, NT = kBlkNT, NW = kBlkNW, PLANE = kBlkPlane, GP = 2 * kBlkG;

  const int64_t bdrop = blockIdx.x / ((int64_t)P.n_split * n_pairs);
  const int rem = (int)(blockIdx.x - bdrop * P.n_split * n_pairs);
  const int pair = rem / P.n_split, split = rem - pair * P.n_split;
  int bi = 0, q0 = pair;
  while (q0 >= nb - bi) { q0 -= nb - bi; ++bi; }
  const int bj = bi + q0;
  const bool diag = bi == bj;
  const int64_t drop = bdrop;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int K = P.K;
  for (int u = tid; u < 2 * kBlkU; u += NT) {
    const int gu = (u < kBlkU ? bi * kBlkU + u : bj * kBlkU + (u - kBlkU));
    if (gu < K) {
      const xl::UserC uc = xl::make_user(P.pos + (drop * K + gu) * 3, KIND, P.sqrt_beta0);
      su[u] = make_double4(uc.xz2, uc.y, uc.z, uc.amp);
    } else {
      su[u] = make_double4(1.0, 0.0, 0.0, 0.0);  // padded user: zero amplitude
    }
  }
  if (tid == 0) {
    for (int i = 0; i < kBlkNBUF; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mt_smem_u32(&mb_full[i])), "r"(NT));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mt_smem_u32(&mb_empty[i])), "r"(NT));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // warp w on sub-partition s = w % 4, j = w / 4: ga = s or 7 - s, gb = 4 (j / 2) + k.
  // Jobs on planes that hold only padded users, and the lower-half jobs of a diagonal
  // block, issue no DMMAs: a warp's active jobs are a contiguous k range [klo, khi)
  // dispatched to a compile-time loop (a predicated-off DMMA would still hold the
  // pipe).  ga in {s, 7 - s} gives every sub-partition 9 of the 36 diagonal jobs.
  const int sp = warp & 3, wj = warp >> 2;
  const int ga = (wj & 1) ? 7 - sp : sp, gb0 = 4 * (wj >> 1);
  const int aoff = ga * 32 + lane;
  const int pa = min(kBlkG, (K - bi * kBlkU + 7) >> 3), pb = min(kBlkG, (K - bj * kBlkU + 7) >> 3);
  int boff[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) boff[k] = ((diag ? 0 : kBlkG) + gb0 + k) * 32 + lane;
  const int klo = (ga >= pa) ? 4 : (diag ? max(0, ga - gb0) : 0);
  const int khi = min(4, pb - gb0);
  const int kcase = (klo < khi) ? klo * 5 + khi : 0;  // 0: no active job
  const int rows = S * (diag ? kBlkG : GP);  // generated 32-lane rows per tile
  __syncthreads();
  const double c4 = 4.0 * P.inv_lambda;
  const bool n_odd = (P.N & 1) != 0;

  const int s0 = (int)min((int64_t)split * P.chunk, P.N);
  const int s1 = (int)min(P.N, (int64_t)s0 + P.chunk);
  const int NP = K * (K + 1) / 2;
  int lv0 = 0;
  uint32_t T = 0;
  for (int l = 0; l < P.n_lvl; ++l) {
    const int lv1 = (int)P.lvl_end[l];
    const int a = max(lv0, s0), b = min(lv1, s1);
    lv0 = lv1;
    double acc[4][4][2];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int m = 0; m < 4; ++m) acc[k][m][0] = acc[k][m][1] = 0.0;
    auto generate = [&](int t0, int buf) {
      double *gre = dsm + buf * (2 * PLANE), *gim = gre + PLANE;
#pragma unroll
      for (int i = 0; i < (S * GP) / NW; ++i) {
        const int row = warp + i * NW;  // row = s * GP + g
        if (row < rows) {
          const int g = diag ? (row % kBlkG) : (row % GP);
          const int st = diag ? (row / kBlkG) : (row / GP);
          const int t = t0 + 4 * st + (lane & 3);
          const bool valid = t < b;
          const ElemPos ep = element_pos32<KIND>(P, valid ? t : a, fd, n_odd);
          const double4 uc = su[8 * g + (lane >> 2)];
          const double dy = ep.y - uc.y;
          double r2 = fma(dy, dy, uc.x);
          if (KIND != XLMIMO_ULA) {
            const double dz = ep.z - uc.z;
            r2 = fma(dz, dz, r2);
          }
          double hr, hi;
          xl::coef_fast(r2, valid ? uc.w : 0.0, c4, hr, hi);
          const int orow = st * GP + g;  // storage row: step-major, 16 planes per step
          gre[orow * 32 + lane] = hr;
          gim[orow * 32 + lane] = hi;
        }
      }
    };
    auto consume_r = [&](auto kl, auto kh, int buf) {
      constexpr int KL = decltype(kl)::value, KH = decltype(kh)::value;
      const double *cre = dsm + buf * (2 * PLANE), *cim = cre + PLANE;
#pragma unroll
      for (int si = 0; si < S; ++si) {
        const int so = si * GP * 32;
        const double ar = cre[so + aoff], ai = cim[so + aoff];
#pragma unroll
        for (int k = KL; k < KH; ++k) {
          const double br = cre[so + boff[k]], bim = cim[so + boff[k]];
          dmma(acc[k][0], ar, br);
          dmma(acc[k][1], ai, bim);
          dmma(acc[k][2], ar, bim);
          dmma(acc[k][3], ai, br);
        }
      }
    };
    using I0 = std::integral_constant<int, 0>;
    using I1 = std::integral_constant<int, 1>;
    using I2 = std::integral_constant<int, 2>;
    using I3 = std::integral_constant<int, 3>;
    using I4 = std::integral_constant<int, 4>;
    auto consume = [&](int buf) {
      switch (kcase) {  // klo * 5 + khi, warp-uniform
        case 4: consume_r(I0{}, I4{}, buf); break;
        case 1: consume_r(I0{}, I1{}, buf); break;
        case 2: consume_r(I0{}, I2{}, buf); break;
        case 3: consume_r(I0{}, I3{}, buf); break;
        case 7: consume_r(I1{}, I2{}, buf); break;
        case 8: consume_r(I1{}, I3{}, buf); break;
        case 9: consume_r(I1{}, I4{}, buf); break;
        case 13: consume_r(I2{}, I3{}, buf); break;
        case 14: consume_r(I2{}, I4{}, buf); break;
        case 19: consume_r(I3{}, I4{}, buf); break;
        default: break;
      }
    };
    const int n = b > a ? (b - a + 4 * S - 1) / (4 * S) : 0;
    auto produce = [&](int i) {
      const uint32_t tt = T + i;
      const int bb = (int)(tt % kBlkNBUF);
      if (tt >= kBlkNBUF) mt_wait(&mb_empty[bb], (tt / kBlkNBUF - 1) & 1);
      generate(a + i * 4 * S, bb);
      mt_arrive(&mb_full[bb]);
    };
#pragma unroll
    for (int i = 0; i < kBlkNBUF - 1; ++i)
      if (i < n) produce(i);
    for (int i = 0; i < n; ++i) {
      if (i + kBlkNBUF - 1 < n) produce(i + kBlkNBUF - 1);
      const uint32_t tt = T + i;
      const int bb = (int)(tt % kBlkNBUF);
      mt_wait(&mb_full[bb], (tt / kBlkNBUF) & 1);
      consume(bb);
      mt_arrive(&mb_empty[bb]);
    }
    T += n;
    __syncthreads();  // every warp's DMMAs done before the stage aliases the tiles
    // stage [job q = ga*8 + gb][m][8][8] (C fragment: row lane/4, cols 2(lane%4) + {0,1})
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int q = ga * kBlkG + gb0 + k;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        double *st = dsm + (q * 4 + m) * 64 + (lane >> 2) * 8 + 2 * (lane & 3);
        st[0] = acc[k][m][0];
        st[1] = acc[k][m][1];
      }
    }
    __syncthreads();
    double *out = P.ws + (((size_t)drop * P.n_split + split) * P.n_lvl + l) * (size_t)(2 * NP);
    for (int e = tid; e < kBlkU * kBlkU; e += NT) {
      const int ua = e >> 6, ub = e & 63;
      const int i = bi * kBlkU + ua, j = bj * kBlkU + ub;
      if (i >= K || j >= K || (diag && ub < ua)) continue;
      const int q = (ua >> 3) * kBlkG + (ub >> 3), f = (ua & 7) * 8 + (ub & 7);
      const double *st = dsm + q * 4 * 64 + f;
      const double re = st[0] + st[64];
      const double im = st[128] - st[192];
      const int64_t p = (int64_t)i * K - (int64_t)i * (i - 1) / 2 + (j - i);
      out[2 * p] = re;
      out[2 * p + 1] = (i == j) ? 0.0 : im;
    }
    __syncthreads();
  }
}

// Row-wise reduce for large K: block (drop, row i), threads over j >= i; sums splits in
// fixed order per level, prefix over levels, Hermitian mirror, Im diag = 0.
__global__ void __launch_bounds__(256) gram_reduce_rows_kernel(const double *ws, int K, int n_split, int n_lvl,
                                                               double *out) {
  const int64_t drop = blockIdx.x / K;
  const int i = (int)(blockIdx.x - drop * K);
  const int64_t NP = (int64_t)K * (K + 1) / 2;
  const int64_t base = (int64_t)i * K - (int64_t)i * (i - 1) / 2 - i;
  for (int j = i + threadIdx.x; j < K; j += blockDim.x) {
    const int64_t p = base + j;
    double re = 0.0, im = 0.0;
    for (int l = 0; l < n_lvl; ++l) {
      for (int s = 0; s < n_split; ++s) {
        const double *w = ws + (((size_t)drop * n_split + s) * n_lvl + l) * (size_t)(2 * NP) + 2 * p;
        re += w[0];
        im += w[1];
      }
      double *g = out + ((size_t)drop * n_lvl + l) * (size_t)K * K * 2;
      g[((size_t)i * K + j) * 2] = re;
      g[((size_t)i * K + j) * 2 + 1] = (i == j) ? 0.0 : im;
      g[((size_t)j * K + i) * 2] = re;
      g[((size_t)j * K + i) * 2 + 1] = (i == j) ? 0.0 : -im;
    }
  }
}

// ------------------------------------------------------------------ kernel B
template <int KP>
struct TiledCfg {
  static constexpr int NB = KP / 4;
  static constexpr int NBP = NB * (NB + 1) / 2;
  // smallest power-of-two group count with NBP * G >= 256 (G <= 32 lanes of one warp)
  static constexpr int G = (NBP >= 256) ? 1 : (NBP * 2 >= 256) ? 2 : (NBP * 4 >= 256) ? 4 : (NBP * 8 >= 256) ? 8 : (NBP * 16 >= 256) ? 16 : 32;
  static constexpr int NTASK = NBP * G;
  static constexpr int NT = (NTASK + 31) / 32 * 32;
  static constexpr int T = 32;  // elements per tile
};

template <typename CT>
struct Cplx;
template <>
struct Cplx<double> { using T2 = double2; };
template <>
struct Cplx<float> { using T2 = float2; };

template <int KP, bool FP32, bool FROM_H = false>
__global__ void __launch_bounds__(TiledCfg<KP>::NT, 1) gram_tiled_kernel(GramParams P) {
  using Cfg = TiledCfg<KP>;
  using RT = typename std::conditional<FP32, float, double>::type;
  using RT2 = typename Cplx<RT>::T2;
  constexpr int T = Cfg::T, G = Cfg::G, NT = Cfg::NT, EPT = T / G;
  __shared__ xl::UserC su[KP];
  __shared__ RT2 hs[T][KP];

  const int64_t bdrop = blockIdx.x / P.n_split;
  const int split = blockIdx.x - (int)(bdrop * P.n_split);
  const int64_t drop = P.h_drop0 + bdrop;
  const int tid = threadIdx.x;
  const int K = P.K;
  if (tid < KP) {
    if (tid < K) su[tid] = xl::make_user(P.pos + (drop * K + tid) * 3, P.kind, P.sqrt_beta0);
    else su[tid] = xl::UserC{1.0, 0.0, 0.0, 0.0};  // padded user: zero amplitude
  }
  // task -> (block pair I <= J, group g)
  const bool active = tid < Cfg::NTASK;
  const int bp = tid / G, g = tid - (tid / G) * G;
  int I = 0, J = 0;
  {
    int rem = bp;
    while (rem >= Cfg::NB - I) { rem -= Cfg::NB - I; ++I; }
    J = I + rem;
    if (!active) { I = 0; J = 0; }
  }
  __syncthreads();

  const int64_t s0 = (int64_t)split * P.chunk;
  const int64_t s1 = min(P.N, s0 + P.chunk);
  int64_t lv0 = 0;
  for (int l = 0; l < P.n_lvl; ++l) {
    const int64_t lv1 = P.lvl_end[l];
    const int64_t a = max(lv0, s0), b = min(lv1, s1);
    lv0 = lv1;
    double acc[4][4][2];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
    for (int64_t t0 = a; t0 < b; t0 += T) {
      if (FROM_H) {
        // materialised planar fp32 H[drop][K][2][N]: coalesced along elements
        const float *Hd = P.hmat + (size_t)(drop - P.h_drop0) * K * 2 * P.N;
        for (int c = tid; c < T * KP; c += NT) {
          const int row = c / T, e = c - (c / T) * T;
          const int64_t t = t0 + e;
          RT2 h;
          h.x = 0; h.y = 0;
          if (t < b && row < K) {
            h.x = __ldcs(Hd + ((size_t)row * 2) * P.N + t);
            h.y = __ldcs(Hd + ((size_t)row * 2 + 1) * P.N + t);
          }
          hs[e][row] = h;
        }
      }
      // generation: T x KP coefficients, element-major interleaved complex
      for (int c = tid; c < (FROM_H ? 0 : T * KP); c += NT) {
        const int e = c / KP, row = c - (c / KP) * KP;
        const int64_t t = t0 + e;
        RT2 h;
        h.x = 0; h.y = 0;
        if (t < b) {
          const ElemPos ep = element_pos(P, t);
          const xl::UserC u = su[row];
          const double r2 = dist2(u, ep, P.kind);
          if (FP32) {
            float fr, fi;
            xl::coef_from_r2_f32(r2, u.amp, P.inv_lambda, fr, fi);
            h.x = fr; h.y = fi;
          } else {
            double dr, di;
            xl::coef_fast(r2, u.amp, 4.0 * P.inv_lambda, dr, di);
            h.x = (RT)dr; h.y = (RT)di;
          }
        }
        hs[e][row] = h;
      }
      __syncthreads();
      if (active) {
        RT tacc[4][4][2];
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) tacc[x][y][0] = tacc[x][y][1] = 0;
#pragma unroll 4
        for (int ee = 0; ee < EPT; ++ee) {
          const int e = g + ee * G;
          RT2 hiv[4], hjv[4];
#pragma unroll
          for (int x = 0; x < 4; ++x) hiv[x] = hs[e][4 * I + x];
#pragma unroll
          for (int y = 0; y < 4; ++y) hjv[y] = hs[e][4 * J + y];
#pragma unroll
          for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) {
              tacc[x][y][0] = fma(hiv[x].x, hjv[y].x, fma(hiv[x].y, hjv[y].y, tacc[x][y][0]));
              tacc[x][y][1] = fma(hiv[x].x, hjv[y].y, fma(-hiv[x].y, hjv[y].x, tacc[x][y][1]));
            }
        }
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) {
            acc[x][y][0] += (double)tacc[x][y][0];
            acc[x][y][1] += (double)tacc[x][y][1];
          }
      }
      __syncthreads();
    }
    // reduce over the G lanes of each block pair (contiguous, inside one warp)
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          double v = acc[x][y][c];
#pragma unroll
          for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, G > 1 ? G : 1);
          acc[x][y][c] = v;
        }
    if (active && g == 0) {
      double *out = P.ws + (((size_t)drop * P.n_split + split) * P.n_lvl + l) * (size_t)(K * (K + 1));
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) {
          const int i = 4 * I + x, j = 4 * J + y;
          if (i <= j && j < K) {
            const int p = i * K - i * (i - 1) / 2 + (j - i);
            out[2 * p] = acc[x][y][0];
            out[2 * p + 1] = acc[x][y][1];
          }
        }
    }
  }
}

// ------------------------------------------------------------------ reduce
// ws layout [drop][split][lvl][part][NP][2]; sums (split, part) in fixed order per
// level and accumulates across levels (nested-N prefix sums).
__global__ void __launch_bounds__(256) gram_reduce_kernel(const double *ws, int K, int64_t n_drops, int n_split,
                                                          int n_lvl, int n_part, double *out) {
  const int NP = K * (K + 1) / 2;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n_drops * NP) return;
  const int64_t drop = idx / NP;
  const int p = (int)(idx - drop * NP);
  int i = 0, rem = p;
  while (rem >= K - i) { rem -= K - i; ++i; }
  const int j = i + rem;
  double re = 0.0, im = 0.0;
  for (int l = 0; l < n_lvl; ++l) {
    for (int s = 0; s < n_split; ++s) {
      const double *w = ws + ((((size_t)drop * n_split + s) * n_lvl + l) * n_part) * (size_t)(2 * NP) + 2 * p;
      for (int q = 0; q < n_part; ++q) {
        re += w[(size_t)q * 2 * NP];
        im += w[(size_t)q * 2 * NP + 1];
      }
    }
    double *g = out + ((size_t)drop * n_lvl + l) * (size_t)K * K * 2;
    g[(i * K + j) * 2] = re;
    g[(i * K + j) * 2 + 1] = (i == j) ? 0.0 : im;
    g[(j * K + i) * 2] = re;
    g[(j * K + i) * 2 + 1] = (i == j) ? 0.0 : -im;
  }
}

int choose_split(int64_t n_drops, int64_t N) {
  const int64_t target_blocks = 148 * 8;
  int64_t s = (target_blocks + n_drops - 1) / (n_drops > 0 ? n_drops : 1);
  const int64_t max_s = N / 4096 > 1 ? N / 4096 : 1;
  if (s > max_s) s = max_s;
  if (s < 1) s = 1;
  return (int)s;
}

// BLK kernel (K > 64): one CTA per SM (192 KB of tiles), so aim for >= 2 waves of
// (drop, block pair, split) CTAs; splits keep >= 4096 elements each.
int blk_pairs(int K) {
  const int nb = (K + kBlkU - 1) / kBlkU;
  return nb * (nb + 1) / 2;
}
// K > 64, fp64: the chunked DMMA SYRK (xl_gram_syrk.cu) above 128 users, the
// block-pair kernel below it; XLMIMO_OPT_LARGE_K = 1 (blocks) | 2 (SYRK) overrides.
// measured (35 000 elements, 1000 drops, after the SYRK's 3M form): K = 121 blk 118.1 vs SYRK
// 115.2 ms, K = 128 118.1 vs 115.9 (tools/time_k128.py); MT2 takes K <= 120 (65.6 ms at 120)
constexpr int kSyrkMinK = 121;
// K > 64, fp32: block pairs fed by TMA from materialised, L2-sized chunks of H from
// kStreamPairMinK users on (generation once per coefficient instead of once per pair),
// generated in-kernel below; XLMIMO_OPT_PAIR = 1 (gen) | 2 (stream) overrides.
constexpr int kStreamPairMinK = 129;  // and above kFusedTcMaxK (256): the fused launches win below  // fp16 chunks win from K = 65 (35 000 elements: K = 100 11.7 vs 13.5 ms, 160 9.2 vs
                                      // 14.8, 352 7.7 vs 16.8); up to 128 the in-kernel path stays, its TMEM folding
                                      // keeping E1/E2's K = 100 rates unbiased (R28)
bool use_stream_pair(int K) {
  const int64_t o = xlh::option(XLMIMO_OPT_PAIR);
  if (o == 1) return false;
  if (o == 2) return true;
  return K >= kStreamPairMinK && K > xlh::kFusedTcMaxK;
}
// 64 < K <= 128 fp32: the fused kernel's wide + narrow launches (xl_stream_tc.cu) unless
// XLMIMO_OPT_PAIR = 1 (the block-pair kernel) or 2 (the pair stream) / MATERIALIZED
bool use_fused_wide(const xlh::ArrayP &a, int K, int mode) {
  return !use_stream_pair(K) && mode != XLMIMO_MATERIALIZED && xlh::option(XLMIMO_OPT_PAIR) != 1 &&
         xlh::fused_tc_wide_supported(a, K);
}
bool use_gram_syrk(int K) {
  const int64_t o = xlh::option(XLMIMO_OPT_LARGE_K);
  if (o == 1) return false;
  if (o == 2) return true;
  return K >= kSyrkMinK;
}
int choose_split_blk(int64_t n_drops, int K, int64_t N) {
  const int64_t target = 148 * 2, have = n_drops * blk_pairs(K);
  int64_t s = (target + have - 1) / (have > 0 ? have : 1);
  const int64_t max_s = N / 4096 > 1 ? N / 4096 : 1;
  if (s > max_s) s = max_s;
  if (s < 1) s = 1;
  return (int)s;
}

template <int KT, bool FP32>
void launch_small(const GramParams &P, int64_t n_blocks, cudaStream_t s) {
  gram_small_kernel<KT, 256, FP32><<<(unsigned)n_blocks, 256, 0, s>>>(P);
}

template <bool FP32>
void launch_small_k(int K, const GramParams &P, int64_t n_blocks, cudaStream_t s) {
  switch (K) {
    case 1: launch_small<1, FP32>(P, n_blocks, s); break;
    case 2: launch_small<2, FP32>(P, n_blocks, s); break;
    case 3: launch_small<3, FP32>(P, n_blocks, s); break;
    case 4: launch_small<4, FP32>(P, n_blocks, s); break;
    case 5: launch_small<5, FP32>(P, n_blocks, s); break;
    case 6: launch_small<6, FP32>(P, n_blocks, s); break;
    case 7: launch_small<7, FP32>(P, n_blocks, s); break;
    default: launch_small<8, FP32>(P, n_blocks, s); break;
  }
}

template <int KP, bool FP32>
void launch_tiled(const GramParams &P, int64_t n_blocks, cudaStream_t s) {
  gram_tiled_kernel<KP, FP32><<<(unsigned)n_blocks, TiledCfg<KP>::NT, 0, s>>>(P);
}

template <bool FP32>
void launch_tiled_k(int K, const GramParams &P, int64_t n_blocks, cudaStream_t s) {
  if (K <= 16) launch_tiled<16, FP32>(P, n_blocks, s);
  else if (K <= 32) launch_tiled<32, FP32>(P, n_blocks, s);
  else if (K <= 48) launch_tiled<48, FP32>(P, n_blocks, s);
  else launch_tiled<64, FP32>(P, n_blocks, s);
}

}  // namespace

namespace xlh {

// Which kernel runs, and how many partials per (drop, split, level) it writes.
// Block shapes of the DMMA kernel (XLMIMO_OPT_DMMA_VARIANT selects for tuning):
//   G = 1: 0 -> 256 thr x 4 blocks/SM (<= 64 regs), 1 -> 256 x 6 (<= 40), 2 -> 128 x 8, 3 -> 256 x 2
//   G = 2: 0 -> 256 x 2, 1 -> 256 x 3, 2 -> 128 x 4, 3 -> 256 x 2
int mma_variant() {
  const int64_t v = option(XLMIMO_OPT_DMMA_VARIANT);
  return (v >= 0 && v <= 3) ? (int)v : 0;
}
int mma_nt(int G) { return (mma_variant() == 2) ? 128 : 256; }

struct KernelChoice {
  int which;      // 0 = small/tiled (kernel A / B), 1 = split (A2), 2 = DMMA (M)
  int nt;         // threads per block
  int parts;      // partials per (drop, split, level)
};

// XLMIMO_OPT_GRAM_KERNEL = 1 split | 2 DMMA | 3 CUDA-core overrides the default (tuning /
// A-B tests); XLMIMO_OPT_SPLIT_NT selects the split kernel's block variant.
KernelChoice choose_kernel(const ArrayP &a, int K, int precision) {
  const int64_t env_k = option(XLMIMO_OPT_GRAM_KERNEL);
  const int64_t env_nt = option(XLMIMO_OPT_SPLIT_NT);
  KernelChoice c;
  const bool fp64 = precision == XLMIMO_FP64;
  const bool split_ok = fp64 && a.kind == XLMIMO_ULA && (K == 8 || K == 4);
  const bool mma_ok = fp64 && K <= 16;
  // measured on B200 (cfg2, K = 8): split 20.4 ms < DMMA 23.6 ms < register kernel A 37.7 ms
  c.which = split_ok ? 1 : mma_ok ? 2 : fp64 ? 3 : 0;
  if (env_k == 1 && split_ok) c.which = 1;
  if (env_k == 2 && mma_ok) c.which = 2;
  if (env_k == 3) c.which = 0;
  // split variants (XLMIMO_OPT_SPLIT_NT selects; "nt" is a variant id, threads in kSplitThreads)
  // split default: variant 192 = 128 threads x 3 blocks/SM, two elements per iteration
  // (19.45 ms vs 19.77 for 256 x 2 on cfg2, B200)
  c.nt = (c.which == 1 && K == 8) ? 192 : 256;
  if (c.which == 1 && (env_nt == 64 || env_nt == 128 || env_nt == 192 || env_nt == 256)) c.nt = (int)env_nt;
  if (c.which == 2) c.nt = mma_nt(K <= 8 ? 1 : 2);
  const int threads = (c.which == 1 && (c.nt == 64)) ? 256 : (c.which == 1 && c.nt == 192) ? 128 : c.nt;
  c.parts = c.which == 2 ? threads / 32 : 1;  // the split kernel reduces its warps in the block
  return c;
}

template <int G, int KIND>
void launch_mma(const GramParams &P, int64_t n_blocks, cudaStream_t s) {
  const int v = mma_variant();
  if constexpr (G == 1) {
    switch (v) {
      case 1: gram_mma_kernel<G, 256, 6, KIND><<<(unsigned)n_blocks, 256, 0, s>>>(P); break;
      case 2: gram_mma_kernel<G, 128, 8, KIND><<<(unsigned)n_blocks, 128, 0, s>>>(P); break;
      case 3: gram_mma_kernel<G, 256, 2, KIND><<<(unsigned)n_blocks, 256, 0, s>>>(P); break;
      default: gram_mma_kernel<G, 256, 4, KIND><<<(unsigned)n_blocks, 256, 0, s>>>(P); break;
    }
  } else {
    switch (v) {
      case 1: gram_mma_kernel<G, 256, 3, KIND><<<(unsigned)n_blocks, 256, 0, s>>>(P); break;
      case 2: gram_mma_kernel<G, 128, 4, KIND><<<(unsigned)n_blocks, 128, 0, s>>>(P); break;
      default: gram_mma_kernel<G, 256, 2, KIND><<<(unsigned)n_blocks, 256, 0, s>>>(P); break;
    }
  }
}

// Materialised streaming on tcgen05 (TF32, RNA-pre-rounded H) unless disabled by
// XLMIMO_OPT_STREAM = 1 (CUDA-core fp32 tiled kernel, also the fallback for shapes
// the TMA path does not take: K < 9, N % 4 != 0).
// The tensor-core fp32 paths round each coefficient to TF32 (RNA, 2^-11 relative): a
// Gram entry's normalised error is ~5.6e-4 / sqrt(N) (per-product errors average over
// the N elements), inside the fp32-tier 1e-4 for all K^2 entries only from N ~ 1000 on
// (measured 8.8e-4 at N = 1, 1.7e-4 at N = 33).  Below kTcMinN the CUDA-core fp32
// kernels (or, for K > 64, the fp64 DMMA kernel) run instead.
constexpr int64_t kTcMinN = 1024;

bool materialised_use_tc(int K, int64_t N) {
  if (option(XLMIMO_OPT_STREAM) == 1) return false;
  return N >= kTcMinN && stream_tc_supported(K, N);
}

// Materialised mode: drops per batch so that the planar complex64 H of a batch
// fits an 8 GiB slice of the workspace (cfg5: 16 drops of 512 MiB; cfg3: 4096), so
// one persistent streaming launch has >= ~14 waves of work items.
// fused fp32 exact Gram on tcgen05 (generate -> TF32 smem tiles -> TMEM), single level only
bool use_fused_tc(const ArrayP &a, int K, int precision, int n_lvl) {
  if (option(XLMIMO_OPT_GRAM_KERNEL) == 3) return false;
  const int64_t N = a.kind == XLMIMO_ULA ? a.n_y : a.n_y * a.n_z;
  return precision == XLMIMO_FP32 && n_lvl == 1 && N >= kTcMinN && fused_tc_supported(a, K);
}

// elements per drop as stored: the tiled32 (tcgen05) layout pads N to whole groups of 4 tiles
int64_t mat_npad(int K, int64_t N) { return materialised_use_tc(K, N) ? (N + 127) / 128 * 128 : N; }

int64_t materialised_batch(int64_t N, int K, int64_t n_drops) {
  const int64_t per = mat_npad(K, N) * K * 2 * (int64_t)sizeof(float);
  int64_t b = ((int64_t)8 << 30) / (per > 0 ? per : 1);
  if (b < 1) b = 1;
  return b < n_drops ? b : n_drops;
}

// warp-per-drop kernel W: small single-level fp64 arrays in large batches (XLMIMO_OPT_GRAM_KERNEL
// = 5 forces it where it applies, 1..4 keep the other kernels)
bool use_warp_kernel(const ArrayP &a, int K, int64_t n_drops, int n_lvl, int precision, int mode) {
  const int64_t N = a.kind == XLMIMO_ULA ? a.n_y : a.n_y * a.n_z;
  const int64_t o = option(XLMIMO_OPT_GRAM_KERNEL);
  const bool fits = precision == XLMIMO_FP64 && mode == XLMIMO_FUSED && n_lvl == 1 && K <= 5 && N <= kWarpMaxN;
  if (!fits) return false;
  if (o == 5) return true;
  return o == 0 && n_drops >= kWarpMinDrops;
}

// fp64 fused Gram for 64 < K <= 128 on the MT2 kernel (3M DMMA stars) unless
// XLMIMO_OPT_LARGE_K picks the block-pair (1) or SYRK (2) kernel
constexpr int kMt2MaxK = 128;  // G <= 16 (G = 16 as two launches of 16 stars of 5 or 4)
bool use_mt2_large(const ArrayP &a, int K, int precision, int mode) {
  const int64_t N = a.kind == XLMIMO_ULA ? a.n_y : a.n_y * a.n_z;
  const int64_t o = option(XLMIMO_OPT_LARGE_K), gk = option(XLMIMO_OPT_GRAM_KERNEL);
  return K > xl::kMaxK && K <= kMt2MaxK && precision == XLMIMO_FP64 && mode == XLMIMO_FUSED &&
         N < ((int64_t)1 << 31) && o != 1 && o != 2 && gk != 3 && gk != 4;
}

size_t gram_ws_bytes(const ArrayP &a, int K, int64_t n_drops, int n_lvl, int precision, int mode) {
  const int64_t N = a.kind == XLMIMO_ULA ? a.n_y : a.n_y * a.n_z;
  if (use_warp_kernel(a, K, n_drops, n_lvl, precision, mode)) return 0;
  const int n_split = choose_split(n_drops, N);
  const size_t np = (size_t)K * (K + 1) / 2;
  if (K > xl::kMaxK && !use_mt2_large(a, K, precision, mode)) {
    if (precision == XLMIMO_FP32 && N >= kTcMinN) {  // tcgen05 block pairs (+ H chunks when streamed)
      if (use_fused_wide(a, K, mode)) return (size_t)n_drops * fused_tc_chunks(N, n_drops) * np * 2 * sizeof(double);
      const size_t part = ((size_t)n_drops * fused_tc_pair_chunks(N) * np * 2 * sizeof(double) + 255) / 256 * 256;
      const bool stream = use_stream_pair(K) || mode == XLMIMO_MATERIALIZED;
      return part + (stream && n_drops > 0 ? stream_pair_h_bytes(K, n_drops, N) : 0);
    }
    if (use_gram_syrk(K)) return gram_syrk_ws_bytes(K, n_drops, n_lvl);
    return (size_t)n_drops * choose_split_blk(n_drops, K, N) * n_lvl * np * 2 * sizeof(double);
  }
  if (mode == XLMIMO_MATERIALIZED) {
    const int parts = materialised_use_tc(K, N) ? stream_tc_chunks(N) * stream_tc_parts(K) : n_split;
    const size_t part = ((size_t)n_drops * parts * n_lvl * np * 2 * sizeof(double) + 255) / 256 * 256;
    return part + (size_t)materialised_batch(N, K, n_drops) * mat_npad(K, N) * K * 2 * sizeof(float);
  }
  if (use_fused_tc(a, K, precision, n_lvl))
    return (size_t)n_drops * fused_tc_chunks(N, n_drops) * stream_tc_parts(K) * np * 2 * sizeof(double);
  const KernelChoice kc = choose_kernel(a, K, precision);
  return (size_t)n_drops * n_split * n_lvl * kc.parts * np * 2 * sizeof(double);
}

template <int KP>
void launch_tiled_from_h(const GramParams &P, int64_t n_blocks, cudaStream_t s) {
  gram_tiled_kernel<KP, true, true><<<(unsigned)n_blocks, TiledCfg<KP>::NT, 0, s>>>(P);
}

// XLMIMO_MATERIALIZED (fp32 only): per batch of drops, K4a writes H to HBM and the
// streaming kernel reads it back; partials reduced in fp64 as in the fused path.
int launch_materialised(const ArrayP &a, const double *pos, int K, int64_t n_drops, int64_t N, double *out,
                        void *ws, size_t ws_bytes, cudaStream_t s) {
  const size_t need = gram_ws_bytes(a, K, n_drops, 1, XLMIMO_FP32, XLMIMO_MATERIALIZED);
  if (ws_bytes < need || !ws) return set_error(XLMIMO_EWORKSPACE, "gram: workspace %zu < %zu bytes", ws_bytes, need);
  GramParams P;
  memset(&P, 0, sizeof(P));
  P.pos = pos;
  P.ws = (double *)ws;
  P.K = K;
  P.kind = a.kind;
  P.n_y = a.n_y;
  P.n_z = a.kind == XLMIMO_ULA ? 1 : a.n_z;
  P.N = N;
  P.n_split = choose_split(n_drops, N);
  P.chunk = ((N + P.n_split - 1) / P.n_split + 255) / 256 * 256;
  P.n_lvl = 1;
  for (int l = 0; l < kMaxLvl; ++l) P.lvl_end[l] = N;
  P.inv_lambda = 1.0 / a.lambda;
  P.pitch = a.pitch;
  P.sqrt_beta0 = a.sqrt_beta0;
  const size_t np = (size_t)K * (K + 1) / 2;
  const bool tc = materialised_use_tc(K, N);
  const int parts = tc ? stream_tc_chunks(N) : P.n_split;
  const int subparts = tc ? stream_tc_parts(K) : 1;
  const size_t part = ((size_t)n_drops * parts * subparts * np * 2 * sizeof(double) + 255) / 256 * 256;
  float *H = (float *)((char *)ws + part);
  P.hmat = H;
  const int64_t B = materialised_batch(N, K, n_drops);
  for (int64_t d0 = 0; d0 < n_drops; d0 += B) {
    const int nb = (int)(d0 + B <= n_drops ? B : n_drops - d0);
    P.h_drop0 = d0;
    const int64_t n_pad = mat_npad(K, N);
    {
      KTimer tm(s, "h_materialise");
      if (tc && materialise_tc_supported(a)) {  // anchor + fp32-delta generator, TF32 tiles
        const int rc = launch_h_materialise_tc(a, pos, K, N, n_pad, d0, nb, H, s);
        if (rc) return rc;
      } else {
        h_materialise_kernel<<<dim3((unsigned)((n_pad + 255) / 256), (unsigned)nb), 256, 0, s>>>(P, H, n_pad,
                                                                                               tc ? 1 : 0, tc ? 1 : 0);
      }
      tm.stop(s);
      count_launch();
    }
    int rc;
    if (tc) {
      KTimer tm(s, "gram_stream_tc_tf32");
      rc = launch_stream_tc(H, K, n_pad, d0, nb, (double *)ws, s);
      tm.stop(s);
      count_launch();
    } else {
      KTimer tm(s, "gram_stream_fp32");
      const int64_t n_blocks = (int64_t)nb * P.n_split;
      if (K <= 16) launch_tiled_from_h<16>(P, n_blocks, s);
      else if (K <= 32) launch_tiled_from_h<32>(P, n_blocks, s);
      else if (K <= 48) launch_tiled_from_h<48>(P, n_blocks, s);
      else launch_tiled_from_h<64>(P, n_blocks, s);
      tm.stop(s);
      count_launch();
      rc = check_launch("materialised gram");
    }
    if (rc) return rc;
  }
  const int64_t n_items = n_drops * (int64_t)np;
  KTimer tr(s, "gram_reduce");
  gram_reduce_kernel<<<(unsigned)((n_items + 255) / 256), 256, 0, s>>>((const double *)ws, K, n_drops, parts, 1,
                                                                      subparts, out);
  tr.stop(s);
  count_launch();
  return check_launch("gram_reduce_kernel");
}

// K > 64: block-pair DMMA kernel (fp64, fused), then the row-wise reduce.
int launch_gram_blk(const ArrayP &a, const double *pos, int K, int64_t n_drops, const int64_t *lvl_end, int n_lvl,
                    double *out, void *ws, size_t ws_bytes, cudaStream_t s) {
  const int64_t N = lvl_end[n_lvl - 1];
  if (N >= ((int64_t)1 << 31)) return set_error(XLMIMO_EUNSUPPORTED, "gram_exact: K > 64 needs N < 2^31");
  const size_t need = gram_ws_bytes(a, K, n_drops, n_lvl, XLMIMO_FP64, XLMIMO_FUSED);
  if (ws_bytes < need || !ws) return set_error(XLMIMO_EWORKSPACE, "gram: workspace %zu < %zu bytes", ws_bytes, need);
  GramParams P;
  memset(&P, 0, sizeof(P));
  P.pos = pos;
  P.ws = (double *)ws;
  P.K = K;
  P.kind = a.kind;
  P.n_y = a.n_y;
  P.n_z = a.kind == XLMIMO_ULA ? 1 : a.n_z;
  P.N = N;
  P.n_split = choose_split_blk(n_drops, K, N);
  P.chunk = ((N + P.n_split - 1) / P.n_split + 255) / 256 * 256;
  P.n_lvl = n_lvl;
  for (int l = 0; l < kMaxLvl; ++l) P.lvl_end[l] = l < n_lvl ? lvl_end[l] : N;
  P.inv_lambda = 1.0 / a.lambda;
  P.pitch = a.pitch;
  P.sqrt_beta0 = a.sqrt_beta0;
  const int nb = (K + kBlkU - 1) / kBlkU, n_pairs = blk_pairs(K);
  const int64_t n_blocks = n_drops * n_pairs * P.n_split;
  const FastDiv fd = make_fastdiv((uint32_t)P.n_y);
  {
    KTimer tm(s, "gram_fused_dmma_blk_fp64");
    if (a.kind == XLMIMO_ULA) {
      cudaFuncSetAttribute(gram_blk_kernel<XLMIMO_ULA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBlkSmem);
      gram_blk_kernel<XLMIMO_ULA><<<(unsigned)n_blocks, kBlkNT, kBlkSmem, s>>>(P, fd, n_pairs, nb);
    } else {
      cudaFuncSetAttribute(gram_blk_kernel<XLMIMO_UPA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBlkSmem);
      gram_blk_kernel<XLMIMO_UPA><<<(unsigned)n_blocks, kBlkNT, kBlkSmem, s>>>(P, fd, n_pairs, nb);
    }
    tm.stop(s);
    count_launch();
  }
  int rc = check_launch("gram_blk_kernel");
  if (rc) return rc;
  KTimer tr(s, "gram_reduce");
  gram_reduce_rows_kernel<<<(unsigned)(n_drops * K), 256, 0, s>>>((const double *)ws, K, P.n_split, n_lvl, out);
  tr.stop(s);
  count_launch();
  return check_launch("gram_reduce_rows_kernel");
}

int launch_gram_exact(const ArrayP &a, const double *pos, int K, int64_t n_drops, const int64_t *lvl_end,
                      int n_lvl, int precision, int mode, double *out, void *ws, size_t ws_bytes,
                      cudaStream_t s) {
  if (K > xl::kMaxK && !use_mt2_large(a, K, precision, mode)) {
    // materialised for K > 64 = the TMA-fed pair stream over complex64 (TF32) chunks of H
    if (mode == XLMIMO_MATERIALIZED && precision != XLMIMO_FP32)
      return set_error(XLMIMO_EUNSUPPORTED, "gram_exact: XLMIMO_MATERIALIZED is complex64 (XLMIMO_FP32) only");
    if (n_lvl < 1 || n_lvl > kMaxLvl) return set_error(XLMIMO_EINVAL, "gram: n_lvl=%d out of [1,%d]", n_lvl, kMaxLvl);
    if (precision == XLMIMO_FP32 && lvl_end[n_lvl - 1] >= kTcMinN) {
      if (n_lvl != 1 || !fused_tc_supported_geometry(a))
        return set_error(XLMIMO_EUNSUPPORTED, "gram_exact: K=%d fp32 needs one level and a ULA or a UPA with "
                                              "rows a multiple of 8", K);
      if (n_drops == 0) return XLMIMO_OK;
      const int64_t N = lvl_end[0];
      const size_t need = gram_ws_bytes(a, K, n_drops, 1, precision, mode);
      if (ws_bytes < need || !ws) return set_error(XLMIMO_EWORKSPACE, "gram: workspace %zu < %zu bytes", ws_bytes, need);
      int rc;
      const bool wide = use_fused_wide(a, K, mode);
      if (wide) {
        KTimer tm(s, "gram_fused_tc_f16");
        rc = launch_fused_tc(a, pos, K, n_drops, N, (double *)ws, s);
        tm.stop(s);
        count_launch(fused_tc_launches(K));
      } else if (use_stream_pair(K) || mode == XLMIMO_MATERIALIZED) {  // times and counts its own launches
        const size_t part =
            ((size_t)n_drops * fused_tc_pair_chunks(N) * ((size_t)K * (K + 1) / 2) * 2 * sizeof(double) + 255) /
            256 * 256;
        rc = launch_stream_tc_pair(a, pos, K, n_drops, N, (double *)ws, (float *)((char *)ws + part), s);
      } else {
        KTimer tm(s, "gram_fused_tc_pair_tf32");
        rc = launch_fused_tc_pair(a, pos, K, n_drops, N, (double *)ws, s);
        tm.stop(s);
        count_launch();
      }
      if (rc) return rc;
      KTimer tr(s, "gram_reduce");
      gram_reduce_rows_kernel<<<(unsigned)(n_drops * K), 256, 0, s>>>(
          (const double *)ws, K, wide ? fused_tc_chunks(N, n_drops) : fused_tc_pair_chunks(N), 1, out);
      tr.stop(s);
      count_launch();
      return check_launch("gram_reduce_rows_kernel");
    }
    if (n_drops == 0) return XLMIMO_OK;
    if (use_gram_syrk(K)) return launch_gram_syrk(a, pos, K, n_drops, lvl_end, n_lvl, out, ws, ws_bytes, s);
    return launch_gram_blk(a, pos, K, n_drops, lvl_end, n_lvl, out, ws, ws_bytes, s);
  }
  if (mode == XLMIMO_MATERIALIZED) {
    if (precision != XLMIMO_FP32)
      return set_error(XLMIMO_EUNSUPPORTED, "gram_exact: XLMIMO_MATERIALIZED is complex64 (XLMIMO_FP32) only");
    if (n_lvl != 1) return set_error(XLMIMO_EUNSUPPORTED, "gram_exact: materialised mode has no nested levels");
    if (n_drops == 0) return XLMIMO_OK;
    return launch_materialised(a, pos, K, n_drops, lvl_end[0], out, ws, ws_bytes, s);
  }
  if (mode != XLMIMO_FUSED) return set_error(XLMIMO_EINVAL, "gram_exact: mode");
  if (n_lvl < 1 || n_lvl > kMaxLvl) return set_error(XLMIMO_EINVAL, "gram: n_lvl=%d out of [1,%d]", n_lvl, kMaxLvl);
  if (n_drops == 0) return XLMIMO_OK;
  const int64_t N = lvl_end[n_lvl - 1];
  const size_t need = gram_ws_bytes(a, K, n_drops, n_lvl, precision, mode);
  if (ws_bytes < need || (need && !ws))
    return set_error(XLMIMO_EWORKSPACE, "gram: workspace %zu < %zu bytes", ws_bytes, need);
  if (use_warp_kernel(a, K, n_drops, n_lvl, precision, mode)) {
    GramParams P;
    memset(&P, 0, sizeof(P));
    P.pos = pos;
    P.K = K;
    P.kind = a.kind;
    P.n_y = a.n_y;
    P.n_z = a.kind == XLMIMO_ULA ? 1 : a.n_z;
    P.N = N;
    P.inv_lambda = 1.0 / a.lambda;
    P.pitch = a.pitch;
    P.sqrt_beta0 = a.sqrt_beta0;
    KTimer tm(s, "gram_fused_warp_fp64");
    if (a.kind == XLMIMO_ULA) launch_warp_k<XLMIMO_ULA>(P, K, n_drops, out, s);
    else launch_warp_k<XLMIMO_UPA>(P, K, n_drops, out, s);
    tm.stop(s);
    count_launch();
    return check_launch("gram_warp_kernel");
  }
  if (use_fused_tc(a, K, precision, n_lvl)) {
    int rc;
    {
      KTimer tm(s, "gram_fused_tc_f16");
      rc = launch_fused_tc(a, pos, K, n_drops, N, (double *)ws, s);
      tm.stop(s);
      count_launch();
    }
    if (rc) return rc;
    const int64_t n_items = n_drops * (int64_t)K * (K + 1) / 2;
    KTimer tr(s, "gram_reduce");
    gram_reduce_kernel<<<(unsigned)((n_items + 255) / 256), 256, 0, s>>>((const double *)ws, K, n_drops,
                                                                        fused_tc_chunks(N, n_drops), 1, stream_tc_parts(K), out);
    tr.stop(s);
    count_launch();
    return check_launch("gram_reduce_kernel");
  }
  GramParams P;
  memset(&P, 0, sizeof(P));
  P.pos = pos;
  P.ws = (double *)ws;
  P.K = K;
  P.kind = a.kind;
  P.n_y = a.n_y;
  P.n_z = a.kind == XLMIMO_ULA ? 1 : a.n_z;
  P.N = N;
  P.n_split = choose_split(n_drops, N);
  const int64_t T = 256;
  P.chunk = ((N + P.n_split - 1) / P.n_split + T - 1) / T * T;
  P.n_lvl = n_lvl;
  for (int l = 0; l < kMaxLvl; ++l) P.lvl_end[l] = l < n_lvl ? lvl_end[l] : N;
  P.inv_lambda = 1.0 / a.lambda;
  P.pitch = a.pitch;
  P.sqrt_beta0 = a.sqrt_beta0;
  const int64_t n_blocks = n_drops * P.n_split;
  const bool fp32 = precision == XLMIMO_FP32;
  const KernelChoice kc = choose_kernel(a, K, precision);
  KTimer tm(s, kc.which == 1 ? "gram_fused_split_fp64"
               : kc.which == 2 ? "gram_fused_dmma_fp64"
               : kc.which == 3 ? "gram_fused_dmma_tiled_fp64"
               : K <= 8 ? (fp32 ? "gram_fused_small_fp32" : "gram_fused_small_fp64")
                        : (fp32 ? "gram_fused_tiled_fp32" : "gram_fused_tiled_fp64"));
  const bool mt1 = option(XLMIMO_OPT_GRAM_KERNEL) == 4 || N >= ((int64_t)1 << 31);
  if (kc.which == 3 && mt1) {
    switch ((K + 7) / 8) {
      case 3: launch_mt<3>(P, n_blocks, s); break;
      case 4: launch_mt<4>(P, n_blocks, s); break;
      case 5: launch_mt<5>(P, n_blocks, s); break;
      case 6: launch_mt<6>(P, n_blocks, s); break;
      case 7: launch_mt<7>(P, n_blocks, s); break;
      default: launch_mt<8>(P, n_blocks, s); break;
    }
  } else if (kc.which == 3) {
    int rc;
    switch ((K + 7) / 8) {
      case 3: rc = launch_mt2<3>(P, n_blocks, s); break;
      case 4: rc = launch_mt2<4>(P, n_blocks, s); break;
      case 5: rc = launch_mt2<5>(P, n_blocks, s); break;
      case 6: rc = launch_mt2<6>(P, n_blocks, s); break;
      case 7: rc = launch_mt2<7>(P, n_blocks, s); break;
      case 8: rc = launch_mt2<8>(P, n_blocks, s); break;
      case 9: rc = launch_mt2<9>(P, n_blocks, s); break;
      case 10: rc = launch_mt2<10>(P, n_blocks, s); break;
      case 11: rc = launch_mt2<11>(P, n_blocks, s); break;
      case 12: rc = launch_mt2<12>(P, n_blocks, s); break;
      case 13: rc = launch_mt2<13>(P, n_blocks, s); break;
      case 14: rc = launch_mt2<14>(P, n_blocks, s); break;
      case 15: rc = launch_mt2<15>(P, n_blocks, s); break;
      default: rc = launch_mt2<16>(P, n_blocks, s); break;
    }
    if (rc) return rc;
  } else if (kc.which == 2) {
    const bool ula = a.kind == XLMIMO_ULA;
    if (K <= 8) {
      if (ula) launch_mma<1, XLMIMO_ULA>(P, n_blocks, s);
      else launch_mma<1, XLMIMO_UPA>(P, n_blocks, s);
    } else {
      if (ula) launch_mma<2, XLMIMO_ULA>(P, n_blocks, s);
      else launch_mma<2, XLMIMO_UPA>(P, n_blocks, s);
    }
  } else if (kc.which == 1) {
    if (K == 8) {
      switch (kc.nt) {
        case 64: gram_split_kernel<4, 256, 1, 2><<<(unsigned)n_blocks, 256, 0, s>>>(P); break;
        case 128: gram_split_kernel<4, 128, 4><<<(unsigned)n_blocks, 128, 0, s>>>(P); break;
        case 192: gram_split_kernel<4, 128, 3, 2><<<(unsigned)n_blocks, 128, 0, s>>>(P); break;
        default: gram_split_kernel<4, 256, 2><<<(unsigned)n_blocks, 256, 0, s>>>(P); break;
      }
    } else {
      gram_split_kernel<2, 256, 2><<<(unsigned)n_blocks, 256, 0, s>>>(P);
    }
  } else if (K <= 8) {
    if (fp32) launch_small_k<true>(K, P, n_blocks, s);
    else launch_small_k<false>(K, P, n_blocks, s);
  } else {
    if (fp32) launch_tiled_k<true>(K, P, n_blocks, s);
    else launch_tiled_k<false>(K, P, n_blocks, s);
  }
  tm.stop(s);
  count_launch();
  int rc = check_launch("gram_exact kernel");
  if (rc) return rc;
  const int64_t n_items = n_drops * (int64_t)K * (K + 1) / 2;
  KTimer tr(s, "gram_reduce");
  gram_reduce_kernel<<<(unsigned)((n_items + 255) / 256), 256, 0, s>>>((const double *)ws, K, n_drops, P.n_split,
                                                                      n_lvl, kc.parts, out);
  tr.stop(s);
  count_launch();
  return check_launch("gram_reduce_kernel");
}

}  // namespace xlh
