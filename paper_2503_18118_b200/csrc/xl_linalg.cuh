// xl_linalg.cuh -- warp-level dense linear-algebra helpers shared by the
// receiver (xl_rates.cu) and Appendix A (xl_bounds.cu) kernels.
#pragma once

#include "xl_common.cuh"

namespace xlk {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// In-place lower Cholesky of As (column-major, K x K complex) by one warp.
// Returns true on success (uniform across the warp).
template <int RPL>
__device__ __forceinline__ bool warp_cholesky(double2 *As, int K, int lane) {
  for (int j = 0; j < K; ++j) {
    __syncwarp();
    const double piv = As[j * K + j].x;
    if (!(piv > 0.0) || !isfinite(piv)) return false;
    const double ljj = sqrt(piv), inv = 1.0 / ljj;
    __syncwarp();
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int i = lane + 32 * r;
      if (i > j && i < K) {
        double2 v = As[j * K + i];
        v.x *= inv;
        v.y *= inv;
        As[j * K + i] = v;
      } else if (i == j) {
        As[j * K + j] = make_double2(ljj, 0.0);
      }
    }
    __syncwarp();
    // trailing update: A[i][k] -= L[i][j] conj(L[k][j]) for j < k <= i
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int i = lane + 32 * r;
      if (i > j && i < K) {
        const double2 lij = As[j * K + i];
        for (int k = j + 1; k <= i; ++k) {
          const double2 lkj = As[j * K + k];
          double2 a = As[k * K + i];
          // lij * conj(lkj) = (lr kr + li ki) + j (li kr - lr ki)
          a.x -= lij.x * lkj.x + lij.y * lkj.y;
          a.y -= lij.y * lkj.x - lij.x * lkj.y;
          As[k * K + i] = a;
        }
      }
    }
  }
  __syncwarp();
  return true;
}

// Packed column-major lower triangle: column j holds rows j..K-1 at poff(K, j).
__device__ __forceinline__ int poff(int K, int j) { return j * K - j * (j - 1) / 2; }

// In-place lower Cholesky of a packed Hermitian matrix (lower triangle, see poff) by
// one warp, lanes over rows (row i = lane + 32 r): per column j the pivot, the column
// scaled by 1/L_jj, and the rank-1 update of the trailing columns (consecutive lanes
// touch consecutive words; L_kj is a broadcast).  Returns true on success (uniform).
template <int RPL>
__device__ __forceinline__ bool warp_cholesky_packed(double2 *Ls, int K, int lane) {
  for (int j = 0; j < K; ++j) {
    __syncwarp();
    const int oj = poff(K, j);
    const double piv = Ls[oj].x;
    if (!(piv > 0.0) || !isfinite(piv)) return false;
    const double ljj = sqrt(piv), inv = 1.0 / ljj;
    __syncwarp();
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int i = lane + 32 * r;
      if (i > j && i < K) {
        double2 v = Ls[oj + i - j];
        v.x *= inv;
        v.y *= inv;
        Ls[oj + i - j] = v;
      } else if (i == j) {
        Ls[oj] = make_double2(ljj, 0.0);
      }
    }
    __syncwarp();
    // A_ik -= L_ij conj(L_kj), j < k <= i
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int i = lane + 32 * r;
      if (i > j && i < K) {
        const double2 lij = Ls[oj + i - j];
        int ok = oj + (K - j);  // poff(K, j + 1)
        for (int k = j + 1; k <= i; ++k) {
          const double2 lkj = Ls[oj + k - j];
          double2 a = Ls[ok + i - k];
          a.x -= lij.x * lkj.x + lij.y * lkj.y;
          a.y -= lij.y * lkj.x - lij.x * lkj.y;
          Ls[ok + i - k] = a;
          ok += K - k;
        }
      }
    }
  }
  __syncwarp();
  return true;
}

// diag(A^{-1}) from the packed Cholesky factor L of A (destroyed: becomes X = L^{-1}),
// columns j = K-1 .. 0:  X_jj = 1/L_jj,  X_ij = -(sum_{k=j+1..i} X_ik L_kj) / L_jj (i > j),
// [A^{-1}]_jj = sum_{i >= j} |X_ij|^2 (A^{-1} = X^H X).  Lanes over rows; the value for
// column c = lane + 32 r lands in dinv[r] of that lane.
template <int RPL>
__device__ __forceinline__ void warp_inv_diag_packed(double2 *Ls, int K, int lane, double (&dinv)[RPL]) {
#pragma unroll
  for (int r = 0; r < RPL; ++r) dinv[r] = 0.0;
  for (int j = K - 1; j >= 0; --j) {
    const int oj = poff(K, j);
    const double d = 1.0 / Ls[oj].x;
    double2 x[RPL];
    double part = 0.0;
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int i = lane + 32 * r;
      x[r] = make_double2(0.0, 0.0);
      if (i > j && i < K) {
        double xr = 0.0, xi = 0.0;
        int ok = oj + (K - j);  // column k = j + 1
        for (int k = j + 1; k <= i; ++k) {
          const double2 xik = Ls[ok + i - k];  // X_ik (columns > j are inverted)
          const double2 lkj = Ls[oj + k - j];  // L_kj
          xr += xik.x * lkj.x - xik.y * lkj.y;
          xi += xik.x * lkj.y + xik.y * lkj.x;
          ok += K - k;
        }
        x[r] = make_double2(-xr * d, -xi * d);
      } else if (i == j) {
        x[r] = make_double2(d, 0.0);
      }
      part += x[r].x * x[r].x + x[r].y * x[r].y;
    }
    const double s = warp_sum(part);
    __syncwarp();
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int i = lane + 32 * r;
      if (i >= j && i < K) Ls[oj + i - j] = x[r];
      if (r == (j >> 5) && lane == (j & 31)) dinv[r] = s;
    }
    __syncwarp();
  }
}


}  // namespace xlk
