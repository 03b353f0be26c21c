// xl_linalg.cuh -- warp-level dense linear-algebra helpers shared by the
// receiver (xl_rates.cu) and Appendix A (xl_bounds.cu) kernels.
#pragma once

#include "xl_common.cuh"

namespace xlk {

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

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace xlk
