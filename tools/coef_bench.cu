// tools/coef_bench.cu -- throughput of the fused generator's pieces on B200:
//  (a) coef_fast (the full fp64 coefficient), 4 independent per thread
//  (b) MUFU.RSQ64H alone (rsqrt.approx.ftz.f64)
//  (c) rsqrt_nr (MUFU + Householder step)
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -I. -o tools/coef_bench tools/coef_bench.cu
#include <cuda_runtime.h>
#include <cstdio>

#include "paper_2503_18118_b200/csrc/xl_common.cuh"

// the ABI-side host symbols referenced by xl_common.cuh are not needed here
__global__ void k_coef(double *out, int iters) {
  double r2[4], acc = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) r2[c] = 9.0 + threadIdx.x * 1e-3 + c * 0.37;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      double re, im;
      xl::coef_fast(r2[c], 1.0, 373.8, re, im);
      acc += re + im;
      r2[c] += 1e-3;
    }
  }
  if (acc == 1234.5) out[0] = acc;
}

__global__ void k_mufu(double *out, int iters) {
  double x[8], acc = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = 2.0 + threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      double y;
      asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x[c]));
      x[c] = y + 2.0;
    }
  }
#pragma unroll
  for (int c = 0; c < 8; ++c) acc += x[c];
  if (acc == 1234.5) out[0] = acc;
}

__global__ void k_rsq(double *out, int iters) {
  double x[8], acc = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = 2.0 + threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = xl::rsqrt_nr(x[c]) + 2.0;
  }
#pragma unroll
  for (int c = 0; c < 8; ++c) acc += x[c];
  if (acc == 1234.5) out[0] = acc;
}

template <typename F>
float time_it(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f, ms;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  return best;
}

namespace xlh {
void count_launch(uint64_t) {}
}

int main() {
  double *d;
  cudaMalloc(&d, 64);
  const int blocks = 148 * 8, threads = 256, it = 2000;
  const double thr = (double)blocks * threads * it;
  float ta = time_it([&] { k_coef<<<blocks, threads>>>(d, it); });
  float tb = time_it([&] { k_mufu<<<blocks, threads>>>(d, it); });
  float tc = time_it([&] { k_rsq<<<blocks, threads>>>(d, it); });
  const double coefs = thr * 4 / (ta * 1e-3);
  printf("{\"coef_per_s\": %.4e, \"coef_fp64_ops_per_s_model34\": %.4e, \"frac_of_18.6T\": %.3f, "
         "\"mufu_rsq64h_per_s\": %.4e, \"rsqrt_nr_per_s\": %.4e}\n",
         coefs, coefs * 34, coefs * 34 / 18.6e12, thr * 8 / (tb * 1e-3), thr * 8 / (tc * 1e-3));
  return cudaGetLastError() != cudaSuccess;
}
