// tools/dfma_ops.cu -- FP64 pipe throughput vs operand pattern on B200.
//  (a) x = fma(x, a, b), a/b warp-uniform          (the classic peak test)
//  (b) acc = fma(p, q, acc), p/q/acc per-thread      (Gram accumulation pattern)
//  (c) (b) with 2 independent products per acc       (cMAC pattern: 2 chained FMAs)
//  (d) DMUL x = x * a
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/dfma_ops tools/dfma_ops.cu
#include <cuda_runtime.h>
#include <cstdio>

__global__ void k_uniform(double *out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = fma(x[c], a, b);
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += x[c];
  if (s == 1234.5) out[0] = s;
}

__global__ void k_perthread(double *out, int iters) {
  double p[8], q[8], acc[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    p[c] = threadIdx.x * 1e-3 + c;
    q[c] = 1.0 + threadIdx.x * 1e-5 * c;
    acc[c] = 0;
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = fma(p[c], q[(c + 1) & 7], acc[c]);
#pragma unroll
    for (int c = 0; c < 8; ++c) p[c] = fma(p[c], q[c], acc[(c + 3) & 7]);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += acc[c] + p[c];
  if (s == 1234.5) out[0] = s;
}

__global__ void k_cmac(double *out, int iters) {
  // 4 "users" (re, im), 10 complex accumulators as in the Gram kernels
  double hr[4], hi[4], acc[20];
#pragma unroll
  for (int c = 0; c < 4; ++c) { hr[c] = threadIdx.x * 1e-3 + c; hi[c] = 1.0 - c * 1e-3; }
#pragma unroll
  for (int c = 0; c < 20; ++c) acc[c] = 0;
  for (int i = 0; i < iters; ++i) {
    int v = 0;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = a; b < 4; ++b) {
        acc[v] = fma(hr[a], hr[b], fma(hi[a], hi[b], acc[v]));
        acc[v + 1] = fma(hr[a], hi[b], fma(-hi[a], hr[b], acc[v + 1]));
        v += 2;
      }
#pragma unroll
    for (int c = 0; c < 4; ++c) { hr[c] = fma(hr[c], 0.999, 1e-9); hi[c] = fma(hi[c], 0.999, 1e-9); }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 20; ++c) s += acc[c];
  if (s == 1234.5) out[0] = s;
}

__global__ void k_dmul(double *out, int iters, double a) {
  double x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = x[c] * a;
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += x[c];
  if (s == 1234.5) out[0] = s;
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

int main() {
  double *d;
  cudaMalloc(&d, 64);
  const int blocks = 148 * 8, threads = 256, it = 8000;
  const double thr = (double)blocks * threads * it;
  float ta = time_it([&] { k_uniform<<<blocks, threads>>>(d, it, 0.999, 1e-3); });
  float tb = time_it([&] { k_perthread<<<blocks, threads>>>(d, it); });
  float tc = time_it([&] { k_cmac<<<blocks, threads>>>(d, it); });
  float td = time_it([&] { k_dmul<<<blocks, threads>>>(d, it, 0.999); });
  printf("{\"uniform_dfma_per_s\": %.4e, \"perthread_dfma_per_s\": %.4e, \"cmac_pattern_dfma_per_s\": %.4e, "
         "\"dmul_per_s\": %.4e}\n",
         thr * 8 / (ta * 1e-3), thr * 16 / (tb * 1e-3), thr * (40 + 8) / (tc * 1e-3), thr * 8 / (td * 1e-3));
  return cudaGetLastError() != cudaSuccess;
}
