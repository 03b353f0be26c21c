// tools/pipes.cu -- do DMMA (mma.sync m8n8k4 f64) and DFMA share one pipe on B200?
// Times a loop of DFMA chains alone, DMMA alone, and both interleaved in the same
// warps.  t(both) ~ max(t_dfma, t_dmma) => separate pipes; ~ sum => shared.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/pipes tools/pipes.cu
#include <cuda_runtime.h>
#include <cstdio>

template <bool DF, bool DM, int NDF>
__global__ void mix_kernel(double *out, int iters, double a, double b) {
  double x[NDF];
#pragma unroll
  for (int c = 0; c < NDF; ++c) x[c] = threadIdx.x * 1e-3 + c;
  double fa = threadIdx.x * 1e-3, fb = 1.0 + threadIdx.x * 1e-4;
  double c0[2] = {0, 0}, c1[2] = {0, 0}, c2[2] = {0, 0}, c3[2] = {0, 0};
  for (int i = 0; i < iters; ++i) {
    if (DM) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c0[0]), "+d"(c0[1]) : "d"(fa), "d"(fb));
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c1[0]), "+d"(c1[1]) : "d"(fa), "d"(fb));
    }
    if (DF) {
#pragma unroll
      for (int c = 0; c < NDF; ++c) x[c] = fma(x[c], a, b);
    }
    if (DM) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c2[0]), "+d"(c2[1]) : "d"(fa), "d"(fb));
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c3[0]), "+d"(c3[1]) : "d"(fa), "d"(fb));
    }
  }
  double s = c0[0] + c0[1] + c1[0] + c1[1] + c2[0] + c2[1] + c3[0] + c3[1];
#pragma unroll
  for (int c = 0; c < NDF; ++c) s += x[c];
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
  const int blocks = 148 * 4, threads = 256, it = 4000;
  // 16 DFMA chains per iter: 16 DFMA warp-instr; 4 DMMA per iter (1024 FMA per warp)
  float t_df = time_it([&] { mix_kernel<true, false, 16><<<blocks, threads>>>(d, it, 0.999, 1e-3); });
  float t_dm = time_it([&] { mix_kernel<false, true, 16><<<blocks, threads>>>(d, it, 0.999, 1e-3); });
  float t_bo = time_it([&] { mix_kernel<true, true, 16><<<blocks, threads>>>(d, it, 0.999, 1e-3); });
  double n_dfma = (double)blocks * threads * it * 16;
  double n_dmma_fma = (double)blocks * (threads / 32) * it * 4 * 256;
  printf("{\"t_dfma_ms\": %.3f, \"t_dmma_ms\": %.3f, \"t_both_ms\": %.3f, \"dfma_per_s\": %.4e, "
         "\"dmma_fma_per_s\": %.4e, \"both_total_fma_per_s\": %.4e, \"verdict\": \"%s\"}\n",
         t_df, t_dm, t_bo, n_dfma / (t_df * 1e-3), n_dmma_fma / (t_dm * 1e-3),
         (n_dfma + n_dmma_fma) / (t_bo * 1e-3),
         t_bo < 0.8f * (t_df + t_dm) ? "overlap (separate pipes)" : "serialised (shared pipe)");
  return cudaGetLastError() != cudaSuccess;
}
