// tools/dmma_shapes.cu -- fp64 tensor-core throughput of the mma.sync f64 shapes on B200:
// m8n8k4 (what the DMMA kernels use) vs m16n8k4 / m16n8k8 / m16n8k16 (sm_90+), each with
// 8 independent accumulator chains per warp, 8 warps per CTA, 4 CTAs per SM.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/dmma_shapes tools/dmma_shapes.cu
#include <cuda_runtime.h>
#include <cstdio>

template <int SHAPE>
__global__ void __launch_bounds__(256) shape_kernel(double *out, int iters) {
  double a[8], b[4], c[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + 1e-3 * (threadIdx.x + i);
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - 1e-4 * (threadIdx.x + i);
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) c[j][i] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (SHAPE == 0)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a[j]), "d"(b[0]));
      else if (SHAPE == 1)
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      else if (SHAPE == 2)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                     : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) s += c[j][i];
  if (s == 1234.5) out[0] = s;
}

int main() {
  double *d;
  cudaMalloc(&d, 64);
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);  // kHz
  const char *names[4] = {"m8n8k4", "m16n8k4", "m16n8k8", "m16n8k16"};
  const double fma_per[4] = {8 * 8 * 4, 16 * 8 * 4, 16 * 8 * 8, 16 * 8 * 16};
  const int iters[4] = {4096, 2048, 1024, 512};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int sh = 0; sh < 4; ++sh) {
    auto run = [&]() {
      const int grid = sms * 4;
      if (sh == 0) shape_kernel<0><<<grid, 256>>>(d, iters[sh]);
      if (sh == 1) shape_kernel<1><<<grid, 256>>>(d, iters[sh]);
      if (sh == 2) shape_kernel<2><<<grid, 256>>>(d, iters[sh]);
      if (sh == 3) shape_kernel<3><<<grid, 256>>>(d, iters[sh]);
    };
    run();
    cudaDeviceSynchronize();
    float best = 1e30f, ms;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      run();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    const double warps = (double)sms * 4 * 8;
    const double fma = warps * iters[sh] * 8 * fma_per[sh];
    printf("%-9s %8.3f ms  %.2f T FMA/s  %.1f FMA/clk/SM (at %d MHz)\n", names[sh], best, fma / best / 1e9,
           fma / (best * 1e-3) / sms / (clk * 1e3), clk / 1000);
  }
  return 0;
}
