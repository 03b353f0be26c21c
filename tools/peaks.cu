// tools/peaks.cu -- B200 microbenchmarks for the roofline denominators this
// engine uses: FP64 DFMA, FP64 DMMA (m8n8k4), FP32 FFMA,
// MUFU sin, and a read-only HBM stream.  Prints one JSON object.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/peaks tools/peaks.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s\n", cudaGetErrorString(e)); return 1; } } while (0)

template <int CH>
__global__ void dfma_kernel(double *out, int iters, double a, double b) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 1234.5) out[0] = s;
}

template <int CH>
__global__ void ffma_kernel(float *out, int iters, float a, float b) {
  float x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fmaf(x[c], a, b);
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 1234.5f) out[0] = s;
}

__global__ void dmma_kernel(double *out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c0[2] = {0, 0}, c1[2] = {0, 0}, c2[2] = {0, 0}, c3[2] = {0, 0};
  for (int i = 0; i < iters; ++i) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0[0]), "+d"(c0[1]) : "d"(a), "d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c1[0]), "+d"(c1[1]) : "d"(a), "d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c2[0]), "+d"(c2[1]) : "d"(a), "d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c3[0]), "+d"(c3[1]) : "d"(a), "d"(b));
  }
  double s = c0[0] + c0[1] + c1[0] + c1[1] + c2[0] + c2[1] + c3[0] + c3[1];
  if (s == 1234.5) out[0] = s;
}

template <int CH>
__global__ void mufu_kernel(float *out, int iters) {
  float x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = __sinf(x[c]);
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 1234.5f) out[0] = s;
}

__global__ void read_kernel(const double4 *in, size_t n, double *out) {
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const double2 *p2 = reinterpret_cast<const double2 *>(in + i);
    double2 v0 = __ldcs(p2), v1 = __ldcs(p2 + 1);
    double4 v = make_double4(v0.x, v0.y, v1.x, v1.y);
    s += v.x + v.y + v.z + v.w;
  }
  if (s == 1234.5) out[0] = s;
}

__global__ void rsqrt_accuracy_kernel(double *out) {
  // max rel error of rsqrt.approx.f64 over a sweep (for the amplitude design)
  double worst = 0;
  for (int i = 0; i < 4096; ++i) {
    double x = 1.0 + i * (3.0 / 4096) + threadIdx.x * 1e-7;
    double y;
    asm("rsqrt.approx.f64 %0, %1;" : "=d"(y) : "d"(x));
    double ref = 1.0 / sqrt(x);
    double e = fabs(y - ref) / ref;
    worst = e > worst ? e : worst;
  }
  out[threadIdx.x] = worst;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  double *dout;
  CK(cudaMalloc(&dout, 1 << 20));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  const int blocks = sms * 8, threads = 256;
  auto time_it = [&](auto launch) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    return best;
  };
  const int it = 20000;
  float t_dfma = time_it([&] { dfma_kernel<8><<<blocks, threads>>>(dout, it, 0.999, 1e-3); });
  double dfma_rate = (double)blocks * threads * it * 8 / (t_dfma * 1e-3);  // DFMA/s
  float t_ffma = time_it([&] { ffma_kernel<8><<<blocks, threads>>>((float *)dout, it, 0.999f, 1e-3f); });
  double ffma_rate = (double)blocks * threads * it * 8 / (t_ffma * 1e-3);
  const int itm = 5000;
  float t_dmma = time_it([&] { dmma_kernel<<<blocks, threads>>>(dout, itm); });
  double dmma_fma = (double)blocks * (threads / 32) * itm * 4 * 256 / (t_dmma * 1e-3);  // FMA/s (8x8x4 per mma)
  float t_mufu = time_it([&] { mufu_kernel<8><<<blocks, threads>>>((float *)dout, it / 4); });
  double mufu_rate = (double)blocks * threads * (it / 4) * 8 / (t_mufu * 1e-3);
  const size_t bytes = (size_t)4 << 30;
  double4 *buf;
  CK(cudaMalloc(&buf, bytes));
  CK(cudaMemset(buf, 0, bytes));
  float t_rd = time_it([&] { read_kernel<<<sms * 16, 512>>>(buf, bytes / sizeof(double4), dout); });
  double rd_gbs = bytes / (t_rd * 1e-3) / 1e9;
  rsqrt_accuracy_kernel<<<1, 256>>>(dout);
  double h[256];
  cudaMemcpy(h, dout, sizeof(h), cudaMemcpyDeviceToHost);
  double worst = 0;
  for (double v : h) worst = v > worst ? v : worst;
  CK(cudaGetLastError());
  printf("{\"sms\": %d, \"clock_attr_mhz\": %.0f, \"dfma_per_s\": %.4e, \"dfma_per_clk_per_sm_at_attr_clock\": %.2f, "
         "\"ffma_per_s\": %.4e, \"dmma_fma_per_s\": %.4e, \"mufu_sin_per_s\": %.4e, \"hbm_read_gbs\": %.1f, "
         "\"rsqrt_approx_f64_max_rel_err\": %.3e}\n",
         sms, clk / 1e3, dfma_rate, dfma_rate / (sms * clk * 1e3), ffma_rate, dmma_fma, mufu_rate, rd_gbs, worst);
  return 0;
}
