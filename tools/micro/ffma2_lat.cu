// Developer microbenchmark: latency and throughput of FFMA / FFMA2 / FADD2 on B200.
#include <cuda_runtime.h>
#include <cstdio>
__global__ void lat_ffma2(float2* out, float2 a, float2 b, int n, long long* cyc) {
  float2 x = make_float2(threadIdx.x, 1.f);
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) x = __ffma2_rn(a, x, b);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_ffma(float* out, float a, float b, int n, long long* cyc) {
  float x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) x = fmaf(a, x, b);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// throughput: 8 independent chains per thread
__global__ void thr_ffma2(float2* out, float2 a, float2 b, int n) {
  float2 x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = make_float2(threadIdx.x + k, k);
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = __ffma2_rn(a, x[k], b);
  }
  float2 s = x[0];
#pragma unroll
  for (int k = 1; k < 8; ++k) s = __fadd2_rn(s, x[k]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void thr_ffma(float* out, float a, float b, int n) {
  float x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fmaf(a, x[k], b);
  }
  float s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float2* o2; float* o; long long* c;
  cudaMalloc(&o2, 1 << 26); cudaMalloc(&o, 1 << 26); cudaMalloc(&c, 8);
  long long h;
  int n = 1000;
  lat_ffma2<<<1, 32>>>(o2, make_float2(0.999f, 0.999f), make_float2(0.1f, 0.1f), n, c);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("FFMA2 dependent latency: %.2f cycles\n", (double)h / (16.0 * n));
  lat_ffma<<<1, 32>>>(o, 0.999f, 0.1f, n, c);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("FFMA dependent latency: %.2f cycles\n", (double)h / (16.0 * n));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int rep = 0; rep < 2; ++rep) {
    int blocks = sms * 8, thr = 256, it = 2000;
    cudaEventRecord(e0);
    thr_ffma2<<<blocks, thr>>>(o2, make_float2(0.999f, 0.999f), make_float2(0.1f, 0.1f), it);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fma = (double)blocks * thr * it * 64 * 2;   // scalar FMAs (2 per FFMA2)
    printf("FFMA2 throughput: %.1f TFMA/s = %.1f FMA/clk/SM (clock %d MHz)\n", fma / ms / 1e9, fma / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    cudaEventRecord(e0);
    thr_ffma<<<blocks, thr>>>(o, 0.999f, 0.1f, it);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fma = (double)blocks * thr * it * 64;
    printf("FFMA throughput: %.1f TFMA/s = %.1f FMA/clk/SM\n", fma / ms / 1e9, fma / (ms * 1e-3) / sms / (clk * 1e3));
  }
  return 0;
}
