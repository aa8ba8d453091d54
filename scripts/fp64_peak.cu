// fp64 FMA peak microbenchmark (the BSSN roofline denominator).
// Every thread runs 8 independent DFMA chains (enough ILP to cover the pipe latency);
// grid = 148 SMs x 8 CTAs x 256 threads.  Burst: one launch (~50 ms); sustained: launches
// back to back for ~3 s (the power cap settles).  Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256) dfma_loop(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += x[c];
  if (s == 1234.5) out[0] = s;  // keep the chains live
}
int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 8);
  const int blocks = sms * 8, threads = 256, iters = 4000;
  const double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  dfma_loop<<<blocks, threads>>>(d, 100, 0.999999, 1e-7);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  // sustained: ~3 s of back-to-back launches
  int n = (int)(3000.0f / best) + 1;
  cudaEventRecord(e0);
  for (int r = 0; r < n; ++r) dfma_loop<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float tot; cudaEventElapsedTime(&tot, e0, e1);
  printf("{\"what\": \"fp64 DFMA peak (8 chains/thread, %d CTAs x %d)\", \"burst_tflops\": %.3f, "
         "\"sustained_tflops\": %.3f, \"sustained_launches\": %d, \"sms\": %d, \"err\": \"%s\"}\n",
         blocks, threads, flops / (best * 1e-3) / 1e12, flops * n / (tot * 1e-3) / 1e12, n, sms,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
