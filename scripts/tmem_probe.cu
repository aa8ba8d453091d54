// TMEM as per-thread scratch (probe for the BSSN z-queue design): one CTA of 256 threads
// per SM allocates all 512 columns; warps w and w+4 share lanes 32*(w%4)..+31.  Checks a
// store by one warp and a load by its partner after a CTA barrier, then times dependent
// tcgen05.ld.32x32b.x2 (one fp64) + wait::ld round trips and independent batches.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ void tst2(uint32_t taddr, double v) {
  uint32_t lo = __double2loint(v), hi = __double2hiint(v);
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr), "r"(lo), "r"(hi) : "memory");
}
__device__ __forceinline__ double tld2(uint32_t taddr) {
  uint32_t lo, hi;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(taddr) : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  return __hiloint2double(hi, lo);
}
__device__ __forceinline__ void tld8(uint32_t taddr, double* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr) : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int q = 0; q < 4; ++q) v[q] = __hiloint2double(r[2 * q + 1], r[2 * q]);
}
__global__ void __launch_bounds__(256, 1) probe(int* bad, long long* cyc, double* sink, int iters) {
  __shared__ uint32_t taddr_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = taddr_s + ((uint32_t)(32 * (warp & 3)) << 16);
  // correctness: warps 0-3 store 256 doubles per lane, warps 4-7 read them
  if (warp < 4)
    for (int c = 0; c < 256; ++c) tst2(base + 2 * c, (double)(blockIdx.x * 100000 + (warp * 32 + lane) * 256 + c) + 0.25);
  asm volatile("tcgen05.wait::st.sync.aligned;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp >= 4)
    for (int c = 0; c < 256; ++c) {
      const double v = tld2(base + 2 * c);
      if (v != (double)(blockIdx.x * 100000 + ((warp - 4) * 32 + lane) * 256 + c) + 0.25) atomicAdd(bad, 1);
    }
  __syncthreads();
  // latency: dependent single loads (address depends on the previous value)
  double acc = 0.0;
  long long t0 = clock64();
  uint32_t col = 0;
  for (int i = 0; i < iters; ++i) {
    const double v = tld2(base + 2 * col);
    acc += v;
    col = ((uint32_t)v + i) & 127;
  }
  long long t1 = clock64();
  // throughput: 8 x4 loads (32 doubles) per wait
  double a2 = 0.0;
  for (int i = 0; i < iters; ++i) {
    double v[4];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      tld8(base + ((8 * q + i) & 255), v);
      a2 += v[0] + v[1] + v[2] + v[3];
    }
  }
  long long t2 = clock64();
  if (threadIdx.x == 0) { cyc[3 * blockIdx.x] = t1 - t0; cyc[3 * blockIdx.x + 1] = t2 - t1; }
  sink[blockIdx.x * 256 + threadIdx.x] = acc + a2;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr_s));
}
int main() {
  int* bad; long long* cyc; double* sink;
  cudaMalloc(&bad, 4); cudaMemset(bad, 0, 4);
  cudaMalloc(&cyc, 8 * 3 * 148); cudaMalloc(&sink, 8 * 148 * 256);
  const int iters = 1000;
  probe<<<148, 256>>>(bad, cyc, sink, iters);
  cudaError_t e = cudaDeviceSynchronize();
  int hb = -1; long long hc[3 * 148];
  cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hc, cyc, sizeof(hc), cudaMemcpyDeviceToHost);
  printf("{\"tmem_probe\": \"%s\", \"mismatches\": %d, \"dep_ld_cycles\": %.1f, \"batched_cycles_per_x8_ld\": %.2f}\n",
         cudaGetErrorString(e), hb, hc[0] / (double)iters, hc[1] / (8.0 * iters));
  return 0;
}
