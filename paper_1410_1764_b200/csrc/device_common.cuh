// device_common.cuh -- small device helpers shared by the stage, ghost and init kernels.
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>
#include "grid.hpp"

namespace chemora {

// Host helpers for the launchers.  The dynamic shared-memory opt-in is a per-device
// attribute of a kernel, so it is recorded per (kernel, device) -- one process may drive
// several devices -- in a bit mask owned by the call site.
inline cudaError_t smem_optin(const void* fn, int bytes, std::atomic<uint64_t>& done) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

// SM count of the current device (grid sizing of the persistent kernels).
inline int device_sm_count() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return 148;
  return n > 0 ? n : 148;
}

// Store the periodic ghost images of interior value v at (i, j, k) (PAPER.md:345-347
// ghost zones).  `own` is the GF array (interior-origin pointer); the
// z images of the first g planes go to `zlo` at k + nz (the lower neighbour's top ghost
// planes, or our own when the slab is the whole periodic z range) and those of the last g
// planes to `zhi` at k - nz.  Every combination of x/y/z images is written so edges and
// corners equal the doubly/triply wrapped interior value, exactly as the axis-by-axis fill.
// Out of line: only threads near a face call it, and keeping its index arithmetic out of
// the stage kernels' register allocation is worth the call.
static __device__ __noinline__ void store_images_n(double* own, double* zlo, double* zhi, int nx, int ny,
                                            int nz, int g, int64_t px, int64_t plane, int i, int j,
                                            int k, double v) {
  const int xi = i < g ? i + nx : (i >= nx - g ? i - nx : i);
  const int yj = j < g ? j + ny : (j >= ny - g ? j - ny : j);
  const int zk = k < g ? k + nz : (k >= nz - g ? k - nz : k);
  const bool hx = xi != i, hy = yj != j, hz = zk != k;
  if (!(hx | hy | hz)) return;
  double* zb = k < g ? zlo : zhi;
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    if (c && !hz) continue;
    double* base = c ? zb : own;
    const int64_t kk = c ? zk : k;
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      if (b && !hy) continue;
      const int64_t jj = b ? yj : j;
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        if (a && !hx) continue;
        if (!(a | b | c)) continue;
        const int64_t ii = a ? xi : i;
        base[kk * plane + jj * px + ii] = v;
      }
    }
  }
}
__device__ __forceinline__ void store_images(double* own, double* zlo, double* zhi,
                                             const Layout& L, int i, int j, int k, double v) {
  store_images_n(own, zlo, zhi, (int)L.nx, (int)L.ny, (int)L.nz, L.g, L.px, L.plane, i, j, k, v);
}

// Where the periodic ghost images of a point go: `general` -- near a z face (images may go
// to a neighbour slab) or on an x-y edge: the noinline store_images path; `single` -- near
// exactly one x or y face: one image in the same plane at offset `off` from the point.
struct ImageSite {
  bool general, single;
  int64_t off;
};
__device__ __forceinline__ ImageSite image_site(const Layout& L, int i, int j, int k) {
  const int g = L.g;
  const bool nxf = i < g || i >= L.nx - g, nyf = j < g || j >= L.ny - g;
  ImageSite s;
  s.general = k < g || k >= L.nz - g || (nxf && nyf);
  s.single = nxf || nyf;
  s.off = nxf ? (int64_t)(i < g ? L.nx : -L.nx) : (int64_t)(j < g ? L.ny : -L.ny) * L.px;
  return s;
}
// Store the images of value v of one GF (own: that GF's base, c = L.idx(i, j, k)).
__device__ __forceinline__ void put_images(const ImageSite& s, double* own, double* zlo, double* zhi,
                                           const Layout& L, int i, int j, int k, int64_t c, double v) {
  if (s.general) store_images(own, zlo, zhi, L, i, j, k, v);
  else if (s.single) own[c + s.off] = v;
}

__device__ __forceinline__ bool near_face(const Layout& L, int i, int j, int k) {
  const int g = L.g;
  return i < g || j < g || k < g || i >= L.nx - g || j >= L.ny - g || k >= L.nz - g;
}

// Record the first non-finite output: flag = min(step * n_gf + gf).
__device__ __forceinline__ void check_finite(unsigned long long* flag, unsigned long long code,
                                             double v) {
  if (!isfinite(v)) atomicMin(flag, code);
}

}  // namespace chemora
