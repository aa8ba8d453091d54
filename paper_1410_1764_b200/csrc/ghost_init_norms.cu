// ghost_init_norms.cu -- off-hot-path kernels: periodic ghost fill / z-face push
// (SPEC.md:433-441), device initial data (Fig. 1 Init, PAPER.md:632-636;
// DESIGN.md §Inputs) and deterministic reductions (Fig. 1 Energy,
// PAPER.md:642-644).
#include <cuda_runtime.h>
#include <cstdint>
#include "grid.hpp"
#include "kernels.hpp"

namespace chemora {
namespace {

// ------------------------------------------------------------------ ghost fill
__global__ void fill_x(Layout L, double* set) {
  const int64_t rows = L.ny * L.nz;
  const int g = L.g;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= rows * g) return;
  const int s = (int)(t % g);
  const int64_t r = t / g;
  const int64_t j = r % L.ny, k = r / L.ny;
  double* f = set + blockIdx.y * L.gfs;
  f[L.idx(-1 - s, j, k)] = f[L.idx(L.nx - 1 - s, j, k)];
  f[L.idx(L.nx + s, j, k)] = f[L.idx(s, j, k)];
}

__global__ void fill_y(Layout L, double* set) {
  const int g = L.g;
  const int64_t wx = L.nx + 2 * g;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= wx * g * L.nz) return;
  const int64_t i = t % wx - g;
  const int64_t r = t / wx;
  const int s = (int)(r % g);
  const int64_t k = r / g;
  double* f = set + blockIdx.y * L.gfs;
  f[L.idx(i, -1 - s, k)] = f[L.idx(i, L.ny - 1 - s, k)];
  f[L.idx(i, L.ny + s, k)] = f[L.idx(i, s, k)];
}

// z: push this slab's first/last g planes (x/y ghosts included) into the lo/hi
// destinations' top/bottom ghost planes.
__global__ void push_z(Layout L, const double* set, double* lo, double* hi) {
  const int g = L.g;
  const int64_t wx = L.nx + 2 * g, wy = L.ny + 2 * g;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= wx * wy * g) return;
  const int64_t i = t % wx - g;
  const int64_t r = t / wx;
  const int64_t j = r % wy - g;
  const int s = (int)(r / wy);
  const int64_t off = blockIdx.y * L.gfs;
  lo[off + L.idx(i, j, L.nz + s)] = set[off + L.idx(i, j, s)];
  hi[off + L.idx(i, j, -g + s)] = set[off + L.idx(i, j, L.nz - g + s)];
}

// ------------------------------------------------------------------ init
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double hash_uniform(uint64_t seed, uint64_t gf, uint64_t index) {
  const uint64_t z = splitmix64(seed ^ ((gf << 40) + index));
  return (double)(z >> 11) * 0x1.0p-52 - 1.0;
}

__constant__ int c_pw3_k[3][3] = {{1, 2, 3}, {2, -1, 1}, {0, 1, -2}};
__constant__ double c_pw3_a[3] = {1.0, 0.5, 0.25};
__constant__ double c_pw3_ph[3] = {0.0, 0.3, 1.1};

__global__ void init_kernel(Layout L, double* set, InitArgs a) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t j = blockIdx.y;
  const int64_t k = blockIdx.z;
  if (i >= L.nx) return;
  const int64_t kg = a.z0 + k;
  const double x = a.origin[0] + i * a.h[0];
  const double y = a.origin[1] + j * a.h[1];
  const double z = a.origin[2] + kg * a.h[2];
  const int64_t c = L.idx(i, j, k);
  const int nf = L.n_gf;
  if (a.kind == 4) {  // NOISE
    const uint64_t I = (uint64_t)i + (uint64_t)a.gext[0] * ((uint64_t)j + (uint64_t)a.gext[1] * (uint64_t)kg);
    for (int f = 0; f < nf; ++f) set[f * L.gfs + c] = hash_uniform(a.seed, f, I);
    return;
  }
  if (a.kind == 2) {  // PW3 (wave)
    double v[5] = {0, 0, 0, 0, 0};
    for (int m = 0; m < 3; ++m) {
      const int kx = c_pw3_k[m][0], ky = c_pw3_k[m][1], kz = c_pw3_k[m][2];
      const double w = sqrt((double)(kx * kx + ky * ky + kz * kz));
      const double arg = kx * x + ky * y + kz * z + c_pw3_ph[m];
      double s, cs;
      sincos(arg, &s, &cs);
      const double am = c_pw3_a[m];
      v[0] += am * s;
      v[1] += -am * w * cs;
      v[2] += am * kx * cs;
      v[3] += am * ky * cs;
      v[4] += am * kz * cs;
    }
    for (int f = 0; f < 5; ++f) set[f * L.gfs + c] = v[f];
    return;
  }
  if (a.kind == 3) {  // GAUSSIAN (wave)
    const double cx = a.origin[0] + 0.5 * a.gext[0] * a.h[0];
    const double cy = a.origin[1] + 0.5 * a.gext[1] * a.h[1];
    const double cz = a.origin[2] + 0.5 * a.gext[2] * a.h[2];
    const double r2 = (x - cx) * (x - cx) + (y - cy) * (y - cy) + (z - cz) * (z - cz);
    const double A = a.kp[0], Wd = a.kp[1];
    for (int f = 0; f < 5; ++f) set[f * L.gfs + c] = 0.0;
    set[1 * L.gfs + c] = A * exp(-0.5 * r2 / (Wd * Wd));
    return;
  }
  if (a.kind == 6) {  // GAUGE_WAVE (BSSN), kp = {amp, d, shift, t}
    const double amp = a.kp[0], d = a.kp[1], shift = a.kp[2], t = a.kp[3];
    const double pi2 = 6.283185307179586476925286766559;
    const double ph = pi2 * (x + shift * t - t) / d;
    double s, cs;
    sincos(ph, &s, &cs);
    const double H = 1.0 - amp * s;
    const double dHdt = amp * (pi2 / d) * cs, dHdx = -amp * (pi2 / d) * cs;
    const double Kxx = -dHdt / (2.0 * sqrt(H));
    for (int f = 0; f < nf; ++f) set[f * L.gfs + c] = 0.0;
    set[0 * L.gfs + c] = log(H) / 12.0;
    set[1 * L.gfs + c] = pow(H, 2.0 / 3.0);
    set[4 * L.gfs + c] = pow(H, -1.0 / 3.0);
    set[6 * L.gfs + c] = pow(H, -1.0 / 3.0);
    set[7 * L.gfs + c] = Kxx / H;
    set[8 * L.gfs + c] = (2.0 / 3.0) * pow(H, -1.0 / 3.0) * Kxx;
    set[11 * L.gfs + c] = -(1.0 / 3.0) * pow(H, -4.0 / 3.0) * Kxx;
    set[13 * L.gfs + c] = -(1.0 / 3.0) * pow(H, -4.0 / 3.0) * Kxx;
    set[14 * L.gfs + c] = (2.0 / 3.0) * pow(H, -5.0 / 3.0) * dHdx;
    set[17 * L.gfs + c] = sqrt(H);
    set[19 * L.gfs + c] = shift;
    return;
  }
  if (a.kind == 5) {  // MINK_PERT (BSSN)
    const double eps = a.kp[0];
    const double len = a.gext[0] * a.h[0];
    const double pi2 = 6.283185307179586476925286766559;
    for (int f = 0; f < nf; ++f) {
      double v = (f == 1 || f == 4 || f == 6 || f == 17) ? 1.0 : 0.0;
      for (int m = 0; m < 2; ++m) {
        double u[5];
        for (int q = 0; q < 5; ++q) u[q] = (hash_uniform(a.seed, 1000 + f, 8 * m + q) + 1.0) * 0.5;
        int kv[3];
        for (int q = 0; q < 3; ++q) {
          int t = (int)floor(u[q] * 5.0);
          kv[q] = (t > 4 ? 4 : t) - 2;
        }
        if (kv[0] == 0 && kv[1] == 0 && kv[2] == 0) kv[0] = 1;
        const double phase = pi2 * u[3];
        const double amp = 0.5 + 0.5 * u[4];
        const double arg = pi2 * (kv[0] * x + kv[1] * y + kv[2] * z) / len + phase;
        v += eps * amp * sin(arg);
      }
      set[f * L.gfs + c] = v;
    }
    return;
  }
}

// ------------------------------------------------------------------ norms
// Partials per CTA: rows (z, y) are dealt round-robin to kNormBlocks CTAs; each thread
// strides x; then a fixed shared-memory tree.  Everything is a fixed function of the
// geometry, hence deterministic.
__device__ double block_sum(double v, double* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int w = kNormThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  const double r = sh[0];
  __syncthreads();
  return r;
}
__device__ double block_max(double v, double* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int w = kNormThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + w]);
    __syncthreads();
  }
  const double r = sh[0];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kNormThreads) norms_pass1(Layout L, const double* set,
                                                            int system, double* scratch,
                                                            int len) {
  __shared__ double sh[kNormThreads];
  const int64_t rows = L.ny * L.nz;
  double* out = scratch + (int64_t)blockIdx.x * len;
  for (int f = 0; f < L.n_gf; ++f) {
    const double* F = set + f * L.gfs;
    double s2 = 0.0, mx = 0.0, s1 = 0.0;
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
      const int64_t j = r % L.ny, k = r / L.ny;
      for (int64_t i = threadIdx.x; i < L.nx; i += blockDim.x) {
        const double v = F[L.idx(i, j, k)];
        s2 = fma(v, v, s2);
        s1 += v;
        mx = fmax(mx, fabs(v));
      }
    }
    s2 = block_sum(s2, sh);
    s1 = block_sum(s1, sh);
    mx = block_max(mx, sh);
    if (threadIdx.x == 0) { out[3 * f] = s2; out[3 * f + 1] = mx; out[3 * f + 2] = s1; }
  }
  if (system == 1) {
    double e = 0.0;
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
      const int64_t j = r % L.ny, k = r / L.ny;
      for (int64_t i = threadIdx.x; i < L.nx; i += blockDim.x) {
        const int64_t c = L.idx(i, j, k);
        const double a = set[L.gfs + c], b = set[2 * L.gfs + c], d = set[3 * L.gfs + c],
                     q = set[4 * L.gfs + c];
        e += 0.5 * (a * a + b * b + d * d + q * q);
      }
    }
    e = block_sum(e, sh);
    if (threadIdx.x == 0) out[3 * L.n_gf] = e;
  }
}

__global__ void norms_pass2(const double* scratch, int len, int nblocks, double* out) {
  for (int v = threadIdx.x; v < len; v += blockDim.x) {
    const bool is_max = (v % 3 == 1);  // slot 3f+1 = max|f|; the energy slot is 3 n_gf
    double acc = 0.0;
    for (int b = 0; b < nblocks; ++b) {
      const double x = scratch[(int64_t)b * len + v];
      acc = is_max ? fmax(acc, x) : acc + x;
    }
    out[v] = acc;
  }
}

}  // namespace

cudaError_t ghost_fill(const Layout& L, double* set, FaceDst z, cudaStream_t st) {
  const int T = 256;
  const int g = L.g;
  {
    const int64_t n = L.ny * L.nz * g;
    fill_x<<<dim3((unsigned)((n + T - 1) / T), L.n_gf), T, 0, st>>>(L, set);
  }
  {
    const int64_t n = (L.nx + 2 * g) * g * L.nz;
    fill_y<<<dim3((unsigned)((n + T - 1) / T), L.n_gf), T, 0, st>>>(L, set);
  }
  {
    const int64_t n = (L.nx + 2 * g) * (L.ny + 2 * g) * g;
    push_z<<<dim3((unsigned)((n + T - 1) / T), L.n_gf), T, 0, st>>>(L, set, z.lo, z.hi);
  }
  return cudaGetLastError();
}

cudaError_t push_z_planes(const Layout& L, const double* set, FaceDst z, cudaStream_t st) {
  const int T = 256;
  const int64_t n = (L.nx + 2 * L.g) * (L.ny + 2 * L.g) * L.g;
  push_z<<<dim3((unsigned)((n + T - 1) / T), L.n_gf), T, 0, st>>>(L, set, z.lo, z.hi);
  return cudaGetLastError();
}

cudaError_t init_interior(const Layout& L, double* set, const InitArgs& a, cudaStream_t st) {
  dim3 block(128);
  dim3 grid((unsigned)((L.nx + 127) / 128), (unsigned)L.ny, (unsigned)L.nz);
  init_kernel<<<grid, block, 0, st>>>(L, set, a);
  return cudaGetLastError();
}

cudaError_t norms_partial(const Layout& L, const double* set, int system, double* scratch,
                          double* out_dev, cudaStream_t st) {
  const int len = 3 * L.n_gf + (system == 1 ? 1 : 0);
  norms_pass1<<<kNormBlocks, kNormThreads, 0, st>>>(L, set, system, scratch, len);
  norms_pass2<<<1, 128, 0, st>>>(scratch, len, kNormBlocks, out_dev);
  return cudaGetLastError();
}

}  // namespace chemora

// ------------------------------------------------------------------ fused energy monitor
// NEXT-3: the stage-4 kernel leaves one partial of
// sum 1/2 (rho^2 + v.v) per CTA (Fig. 1 "Energy"); one CTA sums them in a
// fixed order (strided per thread, then a fixed tree), so the result is deterministic.
namespace chemora {
namespace {
__global__ void __launch_bounds__(1024) monitor_reduce_kernel(const double* p, int64_t n, double vol, double* out) {
  __shared__ double sh[1024];
  double s = 0.0;
  for (int64_t t = threadIdx.x; t < n; t += 1024) s += p[t];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = vol * sh[0];
}
}  // namespace

cudaError_t monitor_reduce(const double* partials, int64_t n, double vol, double* out, cudaStream_t st) {
  monitor_reduce_kernel<<<1, 1024, 0, st>>>(partials, n, vol, out);
  return cudaGetLastError();
}
}  // namespace chemora
