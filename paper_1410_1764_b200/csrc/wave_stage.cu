// wave_stage.cu -- fused RHS + RK4-stage + ghost-image kernels for the first-order scalar
// wave equation, Eq. 1 (Fig. 1):
//     d_t u = rho,   d_t rho = delta^ij d_i v_j,   d_t v_i = d_i rho
// discretised with centered finite differences of order 2W (4th order
// = W 2 is the default, R2) and advanced by classical RK4 in
// the one-HBM-pass-per-substage y/Q/B/C arrangement of DESIGN.md §RK4:
//   stage 1 (in y):  B = y + dt/2 k1
//   stage 2 (in B):  Q = (y + B)/3 + dt/3 k2 ;  C = y + dt/2 k2 ;  Q.u = dt/6 y.rho + dt/3 B.rho
//   stage 3 (in C):  B = y + dt k3            ;  Q.u += dt/3 C.rho
//   stage 4 (in B):  y = Q + B/3 + dt/6 k4    ;  y.u += Q.u + dt/6 B.rho
// (u is never differentiated, so its stage values are dead and only a carry is kept.)
// Each stage writes the periodic ghost images of its output (fused boundary fill) and,
// for a z-slab, stores its boundary planes into the neighbour's ghost planes.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>
#include "grid.hpp"
#include "kernels.hpp"
#include "device_common.cuh"
#include "tma.cuh"
#include "wave_common.cuh"

namespace chemora {
namespace {

using namespace wave;

// ------------------------------------------------------------------ simple kernel
// One thread per interior point, every stencil operand loaded through the read-only
// path.  Used for RHS-only evaluation, as the variant-1 reference for tile-independence
// tests, and as the fallback for shapes the tiled kernel does not take.
//
// CTA order (`band` > 0): a 1-D grid walked as (x-tile fastest, then `band` y-tiles, then z,
// then the next group of y-tiles).  The CTAs resident at any moment then cover a band of
// band*8 rows over a few consecutive planes, so the z-stencil planes (k +- 1, 2) and the
// y-halo rows are re-read from L2 (a few MB of working set) instead of HBM.  With band = 0
// the grid is the plain 3-D (x-tile, y-tile, z) launch.
template <int STAGE, int W>
__global__ void __launch_bounds__(256) wave_simple(StageLaunch a, WaveK K, double* rhs_dst, int band) {
  const Layout& L = a.L;
  int bx, by, bz;
  if (band > 0) {
    const int ntx = (int)((L.nx + 31) >> 5), nty = (int)((L.ny + blockDim.y - 1) / blockDim.y);
    const int ntz = (int)((a.k_end - a.k_begin + blockDim.z - 1) / blockDim.z);
    int lin = blockIdx.x;
    bx = lin % ntx; lin /= ntx;
    const int byl = lin % band; lin /= band;
    bz = lin % ntz;
    by = (lin / ntz) * band + byl;
    if (by >= nty) return;
  } else {
    bx = blockIdx.x; by = blockIdx.y; bz = blockIdx.z;
  }
  const int i = bx * blockDim.x + threadIdx.x;
  const int j = by * blockDim.y + threadIdx.y;
  const int k = a.k_begin + bz * blockDim.z + threadIdx.z;
  const bool mon = STAGE == 4 && a.mon_partials != nullptr;
  double e = 0.0;  // NEXT-3: energy density of the new state, reduced per CTA
  if (i < L.nx && j < L.ny && k < a.k_end) {
  const int64_t c = L.idx(i, j, k);
  const int64_t gfs = L.gfs;
  const double* in = STAGE == 0 ? a.s.y : (STAGE == 1 ? a.s.y : (STAGE == 2 ? a.s.b : (STAGE == 3 ? a.s.c : a.s.b)));
  const double* rho = in + GRHO * gfs;
  double S[5], kk[5];
#pragma unroll
  for (int f = 1; f <= 4; ++f) S[f] = __ldg(in + f * gfs + c);
  const double dxr = d1<W>(rho, c, 1) * K.ih[0];
  const double dyr = d1<W>(rho, c, L.px) * K.ih[1];
  const double dzr = d1<W>(rho, c, L.plane) * K.ih[2];
  const double dv1 = d1<W>(in + GV1 * gfs, c, 1) * K.ih[0];
  const double dv2 = d1<W>(in + GV2 * gfs, c, L.px) * K.ih[1];
  const double dv3 = d1<W>(in + GV3 * gfs, c, L.plane) * K.ih[2];
  kk[GRHO] = dv1 + dv2 + dv3;
  kk[GV1] = dxr;
  kk[GV2] = dyr;
  kk[GV3] = dzr;
  if (STAGE == 0) {
    const int64_t ni = L.nx * L.ny * L.nz;
    const int64_t o = (int64_t(k) * L.ny + j) * L.nx + i;
    rhs_dst[o] = S[GRHO];
#pragma unroll
    for (int f = 1; f <= 4; ++f) rhs_dst[f * ni + o] = kk[f];
    return;
  }
  double Y[5] = {0, 0, 0, 0, 0}, Qv[5] = {0, 0, 0, 0, 0}, yu = 0.0, qu = 0.0;
  if (STAGE == 2 || STAGE == 3) {
#pragma unroll
    for (int f = 1; f <= 4; ++f) Y[f] = a.s.y[f * gfs + c];
  }
  if (STAGE == 1) {
#pragma unroll
    for (int f = 1; f <= 4; ++f) Y[f] = S[f];
  }
  if (STAGE == 3) qu = a.s.q[c];
  if (STAGE == 4) {
#pragma unroll
    for (int f = 1; f <= 4; ++f) Qv[f] = a.s.q[f * gfs + c];
    qu = a.s.q[c];
    yu = a.s.y[c];
  }
  double* out = STAGE == 1 ? a.s.b : (STAGE == 2 ? a.s.c : (STAGE == 3 ? a.s.b : a.s.y));
  const FaceDst fd = a.img[STAGE > 0 ? STAGE - 1 : 0];
  const bool nf = near_face(L, i, j, k);
  const unsigned long long code0 = a.step * (unsigned long long)L.n_gf;
  auto put = [&](int f, double v) {
    out[f * gfs + c] = v;
    if (nf) store_images(out + f * gfs, fd.lo + f * gfs, fd.hi + f * gfs, L, i, j, k, v);
    if (STAGE == 4) check_finite(a.nan_flag, code0 + f, v);
    if (STAGE == 4 && f >= 1) e = fma(0.5 * v, v, e);  // eps = 1/2 (rho^2 + v.v), Fig. 1
  };
  auto putq = [&](int f, double v) { a.s.q[f * gfs + c] = v; };
  wave_update<STAGE>(K, S, kk, Y, Qv, yu, qu, put, putq);
  }
  if (mon) {
    // deterministic CTA reduction (fixed shuffle tree, then warps in order)
    __shared__ double wsum[32];
    const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) e += __shfl_xor_sync(0xffffffffu, e, off);
    if ((tid & 31) == 0) wsum[tid >> 5] = e;
    __syncthreads();
    if (tid == 0) {
      const int nw = (blockDim.x * blockDim.y * blockDim.z) >> 5;
      double s = 0.0;
      for (int w = 0; w < nw; ++w) s += wsum[w];
      const int ntx = (int)((L.nx + 31) >> 5), nty = (int)((L.ny + blockDim.y - 1) / blockDim.y);
      a.mon_partials[((int64_t)bz * nty + by) * ntx + bx] = s;
    }
  }
}

// ------------------------------------------------------------------ z-march kernel
// 2.5-D: a CTA owns a BX x BY column tile of the x-y plane and marches up a chunk of z
// planes.  The z-stencil operands (rho and v3, the only GFs differentiated along z) live in
// a (2W+1)-deep register queue per thread, so every plane of them is loaded from HBM once;
// x/y neighbours come through L1 (the CTA's own rows) or L2 (tile halos).  Arithmetic is
// instruction-for-instruction that of wave_simple (bitwise identical results).
template <int STAGE, int W, int BX, int BY>
__global__ void __launch_bounds__(BX * BY, 4) wave_zmarch(StageLaunch a, WaveK K, int kchunk) {
  const Layout& L = a.L;
  const int i = blockIdx.x * BX + threadIdx.x;
  const int j = blockIdx.y * BY + threadIdx.y;
  const int kb = a.k_begin + blockIdx.z * kchunk;
  const int ke = min(kb + kchunk, a.k_end);
  if (i >= L.nx || j >= L.ny || kb >= ke) return;
  const int64_t gfs = L.gfs, px = L.px, pl = L.plane;
  const double* in = STAGE == 1 ? a.s.y : (STAGE == 2 ? a.s.b : (STAGE == 3 ? a.s.c : a.s.b));
  const double* __restrict__ rho = in + GRHO * gfs;
  const double* __restrict__ v1 = in + GV1 * gfs;
  const double* __restrict__ v2 = in + GV2 * gfs;
  const double* __restrict__ v3 = in + GV3 * gfs;
  double* out = STAGE == 1 ? a.s.b : (STAGE == 2 ? a.s.c : (STAGE == 3 ? a.s.b : a.s.y));
  const FaceDst fd = a.img[STAGE - 1];
  const unsigned long long code0 = a.step * (unsigned long long)L.n_gf;
  int64_t c = L.idx(i, j, kb);
  double qr[2 * W + 1], qw[2 * W + 1];
#pragma unroll
  for (int q = 0; q < 2 * W; ++q) {
    qr[q] = __ldg(rho + c + (q - W) * pl);
    qw[q] = __ldg(v3 + c + (q - W) * pl);
  }
#pragma unroll 1
  for (int k = kb; k < ke; ++k, c += pl) {
    qr[2 * W] = __ldg(rho + c + W * pl);
    qw[2 * W] = __ldg(v3 + c + W * pl);
    double S[5], kk[5];
    S[GRHO] = qr[W];
    S[GV1] = __ldg(v1 + c);
    S[GV2] = __ldg(v2 + c);
    S[GV3] = qw[W];
    double dzr = 0.0, dv3 = 0.0;
#pragma unroll
    for (int q = W; q >= 1; --q) {
      dzr = fma(D1W<W>::c(q), qr[W + q] - qr[W - q], dzr);
      dv3 = fma(D1W<W>::c(q), qw[W + q] - qw[W - q], dv3);
    }
    const double dxr = d1<W>(rho, c, 1) * K.ih[0];
    const double dyr = d1<W>(rho, c, px) * K.ih[1];
    dzr = dzr * K.ih[2];
    const double dv1 = d1<W>(v1, c, 1) * K.ih[0];
    const double dv2 = d1<W>(v2, c, px) * K.ih[1];
    dv3 = dv3 * K.ih[2];
    kk[GRHO] = dv1 + dv2 + dv3;
    kk[GV1] = dxr;
    kk[GV2] = dyr;
    kk[GV3] = dzr;
    double Y[5] = {0, 0, 0, 0, 0}, Qv[5] = {0, 0, 0, 0, 0}, yu = 0.0, qu = 0.0;
    if (STAGE == 2 || STAGE == 3) {
#pragma unroll
      for (int f = 1; f <= 4; ++f) Y[f] = a.s.y[f * gfs + c];
    }
    if (STAGE == 1) {
#pragma unroll
      for (int f = 1; f <= 4; ++f) Y[f] = S[f];
    }
    if (STAGE == 3) qu = a.s.q[c];
    if (STAGE == 4) {
#pragma unroll
      for (int f = 1; f <= 4; ++f) Qv[f] = a.s.q[f * gfs + c];
      qu = a.s.q[c];
      yu = a.s.y[c];
    }
    const bool nf = near_face(L, i, j, k);
    auto put = [&](int f, double v) {
      out[f * gfs + c] = v;
      if (nf) store_images(out + f * gfs, fd.lo + f * gfs, fd.hi + f * gfs, L, i, j, k, v);
      if (STAGE == 4) check_finite(a.nan_flag, code0 + f, v);
    };
    auto putq = [&](int f, double v) { a.s.q[f * gfs + c] = v; };
    wave_update<STAGE>(K, S, kk, Y, Qv, yu, qu, put, putq);
#pragma unroll
    for (int q = 0; q < 2 * W; ++q) {
      qr[q] = qr[q + 1];
      qw[q] = qw[q + 1];
    }
  }
}

template <int STAGE, int W>
cudaError_t launch_zmarch(const StageLaunch& a, const WaveK& K, cudaStream_t st) {
  constexpr int BX = 32, BY = 8;
  const int nk = a.k_end - a.k_begin;
  if (nk <= 0) return cudaSuccess;
  const int64_t tiles = ((a.L.nx + BX - 1) / BX) * ((a.L.ny + BY - 1) / BY);
  // enough CTAs for ~4 waves of (SMs x 4 resident CTAs), but chunks of >= 8 planes
  int64_t want = (4 * device_sm_count() * 4 + tiles - 1) / tiles;
  int chunk = (int)((nk + want - 1) / want);
  if (chunk < 8) chunk = 8;
  if (chunk > nk) chunk = nk;
  const int nchunks = (nk + chunk - 1) / chunk;
  dim3 grid((unsigned)((a.L.nx + BX - 1) / BX), (unsigned)((a.L.ny + BY - 1) / BY), (unsigned)nchunks);
  wave_zmarch<STAGE, W, BX, BY><<<grid, dim3(BX, BY, 1), 0, st>>>(a, K, chunk);
  return cudaGetLastError();
}

template <int STAGE, int W>
cudaError_t launch_simple(const StageLaunch& a, const WaveK& K, double* dst, cudaStream_t st) {
  const int nk = a.k_end - a.k_begin;
  if (nk <= 0) return cudaSuccess;
  // CTA shape 32 x 8 x 1 (32 x 4 x 2 and 32 x 2 x 4, which keep z neighbours inside the
  // CTA, measured no faster: profiles/r1_wave_design_study.md)
  const int BZ = 1, BY = 8;
  dim3 block(32, BY, BZ);
  const int ntx = (int)((a.L.nx + 31) / 32), nty = (int)((a.L.ny + BY - 1) / BY);
  const int ntz = (nk + BZ - 1) / BZ;
  int band = a.band;
  if (band < 0) {
    // auto: keep ~5 planes x 17 streams of the band under ~40 MB of L2
    const double rows = 40e6 / (5.0 * 17.0 * 8.0 * (double)a.L.nx);
    band = 1;
    while (band * 2 * BY <= rows && band * 2 <= nty) band *= 2;
  }
  if (STAGE == 0 || a.variant == 1) band = 0;
  if (band > 0) {
    const int groups = (nty + band - 1) / band;
    const long long n = (long long)ntx * band * ntz * groups;
    wave_simple<STAGE, W><<<dim3((unsigned)n), block, 0, st>>>(a, K, dst, band);
  } else {
    dim3 grid((unsigned)ntx, (unsigned)nty, (unsigned)ntz);
    wave_simple<STAGE, W><<<grid, block, 0, st>>>(a, K, dst, 0);
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ shared-memory brick kernel
// A CTA of 32 x 8 threads owns a 32 x 8 x NZ brick.  It first copies the stencil operands
// of the brick with their halos into shared memory with coalesced loads -- rho with the
// full x/y/z halo, v1 with the x halo, v2 with the y halo, v3 with the z halo -- then every
// thread evaluates its NZ points (one z column) from shared memory.  Compared with
// wave_simple this replaces ~20 global loads per point by ~8 (the halo amortised over the
// brick) plus shared-memory reads, cutting LSU/L1 traffic.  Same arithmetic, bit-identical.
template <int STAGE, int W, int NZ>
__global__ void __launch_bounds__(256) wave_brick(StageLaunch a, WaveK K) {
  constexpr int TX = 32, TY = 8, RX = TX + 2 * W, RY = TY + 2 * W, RZ = NZ + 2 * W;
  constexpr int NR = RZ * RY * RX, N1 = NZ * TY * RX, N2 = NZ * RY * TX, N3 = RZ * TY * TX;
  extern __shared__ __align__(16) double bsm[];
  double* sR = bsm;
  double* s1 = sR + NR;
  double* s2 = s1 + N1;
  double* s3 = s2 + N2;
  const Layout& L = a.L;
  const int i0 = blockIdx.x * TX, j0 = blockIdx.y * TY, k0 = a.k_begin + blockIdx.z * NZ;
  const int tid = threadIdx.y * TX + threadIdx.x;
  const int64_t gfs = L.gfs;
  const double* in = STAGE == 1 ? a.s.y : (STAGE == 2 ? a.s.b : (STAGE == 3 ? a.s.c : a.s.b));
  const int kmax = a.k_end + W;  // planes beyond k_end + W are never needed
  auto fill = [&](double* dst, const double* src, int nx, int ny, int nz, int ox, int oy, int oz, int n) {
    for (int e = tid; e < n; e += 256) {
      const int x = e % nx, r = e / nx, y = r % ny, z = r / ny;
      const int gi = i0 + x - ox, gj = j0 + y - oy, gk = k0 + z - oz;
      // clamp to the padded box (values outside the interior + ghosts are never used)
      const bool ok = gi < L.nx + L.g && gj < L.ny + L.g && gk < kmax;
      dst[e] = ok ? __ldg(src + L.idx(gi, gj, gk)) : 0.0;
      (void)nz;
    }
  };
  fill(sR, in + GRHO * gfs, RX, RY, RZ, W, W, W, NR);
  fill(s1, in + GV1 * gfs, RX, TY, NZ, W, 0, 0, N1);
  fill(s2, in + GV2 * gfs, TX, RY, NZ, 0, W, 0, N2);
  fill(s3, in + GV3 * gfs, TX, TY, RZ, 0, 0, W, N3);
  __syncthreads();
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int i = i0 + tx, j = j0 + ty;
  if (i >= L.nx || j >= L.ny) return;
  double* out = STAGE == 1 ? a.s.b : (STAGE == 2 ? a.s.c : (STAGE == 3 ? a.s.b : a.s.y));
  const FaceDst fd = a.img[STAGE - 1];
  const unsigned long long code0 = a.step * (unsigned long long)L.n_gf;
#pragma unroll 1
  for (int z = 0; z < NZ; ++z) {
    const int k = k0 + z;
    if (k >= a.k_end) break;
    const int64_t c = L.idx(i, j, k);
    const int cr = ((z + W) * RY + ty + W) * RX + tx + W;
    const int c1 = (z * TY + ty) * RX + tx + W;
    const int c2 = (z * RY + ty + W) * TX + tx;
    const int c3 = ((z + W) * TY + ty) * TX + tx;
    double S[5], kk[5];
    S[GRHO] = sR[cr];
    S[GV1] = s1[c1];
    S[GV2] = s2[c2];
    S[GV3] = s3[c3];
    double dxr = 0.0, dyr = 0.0, dzr = 0.0, dv1 = 0.0, dv2 = 0.0, dv3 = 0.0;
#pragma unroll
    for (int q = W; q >= 1; --q) {
      const double w = D1W<W>::c(q);
      dxr = fma(w, sR[cr + q] - sR[cr - q], dxr);
      dyr = fma(w, sR[cr + q * RX] - sR[cr - q * RX], dyr);
      dzr = fma(w, sR[cr + q * RX * RY] - sR[cr - q * RX * RY], dzr);
      dv1 = fma(w, s1[c1 + q] - s1[c1 - q], dv1);
      dv2 = fma(w, s2[c2 + q * TX] - s2[c2 - q * TX], dv2);
      dv3 = fma(w, s3[c3 + q * TX * TY] - s3[c3 - q * TX * TY], dv3);
    }
    dxr = dxr * K.ih[0];
    dyr = dyr * K.ih[1];
    dzr = dzr * K.ih[2];
    dv1 = dv1 * K.ih[0];
    dv2 = dv2 * K.ih[1];
    dv3 = dv3 * K.ih[2];
    kk[GRHO] = dv1 + dv2 + dv3;
    kk[GV1] = dxr;
    kk[GV2] = dyr;
    kk[GV3] = dzr;
    double Y[5] = {0, 0, 0, 0, 0}, Qv[5] = {0, 0, 0, 0, 0}, yu = 0.0, qu = 0.0;
    if (STAGE == 2 || STAGE == 3) {
#pragma unroll
      for (int f = 1; f <= 4; ++f) Y[f] = a.s.y[f * gfs + c];
    }
    if (STAGE == 1) {
#pragma unroll
      for (int f = 1; f <= 4; ++f) Y[f] = S[f];
    }
    if (STAGE == 3) qu = a.s.q[c];
    if (STAGE == 4) {
#pragma unroll
      for (int f = 1; f <= 4; ++f) Qv[f] = a.s.q[f * gfs + c];
      qu = a.s.q[c];
      yu = a.s.y[c];
    }
    const bool nf = near_face(L, i, j, k);
    auto put = [&](int f, double v) {
      out[f * gfs + c] = v;
      if (nf) store_images(out + f * gfs, fd.lo + f * gfs, fd.hi + f * gfs, L, i, j, k, v);
      if (STAGE == 4) check_finite(a.nan_flag, code0 + f, v);
    };
    auto putq = [&](int f, double v) { a.s.q[f * gfs + c] = v; };
    wave_update<STAGE>(K, S, kk, Y, Qv, yu, qu, put, putq);
  }
}

template <int STAGE, int W>
cudaError_t launch_brick(const StageLaunch& a, const WaveK& K, cudaStream_t st) {
  constexpr int NZ = 4;
  const int nk = a.k_end - a.k_begin;
  if (nk <= 0) return cudaSuccess;
  constexpr int RX = 32 + 2 * W, RY = 8 + 2 * W, RZ = NZ + 2 * W;
  constexpr int bytes = 8 * (RZ * RY * RX + NZ * 8 * RX + NZ * RY * 32 + RZ * 8 * 32);
  static std::atomic<uint64_t> attr_done{0};
  if (cudaError_t e = smem_optin((const void*)wave_brick<STAGE, W, NZ>, bytes, attr_done); e != cudaSuccess) return e;
  dim3 grid((unsigned)((a.L.nx + 31) / 32), (unsigned)((a.L.ny + 7) / 8), (unsigned)((nk + NZ - 1) / NZ));
  wave_brick<STAGE, W, NZ><<<grid, dim3(32, 8, 1), bytes, st>>>(a, K);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ TMA z-march kernel
// The B200-native tiling: a CTA owns a TX x TY tile of the x-y plane and marches up a chunk
// of z planes.  One elected producer thread streams the stencil operands into shared
// memory with TMA (cp.async.bulk.tensor, 4-D maps over a state set [gf][z][y][x]):
//   ring Z (depth 2W+3): per plane, rho with its x/y halo and v3 -- the two GFs that are
//                        differentiated along z, so 2W+1 planes of them stay resident;
//   ring P (depth 3):    per plane, v1 with its x halo and v2 with its y halo.
// Eight consumer warps compute two points per thread per plane from shared memory (x/y/z
// derivatives all from SMEM, no redundant HBM or L2 reads), load the pointwise operands
// (y, Q) with coalesced loads, and store the stage outputs (+ ghost images).  Full/empty
// mbarriers per slot; the producer runs up to 3 planes ahead.  Arithmetic is operation-for-
// operation that of wave_simple (bitwise-identical results; this file has no FMA
// contraction).
template <int W>
struct TmaCfg {
  static constexpr int TX = 32, TY = 16;
  static constexpr int RX = TX + 2 * W, RY = TY + 2 * W;
  static constexpr int RZ = 2 * W + 3, RP = 3;
  static constexpr int r128(int b) { return (b + 127) / 128 * 128; }
  static constexpr int ZRHO_B = r128(RX * RY * 8), ZV3_B = r128(TX * TY * 8), ZSLOT = ZRHO_B + ZV3_B;
  static constexpr int PV1_B = r128(RX * TY * 8), PV2_B = r128(TX * RY * 8), PSLOT = PV1_B + PV2_B;
  static constexpr uint32_t ZBYTES = (RX * RY + TX * TY) * 8;
  static constexpr uint32_t PBYTES = (RX * TY + TX * RY) * 8;
  static constexpr int SMEM = RZ * ZSLOT + RP * PSLOT + (2 * RZ + 2 * RP) * 8;
  static constexpr int NCW = 8;  // consumer warps
};

template <int W>
__device__ __forceinline__ double d1s(const double* f, int c, int s) {
  double acc = 0.0;
#pragma unroll
  for (int q = W; q >= 1; --q) acc = fma(D1W<W>::c(q), f[c + q * s] - f[c - q * s], acc);
  return acc;
}

template <int STAGE, int W>
__global__ void __launch_bounds__(288, 2)
    wave_tma(const __grid_constant__ CUtensorMap tmR, const __grid_constant__ CUtensorMap tmV1,
             const __grid_constant__ CUtensorMap tmV2, const __grid_constant__ CUtensorMap tmC,
             StageLaunch a, WaveK K, int kchunk) {
  using Cf = TmaCfg<W>;
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* zbase = smem;
  unsigned char* pbase = smem + Cf::RZ * Cf::ZSLOT;
  uint64_t* zfull = reinterpret_cast<uint64_t*>(pbase + Cf::RP * Cf::PSLOT);
  uint64_t* zempty = zfull + Cf::RZ;
  uint64_t* pfull = zempty + Cf::RZ;
  uint64_t* pempty = pfull + Cf::RP;
  const Layout& L = a.L;
  const int i0 = blockIdx.x * Cf::TX, j0 = blockIdx.y * Cf::TY;
  const int kb = a.k_begin + blockIdx.z * kchunk;
  const int ke = min(kb + kchunk, a.k_end);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < Cf::RZ; ++s) { mbar_init(zfull + s, 1); mbar_init(zempty + s, Cf::NCW); }
    for (int s = 0; s < Cf::RP; ++s) { mbar_init(pfull + s, 1); mbar_init(pempty + s, Cf::NCW); }
    fence_mbar_init();
  }
  __syncthreads();
  if (kb >= ke) return;
  const int g = L.g;
  const int nk = ke - kb;

  if (warp == Cf::NCW) {  // ---------------- producer
    if (lane == 0) {
      prefetch_tmap(&tmR); prefetch_tmap(&tmV1); prefetch_tmap(&tmV2); prefetch_tmap(&tmC);
      auto loadZ = [&](int t) {  // plane kb - W + t
        const int s = t % Cf::RZ, n = t / Cf::RZ;
        if (n > 0) mbar_wait(zempty + s, (n - 1) & 1);
        unsigned char* dst = zbase + s * Cf::ZSLOT;
        const int zc = g + kb - W + t;
        mbar_arrive_expect_tx(zfull + s, Cf::ZBYTES);
        tma_load_4d(dst, &tmR, zfull + s, kXOff + i0 - W, g + j0 - W, zc, GRHO);
        tma_load_4d(dst + Cf::ZRHO_B, &tmC, zfull + s, kXOff + i0, g + j0, zc, GV3);
      };
      auto loadP = [&](int t) {  // plane kb + t
        const int s = t % Cf::RP, n = t / Cf::RP;
        if (n > 0) mbar_wait(pempty + s, (n - 1) & 1);
        unsigned char* dst = pbase + s * Cf::PSLOT;
        const int zc = g + kb + t;
        mbar_arrive_expect_tx(pfull + s, Cf::PBYTES);
        tma_load_4d(dst, &tmV1, pfull + s, kXOff + i0 - W, g + j0, zc, GV1);
        tma_load_4d(dst + Cf::PV1_B, &tmV2, pfull + s, kXOff + i0, g + j0 - W, zc, GV2);
      };
      for (int t = 0; t < 2 * W; ++t) loadZ(t);
      for (int t = 0; t < nk; ++t) {
        loadZ(t + 2 * W);
        loadP(t);
      }
    }
    return;
  }

  // ---------------- consumers: thread (lane, warp) owns points (lane, warp) and (lane, warp+8)
  const int64_t gfs = L.gfs;
  double* out = STAGE == 1 ? a.s.b : (STAGE == 2 ? a.s.c : (STAGE == 3 ? a.s.b : a.s.y));
  const FaceDst fd = a.img[STAGE - 1];
  const unsigned long long code0 = a.step * (unsigned long long)L.n_gf;
  const int i = i0 + lane;
  for (int t = 0; t < 2 * W; ++t) mbar_wait(zfull + t % Cf::RZ, (t / Cf::RZ) & 1);
#pragma unroll 1
  for (int t = 0; t < nk; ++t) {
    const int k = kb + t;
    // pointwise operands first so their latency overlaps the barrier wait
    double Y[2][5], Qv[2][5], yu[2], qu[2];
    int64_t cc[2];
    bool live[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = j0 + warp + 8 * h;
      live[h] = i < L.nx && j < L.ny;
      cc[h] = L.idx(i, j, k);
#pragma unroll
      for (int f = 0; f < 5; ++f) { Y[h][f] = 0.0; Qv[h][f] = 0.0; }
      yu[h] = 0.0; qu[h] = 0.0;
      if (live[h]) {
        if (STAGE == 2 || STAGE == 3) {
#pragma unroll
          for (int f = 1; f <= 4; ++f) Y[h][f] = a.s.y[f * gfs + cc[h]];
        }
        if (STAGE == 3) qu[h] = a.s.q[cc[h]];
        if (STAGE == 4) {
#pragma unroll
          for (int f = 1; f <= 4; ++f) Qv[h][f] = a.s.q[f * gfs + cc[h]];
          qu[h] = a.s.q[cc[h]];
          yu[h] = a.s.y[cc[h]];
        }
      }
    }
    mbar_wait(zfull + (t + 2 * W) % Cf::RZ, ((t + 2 * W) / Cf::RZ) & 1);
    mbar_wait(pfull + t % Cf::RP, (t / Cf::RP) & 1);
    const double* zr[2 * W + 1];
    const double* zv[2 * W + 1];
#pragma unroll
    for (int q = 0; q <= 2 * W; ++q) {
      const unsigned char* sl = zbase + ((t + q) % Cf::RZ) * Cf::ZSLOT;
      zr[q] = reinterpret_cast<const double*>(sl);
      zv[q] = reinterpret_cast<const double*>(sl + Cf::ZRHO_B);
    }
    const unsigned char* ps = pbase + (t % Cf::RP) * Cf::PSLOT;
    const double* sv1 = reinterpret_cast<const double*>(ps);
    const double* sv2 = reinterpret_cast<const double*>(ps + Cf::PV1_B);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int ty = warp + 8 * h;
      const int cr = (ty + W) * Cf::RX + (lane + W);  // rho box index
      const int cv = ty * Cf::TX + lane;              // centre box index
      double S[5], kk[5];
      S[GRHO] = zr[W][cr];
      S[GV1] = sv1[ty * Cf::RX + lane + W];
      S[GV2] = sv2[(ty + W) * Cf::TX + lane];
      S[GV3] = zv[W][cv];
      double dzr = 0.0, dv3 = 0.0;
#pragma unroll
      for (int q = W; q >= 1; --q) {
        dzr = fma(D1W<W>::c(q), zr[W + q][cr] - zr[W - q][cr], dzr);
        dv3 = fma(D1W<W>::c(q), zv[W + q][cv] - zv[W - q][cv], dv3);
      }
      const double dxr = d1s<W>(zr[W], cr, 1) * K.ih[0];
      const double dyr = d1s<W>(zr[W], cr, Cf::RX) * K.ih[1];
      dzr = dzr * K.ih[2];
      const double dv1 = d1s<W>(sv1, ty * Cf::RX + lane + W, 1) * K.ih[0];
      const double dv2 = d1s<W>(sv2, (ty + W) * Cf::TX + lane, Cf::TX) * K.ih[1];
      dv3 = dv3 * K.ih[2];
      kk[GRHO] = dv1 + dv2 + dv3;
      kk[GV1] = dxr;
      kk[GV2] = dyr;
      kk[GV3] = dzr;
      if (STAGE == 1) {
#pragma unroll
        for (int f = 1; f <= 4; ++f) Y[h][f] = S[f];
      }
      if (live[h]) {
        const int j = j0 + ty;
        const int64_t c = cc[h];
        const bool nf = near_face(L, i, j, k);
        auto put = [&](int f, double v) {
          out[f * gfs + c] = v;
          if (nf) store_images(out + f * gfs, fd.lo + f * gfs, fd.hi + f * gfs, L, i, j, k, v);
          if (STAGE == 4) check_finite(a.nan_flag, code0 + f, v);
        };
        auto putq = [&](int f, double v) { a.s.q[f * gfs + c] = v; };
        wave_update<STAGE>(K, S, kk, Y[h], Qv[h], yu[h], qu[h], put, putq);
      }
    }
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(pempty + t % Cf::RP);
      mbar_arrive(zempty + t % Cf::RZ);  // plane k - W is no longer needed
    }
  }
}

template <int STAGE, int W>
cudaError_t launch_tma(const StageLaunch& a, const WaveK& K, cudaStream_t st) {
  using Cf = TmaCfg<W>;
  const int nk = a.k_end - a.k_begin;
  if (nk <= 0) return cudaSuccess;
  const Layout& L = a.L;
  const double* in = STAGE == 1 ? a.s.y : (STAGE == 2 ? a.s.b : (STAGE == 3 ? a.s.c : a.s.b));
  const double* base = in - L.c0;
  CUtensorMap mR, mV1, mV2, mC;
  if (!encode_set_map(&mR, base, L.px, L.py, L.pz, L.n_gf, L.gfs, Cf::RX, Cf::RY) ||
      !encode_set_map(&mV1, base, L.px, L.py, L.pz, L.n_gf, L.gfs, Cf::RX, Cf::TY) ||
      !encode_set_map(&mV2, base, L.px, L.py, L.pz, L.n_gf, L.gfs, Cf::TX, Cf::RY) ||
      !encode_set_map(&mC, base, L.px, L.py, L.pz, L.n_gf, L.gfs, Cf::TX, Cf::TY))
    return cudaErrorInvalidValue;
  static std::atomic<uint64_t> attr_done{0};
  if (cudaError_t e = smem_optin((const void*)wave_tma<STAGE, W>, Cf::SMEM, attr_done); e != cudaSuccess) return e;
  const int tiles = (int)(((L.nx + Cf::TX - 1) / Cf::TX) * ((L.ny + Cf::TY - 1) / Cf::TY));
  // ~64-plane chunks, but at least ~8 waves of 2 CTAs x SMs when the tile count is small
  int nchunks = (nk + 63) / 64;
  const int want = (8 * 2 * device_sm_count() + tiles - 1) / tiles;
  if (nchunks < want) nchunks = want;
  int chunk = (nk + nchunks - 1) / nchunks;
  if (chunk < 4) chunk = 4;
  if (chunk > nk) chunk = nk;
  nchunks = (nk + chunk - 1) / chunk;
  dim3 grid((unsigned)((L.nx + Cf::TX - 1) / Cf::TX), (unsigned)((L.ny + Cf::TY - 1) / Cf::TY), (unsigned)nchunks);
  wave_tma<STAGE, W><<<grid, 32 * (Cf::NCW + 1), Cf::SMEM, st>>>(mR, mV1, mV2, mC, a, K, chunk);
  return cudaGetLastError();
}

WaveK make_k(const StageLaunch& a) {
  WaveK K;
  for (int d = 0; d < 3; ++d) K.ih[d] = 1.0 / a.h[d];
  K.half = 0.5; K.third = 1.0 / 3.0; K.sixth = 1.0 / 6.0;
  K.dt = a.dt; K.dt2 = a.dt / 2.0; K.dt3 = a.dt / 3.0; K.dt6 = a.dt / 6.0;
  return K;
}

template <int W>
cudaError_t dispatch_stage(const StageLaunch& a, int stage, double* dst, cudaStream_t st) {
  const WaveK K = make_k(a);
  // variant 0 (default) and 1: one thread per point (0: banded CTA order, 1: plain order);
  // 2: register-queue z-march; 3: TMA z-march (W = 2); 4: persistent TMA z-march (any W,
  // wave_tma.cu).  RHS-only uses the simple kernel.
  // the fused energy monitor (NEXT-3) lives in the one-thread-per-point stage-4 kernel
  const bool mon = stage == 4 && a.mon_partials != nullptr;
  if (a.variant == 4 && stage >= 1 && !mon) return wave_tma_stage(a, stage, st);
  if (a.variant == 5 && !mon) {
    switch (stage) {
      case 1: return launch_brick<1, W>(a, K, st);
      case 2: return launch_brick<2, W>(a, K, st);
      case 3: return launch_brick<3, W>(a, K, st);
      case 4: return launch_brick<4, W>(a, K, st);
    }
  }
  if (a.variant == 3 && W == 2 && !mon) {


    switch (stage) {
      case 1: return launch_tma<1, W>(a, K, st);
      case 2: return launch_tma<2, W>(a, K, st);
      case 3: return launch_tma<3, W>(a, K, st);
      case 4: return launch_tma<4, W>(a, K, st);
    }
  }
  if (a.variant == 2 && !mon) {
    switch (stage) {
      case 1: return launch_zmarch<1, W>(a, K, st);
      case 2: return launch_zmarch<2, W>(a, K, st);
      case 3: return launch_zmarch<3, W>(a, K, st);
      case 4: return launch_zmarch<4, W>(a, K, st);
    }
  }
  switch (stage) {
    case 0: return launch_simple<0, W>(a, K, dst, st);
    case 1: return launch_simple<1, W>(a, K, dst, st);
    case 2: return launch_simple<2, W>(a, K, dst, st);
    case 3: return launch_simple<3, W>(a, K, dst, st);
    case 4: return launch_simple<4, W>(a, K, dst, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t dispatch(const StageLaunch& a, int stage, double* dst, cudaStream_t st) {
  switch (a.fd_order) {
    case 2: return dispatch_stage<1>(a, stage, dst, st);
    case 4: return dispatch_stage<2>(a, stage, dst, st);
    case 6: return dispatch_stage<3>(a, stage, dst, st);
    case 8: return dispatch_stage<4>(a, stage, dst, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

bool encode_set_map(CUtensorMap* out, const double* set_base, int64_t px, int64_t py, int64_t pz,
                    int64_t n_gf, int64_t gfs, unsigned bx, unsigned by, unsigned bg) {
  typedef CUresult (*PFN_encode)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static PFN_encode fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess || !f)
      return false;
    fn = reinterpret_cast<PFN_encode>(f);
  }
  const cuuint64_t dims[4] = {(cuuint64_t)px, (cuuint64_t)py, (cuuint64_t)pz, (cuuint64_t)n_gf};
  const cuuint64_t strides[3] = {(cuuint64_t)(px * 8), (cuuint64_t)(px * py * 8), (cuuint64_t)(gfs * 8)};
  const cuuint32_t box[4] = {bx, by, 1, bg};
  // L2 promotion: interior rows start on 128-byte (not 256-byte) boundaries, so 256-byte
  // promotion would fetch a neighbour tile's half line with every row (measured: up to 2x
  // DRAM reads): no promotion.
  const CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_NONE;
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return fn(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(set_base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t wave_stage(const StageLaunch& a, int stage, cudaStream_t st) {
  return dispatch(a, stage, nullptr, st);
}

cudaError_t wave_rhs(const StageLaunch& a, double* dst, cudaStream_t st) {
  return dispatch(a, 0, dst, st);
}

}  // namespace chemora
