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
  // variants 0 and 1: one thread per point (0: banded CTA order, 1: plain order); 4:
  // persistent TMA z-march (any W, wave_tma.cu); the stage pairs (8) are launched by the
  // step driver (wave_fused3.cu).  RHS-only uses the simple kernel.  The fused energy
  // monitor (NEXT-3) lives in the one-thread-per-point stage-4 kernel.
  const bool mon = stage == 4 && a.mon_partials != nullptr;
  if (a.variant == 4 && stage >= 1 && !mon) return wave_tma_stage(a, stage, st);
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
