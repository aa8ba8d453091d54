// bssn_fused.cu -- BSSN kernel variant 4 (default): ONE fused kernel per RK stage, the
// derivatives computed on chip where the algebra needs them -- no derivative table in HBM.
//
// The paper's Einstein kernels are "too large in data and instructions" and need fission
// (PAPER.md:537-547, 699-700); on B200 the round-1 fission went through an HBM table of 136
// derivative slots per point (5.8x the algorithmic DRAM traffic).  Here the data that makes
// the fused kernel too large is split across the SM's three on-chip stores instead:
//
//   * shared memory holds the current z-plane of ALL 25 GFs on a 16x8 tile with a 3-point
//     halo (one TMA box (24, 14, 1, 1) per GF, double-buffered so the next plane streams in
//     while this one is used): every x and y stencil (D1, D2, upwind, mixed xy) reads it;
//   * TENSOR MEMORY holds each point's own z-column window, planes k-3 .. k+3 of all 25 GFs
//     (TMEM lane = point, 16 columns per GF; 400 of the 512 columns), shifted by one plane per
//     step: the z stencils (D1, D2, upwind) read it with one tcgen05.ld per GF;
//   * small shared helper planes hold the inner derivatives of the mixed stencils (D1_y on
//     the x-extended tile for d_x d_y, D1_z on the x- and y-extended tile for d_x d_z and
//     d_y d_z; the tile interior from the TMEM windows, the 2-point frame from L2).
//
// The CTA (one per SM, persistent over (tile, z-chunk) items) has 256 threads: every point
// of the tile is served by two threads in warps w and w+4, which share the TMEM lanes of the
// point -- one runs the curvature group G2 (trK, At, A), the other the kinematic + shift
// group G13 (phi, gt, alpha, beta, Xt, B) of bssn_point, each followed by its RK4 update.
// HBM traffic is the one-pass-per-stage floor plus L2-resident halo re-reads.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include "bssn_common.cuh"
#include "tma.cuh"

namespace chemora {
namespace {

constexpr int FX = 16, FY = 8, FPT = FX * FY;          // tile points = TMEM lanes used
constexpr int FR = 3;                                  // halo (upwind radius)
// the x halo is stored 4 wide so every TMA box row starts 16-byte aligned in global memory
// (an odd fp64 start column faults the bulk-tensor copy) and spans 24 doubles
constexpr int FRX = 4;
constexpr int FSX = FX + 2 * FRX, FSY = FY + 2 * FR, FPL = FSX * FSY;   // 24 x 14
// two threads per point: the curvature group G2 and the kinematic + shift group G13 at 255
// registers, 8 warps per SM (three groups at 168 registers, 12 warps, spilled and measured
// slower: profiles/r2_bssn_summary.md)
constexpr int NGRP = 2;
constexpr int FNT = NGRP * FPT;                        // (point, group) threads
constexpr int NWARP = FNT / 32;
constexpr int NMIX = 11;                               // GFs with mixed second derivatives
constexpr int HXW = FX + 4;                            // x-extended helper rows: i = -2 .. FX+1
constexpr int HYH = FY + 4;                            // y-extended helper columns: j = -2 .. FY+1
constexpr int TILE_BYTES = NV * FPL * 8;               // one plane of all GFs (67200 B)
constexpr int FPLS = (FPL * 8 + 127) / 128 * 16;       // GF plane stride in the tile: 128-byte aligned (336)
constexpr int TILE_STRIDE = (NV * FPLS * 8 + 1023) / 1024 * 1024;
constexpr int GZX_N = NMIX * FY * HXW, GZY_N = NMIX * HYH * FX, GYX_N = NMIX * FY * HXW;
constexpr int NMON = 14;                               // constraint monitor: [sum c_q^2, max|c_q|] x 7
// the own-column feed of plane k+3: the tile interior of that plane, one TMA box (16, 8) per GF,
// streamed in one iteration ahead into a double buffer
constexpr int FEED_PL = FPT;                            // doubles per GF (1 KB)
constexpr int FEED_STRIDE = NV * FEED_PL * 8;           // bytes per buffer (25.6 KB)
constexpr int SMEM_FUSED = 2 * TILE_STRIDE + 2 * FEED_STRIDE + 8 * (GZX_N + GZY_N + GYX_N) + 64 + 8 * NWARP * NMON;
// TMEM window feed split over the groups: [0, 13) [13, 25) -- the 11 GFs with mixed
// derivatives stay with one group each (phi, gt: G2's threads; alpha, beta: G13's)
constexpr int FEED_B1 = 13;
constexpr int FEEDN = 13;                              // max GFs fed by one thread
constexpr int NFRAME = 2 * 2 * FY + 2 * 2 * FX;        // 2-point x- and y-frames of the tile: 96
constexpr int NFI = (NMIX * NFRAME + FNT - 1) / FNT;   // frame items per thread (5)

// ---- TMEM (tcgen05) helpers: each thread reads / writes its own lane
__device__ __forceinline__ void tm_ld16(uint32_t ta, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(ta)
      : "memory");
}
__device__ __forceinline__ void tm_st16(uint32_t ta, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tm_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ double dbl(uint32_t lo, uint32_t hi) { return __hiloint2double((int)hi, (int)lo); }
__device__ __forceinline__ void cta_sync_tm() {
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
}

// z-window of GF gf: planes k-3 .. k+3 (slots 0..6) of the thread's point
struct ZWin {
  double w[7];
};
__device__ __forceinline__ ZWin zwin(uint32_t tb, int gf) {
  uint32_t r[16];
  tm_ld16(tb + 16u * (uint32_t)gf, r);
  tm_wait_ld();
  ZWin z;
#pragma unroll
  for (int s = 0; s < 7; ++s) z.w[s] = dbl(r[2 * s], r[2 * s + 1]);
  return z;
}

// Derivative provider of the fused kernel (same operation order as StencilP: D1raw, D2raw,
// D11raw with the outer sum along the first axis of the pair, ADVraw).
struct FusedP {
  const double* t;     // plane-k tile of all GFs, [gf][FSY][FSX], GF stride FPLS
  int c;               // own point's offset in a GF plane of the tile
  const double* gzx;   // [NMIX][FY][HXW]   D1raw_z, x-extended
  const double* gzy;   // [NMIX][HYH][FX]   D1raw_z, y-extended
  const double* gyx;   // [NMIX][FY][HXW]   D1raw_y, x-extended
  int hx, hy;          // own point's offsets in the x- / y-extended helper planes
  uint32_t tb;         // TMEM address of the point's lane, column 0
  __device__ __forceinline__ double v(int gf) const { return t[gf * FPLS + c]; }
  __device__ __forceinline__ double d1(const BssnK& K, int gf, int l) const {
    if (l == 2) {
      const ZWin z = zwin(tb, gf);
      return (8.0 * (z.w[4] - z.w[2]) - (z.w[5] - z.w[1])) * K.i12h[2];
    }
    const double* f = t + gf * FPLS + c;
    const int s = l == 0 ? 1 : FSX;
    return (8.0 * (f[s] - f[-s]) - (f[2 * s] - f[-2 * s])) * K.i12h[l];
  }
  __device__ __forceinline__ double dd(const BssnK& K, int gf, int l, int m, double f0) const {
    if (l == m) {
      if (l == 2) {
        const ZWin z = zwin(tb, gf);
        return (16.0 * (z.w[4] + z.w[2]) - (z.w[5] + z.w[1]) - 30.0 * f0) * K.i12h2[2];
      }
      const double* f = t + gf * FPLS + c;
      const int s = l == 0 ? 1 : FSX;
      return (16.0 * (f[s] + f[-s]) - (f[2 * s] + f[-2 * s]) - 30.0 * f0) * K.i12h2[l];
    }
    const int e = ddi(gf);
    const double* g;
    int s;
    if (m == 1) { g = gyx + e * (FY * HXW) + hx; s = 1; }          // (x, y): outer x of D1_y
    else if (l == 0) { g = gzx + e * (FY * HXW) + hx; s = 1; }     // (x, z): outer x of D1_z
    else { g = gzy + e * (HYH * FX) + hy; s = FX; }                // (y, z): outer y of D1_z
    return (8.0 * (g[s] - g[-s]) - (g[2 * s] - g[-2 * s])) * K.i144hh[l + m - 1];
  }
  __device__ __forceinline__ double adv(const BssnK& K, int gf, const double* beta, double f0) const {
    const double* f = t + gf * FPLS + c;
    double r = 0.0;
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const int s = a == 0 ? 1 : FSX;
      const double a1 = f[s], b1 = f[-s], a2 = f[2 * s], b2 = f[-2 * s], a3 = f[3 * s], b3 = f[-3 * s];
      const double S = 21.0 * (a1 - b1) - 6.0 * (a2 - b2) + (a3 - b3);
      const double A = 15.0 * (a1 + b1) - 6.0 * (a2 + b2) + (a3 + b3) - 20.0 * f0;
      r = fma(fma(beta[a], S, fabs(beta[a]) * A), K.i24h[a], r);
    }
    const ZWin z = zwin(tb, gf);
    const double S = 21.0 * (z.w[4] - z.w[2]) - 6.0 * (z.w[5] - z.w[1]) + (z.w[6] - z.w[0]);
    const double A = 15.0 * (z.w[4] + z.w[2]) - 6.0 * (z.w[5] + z.w[1]) + (z.w[6] + z.w[0]) - 20.0 * f0;
    return fma(fma(beta[2], S, fabs(beta[2]) * A), K.i24h[2], r);
  }
};

// stage-input values at the point from the shared plane tile (RK update operands)
struct TileIn {
  const double* t;
  int c;
  __device__ __forceinline__ double operator()(int v) const { return t[v * FPLS + c]; }
};

struct FusedMaps {
  CUtensorMap in;    // the stage input set, box (FSX, FSY, 1, 1)
  CUtensorMap feed;  // the same set, box (FX, FY, 1, 1): the tile interior (the TMEM feed)
};

// MON: the stage-1 instantiation with the fused constraint monitor (a separate kernel, so the
// default one carries neither its code nor its registers)
template <int STAGE, bool MON>
__global__ void __launch_bounds__(FNT, 1)
    bssn_fused(const __grid_constant__ FusedMaps M, StageLaunch a, BssnK K, int ntx, int nty, int chunk,
               int nitems, double* rhs_dst) {
  extern __shared__ __align__(1024) unsigned char smem[];
  double* tiles = reinterpret_cast<double*>(smem);                       // 2 x TILE_STRIDE bytes
  double* feeds = reinterpret_cast<double*>(smem + 2 * TILE_STRIDE);      // 2 x FEED_STRIDE bytes
  double* gzx = reinterpret_cast<double*>(smem + 2 * TILE_STRIDE + 2 * FEED_STRIDE);
  double* gzy = gzx + GZX_N;
  double* gyx = gzy + GZY_N;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(gyx + GYX_N);           // 2 tile + 2 feed mbarriers
  uint64_t* fbar = mbar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mbar + 4);
  double* macc = reinterpret_cast<double*>(smem + 2 * TILE_STRIDE + 2 * FEED_STRIDE + 8 * (GZX_N + GZY_N + GYX_N) + 64);
  constexpr bool monitor = STAGE == 1 && MON;
  const Layout& L = a.L;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int grp = warp >> 2;                     // 0: G2; 1: G13 (2 groups) or G1; 2: G3
  const int p = (warp & 3) * 32 + lane;          // point of the tile (= TMEM lane)
  const int tx = p % FX, ty = p / FX;
  if (monitor && tid < NWARP * NMON) macc[tid] = 0.0;  // ordered before use by the first CTA barrier
  const double* in = stage_input<STAGE>(a);
  const int ntiles = ntx * nty;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int q = 0; q < 2; ++q) { mbar_init(&mbar[q], 1); mbar_init(&fbar[q], 1); }
    fence_mbar_init();
    prefetch_tmap(&M.in);
    prefetch_tmap(&M.feed);
  }
  cta_sync_tm();
  const uint32_t tb = *tmem_slot + ((uint32_t)((warp & 3) * 32) << 16);

  // (item, plane) sequence of this CTA: items it = blockIdx.x + q * gridDim.x, chunk-major
  auto item_geom = [&](int it, int& i0, int& j0, int& kb, int& ke) {
    const int ch = it / ntiles, tile = it % ntiles;
    i0 = (tile % ntx) * FX;
    j0 = (tile / ntx) * FY;
    kb = a.k_begin + ch * chunk;
    ke = min(kb + chunk, a.k_end);
  };
  auto issue_tile = [&](int buf, int i0, int j0, int k) {
    mbar_arrive_expect_tx(&mbar[buf], (uint32_t)TILE_BYTES);
#pragma unroll 1
    for (int q = 0; q < NV; ++q)  // one box per GF (a GF plane per 128-byte aligned slot)
      tma_load_4d(tiles + (size_t)buf * (TILE_STRIDE / 8) + q * FPLS, &M.in, &mbar[buf], kXOff + i0 - FRX,
                  L.g + j0 - FR, L.g + k, q);
  };
  auto issue_feed = [&](int buf, int i0, int j0, int k) {  // tile interior of plane k, all GFs
    mbar_arrive_expect_tx(&fbar[buf], (uint32_t)FEED_STRIDE);
#pragma unroll 1
    for (int q = 0; q < NV; ++q)
      tma_load_4d(feeds + (size_t)buf * (FEED_STRIDE / 8) + q * FEED_PL, &M.feed, &fbar[buf], kXOff + i0, L.g + j0,
                  L.g + k, q);
  };
  uint32_t fphase = 0;  // parity bit per feed buffer
  const int64_t gfs = L.gfs;
  const int xlo = -L.g, xhi = (int)L.nx + L.g - 1, ylo = -L.g, yhi = (int)L.ny + L.g - 1;
  uint32_t phase = 0;  // parity bit per tile buffer
  int n = 0;           // planes processed by this CTA (buffer = n & 1)
  if (tid == 0 && (int)blockIdx.x < nitems) {
    int i0, j0, kb, ke;
    item_geom(blockIdx.x, i0, j0, kb, ke);
    issue_tile(0, i0, j0, kb);
    issue_feed(0, i0, j0, kb + 3);
  }
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    int i0, j0, kb, ke;
    item_geom(it, i0, j0, kb, ke);
    const int i = i0 + tx, j = j0 + ty;
    const bool live = i < L.nx && j < L.ny;
    // dead lanes (past the interior of a ragged tile) keep their own column while it lies in
    // the ghost zone: live neighbours read their D1_z through the mixed-derivative helpers
    const int ic = min(i, xhi), jc = min(j, yhi);
    const double* col = in + (int64_t)jc * L.px + ic;                   // own column, plane 0, GF 0
    const int g_lo = grp == 0 ? 0 : FEED_B1, g_hi = grp == 0 ? FEED_B1 : NV;  // this thread's feed GFs
    // frame item geometry of this thread, recomputed per plane (cheap integer work; keeping
    // it live across the algebra would cost registers)
    auto frame_item = [&](int m, int& dst) -> int64_t {
      const int q = tid + m * FNT;
      const int e = q / NFRAME, f = q % NFRAME;
      int ii, jj;
      if (f < 4 * FY) { jj = f >> 2; const int cc = f & 3; ii = cc < 2 ? cc - 2 : FX + cc - 2; }
      else { const int f2 = f - 4 * FY; ii = f2 % FX; const int rr = f2 / FX; jj = rr < 2 ? rr - 2 : FY + rr - 2; }
      const int gx = min(max(i0 + ii, xlo), xhi), gy = min(max(j0 + jj, ylo), yhi);
      dst = f < 4 * FY ? e * (FY * HXW) + jj * HXW + ii + 2 : GZX_N + e * (HYH * FX) + (jj + 2) * FX + ii;
      return ddgf(e) * gfs + (int64_t)gy * L.px + gx;
    };
    // ---- window fill: planes kb-4 .. kb+2 into slots 0..6 (slot 0 is dropped by the first shift)
    __syncwarp();
    for (int gf = g_lo; gf < g_hi; ++gf) {
      uint32_t r[16];
#pragma unroll
      for (int s = 0; s < 7; ++s) {
        const int kk = max(kb - 4 + s, -L.g);
        const double v = __ldg(col + gf * gfs + (int64_t)kk * L.plane);
        r[2 * s] = (uint32_t)__double2loint(v);
        r[2 * s + 1] = (uint32_t)__double2hiint(v);
      }
      r[14] = r[15] = 0u;
      tm_st16(tb + 16u * (uint32_t)gf, r);
    }
    tm_wait_st();
    for (int k = kb; k < ke; ++k, ++n) {
      const int buf = n & 1;
      // ---- next plane's tile (this item's k+1, or the next item's first plane) into the other
      // buffer: its last reader (plane n-1) finished at the end-of-plane barrier
      if (tid == 0) {  // and the next plane's TMEM feed (plane k+4, or the next item's kb+3)
        if (k + 1 < ke) {
          issue_tile(buf ^ 1, i0, j0, k + 1);
          issue_feed(buf ^ 1, i0, j0, k + 4);
        } else if (it + (int)gridDim.x < nitems) {
          int ni0, nj0, nkb, nke;
          item_geom(it + gridDim.x, ni0, nj0, nkb, nke);
          issue_tile(buf ^ 1, ni0, nj0, nkb);
          issue_feed(buf ^ 1, ni0, nj0, nkb + 3);
        }
      }
      // ---- all global loads of the plane first (one exposed latency): the D1_z frame operands
      // (planes k+-1, k+-2 around the tile, L2-resident) ...
      double fv[NFI][4];
      int fdst[NFI];
#pragma unroll
      for (int m = 0; m < NFI; ++m)
        if (tid + m * FNT < NMIX * NFRAME) {
          const double* s0 = in + frame_item(m, fdst[m]) + (int64_t)k * L.plane;
          fv[m][0] = __ldg(s0 - 2 * L.plane);
          fv[m][1] = __ldg(s0 - L.plane);
          fv[m][2] = __ldg(s0 + L.plane);
          fv[m][3] = __ldg(s0 + 2 * L.plane);
        }
      // ... the RK update's pointwise operands of y / Q pulled into L1 ...
      if (STAGE >= 2 && STAGE <= 4 && live) {
        const double* pre = (STAGE == 4 ? a.s.q : a.s.y) + L.idx(i, j, k);
#pragma unroll
        for (int v = 0; v < NV; ++v)
          if (grp == 0 ? in_group(2, v) : in_group(13, v))
            asm volatile("prefetch.global.L1 [%0];" ::"l"(pre + v * gfs));
      }
      // ... the own column two planes ahead of the feed pulled into L2 (its first touch is
      // an HBM round trip; the feed itself arrives by TMA one plane ahead)
      {
        const int kp = min(k + 5, (int)L.nz + L.g - 1);
        for (int gf = g_lo; gf < g_hi; ++gf)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(col + gf * gfs + (int64_t)kp * L.plane));
      }
      mbar_wait(&mbar[buf], (phase >> buf) & 1u);
      phase ^= 1u << buf;
      const double* t = tiles + (size_t)buf * (TILE_STRIDE / 8);
      // ---- helper: D1raw_y on the x-extended tile (inner derivative of d_x d_y), from the tile
      for (int q = tid; q < GYX_N; q += FNT) {
        const int e = q / (FY * HXW), rem = q % (FY * HXW);
        const int jj = rem / HXW, ii = rem % HXW - 2;
        const double* f = t + ddgf(e) * FPLS + (jj + FR) * FSX + (ii + FRX);
        gyx[q] = 8.0 * (f[FSX] - f[-FSX]) - (f[2 * FSX] - f[-2 * FSX]);
      }
      // ---- helper: D1raw_z on the 2-point frame around the tile (operands loaded above)
#pragma unroll
      for (int m = 0; m < NFI; ++m)
        if (tid + m * FNT < NMIX * NFRAME) gzx[fdst[m]] = 8.0 * (fv[m][2] - fv[m][1]) - (fv[m][3] - fv[m][0]);
      // ---- TMEM window shift (planes k-3 .. k+3) with the new plane k+3 (from the TMA feed
      // buffer), and D1raw_z of the mixed GFs at the own point into the interior of the z
      // helpers.  tcgen05.ld/st are .sync.aligned: reconverge the warp after the
      // thread-dependent helper loops first
      mbar_wait(&fbar[buf], (fphase >> buf) & 1u);
      fphase ^= 1u << buf;
      const double* fb = feeds + (size_t)buf * (FEED_STRIDE / 8) + ty * FX + tx;
      __syncwarp();
#pragma unroll
      for (int q = 0; q < FEEDN; ++q) {
        const int gf = g_lo + q;
        if (gf >= g_hi) continue;
        uint32_t r[16];
        tm_ld16(tb + 16u * (uint32_t)gf, r);
        tm_wait_ld();
        // old slots: planes k-4 .. k+2
        const int e = ddi(gf);
        if (e >= 0) {
          const double v = 8.0 * (dbl(r[10], r[11]) - dbl(r[6], r[7])) - (dbl(r[12], r[13]) - dbl(r[4], r[5]));
          gzx[e * (FY * HXW) + ty * HXW + tx + 2] = v;
          gzy[e * (HYH * FX) + (ty + 2) * FX + tx] = v;
        }
        uint32_t w[16];
#pragma unroll
        for (int s = 0; s < 12; ++s) w[s] = r[s + 2];
        const double fv = fb[gf * FEED_PL];
        w[12] = (uint32_t)__double2loint(fv);
        w[13] = (uint32_t)__double2hiint(fv);
        w[14] = w[15] = 0u;
        tm_st16(tb + 16u * (uint32_t)gf, w);
      }
      tm_wait_st();
      cta_sync_tm();
      // ---- the RHS algebra of this thread's group from the on-chip derivatives, and its RK4
      // update (pointwise operands from global memory, outputs + ghost images to global)
      FusedP P{t, (ty + FR) * FSX + tx + FRX, gzx, gzy, gyx, ty * HXW + tx + 2, (ty + 2) * FX + tx, tb};
      const int64_t c = L.idx(i, j, k);
      double r[NV];
      const TileIn tin{t, P.c};
      if (grp == 0) {
        bssn_point<2>(P, K, r);
        if (live) bssn_update_src<STAGE, 2, TileIn, true>(a, K, r, tin, c, i, j, k, rhs_dst);
      } else {
        bssn_point<13>(P, K, r);
        if (live) bssn_update_src<STAGE, 13, TileIn, true>(a, K, r, tin, c, i, j, k, rhs_dst);
      }
      if constexpr (monitor) {
        // NEXT-3 fused constraint monitor: H, M^i, G^i of the state entering
        // this step (stage 1's input, already on chip), reduced per warp in a fixed order
        {  // H by the G2 warps, M and G by the G13 warps
          double cv[7];
          if (grp == 0) bssn_constraint_point<1>(P, K, cv);
          else bssn_constraint_point<2>(P, K, cv);
#pragma unroll
          for (int q = 0; q < 7; ++q) {
            if ((grp == 0) != (q == 0)) continue;
            const double v = live ? cv[q] : 0.0;
            double s2 = v * v, mx = fabs(v);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              s2 += __shfl_xor_sync(0xffffffffu, s2, o);
              mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            }
            if (lane == 0) {
              macc[warp * NMON + 2 * q] += s2;
              macc[warp * NMON + 2 * q + 1] = fmax(macc[warp * NMON + 2 * q + 1], mx);
            }
          }
        }
      }
      cta_sync_tm();
    }
  }
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(*tmem_slot));
  if (monitor && tid < NMON) {  // warps in order: deterministic per-CTA partials
    double v = macc[tid];
    for (int w = 1; w < NWARP; ++w) v = (tid & 1) ? fmax(v, macc[w * NMON + tid]) : v + macc[w * NMON + tid];
    a.mon_partials[(int64_t)blockIdx.x * NMON + tid] = v;
  }
}

// z chunks: the fewest that fill the SMs in near-whole waves (each item re-reads a 7-plane
// window prologue, so longer chunks waste less); grid = min(items, SMs)
struct FusedPlan {
  int ntx, nty, chunk, nitems, grid;
};
FusedPlan fused_plan(const Layout& L, int nk) {
  FusedPlan p;
  const int nsm = device_sm_count();
  p.ntx = (int)((L.nx + FX - 1) / FX);
  p.nty = (int)((L.ny + FY - 1) / FY);
  const int ntiles = p.ntx * p.nty;
  int best_c = 1;
  double best = -1.0;
  for (int cnum = 1; cnum <= 8 && cnum <= nk; ++cnum) {
    const int chunk = (nk + cnum - 1) / cnum;
    const int items = ntiles * ((nk + chunk - 1) / chunk);
    const int waves = (items + nsm - 1) / nsm;
    const double eff = (double)items / ((double)waves * nsm) * (double)chunk / (chunk + 7.0);
    if (eff > best + 1e-3) { best = eff; best_c = cnum; }
  }
  p.chunk = (nk + best_c - 1) / best_c;
  p.nitems = ntiles * ((nk + p.chunk - 1) / p.chunk);
  p.grid = p.nitems < nsm ? p.nitems : nsm;
  return p;
}

template <int STAGE>
cudaError_t launch_fused(const StageLaunch& a, const BssnK& K, double* dst, cudaStream_t st) {
  const Layout& L = a.L;
  const int nk = a.k_end - a.k_begin;
  if (nk <= 0) return cudaSuccess;
  if (L.g < FR) return cudaErrorInvalidValue;
#ifdef CHEMORA_DEBUG_FUSED
  fprintf(stderr, "launch_fused<%d> enter\n", STAGE);
#endif
  FusedMaps M;
  const double* in = stage_input<STAGE>(a);
  if (!encode_set_map(&M.in, in - L.c0, L.px, L.py, L.pz, L.n_gf, L.gfs, FSX, FSY, 1) ||
      !encode_set_map(&M.feed, in - L.c0, L.px, L.py, L.pz, L.n_gf, L.gfs, FX, FY, 1))
    return cudaErrorInvalidValue;
#ifdef CHEMORA_DEBUG_FUSED
  fprintf(stderr, "launch_fused<%d> encoded\n", STAGE);
#endif
  const bool mon = STAGE == 1 && a.mon_partials != nullptr;
  const void* fn = (const void*)bssn_fused<STAGE, false>;
  if constexpr (STAGE == 1)
    if (mon) fn = (const void*)bssn_fused<1, true>;
  static std::atomic<uint64_t> attr_done[2];
  if (cudaError_t e = smem_optin(fn, SMEM_FUSED, attr_done[mon ? 1 : 0]); e != cudaSuccess) return e;
#ifdef CHEMORA_DEBUG_FUSED
  fprintf(stderr, "launch_fused<%d> optin\n", STAGE);
#endif
  const FusedPlan p = fused_plan(L, nk);
  const int ntx = p.ntx, nty = p.nty, chunk = p.chunk, nitems = p.nitems, grid = p.grid;
#ifdef CHEMORA_DEBUG_FUSED
  fprintf(stderr, "launch_fused<%d> grid %d items %d chunk %d smem %d\n", STAGE, grid, nitems, chunk, SMEM_FUSED);
#endif
  if constexpr (STAGE == 1) {
    if (mon) bssn_fused<1, true><<<grid, FNT, SMEM_FUSED, st>>>(M, a, K, ntx, nty, chunk, nitems, dst);
    else bssn_fused<1, false><<<grid, FNT, SMEM_FUSED, st>>>(M, a, K, ntx, nty, chunk, nitems, dst);
  } else {
    bssn_fused<STAGE, false><<<grid, FNT, SMEM_FUSED, st>>>(M, a, K, ntx, nty, chunk, nitems, dst);
  }
  if (STAGE >= 1) {  // z ghost planes of the stage output (own wrap or the neighbours' slabs)
    double* out = const_cast<double*>(STAGE == 1 ? a.s.b : (STAGE == 2 ? a.s.c : (STAGE == 3 ? a.s.b : a.s.y)));
    if (cudaError_t e = push_z_planes(L, out, a.img[STAGE - 1], st); e != cudaSuccess) return e;
  }
#ifdef CHEMORA_DEBUG_FUSED
  {
    cudaError_t e1 = cudaGetLastError();
    cudaError_t e2 = cudaDeviceSynchronize();
    fprintf(stderr, "launch_fused<%d>: launch %s, sync %s\n", STAGE, cudaGetErrorString(e1), cudaGetErrorString(e2));
    return e1 != cudaSuccess ? e1 : e2;
  }
#endif
  return cudaGetLastError();
}

}  // namespace

int bssn_fused_grid(const Layout& L, int nk) { return fused_plan(L, nk).grid; }

cudaError_t bssn_fused_stage(const StageLaunch& a, int stage, double* dst, cudaStream_t st) {
  const BssnK K = make_k(a, a.hparams);
  switch (stage) {
    case 0: return launch_fused<0>(a, K, dst, st);
    case 1: return launch_fused<1>(a, K, dst, st);
    case 2: return launch_fused<2>(a, K, dst, st);
    case 3: return launch_fused<3>(a, K, dst, st);
    case 4: return launch_fused<4>(a, K, dst, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace chemora
