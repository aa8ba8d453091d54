// bssn_stage.cu -- fused RHS + RK4-stage + ghost-image kernels for the 25-GF BSSN-like
// Einstein system ("the Einstein equations ...
// several thousand floating point operations to evaluate the RHS at a single grid
// point"; reading R7), 4th-order centered D1/D2/mixed stencils and 4th-order
// lopsided upwind advection (R6), advanced by the same one-pass y/Q/B/C RK4
// arrangement as the wave kernels (every BSSN GF is a stencil input):
//   stage 1 (in y): B = y + dt/2 k1
//   stage 2 (in B): Q = (y + B)/3 + dt/3 k2 ; C = y + dt/2 k2
//   stage 3 (in C): B = y + dt k3
//   stage 4 (in B): y = Q + B/3 + dt/6 k4
//
// The RHS algebra (bssn_point) is written once, on symmetric-packed tensors (xx, xy, xz,
// yy, yz, zz), against a derivative *provider*:
//   StencilP -- every derivative evaluated from global memory at the point (used by the
//               one-thread-per-point kernels: fused G0 and fissioned G1/G2/G3);
//   TabP     -- derivatives read from a shared-memory table that the CTA filled first
//               (the two-phase kernel: phase 1 computes the 161 point values, first and
//               second derivatives and advection terms of 32 points with fully parallel,
//               register-light stencil evaluations; phase 2 runs the algebra, two threads
//               per point splitting the equations).
// Advection is evaluated branch-free as beta * S f + |beta| * A f with S = (D+ + D-)/2 and
// A = (D+ - D-)/2 (identical to max(beta,0) D+ + min(beta,0) D-).
#include <cuda_runtime.h>
#include <cstdint>
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include "grid.hpp"
#include "kernels.hpp"
#include "device_common.cuh"

#include "bssn_common.cuh"

namespace chemora {
namespace {

template <int NP>
struct TabP {
  const double* tab;  // [NSLOT][NP]
  int pt;
  __device__ __forceinline__ double v(int gf) const { return tab[gf * NP + pt]; }
  __device__ __forceinline__ double d1(const BssnK&, int gf, int l) const { return tab[(T_D1 + 3 * d1i(gf) + l) * NP + pt]; }
  __device__ __forceinline__ double dd(const BssnK&, int gf, int l, int m, double) const {
    return tab[(T_DD + 6 * ddi(gf) + sy(l, m)) * NP + pt];
  }
  __device__ __forceinline__ double adv(const BssnK&, int gf, const double*, double) const { return tab[(T_ADV + gf) * NP + pt]; }
};
constexpr int kConThreads = 128;
__global__ void __launch_bounds__(kConThreads) bssn_constraints_kernel(Layout L, const double* in, BssnK K,
                                                                       double* fields, double* part) {
  __shared__ double sh[kConThreads / 32][14];
  double acc[14];
#pragma unroll
  for (int q = 0; q < 14; ++q) acc[q] = 0.0;
  const int64_t ni = L.nx * L.ny * L.nz;
  for (int64_t p = (int64_t)blockIdx.x * kConThreads + threadIdx.x; p < ni; p += (int64_t)gridDim.x * kConThreads) {
    const int i = (int)(p % L.nx);
    const int j = (int)((p / L.nx) % L.ny);
    const int k = (int)(p / (L.nx * L.ny));
    StencilP P{in, L.gfs, L.idx(i, j, k), {{1, L.px, L.plane}}};
    double c[7];
    bssn_constraint_point(P, K, c);
#pragma unroll
    for (int q = 0; q < 7; ++q) {
      if (fields) fields[q * ni + p] = c[q];
      acc[2 * q] = fma(c[q], c[q], acc[2 * q]);
      acc[2 * q + 1] = fmax(acc[2 * q + 1], fabs(c[q]));
    }
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < 14; ++q) {
    double v = acc[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double u = __shfl_xor_sync(0xffffffffu, v, o);
      v = (q & 1) ? fmax(v, u) : v + u;
    }
    if (lane == 0) sh[w][q] = v;
  }
  __syncthreads();
  if (threadIdx.x < 14) {
    const int q = threadIdx.x;
    double v = sh[0][q];
    for (int ww = 1; ww < kConThreads / 32; ++ww) v = (q & 1) ? fmax(v, sh[ww][q]) : v + sh[ww][q];
    part[(int64_t)blockIdx.x * 14 + q] = v;
  }
}

__global__ void bssn_constraints_combine(const double* part, int nblocks, double* out) {
  const int q = threadIdx.x;
  if (q >= 14) return;
  double v = 0.0;
  for (int b = 0; b < nblocks; ++b) v = (q & 1) ? fmax(v, part[(int64_t)b * 14 + q]) : v + part[(int64_t)b * 14 + q];
  out[q] = v;
}

// ------------------------------------------------------------------ one thread per point
// Computes the RHS group G (stencils from global memory) and the RK4 stage update of that
// group's GFs.  G = 0: the fused single kernel; G = 1, 2, 3: the fissioned kernels.
// register budget per group (128-thread CTAs): unconstrained -- capping G1 at 128 and G3
// at 168 registers measured slower (0.188 vs 0.221 G updates/s at 192^3: spills)
template <int G> struct MinBlocks { static constexpr int value = 1; };

template <int STAGE, int G>
__global__ void __launch_bounds__(128, MinBlocks<G>::value) bssn_simple(StageLaunch a, BssnK K, double* rhs_dst) {
  const Layout& L = a.L;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  const int k = a.k_begin + blockIdx.z * blockDim.z + threadIdx.z;
  if (i >= L.nx || j >= L.ny || k >= a.k_end) return;
  const int64_t c = L.idx(i, j, k);
  const double* in = stage_input<STAGE>(a);
  StencilP P{in, L.gfs, c, {{1, L.px, L.plane}}};
  double r[NV];
  bssn_point<G>(P, K, r);
  bssn_update<STAGE, G>(a, K, r, in, c, i, j, k, rhs_dst);
}

// ------------------------------------------------------------------ two-phase table kernel
// CTA = 32 consecutive x points of one row (TP points), 64 threads.  Phase 1: the 161
// table slots of the 32 points are computed by the 2 warps slot by slot (each warp one
// slot for its 32 points: coalesced loads, a handful of live registers, many independent
// loads in flight).  Phase 2: warp 0 runs the curvature group G2 (trK, At, A), warp 1 the
// kinematic + shift groups G1 + G3, both reading derivatives from the table.
constexpr int TP = 32;
template <int STAGE>
__global__ void __launch_bounds__(64) bssn_tab(StageLaunch a, BssnK K, double* rhs_dst) {
  __shared__ double tab[NSLOT * TP];
  const Layout& L = a.L;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i = blockIdx.x * TP + lane;
  const int j = blockIdx.y;
  const int k = a.k_begin + blockIdx.z;
  const bool live = i < L.nx;
  const int ic = live ? i : L.nx - 1;  // dead lanes recompute a valid point (discarded)
  const int64_t c = L.idx(ic, j, k);
  const int64_t gfs = L.gfs;
  const double* in = stage_input<STAGE>(a);
  const int64_t st[3] = {1, L.px, L.plane};
  // phase 1 -- point values first (the advection slots need beta, the D2 slots f0)
  for (int s = warp; s < T_D1; s += 2) tab[s * TP + lane] = ld(in + s * gfs + c);
  __syncthreads();
  double beta[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) beta[q] = tab[(V_BETA + q) * TP + lane];
  // first derivatives: 15 GFs x 3 axes, the warp's 3 axes of one GF per iteration (12
  // independent loads in flight per thread)
#pragma unroll 1
  for (int e = warp; e < 15; e += 2) {
    const double* f = in + d1gf(e) * gfs;
    const double a0 = D1raw(f, c, st[0]), a1 = D1raw(f, c, st[1]), a2 = D1raw(f, c, st[2]);
    tab[(T_D1 + 3 * e + 0) * TP + lane] = a0 * K.i12h[0];
    tab[(T_D1 + 3 * e + 1) * TP + lane] = a1 * K.i12h[1];
    tab[(T_D1 + 3 * e + 2) * TP + lane] = a2 * K.i12h[2];
  }
  // second derivatives: 11 GFs x 6 pairs, all six of one GF per iteration
#pragma unroll 1
  for (int e = warp; e < 11; e += 2) {
    const int gf = ddgf(e);
    const double* f = in + gf * gfs;
    const double f0 = tab[gf * TP + lane];
    const double xx = D2raw(f, c, st[0], f0), yy = D2raw(f, c, st[1], f0), zz = D2raw(f, c, st[2], f0);
    const double xy = D11raw(f, c, st[0], st[1]), xz = D11raw(f, c, st[0], st[2]), yz = D11raw(f, c, st[1], st[2]);
    double* o = tab + (T_DD + 6 * e) * TP + lane;
    o[0 * TP] = xx * K.i12h2[0];
    o[1 * TP] = xy * K.i144hh[0];
    o[2 * TP] = xz * K.i144hh[1];
    o[3 * TP] = yy * K.i12h2[1];
    o[4 * TP] = yz * K.i144hh[2];
    o[5 * TP] = zz * K.i12h2[2];
  }
  // advection terms, two GFs per iteration
#pragma unroll 1
  for (int gf = warp; gf < NV; gf += 4) {
    double r[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int v = gf + 2 * u < NV ? gf + 2 * u : gf;
      const double f0 = tab[v * TP + lane];
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < 3; ++q) acc = fma(ADVraw(in + v * gfs, c, st[q], f0, beta[q]), K.i24h[q], acc);
      r[u] = acc;
    }
    tab[(T_ADV + gf) * TP + lane] = r[0];
    if (gf + 2 < NV) tab[(T_ADV + gf + 2) * TP + lane] = r[1];
  }
  __syncthreads();
  // phase 2 -- the algebra from the table, two equation groups per point
  TabP<TP> P{tab, lane};
  double r[NV];
  if (warp == 0) {
    bssn_point<2>(P, K, r);
    if (live) bssn_update<STAGE, 2>(a, K, r, in, c, i, j, k, rhs_dst);
  } else {
    bssn_point<13>(P, K, r);
    if (live) bssn_update<STAGE, 13>(a, K, r, in, c, i, j, k, rhs_dst);
  }
}

// ------------------------------------------------------------------ derivative table in HBM
// Variant 3: the kernel fission of PAPER.md:537-547 taken to the derivative/algebra
// boundary.  A stencil-only kernel writes the 136 derivative slots of every interior point
// (45 D1, 66 second derivatives, 25 advection terms; the layout of the SMEM table above
// minus the point values) to an HBM table [slot][point]; the algebra kernels then read point
// values from the stage input and derivatives from the table -- pointwise and coalesced, so
// the register-heavy algebra has no stencil loads in flight.  Table traffic: 136 x 8 B
// written + read per point per stage.
constexpr int NTAB = NSLOT - T_D1;            // 136
// Derivative kernel: one CTA per (32 x 8 tile, z chunk of DZC planes, GF), 4 CTAs per SM.
// It marches the chunk with an 8-plane shared-memory ring of the GF's planes (tile + 3-point
// halo; cp.async, two planes in flight), so every stencil operand is read from HBM/L2 once
// per CTA; the own column's z stencils come from a register queue, the own x row and y
// column are read from the ring once per plane, and the inner derivatives of the mixed
// second derivatives are computed once per plane for the whole tile.  It writes all table
// slots of that GF (D1 if differentiated, the 6 second derivatives if twice differentiated,
// the advection term) with streaming stores.  Same operation order as StencilP (D1raw,
// D2raw, D11raw, ADVraw).  Design steps and probes: profiles/r1_bssn_summary.md.
constexpr int DT_X = 32, DT_Y = 8, DR = 3, DSX = DT_X + 2 * DR, DSY = DT_Y + 2 * DR, DPL = DSX * DSY;
constexpr int DZC = 32, DRING = 8, DNT = DT_X * DT_Y;

template <int STAGE>
__global__ void __launch_bounds__(DNT, 1024 / DNT) bssn_deriv(StageLaunch a, BssnK K, int ntx, int nty, int dzc) {
  extern __shared__ __align__(16) double dring[];
  double (*ring)[DPL] = reinterpret_cast<double (*)[DPL]>(dring);
  double* gzb = dring + DRING * DPL;   // D1raw_z f on the whole plane (tile + halo)
  double* gyb = gzb + DPL;             // D1raw_y f on the tile rows, all DSX columns
  const Layout& L = a.L;
  const int gf = blockIdx.x;  // GFs fastest: the 25 CTAs of a tile run together (beta from L2)
  const int t = blockIdx.y;
  const int bx = t % ntx, by = (t / ntx) % nty, ch = t / (ntx * nty);
  const int i0 = bx * DT_X, j0 = by * DT_Y;
  const int kb = a.k_begin + ch * dzc, ke = min(kb + dzc, a.k_end);
  const double* in = stage_input<STAGE>(a);
  const double* f = in + gf * L.gfs;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int i = i0 + tx, j = j0 + ty;
  const bool live = i < L.nx && j < L.ny;
  const int64_t ni = L.nx * L.ny * L.nz;
  const int xmax = (int)L.nx + L.g - 1, ymax = (int)L.ny + L.g - 1;
  // asynchronous plane copies (cp.async, one commit group per plane): the copies of planes
  // k + 4 and k + 5 overlap the computation of plane k
  // this thread's elements of a ring plane are the same for every plane: their in-plane
  // offsets are computed once (the plane loop then only adds the plane base)
  constexpr int NE = (DPL + DNT - 1) / DNT;
  int xyo[NE];
#pragma unroll
  for (int m = 0; m < NE; ++m) {
    const int e = threadIdx.x + m * DNT;
    const int x = min(i0 - DR + e % DSX, xmax), y = min(j0 - DR + e / DSX, ymax);
    xyo[m] = y * (int)L.px + x;
  }
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(dring) + 8u * threadIdx.x;
  auto load = [&](int plane) {  // always commits a group (empty past the chunk's last plane)
    if (plane < ke + DR) {
      const uint32_t dst = ring_s + 8u * DPL * (uint32_t)((plane + DRING) & (DRING - 1));
      const double* src = f + (int64_t)plane * L.plane;
#pragma unroll
      for (int m = 0; m < NE; ++m)
        if (m < NE - 1 || threadIdx.x + m * DNT < DPL)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst + 8u * m * DNT), "l"(src + xyo[m])
                       : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  const int e1 = d1i(gf), e2 = ddi(gf);
  // Ring use at plane k: k-2 .. k+2 (the shared D1_z of the mixed derivatives), k + 3 (the
  // own column's z queue); so two planes can be in flight: k + 4 and k + 5 (slot of k - 3).
  for (int q = -DR; q <= DR; ++q) load(kb + q);
  const int c = (ty + DR) * DSX + tx + DR;
  double* tab = a.dtab;
  double zq[2 * DR + 1];  // this thread's column at planes k-3 .. k+3 (z stencils from registers)
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 2 * DR; ++q) zq[q] = ring[(kb - DR + q + DRING) & (DRING - 1)][c];
  load(kb + DR + 1);
  // own-point addresses, advanced by one plane per iteration
  const int64_t nxy = (int64_t)L.nx * L.ny;
  int64_t o = (int64_t(kb) * L.ny + j) * L.nx + i;  // table index of the own point
  double* const t_d1 = tab + (int64_t)(3 * max(e1, 0)) * ni;
  double* const t_dd = tab + (int64_t)(45 + 6 * max(e2, 0)) * ni;
  double* const t_adv = tab + (int64_t)(111 + gf) * ni;
  const double* bb = in + V_BETA * L.gfs + L.idx(i, j, kb);
  for (int k = kb; k < ke; ++k) {
    asm volatile("cp.async.wait_group 1;" ::: "memory");  // plane k + 3 has landed (k + 4 may not)
    __syncthreads();  // ... for every thread, and plane k - 3's slot is no longer read
    zq[2 * DR] = ring[(k + DR + DRING) & (DRING - 1)][c];
    load(k + DR + 2);
    if (e2 >= 0) {
      // inner derivatives of the mixed second derivatives, shared by the tile: D1_z on the
      // plane (for d_x d_z at x-halo columns and d_y d_z at y-halo rows), D1_y on the rows
      const double* rm2 = ring[(k - 2 + DRING) & (DRING - 1)] + threadIdx.x;
      const double* rm1 = ring[(k - 1 + DRING) & (DRING - 1)] + threadIdx.x;
      const double* rp1 = ring[(k + 1 + DRING) & (DRING - 1)] + threadIdx.x;
      const double* rp2 = ring[(k + 2 + DRING) & (DRING - 1)] + threadIdx.x;
#pragma unroll
      for (int m = 0; m < NE; ++m)
        if (m < NE - 1 || threadIdx.x + m * DNT < DPL)
          gzb[threadIdx.x + m * DNT] = 8.0 * (rp1[m * DNT] - rm1[m * DNT]) - (rp2[m * DNT] - rm2[m * DNT]);
      const double* r0 = ring[(k + DRING) & (DRING - 1)] + DR * DSX + threadIdx.x;
      constexpr int NEY = (DT_Y * DSX + DNT - 1) / DNT;
#pragma unroll
      for (int m = 0; m < NEY; ++m)
        if (m < NEY - 1 || threadIdx.x + m * DNT < DT_Y * DSX) {
          const double* q = r0 + m * DNT;
          gyb[threadIdx.x + m * DNT] = 8.0 * (q[DSX] - q[-DSX]) - (q[2 * DSX] - q[-2 * DSX]);
        }
      __syncthreads();
    }
    if (live) {
      // the x row and y column of the own plane, read from shared memory once: the D1, D2
      // and advection stencils of an axis share these operands, and the table stores in
      // between would otherwise force the compiler to re-read them (generic-pointer aliasing)
      const double* own = ring[(k + DRING) & (DRING - 1)] + c;
      double xr[2 * DR + 1], yr[2 * DR + 1];
#pragma unroll
      for (int q = 0; q <= 2 * DR; ++q) {
        xr[q] = q == DR ? zq[DR] : own[q - DR];
        yr[q] = q == DR ? zq[DR] : own[(q - DR) * DSX];
      }
      auto F = [&](int dx, int dy, int dz) {
        return (dx == 0 && dy == 0) ? zq[dz + DR] : (dy == 0 && dz == 0) ? xr[dx + DR] : yr[dy + DR];
      };
      auto D1 = [&](int ax, int ox, int oy, int oz) {  // D1raw along axis ax at offset (ox,oy,oz)
        const int sx = ax == 0, sy_ = ax == 1, sz = ax == 2;
        return 8.0 * (F(ox + sx, oy + sy_, oz + sz) - F(ox - sx, oy - sy_, oz - sz)) -
               (F(ox + 2 * sx, oy + 2 * sy_, oz + 2 * sz) - F(ox - 2 * sx, oy - 2 * sy_, oz - 2 * sz));
      };
      const double f0 = F(0, 0, 0);
      if (e1 >= 0) {
#pragma unroll
        for (int l = 0; l < 3; ++l) __stcs(t_d1 + l * ni + o, D1(l, 0, 0, 0) * K.i12h[l]);
      }
      if (e2 >= 0) {
        double* tt = t_dd + o;
#pragma unroll
        for (int p = 0; p < 6; ++p) {
          const int l = sI(p), m = sJ(p);
          double v;
          if (l == m) {
            const int sx = l == 0, sy_ = l == 1, sz = l == 2;
            v = (16.0 * (F(sx, sy_, sz) + F(-sx, -sy_, -sz)) - (F(2 * sx, 2 * sy_, 2 * sz) + F(-2 * sx, -2 * sy_, -2 * sz)) -
                 30.0 * f0) * K.i12h2[l];
          } else {
            // outer D1 along l of the inner D1raw along m, read from the shared buffers
            const double* gb = (m == 1) ? gyb + ty * DSX + tx + DR : gzb + c;
            const int so = (l == 0) ? 1 : DSX;   // (l, m) = (x, y), (x, z) or (y, z)
            const double p1 = gb[so], m1 = gb[-so], p2 = gb[2 * so], m2 = gb[-2 * so];
            v = (8.0 * (p1 - m1) - (p2 - m2)) * K.i144hh[l + m - 1];
          }
          __stcs(tt + p * ni, v);
        }
      }
      double r = 0.0;
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const int sx = q == 0, sy_ = q == 1, sz = q == 2;
        const double beta = ld(bb + q * L.gfs);
        const double a1 = F(sx, sy_, sz), b1 = F(-sx, -sy_, -sz);
        const double a2 = F(2 * sx, 2 * sy_, 2 * sz), b2 = F(-2 * sx, -2 * sy_, -2 * sz);
        const double a3 = F(3 * sx, 3 * sy_, 3 * sz), b3 = F(-3 * sx, -3 * sy_, -3 * sz);
        const double S = 21.0 * (a1 - b1) - 6.0 * (a2 - b2) + (a3 - b3);
        const double A = 15.0 * (a1 + b1) - 6.0 * (a2 + b2) + (a3 + b3) - 20.0 * f0;
        r = fma(fma(beta, S, fabs(beta) * A), K.i24h[q], r);
      }
      __stcs(t_adv + o, r);
    }
#pragma unroll
    for (int q = 0; q < 2 * DR; ++q) zq[q] = zq[q + 1];
    o += nxy;
    bb += L.plane;
  }
}

struct HbmP {
  const double* in;
  int64_t gfs, c;
  const double* tab;
  int64_t ni, o;
  __device__ __forceinline__ double v(int gf) const { return ld(in + gf * gfs + c); }
  __device__ __forceinline__ double d1(const BssnK&, int gf, int l) const {
    return __ldcs(tab + (3 * d1i(gf) + l) * ni + o);
  }
  __device__ __forceinline__ double dd(const BssnK&, int gf, int l, int m, double) const {
    return __ldcs(tab + (45 + 6 * ddi(gf) + sy(l, m)) * ni + o);
  }
  __device__ __forceinline__ double adv(const BssnK&, int gf, const double*, double) const {
    return __ldcs(tab + (111 + gf) * ni + o);
  }
};

template <int STAGE, int G, int MB>
__global__ void __launch_bounds__(128, MB) bssn_alg(StageLaunch a, BssnK K, double* rhs_dst) {
  const Layout& L = a.L;
  const int i = blockIdx.x * 32 + threadIdx.x;
  const int j = blockIdx.y * 4 + threadIdx.y;
  const int k = a.k_begin + blockIdx.z;
  if (i >= L.nx || j >= L.ny) return;
  const int64_t c = L.idx(i, j, k);
  const double* in = stage_input<STAGE>(a);
  HbmP P{in, L.gfs, c, a.dtab, L.nx * L.ny * L.nz, (int64_t(k) * L.ny + j) * L.nx + i};
  double r[NV];
  bssn_point<G>(P, K, r);
  bssn_update<STAGE, G>(a, K, r, in, c, i, j, k, rhs_dst);
}

template <int STAGE>
cudaError_t launch_hbm(const StageLaunch& a, const BssnK& K, double* dst, cudaStream_t st) {
  const int nk = a.k_end - a.k_begin;
  if (nk <= 0) return cudaSuccess;
  if (!a.dtab) return cudaErrorInvalidValue;
  const dim3 block(32, 4, 1);
  const unsigned gx = (unsigned)((a.L.nx + 31) / 32), gy = (unsigned)((a.L.ny + 3) / 4);
  {
    const int ntx = (int)((a.L.nx + DT_X - 1) / DT_X), nty = (int)((a.L.ny + DT_Y - 1) / DT_Y);
    constexpr int dzc = DZC;  // z planes per CTA (profiles/r1_bssn_summary.md: 32 measured best)
    const int nch = (nk + dzc - 1) / dzc;
    constexpr int smem = (DRING * DPL + DPL + DT_Y * DSX) * 8;
    static std::atomic<uint64_t> attr_done{0};
    if (cudaError_t e = smem_optin((const void*)bssn_deriv<STAGE>, smem, attr_done); e != cudaSuccess) return e;
    bssn_deriv<STAGE><<<dim3(NV, (unsigned)(ntx * nty * nch), 1), DNT, smem, st>>>(a, K, ntx, nty, dzc);
  }
  // algebra kernels at 2 resident CTAs per SM (up to 255 registers, spill-free: measured
  // best against 3 and 4 CTAs/SM, profiles/r1_bssn_summary.md)
  const dim3 grid(gx, gy, (unsigned)nk);
  bssn_alg<STAGE, 2, 2><<<grid, block, 0, st>>>(a, K, dst);
  bssn_alg<STAGE, 13, 2><<<grid, block, 0, st>>>(a, K, dst);
  return cudaGetLastError();
}

template <int STAGE, int G>
cudaError_t launch(const StageLaunch& a, const BssnK& K, double* dst, cudaStream_t st) {
  const int nk = a.k_end - a.k_begin;
  if (nk <= 0) return cudaSuccess;
  constexpr int bdim[3] = {32, 4, 1};  // CTA shape (128 threads)
  dim3 block(bdim[0], bdim[1], bdim[2]);
  dim3 grid((unsigned)((a.L.nx + bdim[0] - 1) / bdim[0]), (unsigned)((a.L.ny + bdim[1] - 1) / bdim[1]),
            (unsigned)((nk + bdim[2] - 1) / bdim[2]));
  bssn_simple<STAGE, G><<<grid, block, 0, st>>>(a, K, dst);
  return cudaGetLastError();
}

template <int STAGE>
cudaError_t launch_tab(const StageLaunch& a, const BssnK& K, double* dst, cudaStream_t st) {
  const int nk = a.k_end - a.k_begin;
  if (nk <= 0) return cudaSuccess;
  dim3 grid((unsigned)((a.L.nx + TP - 1) / TP), (unsigned)a.L.ny, (unsigned)nk);
  bssn_tab<STAGE><<<grid, 64, 0, st>>>(a, K, dst);
  return cudaGetLastError();
}

template <int STAGE>
cudaError_t launch_stage(const StageLaunch& a, const BssnK& K, double* dst, cudaStream_t st) {
  // variant 0: two-phase SMEM table kernel; 2: the fissioned kernels G1, G2, G3; 3: HBM
  // derivative table + algebra kernels.  (Variant 1, the fused single kernel, spilled 33 KB
  // per thread and ran 8x slower -- the NEXT-2 fission result, profiles/r1_bssn_summary.md --
  // and is gone.)
  if (a.variant == 3) return launch_hbm<STAGE>(a, K, dst, st);
  if (a.variant == 2) {
    cudaError_t e = launch<STAGE, 1>(a, K, dst, st);
    if (e == cudaSuccess) e = launch<STAGE, 2>(a, K, dst, st);
    if (e == cudaSuccess) e = launch<STAGE, 3>(a, K, dst, st);
    return e;
  }
  return launch_tab<STAGE>(a, K, dst, st);
}

cudaError_t dispatch(const StageLaunch& a, int stage, double* dst, cudaStream_t st, const double* hparams) {
  if (a.variant == 4) return bssn_fused_stage(a, stage, dst, st);
  const BssnK K = make_k(a, hparams);
  switch (stage) {
    case 0: return launch_stage<0>(a, K, dst, st);
    case 1: return launch_stage<1>(a, K, dst, st);
    case 2: return launch_stage<2>(a, K, dst, st);
    case 3: return launch_stage<3>(a, K, dst, st);
    case 4: return launch_stage<4>(a, K, dst, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t bssn_stage(const StageLaunch& a, int stage, cudaStream_t st) {
  return dispatch(a, stage, nullptr, st, a.hparams);
}
cudaError_t bssn_rhs(const StageLaunch& a, double* dst, cudaStream_t st) {
  return dispatch(a, 0, dst, st, a.hparams);
}
cudaError_t bssn_constraints_reduce(const double* part, int nblocks, double* out14, cudaStream_t st) {
  bssn_constraints_combine<<<1, 32, 0, st>>>(part, nblocks, out14);
  return cudaGetLastError();
}

cudaError_t bssn_constraints(const StageLaunch& a, double* fields, double* scratch, double* out_dev,
                             cudaStream_t st) {
  const BssnK K = make_k(a, a.hparams);
  bssn_constraints_kernel<<<kNormBlocks, kConThreads, 0, st>>>(a.L, a.s.y, K, fields, scratch);
  bssn_constraints_combine<<<1, 32, 0, st>>>(scratch, kNormBlocks, out_dev);
  return cudaGetLastError();
}

}  // namespace chemora
