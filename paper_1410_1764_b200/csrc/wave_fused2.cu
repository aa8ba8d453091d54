// wave_fused2.cu -- kernel variant 7: the temporally blocked RK4 stage pairs of wave_fused.cu
// (Eq. 1) on 32x16 tiles with two output rows per thread.
//
// Same arithmetic, same HBM traffic per point (A: 4 reads + 9 writes, B: 14 reads + 5
// writes); what changes is the shape of the work.  With one 9-warp CTA per SM (the rings
// fill the shared memory) the 32x8 kernel is latency-bound: every warp has one point's
// dependent chain per plane.  Here every thread carries two independent chains (rows w and
// w + 8 of the tile for warp w) and the halo recompute per point drops (intermediate
// elements per point 4.6 instead of 5.3; TMA box bytes per point 6.9 instead of 8.3 doubles).
// To fit the shared memory: the second stage runs 2 planes behind the first (two CTA
// barriers per plane), the stage-3 u carry is folded into kernel A (Q.u already holds
// dt/6 y.rho + dt/3 Y2.rho + dt/3 C.rho), and the pointwise operands of the second stage
// (A: y, B: Q and y.u at the output points) are plain global loads issued before the first
// stage, so the P ring holds one plane and the Z ring gets the prefetch depth.
// Bit-identical to the stagewise path (no FMA contraction in this file).
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

constexpr int TX = 32, TY = 16, NCW = 8, NT = 32 * (NCW + 1), NTC = 32 * NCW;
constexpr int W = 2;   // 4th-order stencils
constexpr int H = 4;   // input halo: two stacked radius-2 stencils
constexpr int RY = TY / NCW;   // output rows per thread (2)
constexpr int r128(int b) { return (b + 127) / 128 * 128; }

// input box geometries (x extent, y extent); origins (-4,-4) rho, (-2,-2) v3, (-4,-2) v1,
// (-2,-4) v2
constexpr int BR_X = TX + 2 * H, BR_Y = TY + 2 * H;      // 40 x 24
constexpr int B3_X = TX + 2 * W, B3_Y = TY + 2 * W;      // 36 x 20
constexpr int B1_X = TX + 2 * H, B1_Y = TY + 2 * W;      // 40 x 20
constexpr int B2_X = TX + 2 * W, B2_Y = TY + 2 * H;      // 36 x 24
// intermediate-state geometries; origins (-2,-2), (-2,0), (0,-2), (0,0)
constexpr int IR_X = TX + 2 * W, IR_Y = TY + 2 * W;      // 36 x 20
constexpr int I1_X = TX + 2 * W, I1_Y = TY;              // 36 x 16
constexpr int I2_X = TX, I2_Y = TY + 2 * W;              // 32 x 20
constexpr int I3_X = TX, I3_Y = TY;                      // 32 x 16
constexpr int NIR = IR_X * IR_Y, NI1 = I1_X * I1_Y, NI2 = I2_X * I2_Y, NI3 = I3_X * I3_Y;
constexpr int ER = (NIR + NTC - 1) / NTC, E1 = (NI1 + NTC - 1) / NTC, E2 = (NI2 + NTC - 1) / NTC,
              E3 = NI3 / NTC;
static_assert(NI3 % NTC == 0, "tile geometry");

constexpr int ZR_B = r128(BR_X * BR_Y * 8), Z3_B = r128(B3_X * B3_Y * 8);
constexpr int ZSLOT = ZR_B + Z3_B;
constexpr uint32_t ZBYTES = (BR_X * BR_Y + B3_X * B3_Y) * 8;
constexpr int P1_B = r128(B1_X * B1_Y * 8), P2_B = r128(B2_X * B2_Y * 8);
constexpr int PY_R = r128(NIR * 8), PY_1 = r128(NI1 * 8), PY_2 = r128(NI2 * 8), PY_3 = r128(NI3 * 8);
constexpr int IR_B = r128(NIR * 8), I1_B = r128(NI1 * 8);
constexpr int IZ_B = IR_B + r128(NI3 * 8);   // intermediate z ring slot (rho, v3)
constexpr int IP_B = I1_B + r128(NI2 * 8);   // intermediate p ring slot (v1, v2)
constexpr int LAG = 2;                        // second stage at k = p - 2
constexpr int RI_Z = 5, RI_P = 3;

template <bool B> struct Geo {
  // input rings: Z (rho, v3 boxes) holds planes p-2 .. p+2 + prefetch (A: 4, B: 1); P (v1,
  // v2 boxes, and for B the y boxes) holds plane p + 1 prefetch
  static constexpr int RZ = B ? 6 : 9;
  static constexpr int RP = 2;
  static constexpr int PSLOT = P1_B + P2_B + (B ? PY_R + PY_1 + PY_2 + PY_3 : 0);
  static constexpr uint32_t PBYTES = (B1_X * B1_Y + B2_X * B2_Y + (B ? NIR + NI1 + NI2 + NI3 : 0)) * 8;
  static constexpr int OFF_P = RZ * ZSLOT;
  static constexpr int OFF_IZ = OFF_P + RP * PSLOT;
  static constexpr int OFF_IP = OFF_IZ + RI_Z * IZ_B;
  static constexpr int OFF_BAR = OFF_IP + RI_P * IP_B;
  static constexpr int NBAR = 2 * RZ + 2 * RP;
  static constexpr int SMEM = OFF_BAR + NBAR * 8;
  static_assert(SMEM <= 232448, "shared memory");
};

struct FMaps {
  CUtensorMap rho, v3, v1, v2;       // stencil input set (A: y, B: C)
  CUtensorMap yr, y1, y2, y3;        // B: y on the intermediate geometries
};

__device__ __forceinline__ double d1s_(const double* f, int c, int s) {
  double acc = 0.0;
#pragma unroll
  for (int q = W; q >= 1; --q) acc = fma(D1W<W>::c(q), f[c + q * s] - f[c - q * s], acc);
  return acc;
}

__device__ __forceinline__ void cbar() { asm volatile("bar.sync 1, %0;" ::"r"(NTC) : "memory"); }

template <bool B>
__global__ void __launch_bounds__(NT, 1)
    wave_fused2(const __grid_constant__ FMaps M, StageLaunch a, WaveK K, int kchunk, int ntx, int nty, int nitems) {
  using G = Geo<B>;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + G::OFF_BAR);
  uint64_t* zfull = bars;
  uint64_t* zempty = zfull + G::RZ;
  uint64_t* pfull = zempty + G::RZ;
  uint64_t* pempty = pfull + G::RP;
  const Layout& L = a.L;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < G::RZ; ++s) { mbar_init(zfull + s, 1); mbar_init(zempty + s, NCW); }
    for (int s = 0; s < G::RP; ++s) { mbar_init(pfull + s, 1); mbar_init(pempty + s, NCW); }
    fence_mbar_init();
  }
  __syncthreads();
  const int g = L.g;
  const int nkall = a.k_end - a.k_begin;

  if (warp == NCW) {  // ------------------------------------------------------ producer
    if (lane != 0) return;
    uint32_t nz = 0, np = 0;
    for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
      const int bx = item % ntx, by = (item / ntx) % nty, ch = item / (ntx * nty);
      const int kb = a.k_begin + ch * kchunk;
      const int nk = min(kchunk, a.k_begin + nkall - kb);
      const int xo = kXOff + bx * TX, yo = g + by * TY;
      auto loadZ = [&](int plane) {
        const uint32_t s = nz % G::RZ, n = nz / G::RZ;
        if (n > 0) mbar_wait_suspend(zempty + s, (n - 1) & 1);
        unsigned char* d = smem + s * ZSLOT;
        mbar_arrive_expect_tx(zfull + s, ZBYTES);
        tma_load_4d(d, &M.rho, zfull + s, xo - H, yo - H, g + plane, GRHO);
        tma_load_4d(d + ZR_B, &M.v3, zfull + s, xo - W, yo - W, g + plane, GV3);
        ++nz;
      };
      auto loadP = [&](int plane) {
        const uint32_t s = np % G::RP, n = np / G::RP;
        if (n > 0) mbar_wait_suspend(pempty + s, (n - 1) & 1);
        unsigned char* d = smem + G::OFF_P + s * G::PSLOT;
        uint64_t* bar = pfull + s;
        mbar_arrive_expect_tx(bar, G::PBYTES);
        tma_load_4d(d, &M.v1, bar, xo - H, yo - W, g + plane, GV1);
        tma_load_4d(d + P1_B, &M.v2, bar, xo - W, yo - H, g + plane, GV2);
        if (B) {
          unsigned char* e = d + P1_B + P2_B;
          tma_load_4d(e, &M.yr, bar, xo - W, yo - W, g + plane, GRHO);
          tma_load_4d(e + PY_R, &M.y1, bar, xo - W, yo, g + plane, GV1);
          tma_load_4d(e + PY_R + PY_1, &M.y2, bar, xo, yo - W, g + plane, GV2);
          tma_load_4d(e + PY_R + PY_1 + PY_2, &M.y3, bar, xo, yo, g + plane, GV3);
        }
        ++np;
      };
      for (int pl = kb - 4; pl < kb; ++pl) loadZ(pl);
      for (int j = 0; j < nk + 4; ++j) {
        loadZ(kb + j);      // input plane p + 2 for p = kb - 2 + j
        loadP(kb - 2 + j);  // P plane p
      }
    }
    return;
  }

  // --------------------------------------------------------------------------- consumers
  const int tid = threadIdx.x;
  const int64_t gfs = L.gfs;
  // first-stage elements of this thread (e = tid + u * NTC; past-the-end ones clamped and
  // not stored)
  int rR_c1[ER], rR_c2[ER], rR_c3[ER], rR_b[ER];
#pragma unroll
  for (int u = 0; u < ER; ++u) {
    const int e = min(tid + u * NTC, NIR - 1);
    const int x = e % IR_X, y = e / IR_X;
    rR_c1[u] = y * B1_X + x + 2;
    rR_c2[u] = (y + 2) * B2_X + x;
    rR_c3[u] = y * B3_X + x;
    rR_b[u] = (y + 2) * BR_X + x + 2;
  }
  int r1_cr[E1], r1_b[E1];
#pragma unroll
  for (int u = 0; u < E1; ++u) {
    const int e = min(tid + u * NTC, NI1 - 1);
    const int x = e % I1_X, y = e / I1_X;
    r1_cr[u] = (y + 4) * BR_X + x + 2;
    r1_b[u] = (y + 2) * B1_X + x + 2;
  }
  int r2_cr[E2], r2_b[E2];
#pragma unroll
  for (int u = 0; u < E2; ++u) {
    const int e = min(tid + u * NTC, NI2 - 1);
    const int x = e % I2_X, y = e / I2_X;
    r2_cr[u] = (y + 2) * BR_X + x + 4;
    r2_b[u] = (y + 2) * B2_X + x + 2;
  }
  // second stage: points (ti, tj) and (ti, tj + NCW); per-row offsets are immediates
  const int ti = lane, tj = warp;
  const int s_cr = (tj + 2) * IR_X + ti + 2, s_c1 = tj * I1_X + ti + 2, s_c2 = (tj + 2) * I2_X + ti,
            s_c3 = tj * I3_X + ti;
  const double cdt = B ? K.dt : K.dt2;
  double* const sm = reinterpret_cast<double*>(smem);
  constexpr int ZSD = ZSLOT / 8, ZR_D = ZR_B / 8, PSD = G::PSLOT / 8, P1D = P1_B / 8, P2D = P2_B / 8;
  constexpr int IZD = IZ_B / 8, IPD = IP_B / 8, IR_D = IR_B / 8, I1_D = I1_B / 8;
  constexpr int OFF_PD = G::OFF_P / 8, OFF_IZD = G::OFF_IZ / 8, OFF_IPD = G::OFF_IP / 8;
  constexpr int PYR = PY_R / 8, PY1 = PY_1 / 8, PY2 = PY_2 / 8;

  uint32_t nz = 0, np = 0;
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    const int bx = item % ntx, by = (item / ntx) % nty, ch = item / (ntx * nty);
    const int i0 = bx * TX, j0 = by * TY;
    const int kb = a.k_begin + ch * kchunk;
    const int nk = min(kchunk, a.k_begin + nkall - kb);
    const uint32_t z0 = nz, p0 = np;  // ring index of input plane kb-4, of P plane kb-2
    for (int q = 0; q < 4; ++q) mbar_wait(zfull + (z0 + q) % G::RZ, ((z0 + q) / G::RZ) & 1);
    const int i = i0 + ti;
    int jr[RY];
    bool live[RY];
    int64_t cglob[RY];
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      jr[r] = j0 + tj + r * NCW;
      live[r] = i < L.nx && jr[r] < L.ny;
      cglob[r] = L.idx(i, jr[r], kb);
    }
    int zsl[5];
#pragma unroll
    for (int q = 0; q < 5; ++q) zsl[q] = (int)((z0 + q) % G::RZ);
    int psl = (int)(p0 % G::RP);             // P slot of plane p
    int zph = (int)(((z0 + 4) / G::RZ) & 1);
    int pph = (int)((p0 / G::RP) & 1);
    int izs[5] = {0, 0, 0, 0, 0};
    int ips[3] = {0, 0, 0};
#pragma unroll 1
    for (int jj = 0; jj < nk + 4; ++jj) {
      const int p = kb - 2 + jj;
      const int k = p - LAG;
      const bool second = k >= kb;
#pragma unroll
      for (int q = 0; q < 4; ++q) izs[q] = izs[q + 1];
      izs[4] = jj % RI_Z;
      ips[0] = ips[1];
      ips[1] = ips[2];
      ips[2] = jj % RI_P;
      // pointwise operands of the second stage, from global memory, in flight during the
      // first stage (A: y at plane k; B: Q and y.u)
      double Qv[RY][5], yu[RY], qu[RY];
      if (second) {
#pragma unroll
        for (int r = 0; r < RY; ++r) {
          if (!live[r]) continue;
#pragma unroll
          for (int f = 1; f <= 4; ++f) Qv[r][f] = __ldg((B ? a.s.q : a.s.y) + f * gfs + cglob[r]);
          if (B) {
            qu[r] = __ldg(a.s.q + cglob[r]);
            yu[r] = __ldg(a.s.y + cglob[r]);
          }
        }
      }
      mbar_wait(zfull + zsl[4], zph);
      mbar_wait(pfull + psl, pph);
      const double* zR[5];
      const double* z3[5];
#pragma unroll
      for (int q = 0; q < 5; ++q) {
        zR[q] = sm + zsl[q] * ZSD;
        z3[q] = zR[q] + ZR_D;
      }
      const double* s1 = sm + OFF_PD + psl * PSD;
      const double* s2 = s1 + P1D;
      const double* sy = s2 + P2D;  // B only
      double* IR = sm + OFF_IZD + izs[4] * IZD;
      double* I3 = IR + IR_D;
      double* I1 = sm + OFF_IPD + ips[2] * IPD;
      double* I2 = I1 + I1_D;
      cbar();  // the intermediate slots being overwritten are no longer read
      // ---- intermediate state at plane p: Y2 = y + dt/2 k1(y) (A) or Y4 = y + dt k3(C) (B)
#pragma unroll
      for (int u = 0; u < ER; ++u) {
        const int e = tid + u * NTC;
        if (u == ER - 1 && e >= NIR) continue;
        const double dv1 = d1s_(s1, rR_c1[u], 1) * K.ih[0];
        const double dv2 = d1s_(s2, rR_c2[u], B2_X) * K.ih[1];
        double dv3 = 0.0;
#pragma unroll
        for (int q = W; q >= 1; --q) dv3 = fma(D1W<W>::c(q), z3[2 + q][rR_c3[u]] - z3[2 - q][rR_c3[u]], dv3);
        dv3 = dv3 * K.ih[2];
        const double kr = dv1 + dv2 + dv3;
        const double base = B ? sy[e] : zR[2][rR_b[u]];
        IR[e] = fma(cdt, kr, base);
      }
#pragma unroll
      for (int u = 0; u < E1; ++u) {
        const int e = tid + u * NTC;
        if (u == E1 - 1 && e >= NI1) continue;
        const double kr = d1s_(zR[2], r1_cr[u], 1) * K.ih[0];
        const double base = B ? sy[PYR + e] : s1[r1_b[u]];
        I1[e] = fma(cdt, kr, base);
      }
#pragma unroll
      for (int u = 0; u < E2; ++u) {
        const int e = tid + u * NTC;
        if (u == E2 - 1 && e >= NI2) continue;
        const double kr = d1s_(zR[2], r2_cr[u], BR_X) * K.ih[1];
        const double base = B ? sy[PYR + PY1 + e] : s2[r2_b[u]];
        I2[e] = fma(cdt, kr, base);
      }
#pragma unroll
      for (int u = 0; u < E3; ++u) {
        const int e = tid + u * NTC;
        const int cr = (e / I3_X + 4) * BR_X + e % I3_X + 4;
        double dzr = 0.0;
#pragma unroll
        for (int q = W; q >= 1; --q) dzr = fma(D1W<W>::c(q), zR[2 + q][cr] - zR[2 - q][cr], dzr);
        const double kr = dzr * K.ih[2];
        const double base = B ? sy[PYR + PY1 + PY2 + e] : z3[2][(e / I3_X + 2) * B3_X + e % I3_X + 2];
        I3[e] = fma(cdt, kr, base);
      }
      cbar();  // the intermediate plane p is complete
      // ---- second stage at plane k = p - 2 for the thread's two points
      if (second) {
        const double* iR[5];
        const double* i3[5];
#pragma unroll
        for (int q = 0; q < 5; ++q) {
          iR[q] = sm + OFF_IZD + izs[q] * IZD;
          i3[q] = iR[q] + IR_D;
        }
        const double* i1 = sm + OFF_IPD + ips[0] * IPD;
        const double* i2 = i1 + I1_D;
#pragma unroll
        for (int r = 0; r < RY; ++r) {
          const int dr = r * NCW;
          const int cr = s_cr + dr * IR_X, c1 = s_c1 + dr * I1_X, c2 = s_c2 + dr * I2_X, c3 = s_c3 + dr * I3_X;
          double S[5], kk[5];
          S[GRHO] = iR[2][cr];
          S[GV1] = i1[c1];
          S[GV2] = i2[c2];
          S[GV3] = i3[2][c3];
          double dzr = 0.0, dv3 = 0.0;
#pragma unroll
          for (int q = W; q >= 1; --q) {
            dzr = fma(D1W<W>::c(q), iR[2 + q][cr] - iR[2 - q][cr], dzr);
            dv3 = fma(D1W<W>::c(q), i3[2 + q][c3] - i3[2 - q][c3], dv3);
          }
          const double dxr = d1s_(iR[2], cr, 1) * K.ih[0];
          const double dyr = d1s_(iR[2], cr, IR_X) * K.ih[1];
          dzr = dzr * K.ih[2];
          const double dv1 = d1s_(i1, c1, 1) * K.ih[0];
          const double dv2 = d1s_(i2, c2, I2_X) * K.ih[1];
          dv3 = dv3 * K.ih[2];
          kk[GRHO] = dv1 + dv2 + dv3;
          kk[GV1] = dxr;
          kk[GV2] = dyr;
          kk[GV3] = dzr;
          if (!live[r]) continue;
          const int64_t c = cglob[r];
          const int j = jr[r];
          double v[5];
          if (!B) {
            const double* Y = Qv[r];   // y at the output point (plane k)
            // stage 2 (wave_update<2>) and the stage-3 u carry, in the stagewise order
            double* outc = a.s.c;
            double* outq = a.s.q;
#pragma unroll
            for (int f = 1; f <= 4; ++f) {
              outq[f * gfs + c] = fma(K.dt3, kk[f], (Y[f] + S[f]) * K.third);
              v[f] = fma(K.dt2, kk[f], Y[f]);
              outc[f * gfs + c] = v[f];
            }
            const double qu2 = fma(K.dt3, S[1], K.dt6 * Y[1]);
            outq[c] = fma(K.dt3, v[1], qu2);
            if (near_face(L, i, j, k)) {
              const FaceDst fd = a.img[1];
#pragma unroll 1
              for (int f = 1; f <= 4; ++f)
                store_images(outc + f * gfs, fd.lo + f * gfs, fd.hi + f * gfs, L, i, j, k, v[f]);
            }
          } else {
            // stage 4 (wave_update<4>); the new state goes to the scratch set
            double* outy = a.s.b;
#pragma unroll
            for (int f = 1; f <= 4; ++f) v[f] = fma(K.dt6, kk[f], fma(S[f], K.third, Qv[r][f]));
            v[0] = fma(K.dt6, S[1], yu[r] + qu[r]);
#pragma unroll
            for (int f = 0; f <= 4; ++f) outy[f * gfs + c] = v[f];
            if (near_face(L, i, j, k)) {
              const FaceDst fd = a.img[0];
#pragma unroll 1
              for (int f = 0; f <= 4; ++f)
                store_images(outy + f * gfs, fd.lo + f * gfs, fd.hi + f * gfs, L, i, j, k, v[f]);
            }
            if (isnan((v[0] - v[0]) + (v[1] - v[1]) + (v[2] - v[2]) + (v[3] - v[3]) + (v[4] - v[4]))) {
              const unsigned long long code0 = a.step * (unsigned long long)L.n_gf;
#pragma unroll 1
              for (int f = 0; f <= 4; ++f) check_finite(a.nan_flag, code0 + f, v[f]);
            }
          }
        }
#pragma unroll
        for (int r = 0; r < RY; ++r) cglob[r] += L.plane;
      }
      // ---- release what this warp has finished reading
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(pempty + psl);                    // P plane p (first stage only)
        mbar_arrive(zempty + zsl[0]);                 // input plane p - 2
      }
      // ---- advance the rings
#pragma unroll
      for (int q = 0; q < 4; ++q) zsl[q] = zsl[q + 1];
      zsl[4] = zsl[3] + 1 == G::RZ ? 0 : zsl[3] + 1;
      if (zsl[4] == 0) zph ^= 1;
      psl = psl + 1 == G::RP ? 0 : psl + 1;
      if (psl == 0) pph ^= 1;
    }
    // input planes ke .. ke+3 were only read
    __syncwarp();
    if (lane == 0)
      for (int q = 0; q < 4; ++q) mbar_arrive(zempty + (z0 + nk + 4 + q) % G::RZ);
    nz = z0 + nk + 8;
    np = p0 + nk + 4;
  }
}

bool enc(CUtensorMap* m, const double* set, const Layout& L, unsigned bx, unsigned by) {
  return encode_set_map(m, set - L.c0, L.px, L.py, L.pz, L.n_gf, L.gfs, bx, by, 1);
}

WaveK make_k(const StageLaunch& a) {
  WaveK K;
  for (int d = 0; d < 3; ++d) K.ih[d] = 1.0 / a.h[d];
  K.half = 0.5; K.third = 1.0 / 3.0; K.sixth = 1.0 / 6.0;
  K.dt = a.dt; K.dt2 = a.dt / 2.0; K.dt3 = a.dt / 3.0; K.dt6 = a.dt / 6.0;
  return K;
}

template <bool B>
cudaError_t launch(const StageLaunch& a, cudaStream_t st) {
  using G = Geo<B>;
  const int nk = a.k_end - a.k_begin;
  if (nk <= 0) return cudaSuccess;
  const Layout& L = a.L;
  const double* in = B ? a.s.c : a.s.y;
  FMaps M;
  bool ok = enc(&M.rho, in, L, BR_X, BR_Y) && enc(&M.v3, in, L, B3_X, B3_Y) && enc(&M.v1, in, L, B1_X, B1_Y) &&
            enc(&M.v2, in, L, B2_X, B2_Y) && enc(&M.yr, a.s.y, L, IR_X, IR_Y) && enc(&M.y1, a.s.y, L, I1_X, I1_Y) &&
            enc(&M.y2, a.s.y, L, I2_X, I2_Y) && enc(&M.y3, a.s.y, L, I3_X, I3_Y);
  if (!ok) return cudaErrorInvalidValue;
  static std::atomic<uint64_t> attr_done{0};
  if (cudaError_t e = smem_optin((const void*)wave_fused2<B>, G::SMEM, attr_done); e != cudaSuccess) return e;
  const int nsm = device_sm_count();
  const int ntx = (int)((L.nx + TX - 1) / TX), nty = (int)((L.ny + TY - 1) / TY);
  static int zc = 0;
  if (!zc) {
    const char* e = getenv("CHEMORA_FUSED_CHUNK");
    zc = e ? atoi(e) : 128;
    if (zc < 4) zc = 128;
  }
  int nchunks = (nk + zc - 1) / zc;
  const int want = (8 * nsm + ntx * nty - 1) / (ntx * nty);
  if (nchunks < want) nchunks = want;
  int chunk = (nk + nchunks - 1) / nchunks;
  if (chunk < 2) chunk = 2;
  if (chunk > nk) chunk = nk;
  nchunks = (nk + chunk - 1) / chunk;
  const int nitems = ntx * nty * nchunks;
  const int grid = nitems < nsm ? nitems : nsm;
  const WaveK K = make_k(a);
  wave_fused2<B><<<grid, NT, G::SMEM, st>>>(M, a, K, chunk, ntx, nty, nitems);
  return cudaGetLastError();
}

}  // namespace

cudaError_t wave_fused2_pair(const StageLaunch& a, int pair, cudaStream_t st) {
  if (a.fd_order != 4) return cudaErrorInvalidValue;
  return pair == 0 ? launch<false>(a, st) : launch<true>(a, st);
}

}  // namespace chemora
