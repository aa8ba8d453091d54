// wave_fused3.cu -- kernel variant 8: the temporally blocked RK4 stage pairs of
// the round-1 pair kernel (Eq. 1) with the z stencils of each thread's
// own column taken from register queues (2.5-D z-march inside the temporal blocking).
//
// Every consumer thread owns one output point (ti, tj) of the 32x8 tile, and with it the
// intermediate values at that point (rho, v1, v2, v3); the 176 / 32 / 128 halo elements of
// the intermediate rho / v1 / v2 planes are spread over the other threads.  The thread keeps
// its own intermediate rho and v3 for planes p-5 .. p-1 in registers, so the second stage's
// z stencils and centres need no shared loads and the intermediate v3 never goes to shared
// memory.  (Keeping the input rho/v3 column in registers too exceeds the 168-register cap
// of the 9-warp CTA: measured slower.)  Same arithmetic in the
// same order as the one-kernel-per-stage path (bit-identical; no FMA contraction).
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

constexpr int TX = 32, TY = 8, NCW = 8, NT = 32 * (NCW + 1);
constexpr int W = 2;   // 4th-order stencils (fd_order 4 only)
constexpr int H = 4;   // input halo: two stacked radius-2 stencils
constexpr int r128(int b) { return (b + 127) / 128 * 128; }

// input box geometries (x extent, y extent, x origin offset, y origin offset)
constexpr int BR_X = TX + 2 * H, BR_Y = TY + 2 * H;      // rho   (40 x 16), origin (-4,-4)
constexpr int B3_X = TX + 2 * W, B3_Y = TY + 2 * W;      // v3    (36 x 12), origin (-2,-2)
constexpr int B1_X = TX + 2 * H, B1_Y = TY + 2 * W;      // v1    (40 x 12), origin (-4,-2)
constexpr int B2_X = TX + 2 * W, B2_Y = TY + 2 * H;      // v2    (36 x 16), origin (-2,-4)
// intermediate-state geometries
constexpr int IR_X = TX + 2 * W, IR_Y = TY + 2 * W;      // rho   (36 x 12), origin (-2,-2)
constexpr int I1_X = TX + 2 * W, I1_Y = TY;              // v1    (36 x 8),  origin (-2, 0)
constexpr int I2_X = TX, I2_Y = TY + 2 * W;              // v2    (32 x 12), origin ( 0,-2)
constexpr int I3_X = TX, I3_Y = TY;                      // v3    (32 x 8)
// pointwise boxes of kernel B (y on the intermediate geometries, Q and y.u centres)
constexpr int C1 = TX * TY;

constexpr int ZR_B = r128(BR_X * BR_Y * 8), Z3_B = r128(B3_X * B3_Y * 8);
constexpr int ZSLOT = ZR_B + Z3_B;
constexpr uint32_t ZBYTES = (BR_X * BR_Y + B3_X * B3_Y) * 8;
constexpr int P1_B = r128(B1_X * B1_Y * 8), P2_B = r128(B2_X * B2_Y * 8);
constexpr int PY_R = r128(IR_X * IR_Y * 8), PY_1 = r128(I1_X * I1_Y * 8), PY_2 = r128(I2_X * I2_Y * 8),
              PY_3 = r128(I3_X * I3_Y * 8);
constexpr int IZ_B = r128(IR_X * IR_Y * 8);  // intermediate rho ring slot (v3 lives in registers)
constexpr int IP_B = r128(I1_X * I1_Y * 8) + r128(I2_X * I2_Y * 8);  // intermediate p ring slot
// The second stage runs 3 planes behind the first (k = p - 3), so within one iteration the
// two stages touch disjoint intermediate slots.  The intermediate rings hold 5 planes
// (p-4 .. p): iteration t writes slot t mod 5, which the second stage last read in iteration
// t-2, and reads the slot written in t-3.  So the warps need not meet at a CTA barrier every
// plane: each arrives on a per-iteration mbarrier when done and, before writing, waits only
// until every warp has finished iteration t-2 (the warps may drift one plane apart).
constexpr int LAG = 3;
constexpr int RI_Z = 5, RI_P = 5;
constexpr int ND = 4;               // per-iteration "done" mbarriers, used round robin
// items (tile x z-chunk) are handed out dynamically (an atomic counter, in order), so the
// items in flight at any time are neighbours in (x, y): their shared halo rows are read by
// both while still in L2.  (With a static round-robin assignment the persistent CTAs drift
// apart by tens of planes over a launch and the halos are read from HBM twice.)  The
// producer passes each item index to its consumers through a small shared queue, published
// by the mbarrier of the item's first input plane.
constexpr int IQ = 4;

template <bool B> struct Geo {
  // input ring depths: resident windows are Z: planes p-3 .. p+2 (6), P: p-3 .. p (A) or p
  // (B), Q: k (B); the rest is prefetch
  static constexpr int RZ = B ? 8 : 10;
  static constexpr int RP = B ? 3 : 8;
  static constexpr int RQ = B ? 3 : 1;  // (A: one unused slot pair keeps the ring arithmetic defined)
  static constexpr int PSLOT = P1_B + P2_B + (B ? PY_R + PY_1 + PY_2 + PY_3 : 0);
  static constexpr uint32_t PBYTES =
      (B1_X * B1_Y + B2_X * B2_Y + (B ? IR_X * IR_Y + I1_X * I1_Y + I2_X * I2_Y + I3_X * I3_Y : 0)) * 8;
  static constexpr int QSLOT = B ? r128(6 * C1 * 8) : 0;  // Q (u, rho, v1..3) + y.u
  static constexpr uint32_t QBYTES = B ? 6 * C1 * 8 : 0;
  static constexpr int OFF_P = RZ * ZSLOT;
  static constexpr int OFF_Q = OFF_P + RP * PSLOT;
  static constexpr int OFF_IZ = OFF_Q + RQ * QSLOT;
  static constexpr int OFF_IP = OFF_IZ + RI_Z * IZ_B;
  static constexpr int OFF_BAR = OFF_IP + RI_P * IP_B;
  static constexpr int NBAR = 2 * RZ + 2 * RP + 2 * RQ + ND;
  static constexpr int OFF_ITEMQ = OFF_BAR + NBAR * 8;
  static constexpr int OFF_RED = OFF_ITEMQ + 4 * IQ + 8;  // energy partials, 2 x NCW doubles
  static constexpr int SMEM = OFF_RED + 16 * NCW;
  static_assert(SMEM <= 232448, "shared memory");
};

struct FMaps {
  CUtensorMap rho, v3, v1, v2;       // stencil input set (A: y, B: C)
  CUtensorMap yr, y1, y2, y3;        // B: y on the intermediate geometries
  CUtensorMap q5, yu;                // B: Q centres (5 GFs) and y.u centre
};

// shared-memory centered D1 (no 1/h), same operation order as wave::d1
__device__ __forceinline__ double d1s_(const double* f, int c, int s) {
  double acc = 0.0;
#pragma unroll
  for (int q = W; q >= 1; --q) acc = fma(D1W<W>::c(q), f[c + q * s] - f[c - q * s], acc);
  return acc;
}

__device__ __forceinline__ void cbar() { asm volatile("bar.sync 1, %0;" ::"r"(32 * NCW) : "memory"); }

// MON: kernel B with the fused energy monitor (its own instantiation: the default kernel
// carries none of the monitor's work)
template <bool B, bool MON>
__global__ void __launch_bounds__(NT, 1)
    wave_fused3(const __grid_constant__ FMaps M, StageLaunch a, WaveK K, int kchunk, int ntx, int nty, int nitems) {
  using G = Geo<B>;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + G::OFF_BAR);
  uint64_t* zfull = bars;
  uint64_t* zempty = zfull + G::RZ;
  uint64_t* pfull = zempty + G::RZ;
  uint64_t* pempty = pfull + G::RP;
  uint64_t* qfull = pempty + G::RP;
  uint64_t* qempty = qfull + G::RQ;
  uint64_t* done = qempty + G::RQ;
  int* itemq = reinterpret_cast<int*>(smem + G::OFF_ITEMQ);
  const Layout& L = a.L;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < G::RZ; ++s) { mbar_init(zfull + s, 1); mbar_init(zempty + s, NCW); }
    for (int s = 0; s < G::RP; ++s) { mbar_init(pfull + s, 1); mbar_init(pempty + s, NCW); }
    for (int s = 0; s < G::RQ; ++s) { mbar_init(qfull + s, 1); mbar_init(qempty + s, NCW); }
    for (int s = 0; s < ND; ++s) mbar_init(done + s, NCW);
    fence_mbar_init();
  }
  __syncthreads();
  const int g = L.g;
  const int nkall = a.k_end - a.k_begin;

  if (warp == NCW) {  // ------------------------------------------------------ producer
    if (lane != 0) return;
    uint32_t nz = 0, np = 0, nq = 0, nit = 0;
    for (;;) {
      const int item = (int)atomicAdd(a.sched, 1ull);
      {  // the item index (or the end marker) travels with the item's first input slot
        const uint32_t s = nz % G::RZ, n = nz / G::RZ;
        if (n > 0) mbar_wait_suspend(zempty + s, (n - 1) & 1);
        itemq[nit % IQ] = item;
        ++nit;
        if (item >= nitems) {
          mbar_arrive(zfull + s);  // completes the slot's phase with no data: end of work
          break;
        }
      }
      const int bx = item % ntx, by = (item / ntx) % nty, ch = item / (ntx * nty);
      const int i0 = bx * TX, j0 = by * TY;
      const int kb = a.k_begin + ch * kchunk;
      const int nk = min(kchunk, a.k_begin + nkall - kb);
      const int xo = kXOff + i0, yo = g + j0;
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
      auto loadQ = [&](int plane) {
        const uint32_t s = nq % G::RQ, n = nq / G::RQ;
        if (n > 0) mbar_wait_suspend(qempty + s, (n - 1) & 1);
        unsigned char* d = smem + G::OFF_Q + s * G::QSLOT;
        mbar_arrive_expect_tx(qfull + s, G::QBYTES);
        tma_load_4d(d, &M.q5, qfull + s, xo, yo, g + plane, GU);
        tma_load_4d(d + 5 * C1 * 8, &M.yu, qfull + s, xo, yo, g + plane, GU);
        ++nq;
      };
      // intermediate planes p = kb-2 .. kb+nk+1 need input planes p-2 .. p+2
      for (int pl = kb - 4; pl < kb; ++pl) loadZ(pl);
      for (int j = 0; j < nk + 4; ++j) {
        const int p = kb - 2 + j;
        loadZ(p + 2);
        loadP(p);
        if (B && p - LAG >= kb) loadQ(p - LAG);
      }
      if (B)
        for (int k = kb + nk + 2 - LAG; k < kb + nk; ++k) loadQ(k);
    }
    // the last CTA to finish fetching resets the scheduler for the next launch
    if (atomicAdd(a.sched + 1, 1ull) == gridDim.x - 1) {
      a.sched[0] = 0ull;
      a.sched[1] = 0ull;
    }
    return;
  }

  // --------------------------------------------------------------------------- consumers
  const int tid = threadIdx.x;
  const int64_t gfs = L.gfs;
  constexpr int NTC = 32 * NCW;
  const int ti = lane, tj = warp;  // this thread's output point of the tile
  // the own point in the input boxes (origins: rho (-4,-4), v1 (-4,-2), v2 (-2,-4), v3 (-2,-2))
  const int o_r = (tj + 4) * BR_X + ti + 4, o_1 = (tj + 2) * B1_X + ti + 4;
  const int o_2 = (tj + 4) * B2_X + ti + 2, o_3 = (tj + 2) * B3_X + ti + 2;
  // ... and in the intermediate geometries (IR (-2,-2), I1 (-2,0), I2 (0,-2))
  const int e_R = (tj + 2) * IR_X + ti + 2, e_1 = tj * I1_X + ti + 2, e_2 = (tj + 2) * I2_X + ti;
  const int cc = tj * TX + ti;
  // halo elements: IR ring of the 36x12 plane minus the 32x8 interior (176, threads 64..239),
  // I1 columns x in {0,1,34,35} (32, warp 0), I2 rows y in {0,1,10,11} (128, threads 0..63 x 2)
  const bool hR = tid >= 64 && tid < 64 + (IR_X * IR_Y - TX * TY);
  int hR_c1 = 0, hR_c2 = 0, hR_c3 = 0, hR_b = 0, hR_e = 0;
  {
    const int h = hR ? tid - 64 : 0;
    int x, y;
    if (h < 2 * IR_X) { y = h / IR_X; x = h % IR_X; }
    else if (h < 4 * IR_X) { y = IR_Y - 2 + (h - 2 * IR_X) / IR_X; x = (h - 2 * IR_X) % IR_X; }
    else { const int q = h - 4 * IR_X; y = 2 + q / 4; x = (q % 4) < 2 ? q % 4 : IR_X - 4 + q % 4; }
    hR_c1 = y * B1_X + x + 2; hR_c2 = (y + 2) * B2_X + x; hR_c3 = y * B3_X + x;
    hR_b = (y + 2) * BR_X + x + 2; hR_e = y * IR_X + x;
  }
  const bool h1 = tid < 32;
  int h1_cr, h1_b, h1_e;
  {
    const int y = tid / 4 % I1_Y, q = tid % 4, x = q < 2 ? q : I1_X - 4 + q;
    h1_cr = (y + 4) * BR_X + x + 2; h1_b = (y + 2) * B1_X + x + 2; h1_e = y * I1_X + x;
  }
  const bool h2 = tid < 64;
  int h2_cr[2], h2_b[2], h2_e[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int h = (tid % 64) + 64 * u, r = h / I2_X, x = h % I2_X, y = r < 2 ? r : I2_Y - 4 + r;
    h2_cr[u] = (y + 2) * BR_X + x + 4; h2_b[u] = (y + 2) * B2_X + x + 2; h2_e[u] = y * I2_X + x;
  }
  static_assert(IR_X * IR_Y - TX * TY == 176 && IR_X * IR_Y - TX * TY <= NTC - 64, "halo map");
  const double cdt = B ? K.dt : K.dt2;
  double* const sm = reinterpret_cast<double*>(smem);
  constexpr int ZSD = ZSLOT / 8, ZR_D = ZR_B / 8, PSD = G::PSLOT / 8, P1D = P1_B / 8, P2D = P2_B / 8;
  constexpr int IZD = IZ_B / 8, IPD = IP_B / 8, I1_D = r128(I1_X * I1_Y * 8) / 8;
  constexpr int OFF_PD = G::OFF_P / 8, OFF_QD = G::OFF_Q / 8, OFF_IZD = G::OFF_IZ / 8, OFF_IPD = G::OFF_IP / 8;
  constexpr int PYR = PY_R / 8, PY1 = PY_1 / 8, PY2 = PY_2 / 8;
  const double C1W = D1W<W>::c(1), C2W = D1W<W>::c(2);

  double eacc = 0.0;  // this thread's energy sum over the current item (B, monitor on)
  uint32_t bad = 0;   // B: bit f set once GF f produced a non-finite value (reported at the end)
  uint32_t nz = 0, np = 0, nq = 0, nit = 0;
  uint32_t t = 0;  // iterations of this CTA's warps over all items
  int wslot = 0;   // t mod RI_Z: the intermediate slot written in iteration t
  for (;;) {
    const uint32_t z0 = nz, p0 = np;  // ring index of input plane kb-4, of P plane kb-2
    mbar_wait(zfull + z0 % G::RZ, (z0 / G::RZ) & 1);  // the item's first input plane, or the end
    const int item = itemq[nit % IQ];
    ++nit;
    if (item >= nitems) break;
    const int bx = item % ntx, by = (item / ntx) % nty, ch = item / (ntx * nty);
    const int i0 = bx * TX, j0 = by * TY;
    const int kb = a.k_begin + ch * kchunk;
    const int nk = min(kchunk, a.k_begin + nkall - kb);
    for (int q = 0; q < 4; ++q) mbar_wait(zfull + (z0 + q) % G::RZ, ((z0 + q) / G::RZ) & 1);
    const int i = i0 + ti, j = j0 + tj;
    const bool live = i < L.nx && j < L.ny;
    int64_t cglob = L.idx(i, j, kb);  // global offset of this thread's point at plane k
    // ghost images (see image_site): the x/y part is fixed for the item; only warps with a
    // point near an x or y face -- or any warp on a plane near a z face -- store images
    const bool nxf = i < L.g || i >= L.nx - L.g, nyf = j < L.g || j >= L.ny - L.g;
    const int64_t ioff = nxf ? (int64_t)(i < L.g ? L.nx : -L.nx) : (int64_t)(j < L.g ? L.ny : -L.ny) * L.px;
    const bool img_xy = __any_sync(0xffffffffu, live && (nxf || nyf));
    int zsl[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) zsl[q] = (int)((z0 + G::RZ + q - 1) % G::RZ);
    int zph = (int)(((z0 + 4) / G::RZ) & 1);    // phase of the input slot zsl[5]
    int psl = (int)(p0 % G::RP);                // P slot of plane p
    int pph = (int)((p0 / G::RP) & 1);
    int pslk = psl;                             // P slot of plane k = p - 3 (A, jj >= 3)
    int izs[4] = {0, 0, 0, 0};                  // intermediate rho slots of planes p-3 .. p
    int ips[4] = {0, 0, 0, 0};                  // intermediate v1/v2 slots of planes p-3 .. p
    // register queues (see the file header); index 0 is the oldest plane
    double qIR[5], qI3[5];
#pragma unroll
    for (int q = 0; q < 5; ++q) { qIR[q] = 0.0; qI3[q] = 0.0; }
#pragma unroll 1
    for (int jj = 0; jj < nk + 4 + 1; ++jj) {
      const int p = kb - 2 + jj;
      const bool first = jj < nk + 4;           // intermediate plane p is needed
      const int k = p - LAG;
      const bool second = k >= kb;              // output plane k
#pragma unroll
      for (int q = 0; q < 3; ++q) izs[q] = izs[q + 1];
      izs[3] = wslot;
#pragma unroll
      for (int q = 0; q < 3; ++q) ips[q] = ips[q + 1];
      ips[3] = wslot;
      // every warp has finished iteration t-2: the slot written now was last read there, and
      // the slot read now (written in t-3) is complete
      if (t >= 2) mbar_wait(done + (t - 2) % ND, ((t - 2) / ND) & 1);
      double IRown = 0.0, I3own = 0.0;
      if (first) {
        mbar_wait(zfull + zsl[5], zph);
        mbar_wait(pfull + psl, pph);
        const double* zR[5];
        const double* z3[5];
#pragma unroll
        for (int q = 0; q < 5; ++q) {
          zR[q] = sm + zsl[q + 1] * ZSD;
          z3[q] = zR[q] + ZR_D;
        }
        const double* s1 = sm + OFF_PD + psl * PSD;
        const double* s2 = s1 + P1D;
        const double* sy = s2 + P2D;  // B only
        double* IR = sm + OFF_IZD + izs[3] * IZD;
        double* I1 = sm + OFF_IPD + ips[3] * IPD;
        double* I2 = I1 + I1_D;
        // ---- intermediate state at plane p: Y2 = y + dt/2 k1(y) (A) or Y4 = y + dt k3(C) (B)
        {  // rho at the own point; z neighbours of v3 from the queue (planes p-2 .. p+2)
          const double dv1 = d1s_(s1, o_1, 1) * K.ih[0];
          const double dv2 = d1s_(s2, o_2, B2_X) * K.ih[1];
          double dv3 = 0.0;
          dv3 = fma(C2W, z3[4][o_3] - z3[0][o_3], dv3);
          dv3 = fma(C1W, z3[3][o_3] - z3[1][o_3], dv3);
          dv3 = dv3 * K.ih[2];
          const double kr = dv1 + dv2 + dv3;
          const double base = B ? sy[e_R] : zR[2][o_r];
          IRown = fma(cdt, kr, base);
          IR[e_R] = IRown;
        }
        if (hR) {  // rho at the halo element
          const double dv1 = d1s_(s1, hR_c1, 1) * K.ih[0];
          const double dv2 = d1s_(s2, hR_c2, B2_X) * K.ih[1];
          double dv3 = 0.0;
          dv3 = fma(C2W, z3[4][hR_c3] - z3[0][hR_c3], dv3);
          dv3 = fma(C1W, z3[3][hR_c3] - z3[1][hR_c3], dv3);
          dv3 = dv3 * K.ih[2];
          const double kr = dv1 + dv2 + dv3;
          const double base = B ? sy[hR_e] : zR[2][hR_b];
          IR[hR_e] = fma(cdt, kr, base);
        }
        {  // v1, v2 at the own point
          const double k1v = d1s_(zR[2], o_r, 1) * K.ih[0];
          I1[e_1] = fma(cdt, k1v, B ? sy[PYR + e_1] : s1[o_1]);
          const double k2v = d1s_(zR[2], o_r, BR_X) * K.ih[1];
          I2[e_2] = fma(cdt, k2v, B ? sy[PYR + PY1 + e_2] : s2[o_2]);
        }
        if (h1) {
          const double kr = d1s_(zR[2], h1_cr, 1) * K.ih[0];
          I1[h1_e] = fma(cdt, kr, B ? sy[PYR + h1_e] : s1[h1_b]);
        }
        if (h2) {
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const double kr = d1s_(zR[2], h2_cr[u], BR_X) * K.ih[1];
            I2[h2_e[u]] = fma(cdt, kr, B ? sy[PYR + PY1 + h2_e[u]] : s2[h2_b[u]]);
          }
        }
        {  // v3 at the own point: z neighbours of rho from the queue; stays in registers
          double dzr = 0.0;
          dzr = fma(C2W, zR[4][o_r] - zR[0][o_r], dzr);
          dzr = fma(C1W, zR[3][o_r] - zR[1][o_r], dzr);
          const double kr = dzr * K.ih[2];
          const double base = B ? sy[PYR + PY1 + PY2 + cc] : z3[2][o_3];
          I3own = fma(cdt, kr, base);
        }
      }
      // ---- second stage at plane k = p - 3: x/y neighbours from the intermediate planes in
      // shared memory, z neighbours (planes k-2 .. k+2) from the register queues
      if (second) {
        const double* iRk = sm + OFF_IZD + izs[0] * IZD;
        const double* i1 = sm + OFF_IPD + ips[0] * IPD;
        const double* i2 = i1 + I1_D;
        double S[5], kk[5];
        S[GRHO] = qIR[2];
        S[GV1] = i1[e_1];
        S[GV2] = i2[e_2];
        S[GV3] = qI3[2];
        double dzr = 0.0, dv3 = 0.0;
        dzr = fma(C2W, qIR[4] - qIR[0], dzr);
        dv3 = fma(C2W, qI3[4] - qI3[0], dv3);
        dzr = fma(C1W, qIR[3] - qIR[1], dzr);
        dv3 = fma(C1W, qI3[3] - qI3[1], dv3);
        const double dxr = d1s_(iRk, e_R, 1) * K.ih[0];
        const double dyr = d1s_(iRk, e_R, IR_X) * K.ih[1];
        dzr = dzr * K.ih[2];
        const double dv1 = d1s_(i1, e_1, 1) * K.ih[0];
        const double dv2 = d1s_(i2, e_2, I2_X) * K.ih[1];
        dv3 = dv3 * K.ih[2];
        kk[GRHO] = dv1 + dv2 + dv3;
        kk[GV1] = dxr;
        kk[GV2] = dyr;
        kk[GV3] = dzr;
        double Y[5] = {0, 0, 0, 0, 0}, Qv[5] = {0, 0, 0, 0, 0}, yu = 0.0, qu = 0.0;
        if (!B) {
          // y at plane k: input plane k (Z slot), P plane k
          const double* zk = sm + zsl[0] * ZSD;
          const double* k1 = sm + OFF_PD + pslk * PSD;
          const double* k2 = k1 + P1D;
          Y[GRHO] = zk[o_r];
          Y[GV1] = k1[o_1];
          Y[GV2] = k2[o_2];
          Y[GV3] = zk[ZR_D + o_3];
        } else {
          mbar_wait(qfull + nq % G::RQ, (nq / G::RQ) & 1);
          const double* qs = sm + OFF_QD + (nq % G::RQ) * (G::QSLOT / 8);
          // u carry of stage 3 (folded): Q.u += dt/3 C.rho, with C.rho at plane k
          qu = fma(K.dt3, (sm + zsl[0] * ZSD)[o_r], qs[cc]);
#pragma unroll
          for (int f = 1; f <= 4; ++f) Qv[f] = qs[f * C1 + cc];
          yu = qs[5 * C1 + cc];
        }
        // ghost images: only warps with a point near an x/y/z face take the image path (the
        // tile rows of the interior -- most warps -- store the new values only)
        const bool kface = k < L.g || k >= L.nz - L.g;
        const ImageSite isite{kface || (nxf && nyf), nxf || nyf, ioff};
        const bool img = img_xy || kface;
        if (live) {
          const int64_t c = cglob;
          if (!B) {
            double* outc = a.s.c;
            const FaceDst fd = a.img[1];
            auto putq = [&](int f, double v) { a.s.q[f * gfs + c] = v; };
            if (img) {
              auto put = [&](int f, double v) {
                outc[f * gfs + c] = v;
                put_images(isite, outc + f * gfs, fd.lo + f * gfs, fd.hi + f * gfs, L, i, j, k, c, v);
              };
              wave_update<2>(K, S, kk, Y, Qv, yu, qu, put, putq);
            } else {
              auto put = [&](int f, double v) { outc[f * gfs + c] = v; };
              wave_update<2>(K, S, kk, Y, Qv, yu, qu, put, putq);
            }
          } else {
            double* outy = a.s.b;  // the new state goes to the scratch set (swapped by the caller)
            const FaceDst fd = a.img[0];
            constexpr bool mon = MON;
            double esq = 0.0;  // rho^2 + v.v of the new state (fused energy monitor)
            double chk = 0.0;  // 0 * v: NaN once any new value is non-finite
            auto putq = [&](int, double) {};
            if (img) {
              auto put = [&](int f, double v) {
                outy[f * gfs + c] = v;
                put_images(isite, outy + f * gfs, fd.lo + f * gfs, fd.hi + f * gfs, L, i, j, k, c, v);
                chk = fma(v, 0.0, chk);
                if (mon && f >= 1) esq += v * v;
              };
              wave_update<4>(K, S, kk, Y, Qv, yu, qu, put, putq);
            } else {
              auto put = [&](int f, double v) {
                outy[f * gfs + c] = v;
                chk = fma(v, 0.0, chk);
                if (mon && f >= 1) esq += v * v;
              };
              wave_update<4>(K, S, kk, Y, Qv, yu, qu, put, putq);
            }
            // (rare) which GFs: re-read the values this thread just stored
            if (chk != 0.0)
#pragma unroll
              for (int f = 0; f < 5; ++f) bad |= (fabs(outy[f * gfs + c]) <= 1.7976931348623157e308 ? 0u : 1u) << f;
            if (MON) eacc += 0.5 * esq;
          }
        }
        cglob += L.plane;
      }
      // intermediate queues: push the own values of plane p
#pragma unroll
      for (int q = 0; q < 4; ++q) { qIR[q] = qIR[q + 1]; qI3[q] = qI3[q + 1]; }
      qIR[4] = IRown;
      qI3[4] = I3own;
      // ---- release what this warp has finished reading
      __syncwarp();
      if (lane == 0) {
        if (B && second) mbar_arrive(qempty + nq % G::RQ);
        if (B) {
          if (first) mbar_arrive(pempty + psl);          // P plane p (first stage only)
        } else if (second) {
          mbar_arrive(pempty + pslk);                     // P plane k
        } else if (jj < 2) {
          mbar_arrive(pempty + psl);                      // planes kb-2, kb-1: no second stage
        }
        if (jj >= 1) mbar_arrive(zempty + zsl[0]);        // input plane p - 3
        mbar_arrive(done + t % ND);                       // this warp is done with iteration t
      }
      ++t;
      wslot = wslot + 1 == RI_Z ? 0 : wslot + 1;
      if (B && second) ++nq;
      // ---- advance the rings
#pragma unroll
      for (int q = 0; q < 5; ++q) zsl[q] = zsl[q + 1];
      zsl[5] = zsl[4] + 1 == G::RZ ? 0 : zsl[4] + 1;
      if (zsl[5] == 0) zph ^= 1;
      if (jj == 2) pslk = (int)(p0 % G::RP);            // plane k of iteration 3 = P index 0
      else if (jj > 2) pslk = pslk + 1 == G::RP ? 0 : pslk + 1;
      psl = psl + 1 == G::RP ? 0 : psl + 1;
      if (psl == 0) pph ^= 1;
    }
    // input planes ke .. ke+3 and (A) P planes ke, ke+1 were only read
    __syncwarp();
    if (lane == 0) {
      if (!B)
        for (int q = 0; q < 2; ++q) mbar_arrive(pempty + (p0 + nk + 2 + q) % G::RP);
      for (int q = 0; q < 4; ++q) mbar_arrive(zempty + (z0 + nk + 4 + q) % G::RZ);
    }
    nz = z0 + nk + 8;
    np = p0 + nk + 4;
    // NEXT-3 fused energy monitor (Fig. 1 "Energy"): one partial per item
    // (tile x z-chunk), a fixed shuffle tree then warps in order, so the per-step energy does
    // not depend on which CTA ran the item
    if (B && MON) {
      double v = eacc;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      double* red = reinterpret_cast<double*>(smem + G::OFF_RED) + (nit & 1) * NCW;  // double-buffered
      if (lane == 0) red[warp] = v;
      cbar();
      if (tid == 0) {
        double sum = 0.0;
        for (int w = 0; w < NCW; ++w) sum += red[w];
        a.mon_partials[item] = sum;
      }
      eacc = 0.0;
    }
  }
  // the first non-finite GF of this thread (the flag keeps min(step * n_gf + gf) over threads)
  if (B && bad) check_finite(a.nan_flag, a.step * (unsigned long long)a.L.n_gf + (unsigned long long)(__ffs(bad) - 1),
                             __longlong_as_double(0x7ff8000000000000ll));
}

bool enc(CUtensorMap* m, const double* set, const Layout& L, unsigned bx, unsigned by, unsigned bg) {
  return encode_set_map(m, set - L.c0, L.px, L.py, L.pz, L.n_gf, L.gfs, bx, by, bg);
}

WaveK make_k(const StageLaunch& a) {
  WaveK K;
  for (int d = 0; d < 3; ++d) K.ih[d] = 1.0 / a.h[d];
  K.half = 0.5; K.third = 1.0 / 3.0; K.sixth = 1.0 / 6.0;
  K.dt = a.dt; K.dt2 = a.dt / 2.0; K.dt3 = a.dt / 3.0; K.dt6 = a.dt / 6.0;
  return K;
}

template <bool B, bool MON>
cudaError_t launch(const StageLaunch& a, cudaStream_t st) {
  using G = Geo<B>;
  const int nk = a.k_end - a.k_begin;
  if (nk <= 0) return cudaSuccess;
  const Layout& L = a.L;
  const double* in = B ? a.s.c : a.s.y;
  FMaps M;
  bool ok = enc(&M.rho, in, L, BR_X, BR_Y, 1) && enc(&M.v3, in, L, B3_X, B3_Y, 1) &&
            enc(&M.v1, in, L, B1_X, B1_Y, 1) && enc(&M.v2, in, L, B2_X, B2_Y, 1) &&
            enc(&M.yr, a.s.y, L, IR_X, IR_Y, 1) && enc(&M.y1, a.s.y, L, I1_X, I1_Y, 1) &&
            enc(&M.y2, a.s.y, L, I2_X, I2_Y, 1) && enc(&M.y3, a.s.y, L, I3_X, I3_Y, 1) &&
            enc(&M.q5, a.s.q, L, TX, TY, 5) && enc(&M.yu, a.s.y, L, TX, TY, 1);
  if (!ok) return cudaErrorInvalidValue;
  static std::atomic<uint64_t> attr_done{0};
  if (cudaError_t e = smem_optin((const void*)wave_fused3<B, MON>, G::SMEM, attr_done); e != cudaSuccess) return e;
  const int nsm = device_sm_count();
  const int ntx = (int)((L.nx + TX - 1) / TX), nty = (int)((L.ny + TY - 1) / TY);
  // z planes per item (128: measured best of 32..512 at 512^3): longer chunks recompute
  // fewer halo planes, shorter ones balance the persistent CTAs better
  constexpr int zc = 128;
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
  wave_fused3<B, MON><<<grid, NT, G::SMEM, st>>>(M, a, K, chunk, ntx, nty, nitems);
  return cudaGetLastError();
}

}  // namespace

cudaError_t wave_fused3_pair(const StageLaunch& a, int pair, cudaStream_t st) {
  if (a.fd_order != 4) return cudaErrorInvalidValue;
  return pair == 0 ? launch<false, false>(a, st)
                   : (a.mon_partials ? launch<true, true>(a, st) : launch<true, false>(a, st));
}

}  // namespace chemora
