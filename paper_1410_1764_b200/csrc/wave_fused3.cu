// wave_fused3.cu -- kernel variant 8: the temporally blocked RK4 stage pairs (Eq. 1,
// PAPER.md:320-327) -- stages 1+2 in kernel A, 3+4 in kernel B -- for stencil
// radius W = 1, 2, 3 (FD orders 2, 4, 6), with the z stencils of each
// thread's own column taken from register queues (2.5-D z-march inside the temporal blocking).
//
// Every consumer thread owns one output point (ti, tj) of the 32x8 tile, and with it the
// intermediate values at that point (rho, v1, v2, v3); the halo elements of the intermediate
// rho / v1 / v2 planes (176 / 32 / 128 at W = 2) are spread over the other threads.  The thread
// keeps its own intermediate rho and v3 for planes p-2W-1 .. p-1 in registers, so the second
// stage's z stencils and centres need no shared loads and the intermediate v3 never goes to
// shared memory.  (Keeping the input rho/v3 column in registers too exceeds the 168-register
// cap of the 9-warp CTA: measured slower.)  Same arithmetic in the same order as the
// one-kernel-per-stage path (bit-identical; no FMA contraction).
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
constexpr int r128(int b) { return (b + 127) / 128 * 128; }
constexpr int C1 = TX * TY;         // points per tile plane
constexpr int IQ = 4;               // item queue (see the producer)
constexpr int ND = 4;               // per-iteration "done" mbarriers, used round robin

// Geometry of the stage pair for stencil radius W (FD order 2W; W = 2: the 4th-order default).
// Boxes are [y][x] planes around the 32x8 tile; a box's x origin is rounded down to an even
// offset (a TMA box whose fp64 rows start at an odd column faults), so for odd W the x-extended
// boxes carry one unused column at each side.
template <int W> struct PG {
  static constexpr int H = 2 * W;                 // input halo: two stacked radius-W stencils
  static constexpr int WX = (W + 1) / 2 * 2;      // x halo of the W-extended boxes, even
  // input boxes (x extent, y extent; x origin, y origin relative to the tile)
  static constexpr int BR_X = TX + 2 * H, BR_Y = TY + 2 * H, BR_OX = -H, BR_OY = -H;     // rho
  static constexpr int B3_X = TX + 2 * WX, B3_Y = TY + 2 * W, B3_OX = -WX, B3_OY = -W;  // v3
  static constexpr int B1_X = TX + 2 * H, B1_Y = TY + 2 * W, B1_OX = -H, B1_OY = -W;     // v1
  static constexpr int B2_X = TX + 2 * WX, B2_Y = TY + 2 * H, B2_OX = -WX, B2_OY = -H;  // v2
  // intermediate-state geometries (the same x rounding: kernel B loads y on them by TMA)
  static constexpr int IR_X = TX + 2 * WX, IR_Y = TY + 2 * W, IR_OX = -WX, IR_OY = -W;  // rho
  static constexpr int I1_X = TX + 2 * WX, I1_Y = TY, I1_OX = -WX, I1_OY = 0;           // v1
  static constexpr int I2_X = TX, I2_Y = TY + 2 * W, I2_OX = 0, I2_OY = -W;             // v2
  static constexpr int I3_X = TX, I3_Y = TY;                                            // v3
  // halo elements computed by the first stage (logical, radius W): the IR ring, the I1 side
  // columns, the I2 top / bottom rows
  static constexpr int NHR = (TX + 2 * W) * (TY + 2 * W) - TX * TY, NH1 = 2 * W * TY, NH2 = 2 * W * TX;
  static constexpr int NH2T = (NH2 + 63) / 64;    // I2 halo elements per thread (threads 0..63)
  static constexpr int ZR_B = r128(BR_X * BR_Y * 8), Z3_B = r128(B3_X * B3_Y * 8);
  static constexpr int ZSLOT = ZR_B + Z3_B;
  static constexpr uint32_t ZBYTES = (BR_X * BR_Y + B3_X * B3_Y) * 8;
  static constexpr int P1_B = r128(B1_X * B1_Y * 8), P2_B = r128(B2_X * B2_Y * 8);
  static constexpr int PY_R = r128(IR_X * IR_Y * 8), PY_1 = r128(I1_X * I1_Y * 8), PY_2 = r128(I2_X * I2_Y * 8),
                       PY_3 = r128(I3_X * I3_Y * 8);
  static constexpr int IZ_B = r128(IR_X * IR_Y * 8);  // intermediate rho ring slot (v3 lives in registers)
  static constexpr int IP_B = r128(I1_X * I1_Y * 8) + r128(I2_X * I2_Y * 8);  // intermediate p ring slot
  // The second stage runs LAG = W+1 planes behind the first (k = p - LAG), so within one
  // iteration the two stages touch disjoint intermediate slots.  The intermediate rings hold
  // LAG+2 planes: iteration t writes slot t mod (LAG+2), which the second stage last read in
  // iteration t-2, and reads the slot written in t-LAG.  So the warps need not meet at a CTA
  // barrier every plane: each arrives on a per-iteration mbarrier when done and, before
  // writing, waits only until every warp has finished iteration t-2 (the warps may drift one
  // plane apart; radius 3: t-1).
  static constexpr int LAG = W + 1;
  // (radius 3: LAG+1 slots -- shared memory is full -- so the warps wait for iteration t-1)
  static constexpr int RI = W <= 2 ? LAG + 2 : LAG + 1;
  static constexpr int DW = RI - LAG;             // before writing in iteration t: wait for t-DW
  static constexpr int NHRT = (NHR + 32 * NCW - 64 - 1) / (32 * NCW - 64);  // IR halo elements per thread
  static_assert(NH1 <= 32 * NCW && W >= 1 && W <= 3, "halo map");
};
// items (tile x z-chunk) are handed out dynamically (an atomic counter, in order), so the
// items in flight at any time are neighbours in (x, y): their shared halo rows are read by
// both while still in L2.  (With a static round-robin assignment the persistent CTAs drift
// apart by tens of planes over a launch and the halos are read from HBM twice.)  The
// producer passes each item index to its consumers through a small shared queue, published
// by the mbarrier of the item's first input plane.

template <int W, bool B> struct Geo {
  using Q = PG<W>;
  // input ring depths: resident windows are Z: planes p-LAG .. p+W, P: p-LAG .. p (A) or p
  // (B), Q: k (B); the rest is prefetch (radius 3: one plane each, to fit 227 KB)
  static constexpr int RZ = W <= 2 ? (B ? 8 : 10) : 2 * W + 3;
  static constexpr int RP = W <= 2 ? (B ? 3 : 8) : (B ? 2 : W + 3);
  static constexpr int RQ = B ? (W <= 2 ? 3 : 2) : 1;  // (A: one unused slot pair keeps the ring arithmetic defined)
  static constexpr int PSLOT = Q::P1_B + Q::P2_B + (B ? Q::PY_R + Q::PY_1 + Q::PY_2 + Q::PY_3 : 0);
  static constexpr uint32_t PBYTES =
      (Q::B1_X * Q::B1_Y + Q::B2_X * Q::B2_Y +
       (B ? Q::IR_X * Q::IR_Y + Q::I1_X * Q::I1_Y + Q::I2_X * Q::I2_Y + Q::I3_X * Q::I3_Y : 0)) * 8;
  static constexpr int QSLOT = B ? r128(6 * C1 * 8) : 0;  // Q (u, rho, v1..3) + y.u
  static constexpr uint32_t QBYTES = B ? 6 * C1 * 8 : 0;
  static constexpr int OFF_P = RZ * Q::ZSLOT;
  static constexpr int OFF_Q = OFF_P + RP * PSLOT;
  static constexpr int OFF_IZ = OFF_Q + RQ * QSLOT;
  static constexpr int OFF_IP = OFF_IZ + Q::RI * Q::IZ_B;
  static constexpr int OFF_BAR = OFF_IP + Q::RI * Q::IP_B;
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
template <int W>
__device__ __forceinline__ double d1s_(const double* f, int c, int s) {
  double acc = 0.0;
#pragma unroll
  for (int q = W; q >= 1; --q) acc = fma(D1W<W>::c(q), f[c + q * s] - f[c - q * s], acc);
  return acc;
}

__device__ __forceinline__ void cbar() { asm volatile("bar.sync 1, %0;" ::"r"(32 * NCW) : "memory"); }

// MON: kernel B with the fused energy monitor (its own instantiation: the default kernel
// carries none of the monitor's work)
template <int W, bool B, bool MON>
__global__ void __launch_bounds__(NT, 1)
    wave_fused3(const __grid_constant__ FMaps M, StageLaunch a, WaveK K, int kchunk, int ntx, int nty, int nitems) {
  using G = Geo<W, B>;
  using Q = PG<W>;
  constexpr int LAG = Q::LAG;
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
        unsigned char* d = smem + s * Q::ZSLOT;
        mbar_arrive_expect_tx(zfull + s, Q::ZBYTES);
        tma_load_4d(d, &M.rho, zfull + s, xo + Q::BR_OX, yo + Q::BR_OY, g + plane, GRHO);
        tma_load_4d(d + Q::ZR_B, &M.v3, zfull + s, xo + Q::B3_OX, yo + Q::B3_OY, g + plane, GV3);
        ++nz;
      };
      auto loadP = [&](int plane) {
        const uint32_t s = np % G::RP, n = np / G::RP;
        if (n > 0) mbar_wait_suspend(pempty + s, (n - 1) & 1);
        unsigned char* d = smem + G::OFF_P + s * G::PSLOT;
        uint64_t* bar = pfull + s;
        mbar_arrive_expect_tx(bar, G::PBYTES);
        tma_load_4d(d, &M.v1, bar, xo + Q::B1_OX, yo + Q::B1_OY, g + plane, GV1);
        tma_load_4d(d + Q::P1_B, &M.v2, bar, xo + Q::B2_OX, yo + Q::B2_OY, g + plane, GV2);
        if (B) {
          unsigned char* e = d + Q::P1_B + Q::P2_B;
          tma_load_4d(e, &M.yr, bar, xo + Q::IR_OX, yo + Q::IR_OY, g + plane, GRHO);
          tma_load_4d(e + Q::PY_R, &M.y1, bar, xo + Q::I1_OX, yo + Q::I1_OY, g + plane, GV1);
          tma_load_4d(e + Q::PY_R + Q::PY_1, &M.y2, bar, xo + Q::I2_OX, yo + Q::I2_OY, g + plane, GV2);
          tma_load_4d(e + Q::PY_R + Q::PY_1 + Q::PY_2, &M.y3, bar, xo, yo, g + plane, GV3);
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
      // intermediate planes p = kb-W .. kb+nk+W-1 need input planes p-W .. p+W
      for (int pl = kb - 2 * W; pl < kb; ++pl) loadZ(pl);
      for (int j = 0; j < nk + 2 * W; ++j) {
        const int p = kb - W + j;
        loadZ(p + W);
        loadP(p);
        if (B && p - LAG >= kb) loadQ(p - LAG);
      }
      if (B)
        for (int k = kb + nk + W - LAG; k < kb + nk; ++k) loadQ(k);
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
  const int ti = lane, tj = warp;  // this thread's output point of the tile
  // offset of logical point (x, y) (relative to the tile) in a box of width sx, origin (ox, oy)
  auto at = [](int x, int y, int sx, int ox, int oy) { return (y - oy) * sx + (x - ox); };
  // the own point in the input boxes and in the intermediate geometries
  const int o_r = at(ti, tj, Q::BR_X, Q::BR_OX, Q::BR_OY), o_1 = at(ti, tj, Q::B1_X, Q::B1_OX, Q::B1_OY);
  const int o_2 = at(ti, tj, Q::B2_X, Q::B2_OX, Q::B2_OY), o_3 = at(ti, tj, Q::B3_X, Q::B3_OX, Q::B3_OY);
  const int e_R = at(ti, tj, Q::IR_X, Q::IR_OX, Q::IR_OY), e_1 = at(ti, tj, Q::I1_X, Q::I1_OX, Q::I1_OY);
  const int e_2 = at(ti, tj, Q::I2_X, Q::I2_OX, Q::I2_OY);
  const int cc = tj * TX + ti;
  // halo elements (logical radius W): the IR ring (threads 64 ..), the I1 side columns
  // (threads 0 ..), the I2 top / bottom rows (threads 0..63, NH2T each)
  int hR_c1[Q::NHRT], hR_c2[Q::NHRT], hR_c3[Q::NHRT], hR_b[Q::NHRT], hR_e[Q::NHRT];
  bool hR[Q::NHRT];
#pragma unroll
  for (int u = 0; u < Q::NHRT; ++u) {
    constexpr int RX = TX + 2 * W;  // logical IR row length
    const int hh = tid - 64 + (32 * NCW - 64) * u;
    hR[u] = tid >= 64 && hh < Q::NHR;
    const int h = hR[u] ? hh : 0;
    int x, y;
    if (h < W * RX) { y = -W + h / RX; x = -W + h % RX; }
    else if (h < 2 * W * RX) { y = TY + (h - W * RX) / RX; x = -W + (h - W * RX) % RX; }
    else { const int q = h - 2 * W * RX, c = q % (2 * W); y = q / (2 * W); x = c < W ? -W + c : TX + c - W; }
    hR_c1[u] = at(x, y, Q::B1_X, Q::B1_OX, Q::B1_OY); hR_c2[u] = at(x, y, Q::B2_X, Q::B2_OX, Q::B2_OY);
    hR_c3[u] = at(x, y, Q::B3_X, Q::B3_OX, Q::B3_OY); hR_b[u] = at(x, y, Q::BR_X, Q::BR_OX, Q::BR_OY);
    hR_e[u] = at(x, y, Q::IR_X, Q::IR_OX, Q::IR_OY);
  }
  const bool h1 = tid < Q::NH1;
  int h1_cr, h1_b, h1_e;
  {
    const int y = tid / (2 * W) % TY, c = tid % (2 * W), x = c < W ? -W + c : TX + c - W;
    h1_cr = at(x, y, Q::BR_X, Q::BR_OX, Q::BR_OY); h1_b = at(x, y, Q::B1_X, Q::B1_OX, Q::B1_OY);
    h1_e = at(x, y, Q::I1_X, Q::I1_OX, Q::I1_OY);
  }
  const bool h2 = tid < 64;
  int h2_cr[Q::NH2T], h2_b[Q::NH2T], h2_e[Q::NH2T];
#pragma unroll
  for (int u = 0; u < Q::NH2T; ++u) {
    const int h = (tid % 64) + 64 * u, r = h / TX % (2 * W), x = h % TX, y = r < W ? -W + r : TY + r - W;
    h2_cr[u] = at(x, y, Q::BR_X, Q::BR_OX, Q::BR_OY); h2_b[u] = at(x, y, Q::B2_X, Q::B2_OX, Q::B2_OY);
    h2_e[u] = at(x, y, Q::I2_X, Q::I2_OX, Q::I2_OY);
  }
  static_assert(Q::NH2 == 64 * Q::NH2T, "I2 halo map");
  const double cdt = B ? K.dt : K.dt2;
  double* const sm = reinterpret_cast<double*>(smem);
  constexpr int ZSD = Q::ZSLOT / 8, ZR_D = Q::ZR_B / 8, PSD = G::PSLOT / 8, P1D = Q::P1_B / 8, P2D = Q::P2_B / 8;
  constexpr int IZD = Q::IZ_B / 8, IPD = Q::IP_B / 8, I1_D = r128(Q::I1_X * Q::I1_Y * 8) / 8;
  constexpr int OFF_PD = G::OFF_P / 8, OFF_QD = G::OFF_Q / 8, OFF_IZD = G::OFF_IZ / 8, OFF_IPD = G::OFF_IP / 8;
  constexpr int PYR = Q::PY_R / 8, PY1 = Q::PY_1 / 8, PY2 = Q::PY_2 / 8;
  constexpr int NZW = 2 * W + 1;  // z window of a stencil: planes -W .. +W

  double eacc = 0.0;  // this thread's energy sum over the current item (B, monitor on)
  uint32_t bad = 0;   // B: bit f set once GF f produced a non-finite value (reported at the end)
  uint32_t nz = 0, np = 0, nq = 0, nit = 0;
  uint32_t t = 0;  // iterations of this CTA's warps over all items
  int wslot = 0;   // t mod RI: the intermediate slot written in iteration t
  for (;;) {
    const uint32_t z0 = nz, p0 = np;  // ring index of input plane kb-2W, of P plane kb-W
    mbar_wait(zfull + z0 % G::RZ, (z0 / G::RZ) & 1);  // the item's first input plane, or the end
    const int item = itemq[nit % IQ];
    ++nit;
    if (item >= nitems) break;
    const int bx = item % ntx, by = (item / ntx) % nty, ch = item / (ntx * nty);
    const int i0 = bx * TX, j0 = by * TY;
    const int kb = a.k_begin + ch * kchunk;
    const int nk = min(kchunk, a.k_begin + nkall - kb);
    for (int q = 0; q < 2 * W; ++q) mbar_wait(zfull + (z0 + q) % G::RZ, ((z0 + q) / G::RZ) & 1);
    const int i = i0 + ti, j = j0 + tj;
    const bool live = i < L.nx && j < L.ny;
    int64_t cglob = L.idx(i, j, kb);  // global offset of this thread's point at plane k
    // ghost images (see image_site): the x/y part is fixed for the item; only warps with a
    // point near an x or y face -- or any warp on a plane near a z face -- store images
    const bool nxf = i < L.g || i >= L.nx - L.g, nyf = j < L.g || j >= L.ny - L.g;
    const int64_t ioff = nxf ? (int64_t)(i < L.g ? L.nx : -L.nx) : (int64_t)(j < L.g ? L.ny : -L.ny) * L.px;
    const bool img_xy = __any_sync(0xffffffffu, live && (nxf || nyf));
    int zsl[NZW + 1];                           // input slots of planes p-LAG .. p+W
#pragma unroll
    for (int q = 0; q <= NZW; ++q) zsl[q] = (int)((z0 + G::RZ + q - 1) % G::RZ);
    int zph = (int)(((z0 + 2 * W) / G::RZ) & 1);  // phase of the input slot zsl[NZW]
    int psl = (int)(p0 % G::RP);                // P slot of plane p
    int pph = (int)((p0 / G::RP) & 1);
    int pslk = psl;                             // P slot of plane k = p - LAG (A, jj >= LAG)
    int izs[LAG + 1] = {};                      // intermediate rho slots of planes p-LAG .. p
    int ips[LAG + 1] = {};                      // intermediate v1/v2 slots of planes p-LAG .. p
    // register queues (see the file header): planes p-2W-1 .. p-1, index 0 the oldest
    double qIR[NZW], qI3[NZW];
#pragma unroll
    for (int q = 0; q < NZW; ++q) { qIR[q] = 0.0; qI3[q] = 0.0; }
#pragma unroll 1
    for (int jj = 0; jj < nk + 2 * W + 1; ++jj) {
      const int p = kb - W + jj;
      const bool first = jj < nk + 2 * W;       // intermediate plane p is needed
      const int k = p - LAG;
      const bool second = k >= kb;              // output plane k
#pragma unroll
      for (int q = 0; q < LAG; ++q) izs[q] = izs[q + 1];
      izs[LAG] = wslot;
#pragma unroll
      for (int q = 0; q < LAG; ++q) ips[q] = ips[q + 1];
      ips[LAG] = wslot;
      // every warp has finished iteration t-DW: the slot written now was last read there, and
      // the slot read now (written in t-LAG) is complete
      if (t >= Q::DW) mbar_wait(done + (t - Q::DW) % ND, ((t - Q::DW) / ND) & 1);
      double IRown = 0.0, I3own = 0.0;
      if (first) {
        mbar_wait(zfull + zsl[NZW], zph);
        mbar_wait(pfull + psl, pph);
        const double* zR[NZW];  // input planes p-W .. p+W
        const double* z3[NZW];
#pragma unroll
        for (int q = 0; q < NZW; ++q) {
          zR[q] = sm + zsl[q + 1] * ZSD;
          z3[q] = zR[q] + ZR_D;
        }
        const double* s1 = sm + OFF_PD + psl * PSD;
        const double* s2 = s1 + P1D;
        const double* sy = s2 + P2D;  // B only
        double* IR = sm + OFF_IZD + izs[LAG] * IZD;
        double* I1 = sm + OFF_IPD + ips[LAG] * IPD;
        double* I2 = I1 + I1_D;
        // ---- intermediate state at plane p: Y2 = y + dt/2 k1(y) (A) or Y4 = y + dt k3(C) (B)
        {  // rho at the own point; z neighbours of v3 from the input planes p-W .. p+W
          const double dv1 = d1s_<W>(s1, o_1, 1) * K.ih[0];
          const double dv2 = d1s_<W>(s2, o_2, Q::B2_X) * K.ih[1];
          double dv3 = 0.0;
#pragma unroll
          for (int q = W; q >= 1; --q) dv3 = fma(D1W<W>::c(q), z3[W + q][o_3] - z3[W - q][o_3], dv3);
          dv3 = dv3 * K.ih[2];
          const double kr = dv1 + dv2 + dv3;
          const double base = B ? sy[e_R] : zR[W][o_r];
          IRown = fma(cdt, kr, base);
          IR[e_R] = IRown;
        }
#pragma unroll
        for (int u = 0; u < Q::NHRT; ++u)
          if (hR[u]) {  // rho at the halo element(s)
            const double dv1 = d1s_<W>(s1, hR_c1[u], 1) * K.ih[0];
            const double dv2 = d1s_<W>(s2, hR_c2[u], Q::B2_X) * K.ih[1];
            double dv3 = 0.0;
#pragma unroll
            for (int q = W; q >= 1; --q) dv3 = fma(D1W<W>::c(q), z3[W + q][hR_c3[u]] - z3[W - q][hR_c3[u]], dv3);
            dv3 = dv3 * K.ih[2];
            const double kr = dv1 + dv2 + dv3;
            const double base = B ? sy[hR_e[u]] : zR[W][hR_b[u]];
            IR[hR_e[u]] = fma(cdt, kr, base);
          }
        {  // v1, v2 at the own point
          const double k1v = d1s_<W>(zR[W], o_r, 1) * K.ih[0];
          I1[e_1] = fma(cdt, k1v, B ? sy[PYR + e_1] : s1[o_1]);
          const double k2v = d1s_<W>(zR[W], o_r, Q::BR_X) * K.ih[1];
          I2[e_2] = fma(cdt, k2v, B ? sy[PYR + PY1 + e_2] : s2[o_2]);
        }
        if (h1) {
          const double kr = d1s_<W>(zR[W], h1_cr, 1) * K.ih[0];
          I1[h1_e] = fma(cdt, kr, B ? sy[PYR + h1_e] : s1[h1_b]);
        }
        if (h2) {
#pragma unroll
          for (int u = 0; u < Q::NH2T; ++u) {
            const double kr = d1s_<W>(zR[W], h2_cr[u], Q::BR_X) * K.ih[1];
            I2[h2_e[u]] = fma(cdt, kr, B ? sy[PYR + PY1 + h2_e[u]] : s2[h2_b[u]]);
          }
        }
        {  // v3 at the own point: z neighbours of rho from the queue; stays in registers
          double dzr = 0.0;
#pragma unroll
          for (int q = W; q >= 1; --q) dzr = fma(D1W<W>::c(q), zR[W + q][o_r] - zR[W - q][o_r], dzr);
          const double kr = dzr * K.ih[2];
          const double base = B ? sy[PYR + PY1 + PY2 + cc] : z3[W][o_3];
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
        S[GRHO] = qIR[W];
        S[GV1] = i1[e_1];
        S[GV2] = i2[e_2];
        S[GV3] = qI3[W];
        double dzr = 0.0, dv3 = 0.0;
#pragma unroll
        for (int q = W; q >= 1; --q) {
          dzr = fma(D1W<W>::c(q), qIR[W + q] - qIR[W - q], dzr);
          dv3 = fma(D1W<W>::c(q), qI3[W + q] - qI3[W - q], dv3);
        }
        const double dxr = d1s_<W>(iRk, e_R, 1) * K.ih[0];
        const double dyr = d1s_<W>(iRk, e_R, Q::IR_X) * K.ih[1];
        dzr = dzr * K.ih[2];
        const double dv1 = d1s_<W>(i1, e_1, 1) * K.ih[0];
        const double dv2 = d1s_<W>(i2, e_2, Q::I2_X) * K.ih[1];
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
      for (int q = 0; q < NZW - 1; ++q) { qIR[q] = qIR[q + 1]; qI3[q] = qI3[q + 1]; }
      qIR[NZW - 1] = IRown;
      qI3[NZW - 1] = I3own;
      // ---- release what this warp has finished reading
      __syncwarp();
      if (lane == 0) {
        if (B && second) mbar_arrive(qempty + nq % G::RQ);
        if (B) {
          if (first) mbar_arrive(pempty + psl);          // P plane p (first stage only)
        } else if (second) {
          mbar_arrive(pempty + pslk);                     // P plane k
        } else if (jj < W) {
          mbar_arrive(pempty + psl);                      // planes kb-W .. kb-1: no second stage
        }
        if (jj >= 1) mbar_arrive(zempty + zsl[0]);        // input plane p - LAG
        mbar_arrive(done + t % ND);                       // this warp is done with iteration t
      }
      ++t;
      wslot = wslot + 1 == Q::RI ? 0 : wslot + 1;
      if (B && second) ++nq;
      // ---- advance the rings
#pragma unroll
      for (int q = 0; q < NZW; ++q) zsl[q] = zsl[q + 1];
      zsl[NZW] = zsl[NZW - 1] + 1 == G::RZ ? 0 : zsl[NZW - 1] + 1;
      if (zsl[NZW] == 0) zph ^= 1;
      if (jj == LAG - 1) pslk = (int)(p0 % G::RP);      // plane k of iteration LAG = P index 0
      else if (jj > LAG - 1) pslk = pslk + 1 == G::RP ? 0 : pslk + 1;
      psl = psl + 1 == G::RP ? 0 : psl + 1;
      if (psl == 0) pph ^= 1;
    }
    // input planes ke .. ke+2W-1 and (A) P planes ke .. ke+W-1 were only read
    __syncwarp();
    if (lane == 0) {
      if (!B)
        for (int q = 0; q < W; ++q) mbar_arrive(pempty + (p0 + nk + W + q) % G::RP);
      for (int q = 0; q < 2 * W; ++q) mbar_arrive(zempty + (z0 + nk + 2 * W + q) % G::RZ);
    }
    nz = z0 + nk + 4 * W;
    np = p0 + nk + 2 * W;
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

template <int W, bool B, bool MON>
cudaError_t launch(const StageLaunch& a, cudaStream_t st) {
  using G = Geo<W, B>;
  using Q = PG<W>;
  const int nk = a.k_end - a.k_begin;
  if (nk <= 0) return cudaSuccess;
  const Layout& L = a.L;
  const double* in = B ? a.s.c : a.s.y;
  FMaps M;
  bool ok = enc(&M.rho, in, L, Q::BR_X, Q::BR_Y, 1) && enc(&M.v3, in, L, Q::B3_X, Q::B3_Y, 1) &&
            enc(&M.v1, in, L, Q::B1_X, Q::B1_Y, 1) && enc(&M.v2, in, L, Q::B2_X, Q::B2_Y, 1) &&
            enc(&M.yr, a.s.y, L, Q::IR_X, Q::IR_Y, 1) && enc(&M.y1, a.s.y, L, Q::I1_X, Q::I1_Y, 1) &&
            enc(&M.y2, a.s.y, L, Q::I2_X, Q::I2_Y, 1) && enc(&M.y3, a.s.y, L, Q::I3_X, Q::I3_Y, 1) &&
            enc(&M.q5, a.s.q, L, TX, TY, 5) && enc(&M.yu, a.s.y, L, TX, TY, 1);
  if (!ok) return cudaErrorInvalidValue;
  static std::atomic<uint64_t> attr_done{0};
  if (cudaError_t e = smem_optin((const void*)wave_fused3<W, B, MON>, G::SMEM, attr_done); e != cudaSuccess)
    return e;
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
  wave_fused3<W, B, MON><<<grid, NT, G::SMEM, st>>>(M, a, K, chunk, ntx, nty, nitems);
  return cudaGetLastError();
}

template <int W>
cudaError_t pair_w(const StageLaunch& a, int pair, cudaStream_t st) {
  return pair == 0 ? launch<W, false, false>(a, st)
                   : (a.mon_partials ? launch<W, true, true>(a, st) : launch<W, true, false>(a, st));
}

}  // namespace

cudaError_t wave_fused3_pair(const StageLaunch& a, int pair, cudaStream_t st) {
  if (a.fd_order == 4) return pair_w<2>(a, pair, st);
  if (a.fd_order == 2) return pair_w<1>(a, pair, st);
  if (a.fd_order == 6) return pair_w<3>(a, pair, st);
  return cudaErrorInvalidValue;
}

}  // namespace chemora
