// wave_tma.cu -- persistent TMA z-march stage kernel for the wave equation (Eq. 1,
// PAPER.md:320-327), the B200-native tiling of the fused RHS + RK4 stage.
//
// One CTA per SM walks a list of work items (x-y tile of TX x TY points, chunk of z planes),
// item order x-tile fastest so the CTAs busy at any moment cover a compact band of the grid
// (their x/y halos are each other's interiors and hit L2).  Per CTA, one elected producer
// thread streams every operand of the stage into shared memory with TMA (4-D tensor maps
// over a state set [gf][z][y][x]), two rings with full/empty mbarriers:
//   ring Z, depth 2W+3: rho with its x/y halo and v3 -- the GFs differentiated along z, so
//                       2W+1 consecutive planes of them stay resident (z reuse on chip);
//   ring P, depth 3:    v1 with its x halo, v2 with its y halo, and the pointwise operands
//                       of the stage (y for stages 2-3, Q and y.u for stage 4) as
//                       multi-GF boxes.
// Sixteen consumer warps compute one point each per plane entirely from shared memory and
// store the stage outputs (+ ghost images, NaN flag) with coalesced global stores.  The
// producer runs up to two planes ahead and across item boundaries, so the HBM pipe never
// drains between items.  Arithmetic is operation-for-operation that of wave_simple
// (bit-identical results; compiled without FMA contraction).
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

constexpr int r128(int b) { return (b + 127) / 128 * 128; }

// pointwise operands per stage (boxes of TX x TY points)
template <int STAGE> struct PW {
  static constexpr int NY = (STAGE == 2 || STAGE == 3) ? 4 : 0;  // y GFs rho..v3
  static constexpr int NQ = STAGE == 4 ? 5 : (STAGE == 3 ? 1 : 0);  // Q GFs (u..v3 or u)
  static constexpr int NU = STAGE == 4 ? 1 : 0;                   // y.u
};

template <int STAGE, int W>
struct Cfg {
  static constexpr int TX = 32, TY = 16, NCW = 16;
  // box halo: the stencil radius rounded up to even, because a TMA box must start on a
  // 16-byte boundary in x (an odd fp64 offset raises an illegal-instruction fault)
  static constexpr int H = (W + 1) / 2 * 2;
  static constexpr int RX = TX + 2 * H, RY = TY + 2 * H;
  static constexpr int RZ = 2 * W + 3;
  static constexpr int C = TX * TY;  // points per tile plane
  static constexpr int ZRHO_B = r128(RX * RY * 8), ZV3_B = r128(C * 8), ZSLOT = ZRHO_B + ZV3_B;
  static constexpr int PV1_B = r128(RX * TY * 8), PV2_B = r128(TX * RY * 8);
  static constexpr int PY_B = r128(PW<STAGE>::NY * C * 8), PQ_B = r128(PW<STAGE>::NQ * C * 8),
                       PU_B = r128(PW<STAGE>::NU * C * 8);
  static constexpr int PSLOT = PV1_B + PV2_B + PY_B + PQ_B + PU_B;
  // three pointwise slots, or two where the radius-4 z ring leaves no room (stage 4, W = 4)
  static constexpr int RP = RZ * ZSLOT + 3 * PSLOT + (2 * RZ + 6) * 8 <= 227 * 1024 ? 3 : 2;
  static constexpr uint32_t ZBYTES = (RX * RY + C) * 8;
  static constexpr uint32_t PBYTES = (RX * TY + TX * RY + (PW<STAGE>::NY + PW<STAGE>::NQ + PW<STAGE>::NU) * C) * 8;
  static constexpr int SMEM = RZ * ZSLOT + RP * PSLOT + (2 * RZ + 2 * RP) * 8 + 16;  // + item queue
  static constexpr int THREADS = 32 * (NCW + 1);
};

struct Maps {
  CUtensorMap rho;   // stencil input set, (RX, RY, 1, 1) box
  CUtensorMap v1;    // (RX, TY, 1, 1)
  CUtensorMap v2;    // (TX, RY, 1, 1)
  CUtensorMap c1;    // stencil input set, (TX, TY, 1, 1)   -> v3
  CUtensorMap y4;    // y set, (TX, TY, 1, 4)               -> y rho..v3 (stages 2, 3)
  CUtensorMap yu;    // y set, (TX, TY, 1, 1)               -> y.u (stage 4)
  CUtensorMap q;     // Q set, (TX, TY, 1, NQ)              -> Q (stage 4: 5 GFs, stage 3: Q.u)
};

template <int W>
__device__ __forceinline__ double d1s(const double* f, int c, int s) {
  double acc = 0.0;
#pragma unroll
  for (int q = W; q >= 1; --q) acc = fma(D1W<W>::c(q), f[c + q * s] - f[c - q * s], acc);
  return acc;
}

template <int STAGE, int W>
__global__ void __launch_bounds__(Cfg<STAGE, W>::THREADS, 1)
    wave_tma2(const __grid_constant__ Maps M, StageLaunch a, WaveK K, int kchunk, int ntx, int nty,
              int nitems) {
  using Cf = Cfg<STAGE, W>;
  using P = PW<STAGE>;
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* zbase = smem;
  unsigned char* pbase = smem + Cf::RZ * Cf::ZSLOT;
  uint64_t* zfull = reinterpret_cast<uint64_t*>(pbase + Cf::RP * Cf::PSLOT);
  uint64_t* zempty = zfull + Cf::RZ;
  uint64_t* pfull = zempty + Cf::RZ;
  uint64_t* pempty = pfull + Cf::RP;
  // items are handed out in order by an atomic counter (as in wave_fused3.cu: the items in
  // flight stay (x,y) neighbours, so shared halo rows are re-read from L2); the producer
  // passes each index to the consumers through this queue, published by the mbarrier of the
  // item's first input plane
  int* itemq = reinterpret_cast<int*>(pempty + Cf::RP);
  constexpr int IQ = 4;
  const Layout& L = a.L;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < Cf::RZ; ++s) { mbar_init(zfull + s, 1); mbar_init(zempty + s, Cf::NCW); }
    for (int s = 0; s < Cf::RP; ++s) { mbar_init(pfull + s, 1); mbar_init(pempty + s, Cf::NCW); }
    fence_mbar_init();
  }
  __syncthreads();
  const int g = L.g;
  const int nkall = a.k_end - a.k_begin;

  if (warp == Cf::NCW) {  // ---------------------------------------------------- producer
    if (lane != 0) return;
    prefetch_tmap(&M.rho); prefetch_tmap(&M.v1); prefetch_tmap(&M.v2); prefetch_tmap(&M.c1);
    if (P::NY) prefetch_tmap(&M.y4);
    if (P::NU) prefetch_tmap(&M.yu);
    if (P::NQ) prefetch_tmap(&M.q);
    uint32_t nz = 0, np = 0, nit = 0;  // running load counters (ring position and phase)
    for (;;) {
      const int item = (int)atomicAdd(a.sched, 1ull);
      {  // the item index (or the end marker) travels with the item's first input slot
        const uint32_t s = nz % Cf::RZ, n = nz / Cf::RZ;
        if (n > 0) mbar_wait(zempty + s, (n - 1) & 1);
        itemq[nit % IQ] = item;
        ++nit;
        if (item >= nitems) {
          mbar_arrive(zfull + s);  // completes the slot's phase with no data: end of work
          break;
        }
      }
      const int bx = item % ntx, by = (item / ntx) % nty, ch = item / (ntx * nty);
      const int i0 = bx * Cf::TX, j0 = by * Cf::TY;
      const int kb = a.k_begin + ch * kchunk;
      const int nk = min(kchunk, a.k_begin + nkall - kb);
      auto loadZ = [&](int plane) {
        const uint32_t s = nz % Cf::RZ, n = nz / Cf::RZ;
        if (n > 0) mbar_wait(zempty + s, (n - 1) & 1);
        unsigned char* dst = zbase + s * Cf::ZSLOT;
        const int zc = g + plane;
        mbar_arrive_expect_tx(zfull + s, Cf::ZBYTES);
        tma_load_4d(dst, &M.rho, zfull + s, kXOff + i0 - Cf::H, g + j0 - Cf::H, zc, GRHO);
        tma_load_4d(dst + Cf::ZRHO_B, &M.c1, zfull + s, kXOff + i0, g + j0, zc, GV3);
        ++nz;
      };
      auto loadP = [&](int plane) {
        const uint32_t s = np % Cf::RP, n = np / Cf::RP;
        if (n > 0) mbar_wait(pempty + s, (n - 1) & 1);
        unsigned char* dst = pbase + s * Cf::PSLOT;
        const int zc = g + plane;
        uint64_t* bar = pfull + s;
        mbar_arrive_expect_tx(bar, Cf::PBYTES);
        tma_load_4d(dst, &M.v1, bar, kXOff + i0 - Cf::H, g + j0, zc, GV1);
        tma_load_4d(dst + Cf::PV1_B, &M.v2, bar, kXOff + i0, g + j0 - Cf::H, zc, GV2);
        unsigned char* d2 = dst + Cf::PV1_B + Cf::PV2_B;
        if (P::NY) tma_load_4d(d2, &M.y4, bar, kXOff + i0, g + j0, zc, GRHO);
        if (P::NQ) tma_load_4d(d2 + Cf::PY_B, &M.q, bar, kXOff + i0, g + j0, zc, GU);
        if (P::NU) tma_load_4d(d2 + Cf::PY_B + Cf::PQ_B, &M.yu, bar, kXOff + i0, g + j0, zc, GU);
        ++np;
      };
      for (int q = -W; q < W; ++q) loadZ(kb + q);
      for (int t = 0; t < nk; ++t) {
        loadZ(kb + t + W);
        loadP(kb + t);
      }
    }
    // the last CTA to finish fetching resets the scheduler for the next launch
    if (atomicAdd(a.sched + 1, 1ull) == gridDim.x - 1) {
      a.sched[0] = 0ull;
      a.sched[1] = 0ull;
    }
    return;
  }

  // ------------------------------------------------------------------------ consumers
  const int64_t gfs = L.gfs;
  double* out = STAGE == 1 ? a.s.b : (STAGE == 2 ? a.s.c : (STAGE == 3 ? a.s.b : a.s.y));
  const FaceDst fd = a.img[STAGE - 1];
  const unsigned long long code0 = a.step * (unsigned long long)L.n_gf;
  const int ty = warp, tx = lane;
  const int cr = (ty + Cf::H) * Cf::RX + (tx + Cf::H);  // rho box index
  const int cv = ty * Cf::TX + tx;              // centre box index
  uint32_t nz = 0, np = 0, nit = 0;
  for (;;) {
    mbar_wait(zfull + nz % Cf::RZ, (nz / Cf::RZ) & 1);  // the item's first input plane, or the end
    const int item = itemq[nit % IQ];
    ++nit;
    if (item >= nitems) break;
    const int bx = item % ntx, by = (item / ntx) % nty, ch = item / (ntx * nty);
    const int i = bx * Cf::TX + tx, j = by * Cf::TY + ty;
    const int kb = a.k_begin + ch * kchunk;
    const int nk = min(kchunk, a.k_begin + nkall - kb);
    const bool live = i < L.nx && j < L.ny;
    const uint32_t z0 = nz;  // ring index of plane kb - W
    for (int q = 0; q < 2 * W; ++q) mbar_wait(zfull + (z0 + q) % Cf::RZ, ((z0 + q) / Cf::RZ) & 1);
#pragma unroll 1
    for (int t = 0; t < nk; ++t) {
      const int k = kb + t;
      const uint32_t zt = z0 + t + 2 * W;
      mbar_wait(zfull + zt % Cf::RZ, (zt / Cf::RZ) & 1);
      mbar_wait(pfull + np % Cf::RP, (np / Cf::RP) & 1);
      const double* zr[2 * W + 1];
      const double* zv[2 * W + 1];
#pragma unroll
      for (int q = 0; q <= 2 * W; ++q) {
        const unsigned char* sl = zbase + ((z0 + t + q) % Cf::RZ) * Cf::ZSLOT;
        zr[q] = reinterpret_cast<const double*>(sl);
        zv[q] = reinterpret_cast<const double*>(sl + Cf::ZRHO_B);
      }
      const unsigned char* ps = pbase + (np % Cf::RP) * Cf::PSLOT;
      const double* sv1 = reinterpret_cast<const double*>(ps);
      const double* sv2 = reinterpret_cast<const double*>(ps + Cf::PV1_B);
      const double* sy = reinterpret_cast<const double*>(ps + Cf::PV1_B + Cf::PV2_B);
      const double* sq = reinterpret_cast<const double*>(ps + Cf::PV1_B + Cf::PV2_B + Cf::PY_B);
      const double* su = reinterpret_cast<const double*>(ps + Cf::PV1_B + Cf::PV2_B + Cf::PY_B + Cf::PQ_B);
      double S[5], kk[5], Y[5] = {0, 0, 0, 0, 0}, Qv[5] = {0, 0, 0, 0, 0}, yu = 0.0, qu = 0.0;
      S[GRHO] = zr[W][cr];
      S[GV1] = sv1[ty * Cf::RX + tx + Cf::H];
      S[GV2] = sv2[(ty + Cf::H) * Cf::TX + tx];
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
      const double dv1 = d1s<W>(sv1, ty * Cf::RX + tx + Cf::H, 1) * K.ih[0];
      const double dv2 = d1s<W>(sv2, (ty + Cf::H) * Cf::TX + tx, Cf::TX) * K.ih[1];
      dv3 = dv3 * K.ih[2];
      kk[GRHO] = dv1 + dv2 + dv3;
      kk[GV1] = dxr;
      kk[GV2] = dyr;
      kk[GV3] = dzr;
      if (STAGE == 1) {
#pragma unroll
        for (int f = 1; f <= 4; ++f) Y[f] = S[f];
      }
      if (P::NY) {
#pragma unroll
        for (int f = 1; f <= 4; ++f) Y[f] = sy[(f - 1) * Cf::C + cv];
      }
      if (STAGE == 3) qu = sq[cv];
      if (STAGE == 4) {
        qu = sq[cv];
#pragma unroll
        for (int f = 1; f <= 4; ++f) Qv[f] = sq[f * Cf::C + cv];
        yu = su[cv];
      }
      // every shared-memory operand is in registers: release the slots before the stores
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(pempty + np % Cf::RP);
        mbar_arrive(zempty + (z0 + t) % Cf::RZ);  // plane k - W is no longer needed
      }
      ++np;
      if (live) {
        const int64_t c = L.idx(i, j, k);
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
    // the item's top 2W planes were only read: free their slots for the next item
    __syncwarp();
    if (lane == 0)
      for (int q = 0; q < 2 * W; ++q) mbar_arrive(zempty + (z0 + nk + q) % Cf::RZ);
    nz = z0 + nk + 2 * W;
  }
}

bool encode(CUtensorMap* m, const double* set_ptr, const Layout& L, unsigned bx, unsigned by, unsigned bg) {
  return encode_set_map(m, set_ptr - L.c0, L.px, L.py, L.pz, L.n_gf, L.gfs, bx, by, bg);
}

template <int STAGE, int W>
cudaError_t launch(const StageLaunch& a, const WaveK& K, cudaStream_t st) {
  using Cf = Cfg<STAGE, W>;
  const int nk = a.k_end - a.k_begin;
  if (nk <= 0) return cudaSuccess;
  const Layout& L = a.L;
  const double* in = STAGE == 1 ? a.s.y : (STAGE == 2 ? a.s.b : (STAGE == 3 ? a.s.c : a.s.b));
  Maps M;
  bool ok = encode(&M.rho, in, L, Cf::RX, Cf::RY, 1) && encode(&M.v1, in, L, Cf::RX, Cf::TY, 1) &&
            encode(&M.v2, in, L, Cf::TX, Cf::RY, 1) && encode(&M.c1, in, L, Cf::TX, Cf::TY, 1) &&
            encode(&M.y4, a.s.y, L, Cf::TX, Cf::TY, 4) && encode(&M.yu, a.s.y, L, Cf::TX, Cf::TY, 1) &&
            encode(&M.q, a.s.q, L, Cf::TX, Cf::TY, PW<STAGE>::NQ > 0 ? PW<STAGE>::NQ : 1);
  if (!ok) return cudaErrorInvalidValue;
  static std::atomic<uint64_t> attr_done{0};
  if (cudaError_t e = smem_optin((const void*)wave_tma2<STAGE, W>, Cf::SMEM, attr_done); e != cudaSuccess) return e;
  const int nsm = device_sm_count();
  const int ntx = (int)((L.nx + Cf::TX - 1) / Cf::TX), nty = (int)((L.ny + Cf::TY - 1) / Cf::TY);
  // chunks of ~64 planes, but enough items for >= 8 per SM (load balance of the round robin)
  const int target = 64;
  int nchunks = (nk + target - 1) / target;
  const int want = (8 * nsm + ntx * nty - 1) / (ntx * nty);
  if (nchunks < want) nchunks = want;
  int chunk = (nk + nchunks - 1) / nchunks;
  if (chunk < 2) chunk = 2;
  if (chunk > nk) chunk = nk;
  nchunks = (nk + chunk - 1) / chunk;
  const int nitems = ntx * nty * nchunks;
  const int grid = nitems < nsm ? nitems : nsm;
  wave_tma2<STAGE, W><<<grid, Cf::THREADS, Cf::SMEM, st>>>(M, a, K, chunk, ntx, nty, nitems);
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
cudaError_t dispatch(const StageLaunch& a, int stage, cudaStream_t st) {
  const WaveK K = make_k(a);
  switch (stage) {
    case 1: return launch<1, W>(a, K, st);
    case 2: return launch<2, W>(a, K, st);
    case 3: return launch<3, W>(a, K, st);
    case 4: return launch<4, W>(a, K, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t wave_tma_stage(const StageLaunch& a, int stage, cudaStream_t st) {
  switch (a.fd_order) {
    case 2: return dispatch<1>(a, stage, st);
    case 4: return dispatch<2>(a, stage, st);
    case 6: return dispatch<3>(a, stage, st);
    case 8: return dispatch<4>(a, stage, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace chemora
