// wave_common.cuh -- pieces shared by the wave stage kernels (wave_stage.cu, wave_tma.cu):
// the centered first-derivative weights of order 2W and the fused RK4 stage update.  Both
// files are compiled without FMA contraction so every tiling computes bit-identical values.
#pragma once
#include <cstdint>

namespace chemora {
namespace wave {

enum { GU = 0, GRHO = 1, GV1 = 2, GV2 = 3, GV3 = 4 };

// Centered first-derivative weights c_s (s = 1..W) of order 2W: D1 f = sum c_s (f_s - f_-s)/h.
template <int W> struct D1W;
template <> struct D1W<1> { static __device__ __forceinline__ double c(int) { return 0.5; } };
template <> struct D1W<2> {
  static __device__ __forceinline__ double c(int s) { return s == 1 ? 2.0 / 3.0 : -1.0 / 12.0; }
};
template <> struct D1W<3> {
  static __device__ __forceinline__ double c(int s) {
    return s == 1 ? 3.0 / 4.0 : (s == 2 ? -3.0 / 20.0 : 1.0 / 60.0);
  }
};
template <> struct D1W<4> {
  static __device__ __forceinline__ double c(int s) {
    return s == 1 ? 4.0 / 5.0 : (s == 2 ? -1.0 / 5.0 : (s == 3 ? 4.0 / 105.0 : -1.0 / 280.0));
  }
};

template <int W>
__device__ __forceinline__ double d1(const double* __restrict__ f, int64_t c, int64_t s) {
  double acc = 0.0;
#pragma unroll
  for (int q = W; q >= 1; --q) acc = fma(D1W<W>::c(q), __ldg(f + c + q * s) - __ldg(f + c - q * s), acc);
  return acc;
}

struct WaveK {
  double ih[3];     // 1/h per axis
  double half, third, sixth, dt, dt2, dt3, dt6;
};

// RK4 stage update of the 4 differentiated GFs and the u carry, given the stage input
// centre values S (rho, v1..3 at index 1..4), the RHS k (index 1..4) and krho_u = S.rho.
// Writes go through `put(gf, value)` for the stage's main output and `putq` for Q.
template <int STAGE, class Put, class PutQ>
__device__ __forceinline__ void wave_update(const WaveK& K, const double* S, const double* k,
                                            const double* Y, const double* Qv, double yu,
                                            double qu, Put put, PutQ putq) {
#pragma unroll
  for (int f = 1; f <= 4; ++f) {
    if (STAGE == 1) put(f, fma(K.dt2, k[f], Y[f]));
    if (STAGE == 2) {
      putq(f, fma(K.dt3, k[f], (Y[f] + S[f]) * K.third));
      put(f, fma(K.dt2, k[f], Y[f]));
    }
    if (STAGE == 3) put(f, fma(K.dt, k[f], Y[f]));
    if (STAGE == 4) put(f, fma(K.dt6, k[f], fma(S[f], K.third, Qv[f])));
  }
  if (STAGE == 2) putq(0, fma(K.dt3, S[1], K.dt6 * Y[1]));
  if (STAGE == 3) putq(0, fma(K.dt3, S[1], qu));
  if (STAGE == 4) put(0, fma(K.dt6, S[1], yu + qu));
}

}  // namespace wave
}  // namespace chemora
