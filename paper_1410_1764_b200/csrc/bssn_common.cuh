// bssn_common.cuh -- the BSSN-like Einstein system's pointwise algebra (
// PAPER.md:686-688; reading R7) written once against a derivative *provider*, the
// 4th-order stencil primitives, the constraint monitors and the RK4 stage update, shared by
// every BSSN kernel design (bssn_stage.cu: one-thread-per-point, SMEM-table and HBM-table
// fissions; bssn_fused.cu: the fused z-marching kernel with TMEM z-windows).
//
// Advection is evaluated branch-free as beta * S f + |beta| * A f with S = (D+ + D-)/2 and
// A = (D+ - D-)/2 (identical to max(beta,0) D+ + min(beta,0) D-, R6).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include "grid.hpp"
#include "kernels.hpp"
#include "device_common.cuh"

namespace chemora {
namespace {
enum {
  V_PHI = 0, V_GT = 1, V_TRK = 7, V_AT = 8, V_XT = 14, V_ALPHA = 17, V_AUX = 18, V_BETA = 19,
  V_B = 22, NV = 25
};

// packed index of the symmetric pair (i, j)
__host__ __device__ constexpr int sy(int i, int j) {
  return i == j ? (i == 0 ? 0 : (i == 1 ? 3 : 5)) : (i + j == 1 ? 1 : (i + j == 2 ? 2 : 4));
}
// multiplicity of a packed symmetric index in a full contraction (1 diagonal, 2 off)
__host__ __device__ constexpr double mult(int s) { return (s == 0 || s == 3 || s == 5) ? 1.0 : 2.0; }
__host__ __device__ constexpr int sI(int s) { return s == 0 ? 0 : (s == 1 ? 0 : (s == 2 ? 0 : (s == 3 ? 1 : (s == 4 ? 1 : 2)))); }
__host__ __device__ constexpr int sJ(int s) { return s == 0 ? 0 : (s == 1 ? 1 : (s == 2 ? 2 : (s == 3 ? 1 : (s == 4 ? 2 : 2)))); }

struct BssnK {
  double i12h[3];     // 1/(12 h_a)
  double i12h2[3];    // 1/(12 h_a^2)
  double i144hh[3];   // 1/(144 h_a h_b) for the pairs (xy, xz, yz) -> index a+b-1
  double i24h[3];     // 1/(24 h_a)
  double dt, dt2, dt3, dt6, third;
  double F_alpha, n_alpha, L, eta_alpha, c_alpha_adv, C_beta, p_beta, S_B, eta, c_beta_adv;
};

struct Strides {
  int64_t s[3];
};

__device__ __forceinline__ double ld(const double* __restrict__ p) { return __ldg(p); }

// centered 4th-order D1 (without the 1/(12h) factor)
__device__ __forceinline__ double D1raw(const double* __restrict__ f, int64_t c, int64_t s) {
  return 8.0 * (ld(f + c + s) - ld(f + c - s)) - (ld(f + c + 2 * s) - ld(f + c - 2 * s));
}
// centered 4th-order D2 (without 1/(12h^2)), given the centre value
__device__ __forceinline__ double D2raw(const double* __restrict__ f, int64_t c, int64_t s, double f0) {
  return 16.0 * (ld(f + c + s) + ld(f + c - s)) - (ld(f + c + 2 * s) + ld(f + c - 2 * s)) - 30.0 * f0;
}
// mixed D1_a D1_b (without 1/(144 h_a h_b))
__device__ __forceinline__ double D11raw(const double* __restrict__ f, int64_t c, int64_t sa, int64_t sb) {
  const double p1 = D1raw(f, c + sa, sb), m1 = D1raw(f, c - sa, sb);
  const double p2 = D1raw(f, c + 2 * sa, sb), m2 = D1raw(f, c - 2 * sa, sb);
  return 8.0 * (p1 - m1) - (p2 - m2);
}
// upwind advection along one axis: beta * S f + |beta| * A f (without 1/(24h))
__device__ __forceinline__ double ADVraw(const double* __restrict__ f, int64_t c, int64_t s, double f0, double beta) {
  const double a1 = ld(f + c + s), b1 = ld(f + c - s);
  const double a2 = ld(f + c + 2 * s), b2 = ld(f + c - 2 * s);
  const double a3 = ld(f + c + 3 * s), b3 = ld(f + c - 3 * s);
  const double S = 21.0 * (a1 - b1) - 6.0 * (a2 - b2) + (a3 - b3);
  const double A = 15.0 * (a1 + b1) - 6.0 * (a2 + b2) + (a3 + b3) - 20.0 * f0;
  return fma(beta, S, fabs(beta) * A);
}

// ------------------------------------------------------------------ derivative table
// slots: [0,25) point values; [25,70) D1 of the 15 differentiated GFs x 3 axes; [70,136)
// second derivatives of the 11 twice-differentiated GFs x 6 pairs; [136,161) Adv(gf).
constexpr int T_D1 = 25, T_DD = 70, T_ADV = 136, NSLOT = 161;
__host__ __device__ constexpr int d1i(int gf) {  // index in the D1 list
  return gf == V_PHI ? 0 : (gf >= V_GT && gf < V_GT + 6) ? 1 + gf - V_GT : gf == V_TRK ? 7
       : gf == V_ALPHA ? 8 : (gf >= V_BETA && gf < V_BETA + 3) ? 9 + gf - V_BETA
       : (gf >= V_XT && gf < V_XT + 3) ? 12 + gf - V_XT : -1;
}
__host__ __device__ constexpr int d1gf(int i) {
  return i == 0 ? V_PHI : i <= 6 ? V_GT + i - 1 : i == 7 ? V_TRK : i == 8 ? V_ALPHA : i <= 11 ? V_BETA + i - 9 : V_XT + i - 12;
}
__host__ __device__ constexpr int ddi(int gf) {  // index in the second-derivative list
  return gf == V_PHI ? 0 : (gf >= V_GT && gf < V_GT + 6) ? 1 + gf - V_GT : gf == V_ALPHA ? 7
       : (gf >= V_BETA && gf < V_BETA + 3) ? 8 + gf - V_BETA : -1;
}
__host__ __device__ constexpr int ddgf(int i) {
  return i == 0 ? V_PHI : i <= 6 ? V_GT + i - 1 : i == 7 ? V_ALPHA : V_BETA + i - 8;
}

struct StencilP {
  const double* in;
  int64_t gfs, c;
  Strides st;
  __device__ __forceinline__ double v(int gf) const { return ld(in + gf * gfs + c); }
  __device__ __forceinline__ double d1(const BssnK& K, int gf, int l) const {
    return D1raw(in + gf * gfs, c, st.s[l]) * K.i12h[l];
  }
  __device__ __forceinline__ double dd(const BssnK& K, int gf, int l, int m, double f0) const {
    return (l == m) ? D2raw(in + gf * gfs, c, st.s[l], f0) * K.i12h2[l]
                    : D11raw(in + gf * gfs, c, st.s[l], st.s[m]) * K.i144hh[l + m - 1];
  }
  __device__ __forceinline__ double adv(const BssnK& K, int gf, const double* beta, double f0) const {
    double r = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a) r = fma(ADVraw(in + gf * gfs, c, st.s[a], f0, beta[a]), K.i24h[a], r);
    return r;
  }
};


// Output groups of the kernel fission (fission is "the most
// important performance optimization" for the Einstein equations).
// G0 = everything; G1 = phi, gt, alpha, beta (kinematics, first derivatives only);
// G2 = trK, At, A (curvature: Ricci, D_i D_j alpha); G3 = Xt, B (second derivatives of
// the shift); G13 = G1 + G3.
__host__ __device__ constexpr bool in_group(int G, int v) {
  return G == 0 ? true
       : G == 1 ? (v == V_PHI || (v >= V_GT && v < V_GT + 6) || v == V_ALPHA || (v >= V_BETA && v < V_BETA + 3))
       : G == 2 ? (v == V_TRK || (v >= V_AT && v < V_AT + 6) || v == V_AUX)
       : G == 3 ? ((v >= V_XT && v < V_XT + 3) || (v >= V_B && v < V_B + 3))
                : (in_group(1, v) || in_group(3, v));
}

// Right-hand sides of group G from the derivative provider P (advection included);
// rhs[v] is written for every v in the group.  App. A.2-A.3.
template <int G, class P>
__device__ __forceinline__ void bssn_point(const P& D, const BssnK& K, double* rhs) {
  constexpr bool g1 = G == 0 || G == 1 || G == 13, g2 = G == 0 || G == 2, g3 = G == 0 || G == 3 || G == 13;
  // ---- point values
  double gt[6], At[6];
#pragma unroll
  for (int s = 0; s < 6; ++s) { gt[s] = D.v(V_GT + s); At[s] = D.v(V_AT + s); }
  const double phi = D.v(V_PHI), trK = D.v(V_TRK), alpha = D.v(V_ALPHA);
  const double Aux = D.v(V_AUX);
  double Xt[3], beta[3], Bv[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) { Xt[i] = D.v(V_XT + i); beta[i] = D.v(V_BETA + i); Bv[i] = D.v(V_B + i); }
  double dbeta[3][3];  // dbeta[l][k] = d_l beta^k
#pragma unroll
  for (int l = 0; l < 3; ++l)
#pragma unroll
    for (int k = 0; k < 3; ++k) dbeta[l][k] = D.d1(K, V_BETA + k, l);
  const double divb = dbeta[0][0] + dbeta[1][1] + dbeta[2][2];

  if (g1) {
    rhs[V_PHI] = (divb - alpha * trK) * (1.0 / 6.0);
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      const int i = sI(s), j = sJ(s);
      double rg = -2.0 * alpha * At[s] - (2.0 / 3.0) * gt[s] * divb;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        rg = fma(gt[sy(i, k)], dbeta[j][k], rg);
        rg = fma(gt[sy(j, k)], dbeta[i][k], rg);
      }
      rhs[V_GT + s] = rg;
    }
    const double apow_n = (K.n_alpha == 1.0) ? alpha : pow(alpha, K.n_alpha);
    rhs[V_ALPHA] = -K.F_alpha * apow_n * (K.L * Aux + (1.0 - K.L) * trK);
    const double apow_p = (K.p_beta == 0.0) ? 1.0 : pow(alpha, K.p_beta);
#pragma unroll
    for (int i = 0; i < 3; ++i)
      rhs[V_BETA + i] = K.C_beta * apow_p * (K.S_B * Bv[i] + (1.0 - K.S_B) * (Xt[i] - K.eta * beta[i]));
  }

  if (g2 || g3) {
    // ---- inverse conformal metric gu = adj(gt) / det(gt)
    const double c00 = gt[3] * gt[5] - gt[4] * gt[4];
    const double c01 = gt[2] * gt[4] - gt[1] * gt[5];
    const double c02 = gt[1] * gt[4] - gt[2] * gt[3];
    const double det = gt[0] * c00 + gt[1] * c01 + gt[2] * c02;
    const double idet = 1.0 / det;
    double gu[6];
    gu[0] = c00 * idet;
    gu[1] = c01 * idet;
    gu[2] = c02 * idet;
    gu[3] = (gt[0] * gt[5] - gt[2] * gt[2]) * idet;
    gu[4] = (gt[1] * gt[2] - gt[0] * gt[4]) * idet;
    gu[5] = (gt[0] * gt[3] - gt[1] * gt[1]) * idet;

    // ---- first derivatives of the metric -> Christoffels (first kind Gl, second kind Gu)
    double Gl[3][6];  // Gl[i][s(j,k)] = 1/2 (d_j gt_ik + d_k gt_ij - d_i gt_jk)
    {
      double dg[3][6];
#pragma unroll
      for (int l = 0; l < 3; ++l)
#pragma unroll
        for (int s = 0; s < 6; ++s) dg[l][s] = D.d1(K, V_GT + s, l);
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int s = 0; s < 6; ++s) {
          const int j = sI(s), k = sJ(s);
          Gl[i][s] = 0.5 * (dg[j][sy(i, k)] + dg[k][sy(i, j)] - dg[i][s]);
        }
    }
    double Gu[3][6];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int s = 0; s < 6; ++s)
        Gu[i][s] = gu[sy(i, 0)] * Gl[0][s] + gu[sy(i, 1)] * Gl[1][s] + gu[sy(i, 2)] * Gl[2][s];
    double Xtn[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      double a = 0.0;
#pragma unroll
      for (int s = 0; s < 6; ++s) a = fma(mult(s) * gu[s], Gu[i][s], a);
      Xtn[i] = a;
    }
    double dphi[3], dalpha[3];
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      dphi[l] = D.d1(K, V_PHI, l);
      dalpha[l] = D.d1(K, V_ALPHA, l);
    }
    // ---- raised At: Am[i][j] = At^i_j (full 3x3), Au = At^ij (sym)
    double Am[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j)
        Am[i][j] = gu[sy(i, 0)] * At[sy(0, j)] + gu[sy(i, 1)] * At[sy(1, j)] + gu[sy(i, 2)] * At[sy(2, j)];
    double Au[6];
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      const int i = sI(s), j = sJ(s);
      Au[s] = Am[i][0] * gu[sy(0, j)] + Am[i][1] * gu[sy(1, j)] + Am[i][2] * gu[sy(2, j)];
    }

    if (g2) {
      const double em4phi = exp(-4.0 * phi);
      double dXt[3][3];  // dXt[l][k] = d_l Xt^k
#pragma unroll
      for (int l = 0; l < 3; ++l)
#pragma unroll
        for (int k = 0; k < 3; ++k) dXt[l][k] = D.d1(K, V_XT + k, l);
      // ---- conformal Ricci tensor R~_ij: -1/2 gu^lm d_l d_m gt_ij, pair (l,m) at a time
      double Rt[6];
#pragma unroll
      for (int s = 0; s < 6; ++s) Rt[s] = 0.0;
#pragma unroll
      for (int p = 0; p < 6; ++p) {
        const int l = sI(p), m = sJ(p);
        const double w = -0.5 * mult(p) * gu[p];
#pragma unroll
        for (int s = 0; s < 6; ++s) Rt[s] = fma(w, D.dd(K, V_GT + s, l, m, gt[s]), Rt[s]);
      }
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        const int i = sI(s), j = sJ(s);
        double r = Rt[s];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          r = fma(0.5 * gt[sy(k, i)], dXt[j][k], r);
          r = fma(0.5 * gt[sy(k, j)], dXt[i][k], r);
          r = fma(0.5 * Xtn[k], Gl[i][sy(j, k)] + Gl[j][sy(i, k)], r);
        }
#pragma unroll
        for (int l = 0; l < 3; ++l)
#pragma unroll
          for (int m = 0; m < 3; ++m) {
            double t = 0.0;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
              t = fma(Gu[k][sy(l, i)], Gl[j][sy(k, m)], t);
              t = fma(Gu[k][sy(l, j)], Gl[i][sy(k, m)], t);
              t = fma(Gu[k][sy(i, m)], Gl[k][sy(l, j)], t);
            }
            r = fma(gu[sy(l, m)], t, r);
          }
        Rt[s] = r;
      }
      // ---- phi terms: D~_i D~_j phi, traces; second derivatives of alpha
      double DDphi[6], DDalpha[6], ddalpha[6];
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        const int i = sI(s), j = sJ(s);
        const double ddp = D.dd(K, V_PHI, i, j, phi);
        const double dda = D.dd(K, V_ALPHA, i, j, alpha);
        ddalpha[s] = dda;
        DDphi[s] = ddp - (Gu[0][s] * dphi[0] + Gu[1][s] * dphi[1] + Gu[2][s] * dphi[2]);
      }
      double gudphi[3];  // gt^kl d_l phi
#pragma unroll
      for (int k = 0; k < 3; ++k) gudphi[k] = gu[sy(k, 0)] * dphi[0] + gu[sy(k, 1)] * dphi[1] + gu[sy(k, 2)] * dphi[2];
      double trDDphi = 0.0, dphi2 = 0.0;
#pragma unroll
      for (int s = 0; s < 6; ++s) trDDphi = fma(mult(s) * gu[s], DDphi[s], trDDphi);
#pragma unroll
      for (int k = 0; k < 3; ++k) dphi2 = fma(gudphi[k], dphi[k], dphi2);
      // D_i D_j alpha with Gamma^k_ij = Gu^k_ij + 2 (delta^k_i d_j phi + delta^k_j d_i phi
      //                                             - gt_ij gt^kl d_l phi)
      const double gdpda = gudphi[0] * dalpha[0] + gudphi[1] * dalpha[1] + gudphi[2] * dalpha[2];
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        const int i = sI(s), j = sJ(s);
        double gam_da = Gu[0][s] * dalpha[0] + Gu[1][s] * dalpha[1] + Gu[2][s] * dalpha[2];
        gam_da += 2.0 * (dalpha[i] * dphi[j] + dalpha[j] * dphi[i] - gt[s] * gdpda);
        DDalpha[s] = ddalpha[s] - gam_da;
      }
      double trDDalpha;
      {
        double s1 = 0.0, s2 = 0.0;
#pragma unroll
        for (int s = 0; s < 6; ++s) s1 = fma(mult(s) * gu[s], ddalpha[s], s1);
#pragma unroll
        for (int k = 0; k < 3; ++k) s2 = fma(Xtn[k], dalpha[k], s2);
        trDDalpha = em4phi * (s1 - s2 + 2.0 * gdpda);
      }
      // ---- X_ij = -D_i D_j alpha + alpha (R~_ij + R^phi_ij)
      double X[6], trX = 0.0;
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        const int i = sI(s), j = sJ(s);
        const double Rphi = -2.0 * DDphi[s] - 2.0 * gt[s] * trDDphi + 4.0 * dphi[i] * dphi[j] - 4.0 * gt[s] * dphi2;
        X[s] = fma(alpha, Rt[s] + Rphi, -DDalpha[s]);
        trX = fma(mult(s) * gu[s], X[s], trX);
      }
      double AA = 0.0;
#pragma unroll
      for (int s = 0; s < 6; ++s) AA = fma(mult(s) * At[s], Au[s], AA);
#pragma unroll
      for (int s = 0; s < 6; ++s) {
        const int i = sI(s), j = sJ(s);
        double ra = em4phi * (X[s] - (1.0 / 3.0) * gt[s] * trX) - (2.0 / 3.0) * At[s] * divb;
        double aam = 0.0;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          ra = fma(At[sy(i, k)], dbeta[j][k], ra);
          ra = fma(At[sy(j, k)], dbeta[i][k], ra);
          aam = fma(At[sy(i, k)], Am[k][j], aam);
        }
        rhs[V_AT + s] = fma(alpha, trK * At[s] - 2.0 * aam, ra);
      }
      rhs[V_TRK] = -trDDalpha + alpha * (AA + trK * trK * (1.0 / 3.0));
    }

    if (g3) {
      double dtrK[3];
#pragma unroll
      for (int l = 0; l < 3; ++l) dtrK[l] = D.d1(K, V_TRK, l);
      double ddivb[3] = {0.0, 0.0, 0.0};  // d_j (d . beta)
      double lapb[3] = {0.0, 0.0, 0.0};   // gt^jk d_j d_k beta^i
#pragma unroll
      for (int p = 0; p < 6; ++p) {
        const int l = sI(p), m = sJ(p);
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const double dd = D.dd(K, V_BETA + i, l, m, beta[i]);
          lapb[i] = fma(mult(p) * gu[p], dd, lapb[i]);
          // d_l d_m beta^i feeds d_j (d.beta) for (j = l, i = m) and (j = m, i = l)
          if (i == m) ddivb[l] += dd;
          if (i == l && l != m) ddivb[m] += dd;
        }
      }
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        double r = lapb[i] + (1.0 / 3.0) * (gu[sy(i, 0)] * ddivb[0] + gu[sy(i, 1)] * ddivb[1] + gu[sy(i, 2)] * ddivb[2]);
        r = fma((2.0 / 3.0) * Xtn[i], divb, r);
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          r = fma(-Xtn[j], dbeta[j][i], r);
          r = fma(-2.0 * Au[sy(i, j)], dalpha[j], r);
          s = fma(6.0 * Au[sy(i, j)], dphi[j], s);
          s = fma(-(2.0 / 3.0) * gu[sy(i, j)], dtrK[j], s);
        }
#pragma unroll
        for (int q = 0; q < 6; ++q) s = fma(mult(q) * Gu[i][q], Au[q], s);
        rhs[V_XT + i] = fma(2.0 * alpha, s, r);
      }
    }
  }

  // ---- advection (App. A.2 Adv) and the gauge couplings that need the full RHS
  auto centre = [&](int v) -> double {
    if (v == V_PHI) return phi;
    if (v >= V_GT && v < V_GT + 6) return gt[v - V_GT];
    if (v == V_TRK) return trK;
    if (v >= V_AT && v < V_AT + 6) return At[v - V_AT];
    if (v >= V_XT && v < V_XT + 3) return Xt[v - V_XT];
    if (v == V_ALPHA) return alpha;
    if (v == V_AUX) return Aux;
    if (v >= V_BETA && v < V_BETA + 3) return beta[v - V_BETA];
    return Bv[v - V_B];
  };
#pragma unroll
  for (int v = 0; v < V_ALPHA; ++v)
    if (in_group(G, v)) rhs[v] += D.adv(K, v, beta, centre(v));
  if (g1) {
    rhs[V_ALPHA] = fma(K.c_alpha_adv, D.adv(K, V_ALPHA, beta, alpha), rhs[V_ALPHA]);
#pragma unroll
    for (int i = 0; i < 3; ++i)
      rhs[V_BETA + i] = fma(K.c_beta_adv, D.adv(K, V_BETA + i, beta, beta[i]), rhs[V_BETA + i]);
  }
  if (g2) rhs[V_AUX] = K.L * (rhs[V_TRK] - K.eta_alpha * Aux) + K.c_alpha_adv * D.adv(K, V_AUX, beta, Aux);
  if (g3) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const double advB = D.adv(K, V_B + i, beta, Bv[i]);
      const double advX = D.adv(K, V_XT + i, beta, Xt[i]);
      rhs[V_B + i] = K.S_B * (rhs[V_XT + i] - K.eta * Bv[i]) + K.c_beta_adv * (advB - advX);
    }
  }
}

// ------------------------------------------------------------------ constraint monitors
// Vacuum BSSN constraints (R16) with
// the RHS's stencils and Ricci tensor:
//   c[0] = H   = e^{-4 phi} gt^ij (R~_ij + R^phi_ij) + 2/3 K^2 - At_ij At^ij
//   c[1+i] = M^i = d_j At^ij + Gt^i_jk At^jk + Gt^j_jk At^ik + 6 At^ij d_j phi - 2/3 gt^ij d_j K
//            (the full conformal divergence D~_j At^ij: det gt is not assumed 1)
//   c[4+i] = G^i = Xt^i - gt^jk Gt^i_jk
// d_j At^ij by the product rule with d_j gt^ab = -gt^ac (d_j gt_cd) gt^db.
// PART: 0 = all seven, 1 = the Hamiltonian only (c[0]), 2 = momentum and Gamma only (c[1..6]).
template <int PART = 0, class P = StencilP>
__device__ __forceinline__ void bssn_constraint_point(const P& D, const BssnK& K, double* c) {
  double gt[6], At[6];
#pragma unroll
  for (int s = 0; s < 6; ++s) { gt[s] = D.v(V_GT + s); At[s] = D.v(V_AT + s); }
  const double phi = D.v(V_PHI), trK = D.v(V_TRK);
  const double c00 = gt[3] * gt[5] - gt[4] * gt[4];
  const double c01 = gt[2] * gt[4] - gt[1] * gt[5];
  const double c02 = gt[1] * gt[4] - gt[2] * gt[3];
  const double idet = 1.0 / (gt[0] * c00 + gt[1] * c01 + gt[2] * c02);
  double gu[6];
  gu[0] = c00 * idet;
  gu[1] = c01 * idet;
  gu[2] = c02 * idet;
  gu[3] = (gt[0] * gt[5] - gt[2] * gt[2]) * idet;
  gu[4] = (gt[1] * gt[2] - gt[0] * gt[4]) * idet;
  gu[5] = (gt[0] * gt[3] - gt[1] * gt[1]) * idet;
  double dg[3][6], Gl[3][6], Gu[3][6], Xtn[3];
#pragma unroll
  for (int l = 0; l < 3; ++l)
#pragma unroll
    for (int s = 0; s < 6; ++s) dg[l][s] = D.d1(K, V_GT + s, l);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      const int j = sI(s), k = sJ(s);
      Gl[i][s] = 0.5 * (dg[j][sy(i, k)] + dg[k][sy(i, j)] - dg[i][s]);
    }
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int s = 0; s < 6; ++s)
      Gu[i][s] = gu[sy(i, 0)] * Gl[0][s] + gu[sy(i, 1)] * Gl[1][s] + gu[sy(i, 2)] * Gl[2][s];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    double a = 0.0;
#pragma unroll
    for (int s = 0; s < 6; ++s) a = fma(mult(s) * gu[s], Gu[i][s], a);
    Xtn[i] = a;
  }
  double dphi[3], dtrK[3];
#pragma unroll
  for (int l = 0; l < 3; ++l) { dphi[l] = D.d1(K, V_PHI, l); dtrK[l] = D.d1(K, V_TRK, l); }
  double Am[3][3], Au[6];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      Am[i][j] = gu[sy(i, 0)] * At[sy(0, j)] + gu[sy(i, 1)] * At[sy(1, j)] + gu[sy(i, 2)] * At[sy(2, j)];
#pragma unroll
  for (int s = 0; s < 6; ++s) {
    const int i = sI(s), j = sJ(s);
    Au[s] = Am[i][0] * gu[sy(0, j)] + Am[i][1] * gu[sy(1, j)] + Am[i][2] * gu[sy(2, j)];
  }
  // ---- Hamiltonian: Ricci scalar as in bssn_point's curvature group
  if (PART != 2) {
    double Rt[6];
#pragma unroll
    for (int s = 0; s < 6; ++s) Rt[s] = 0.0;
#pragma unroll
    for (int p = 0; p < 6; ++p) {
      const int l = sI(p), m = sJ(p);
      const double w = -0.5 * mult(p) * gu[p];
#pragma unroll
      for (int s = 0; s < 6; ++s) Rt[s] = fma(w, D.dd(K, V_GT + s, l, m, gt[s]), Rt[s]);
    }
    double Rsum = 0.0, DDphi[6], trDDphi = 0.0, dphi2 = 0.0;
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      const int i = sI(s), j = sJ(s);
      DDphi[s] = D.dd(K, V_PHI, i, j, phi) - (Gu[0][s] * dphi[0] + Gu[1][s] * dphi[1] + Gu[2][s] * dphi[2]);
      trDDphi = fma(mult(s) * gu[s], DDphi[s], trDDphi);
    }
#pragma unroll
    for (int k = 0; k < 3; ++k)
      dphi2 = fma(gu[sy(k, 0)] * dphi[0] + gu[sy(k, 1)] * dphi[1] + gu[sy(k, 2)] * dphi[2], dphi[k], dphi2);
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      const int i = sI(s), j = sJ(s);
      double r = Rt[s];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        r = fma(0.5 * gt[sy(k, i)], D.d1(K, V_XT + k, j), r);
        r = fma(0.5 * gt[sy(k, j)], D.d1(K, V_XT + k, i), r);
        r = fma(0.5 * Xtn[k], Gl[i][sy(j, k)] + Gl[j][sy(i, k)], r);
      }
#pragma unroll
      for (int l = 0; l < 3; ++l)
#pragma unroll
        for (int m = 0; m < 3; ++m) {
          double t = 0.0;
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            t = fma(Gu[k][sy(l, i)], Gl[j][sy(k, m)], t);
            t = fma(Gu[k][sy(l, j)], Gl[i][sy(k, m)], t);
            t = fma(Gu[k][sy(i, m)], Gl[k][sy(l, j)], t);
          }
          r = fma(gu[sy(l, m)], t, r);
        }
      const double Rphi = -2.0 * DDphi[s] - 2.0 * gt[s] * trDDphi + 4.0 * dphi[i] * dphi[j] - 4.0 * gt[s] * dphi2;
      Rsum = fma(mult(s) * gu[s], r + Rphi, Rsum);
    }
    double AA = 0.0;
#pragma unroll
    for (int s = 0; s < 6; ++s) AA = fma(mult(s) * At[s], Au[s], AA);
    c[0] = exp(-4.0 * phi) * Rsum + (2.0 / 3.0) * trK * trK - AA;
  }
  // ---- momentum and Gamma constraints
  if (PART == 1) return;
  double W[3] = {0.0, 0.0, 0.0}, U[3] = {0.0, 0.0, 0.0}, V[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    double dAt[6];
#pragma unroll
    for (int s = 0; s < 6; ++s) dAt[s] = D.d1(K, V_AT + s, j);
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        W[k] = fma(gu[sy(j, l)], dAt[sy(k, l)], W[k]);      // gt^jl d_j At_kl
        U[k] = fma(dg[j][sy(k, l)], Au[sy(l, j)], U[k]);    // d_j gt_kl At^lj
        V[l] = fma(gu[sy(j, k)], dg[j][sy(k, l)], V[l]);    // gt^jk d_j gt_kl
      }
  }
  double Gjjk[3];  // Gt^j_jk
#pragma unroll
  for (int k = 0; k < 3; ++k) Gjjk[k] = Gu[0][sy(0, k)] + Gu[1][sy(1, k)] + Gu[2][sy(2, k)];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    double m = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      m = fma(Gjjk[k], Au[sy(i, k)], m);
      m = fma(gu[sy(i, k)], W[k] - U[k], m);
      m = fma(-Au[sy(i, k)], V[k], m);
      m = fma(6.0 * Au[sy(i, k)], dphi[k], m);
      m = fma(-(2.0 / 3.0) * gu[sy(i, k)], dtrK[k], m);
    }
#pragma unroll
    for (int q = 0; q < 6; ++q) m = fma(mult(q) * Gu[i][q], Au[q], m);
    c[1 + i] = m;
    c[4 + i] = D.v(V_XT + i) - Xtn[i];
  }
}

// One thread per point over a fixed grid of kNormBlocks CTAs (grid-stride over the
// interior in a fixed order, so the partials -- and the norms -- are deterministic).
// fields (nullable): [7][z][y][x] interior; part: per CTA [sum c_q^2, max |c_q|] x 7.
BssnK make_k(const StageLaunch& a, const double* prm) {
  BssnK K;
  for (int d = 0; d < 3; ++d) {
    K.i12h[d] = 1.0 / (12.0 * a.h[d]);
    K.i12h2[d] = 1.0 / (12.0 * a.h[d] * a.h[d]);
    K.i24h[d] = 1.0 / (24.0 * a.h[d]);
  }
  K.i144hh[0] = 1.0 / (144.0 * a.h[0] * a.h[1]);
  K.i144hh[1] = 1.0 / (144.0 * a.h[0] * a.h[2]);
  K.i144hh[2] = 1.0 / (144.0 * a.h[1] * a.h[2]);
  K.dt = a.dt; K.dt2 = a.dt / 2.0; K.dt3 = a.dt / 3.0; K.dt6 = a.dt / 6.0; K.third = 1.0 / 3.0;
  K.F_alpha = prm[0]; K.n_alpha = prm[1]; K.L = prm[2]; K.eta_alpha = prm[3]; K.c_alpha_adv = prm[4];
  K.C_beta = prm[5]; K.p_beta = prm[6]; K.S_B = prm[7]; K.eta = prm[8]; K.c_beta_adv = prm[9];
  return K;
}

// Source of the stage input's value of GF v at the point: global memory (default) or a
// copy the kernel already holds on chip (bssn_fused.cu: the shared-memory plane tile).
struct GmemIn {
  const double* in;
  int64_t c, gfs;
  __device__ __forceinline__ double operator()(int v) const { return __ldg(in + v * gfs + c); }
};
template <int STAGE, int G, class IN, bool XYONLY = false>
__device__ __forceinline__ void bssn_update_src(const StageLaunch& a, const BssnK& K, const double* r,
                                                const IN& insrc, int64_t c, int i, int j, int k,
                                                double* rhs_dst);
template <int STAGE, int G>
__device__ __forceinline__ void bssn_update(const StageLaunch& a, const BssnK& K, const double* r,
                                            const double* in, int64_t c, int i, int j, int k,
                                            double* rhs_dst) {
  GmemIn src;
  src.in = in;
  src.c = c;
  src.gfs = a.L.gfs;
  bssn_update_src<STAGE, G>(a, K, r, src, c, i, j, k, rhs_dst);
}
// RK4 stage update of the GFs of group G at point c (interior (i,j,k)) and the stores.
// XYONLY: store only the x/y periodic images inline (the launcher pushes the z ghost planes,
// x/y images included, with a separate plane copy after the kernel).
template <int STAGE, int G, class IN, bool XYONLY>
__device__ __forceinline__ void bssn_update_src(const StageLaunch& a, const BssnK& K, const double* r,
                                                const IN& insrc, int64_t c, int i, int j, int k,
                                                double* rhs_dst) {
  const Layout& L = a.L;
  const int64_t gfs = L.gfs;
  if (STAGE == 0) {
    const int64_t ni = L.nx * L.ny * L.nz;
    const int64_t o = (int64_t(k) * L.ny + j) * L.nx + i;
#pragma unroll
    for (int v = 0; v < NV; ++v)
      if (in_group(G, v)) rhs_dst[v * ni + o] = r[v];
    return;
  }
  double* out = STAGE == 1 ? a.s.b : (STAGE == 2 ? a.s.c : (STAGE == 3 ? a.s.b : a.s.y));
  const FaceDst fd = a.img[STAGE - 1];
  // ghost images: a point near exactly one x or y face stores its one periodic image inline;
  // z faces and x-y edges (3 % of the points at 192^3) take the out-of-line general routine
  const ImageSite isite = image_site(L, i, j, k);
  const int gw = L.g;
  const int64_t ddx = i < gw ? L.nx : (i >= L.nx - gw ? -L.nx : 0);
  const int64_t ddy = (j < gw ? L.ny : (j >= L.ny - gw ? -L.ny : 0)) * L.px;
  const unsigned long long code0 = a.step * (unsigned long long)NV;
  // all pointwise operands of the group first: the output stores below may alias them (plain
  // pointers), so loads interleaved with the stores would serialise one memory round trip
  // per GF
  double p0[NV], p1[NV];
  uint32_t bad = 0;  // bit v: GF v non-finite (branch-free check, one report per point)
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    if (!in_group(G, v)) continue;
    const int64_t o = v * gfs + c;
    if (STAGE == 1) p0[v] = insrc(v);
    if (STAGE == 2) { p0[v] = ld(a.s.y + o); p1[v] = insrc(v); }
    if (STAGE == 3) p0[v] = ld(a.s.y + o);
    if (STAGE == 4) { p0[v] = insrc(v); p1[v] = ld(a.s.q + o); }
  }
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    if (!in_group(G, v)) continue;
    const int64_t o = v * gfs + c;
    double val;
    if (STAGE == 1) val = fma(K.dt2, r[v], p0[v]);
    if (STAGE == 2) {
      const double yv = p0[v], sv = p1[v];
      a.s.q[o] = fma(K.dt3, r[v], (yv + sv) * K.third);
      val = fma(K.dt2, r[v], yv);
    }
    if (STAGE == 3) val = fma(K.dt, r[v], p0[v]);
    if (STAGE == 4) val = fma(K.dt6, r[v], fma(p0[v], K.third, p1[v]));
    out[o] = val;
    if (XYONLY) {
      if (ddx) out[o + ddx] = val;
      if (ddy) out[o + ddy] = val;
      if (ddx && ddy) out[o + ddx + ddy] = val;
    } else {
      put_images(isite, out + v * gfs, fd.lo + v * gfs, fd.hi + v * gfs, L, i, j, k, c, val);
    }
    if (STAGE == 4) bad |= (fabs(val) <= 1.7976931348623157e308 ? 0u : 1u) << v;
  }
  if (STAGE == 4 && bad) atomicMin(a.nan_flag, code0 + (unsigned long long)(__ffs(bad) - 1));
}

template <int STAGE>
__host__ __device__ __forceinline__ const double* stage_input(const StageLaunch& a) {
  return (STAGE <= 1) ? a.s.y : (STAGE == 2 ? a.s.b : (STAGE == 3 ? a.s.c : a.s.b));
}


}  // namespace
}  // namespace chemora
