// chemora_oracle.cpp -- the plain, slow, obviously-correct CPU ORACLE.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load this library.  It shares no code with
// the CUDA path (paper_1410_1764_b200/csrc): no headers, helpers, tables or generators.
//
// What it computes (PAPER.md = /root/reference/PAPER.md line numbers):
//   * method of lines + classical RK4 ("a Runge-Kutta method ...
//     calculate the new state vector"), textbook form with k1..k4:
//        fill(y); k1=F(y); Y=y+dt/2 k1; fill(Y); k2=F(Y); Y=y+dt/2 k2; fill(Y);
//        k3=F(Y); Y=y+dt k3; fill(Y); k4=F(Y); y = y + dt/6 (k1 + 2k2 + 2k3 + k4)
//   * periodic ghost fill, axis by axis x, y, z over padded planes (PAPER.md:345-347
//     "ghost zones")
//   * F = Eq. 1, the first-order scalar wave equation (Fig. 1
//     PAPER.md:637-641) discretised with the standard centered 4th-order stencil
//     ("'Standard' Finite Differencing operators of arbitrary order";
//     DESIGN.md reading R2), written literally as (f[-2] - 8 f[-1] + 8 f[+1] - f[+2])/(12 h).
//   * F = the 25-GF BSSN-like system of SURVEY.md App. A (reading R7),
//     transcribed with explicit index loops over full (non-symmetric-packed) 3x3 tensors.
//   * norms: L2 = sqrt(h^3 sum f^2), Linf = max|f|, sum = h^3 sum f,
//     wave energy E = h^3 sum 1/2 (rho^2 + v.v) (Fig. 1 "Energy").
//
// Storage: padded arrays [gf][Nz+2g][Ny+2g][Nx+2g], x fastest, double.  Parallelism:
// an OpenMP `for` over z only; every result is independent of the thread count.
// Built with g++ -O2 -fopenmp -ffp-contract=off (no FMA contraction, no fast-math).
//
// Parity pins: see tests/test_oracle_*.py; every function here is pinned.

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <algorithm>

namespace {

struct Grid {
  int64_t n[3];   // interior extents Nx, Ny, Nz
  int g;          // ghost width
  int64_t p[3];   // padded extents
  double h[3];
  int order = 4;  // accuracy order of the wave system's centered D1 (2, 4, 6, 8)
  Grid(const int64_t* ext, int ghost, const double* sp) {
    for (int a = 0; a < 3; ++a) { n[a] = ext[a]; p[a] = ext[a] + 2 * ghost; h[a] = sp[a]; }
    g = ghost;
  }
  int64_t npad() const { return p[0] * p[1] * p[2]; }
  int64_t nint() const { return n[0] * n[1] * n[2]; }
  // padded index of interior coordinate (i, j, k); ghosts are i in [-g, 0) etc.
  int64_t at(int64_t i, int64_t j, int64_t k) const {
    return ((k + g) * p[1] + (j + g)) * p[0] + (i + g);
  }
  int64_t at_int(int64_t i, int64_t j, int64_t k) const { return (k * n[1] + j) * n[0] + i; }
};

// ---------------------------------------------------------------- ghost fill
// Periodic: each ghost equals the periodic image of the opposite interior edge; applied
// axis by axis (x over interior rows, y over x-padded rows, z over fully padded planes) so
// that edges and corners are the doubly/triply wrapped interior values.
void fill_ghosts_one(double* f, const Grid& G) {
  const int g = G.g;
  const int64_t nx = G.n[0], ny = G.n[1], nz = G.n[2];
  // x
  for (int64_t k = 0; k < nz; ++k)
    for (int64_t j = 0; j < ny; ++j)
      for (int s = 1; s <= g; ++s) {
        f[G.at(-s, j, k)] = f[G.at(nx - s, j, k)];
        f[G.at(nx - 1 + s, j, k)] = f[G.at(s - 1, j, k)];
      }
  // y (all x including ghosts)
  for (int64_t k = 0; k < nz; ++k)
    for (int s = 1; s <= g; ++s)
      for (int64_t i = -g; i < nx + g; ++i) {
        f[G.at(i, -s, k)] = f[G.at(i, ny - s, k)];
        f[G.at(i, ny - 1 + s, k)] = f[G.at(i, s - 1, k)];
      }
  // z (all x, y including ghosts)
  for (int s = 1; s <= g; ++s)
    for (int64_t j = -g; j < ny + g; ++j)
      for (int64_t i = -g; i < nx + g; ++i) {
        f[G.at(i, j, -s)] = f[G.at(i, j, nz - s)];
        f[G.at(i, j, nz - 1 + s)] = f[G.at(i, j, s - 1)];
      }
}

// ---------------------------------------------------------------- stencils
// Centered 4th-order first derivative along axis a at padded index c with stride s:
//   D1 f = (f[-2] - 8 f[-1] + 8 f[+1] - f[+2]) / (12 h)        (SPEC.md:218 (d=1,w=2))
inline double d1(const double* f, int64_t c, int64_t s, double h) {
  return (f[c - 2 * s] - 8.0 * f[c - s] + 8.0 * f[c + s] - f[c + 2 * s]) / (12.0 * h);
}
// Centered first derivatives of order 2, 6 and 8 (the standard operators of PAPER.md:
// 509-514, "Finite Differencing with arbitrary order of accuracy ... run-time option";
// SURVEY.md §8(f) NEXT-1), written out literally:
//   order 2: (f[+1] - f[-1]) / (2h)
//   order 6: (-f[-3] + 9f[-2] - 45f[-1] + 45f[+1] - 9f[+2] + f[+3]) / (60h)
//   order 8: (3f[-4] - 32f[-3] + 168f[-2] - 672f[-1] + 672f[+1] - 168f[+2] + 32f[+3] - 3f[+4]) / (840h)
inline double d1n(const double* f, int64_t c, int64_t s, double h, int order) {
  switch (order) {
    case 2: return (f[c + s] - f[c - s]) / (2.0 * h);
    case 6:
      return (-f[c - 3 * s] + 9.0 * f[c - 2 * s] - 45.0 * f[c - s] + 45.0 * f[c + s] - 9.0 * f[c + 2 * s] +
              f[c + 3 * s]) / (60.0 * h);
    case 8:
      return (3.0 * f[c - 4 * s] - 32.0 * f[c - 3 * s] + 168.0 * f[c - 2 * s] - 672.0 * f[c - s] +
              672.0 * f[c + s] - 168.0 * f[c + 2 * s] + 32.0 * f[c + 3 * s] - 3.0 * f[c + 4 * s]) / (840.0 * h);
    default: return d1(f, c, s, h);
  }
}
// Centered 4th-order second derivative:
//   D2 f = (-f[-2] + 16 f[-1] - 30 f[0] + 16 f[+1] - f[+2]) / (12 h^2)
inline double d2(const double* f, int64_t c, int64_t s, double h) {
  return (-f[c - 2 * s] + 16.0 * f[c - s] - 30.0 * f[c] + 16.0 * f[c + s] - f[c + 2 * s]) /
         (12.0 * h * h);
}
// Mixed derivative d_a d_b f = D1_a (D1_b f): the tensor product of two D1 stencils.
inline double d11(const double* f, int64_t c, int64_t sa, double ha, int64_t sb, double hb) {
  const double w[5] = {1.0, -8.0, 0.0, 8.0, -1.0};
  double acc = 0.0;
  for (int p = -2; p <= 2; ++p) {
    if (p == 0) continue;
    double inner = 0.0;
    for (int q = -2; q <= 2; ++q) {
      if (q == 0) continue;
      inner += w[q + 2] * f[c + p * sa + q * sb];
    }
    acc += w[p + 2] * inner;
  }
  return acc / (144.0 * ha * hb);
}
// Upwind (lopsided) 4th-order first derivatives (reading R6):
//   D+ f = (-3 f[-1] - 10 f[0] + 18 f[+1] - 6 f[+2] + f[+3]) / (12 h)
//   D- f = (-f[-3] + 6 f[-2] - 18 f[-1] + 10 f[0] + 3 f[+1]) / (12 h)
inline double dplus(const double* f, int64_t c, int64_t s, double h) {
  return (-3.0 * f[c - s] - 10.0 * f[c] + 18.0 * f[c + s] - 6.0 * f[c + 2 * s] + f[c + 3 * s]) /
         (12.0 * h);
}
inline double dminus(const double* f, int64_t c, int64_t s, double h) {
  return (-f[c - 3 * s] + 6.0 * f[c - 2 * s] - 18.0 * f[c - s] + 10.0 * f[c] + 3.0 * f[c + s]) /
         (12.0 * h);
}

// ---------------------------------------------------------------- wave RHS (Eq. 1)
// GF order: 0 u, 1 rho, 2 v1, 3 v2, 4 v3.
//   d_t u = rho ;  d_t rho = delta^ij d_i v_j ;  d_t v_i = d_i rho
void wave_rhs(const double* y, double* k, const Grid& G) {
  const int64_t np = G.npad(), ni = G.nint();
  const double* u = y;
  const double* rho = y + 1 * np;
  const double* v1 = y + 2 * np;
  const double* v2 = y + 3 * np;
  const double* v3 = y + 4 * np;
  (void)u;
  const int64_t sx = 1, sy = G.p[0], sz = G.p[0] * G.p[1];
#pragma omp parallel for schedule(static)
  for (int64_t kk = 0; kk < G.n[2]; ++kk)
    for (int64_t j = 0; j < G.n[1]; ++j)
      for (int64_t i = 0; i < G.n[0]; ++i) {
        const int64_t c = G.at(i, j, kk), o = G.at_int(i, j, kk);
        k[0 * ni + o] = rho[c];
        const int q = G.order;
        k[1 * ni + o] = d1n(v1, c, sx, G.h[0], q) + d1n(v2, c, sy, G.h[1], q) + d1n(v3, c, sz, G.h[2], q);
        k[2 * ni + o] = d1n(rho, c, sx, G.h[0], q);
        k[3 * ni + o] = d1n(rho, c, sy, G.h[1], q);
        k[4 * ni + o] = d1n(rho, c, sz, G.h[2], q);
      }
}

// ---------------------------------------------------------------- BSSN RHS
// Variable order (App. A.1): phi, gt(xx,xy,xz,yy,yz,zz), trK, At(6), Xt(3), alpha, A,
// beta(3), B(3).  Gauge parameters (App. A.3): F_alpha, n_alpha, L, eta_alpha, c_alpha_adv,
// C_beta, p_beta, S_B, eta, c_beta_adv.
enum {
  PHI = 0, GT = 1, TRK = 7, AT = 8, XT = 14, ALPHA = 17, AUXA = 18, BETA = 19, BB = 22, NBSSN = 25
};
// symmetric-pair -> packed index (xx,xy,xz,yy,yz,zz)
inline int sym(int i, int j) {
  static const int m[3][3] = {{0, 1, 2}, {1, 3, 4}, {2, 4, 5}};
  return m[i][j];
}

template <typename T> struct BssnParams {
  T F_alpha, n_alpha, L, eta_alpha, c_alpha_adv, C_beta, p_beta, S_B, eta, c_beta_adv;
};

void bssn_rhs(const double* y, double* kout, const Grid& G, const double* prm) {
  const int64_t np = G.npad(), ni = G.nint();
  const int64_t st[3] = {1, G.p[0], G.p[0] * G.p[1]};
  const double* h = G.h;
  BssnParams<double> P{prm[0], prm[1], prm[2], prm[3], prm[4],
                       prm[5], prm[6], prm[7], prm[8], prm[9]};
#pragma omp parallel for schedule(static)
  for (int64_t kk = 0; kk < G.n[2]; ++kk)
    for (int64_t jj = 0; jj < G.n[1]; ++jj)
      for (int64_t ii = 0; ii < G.n[0]; ++ii) {
        const int64_t c = G.at(ii, jj, kk), o = G.at_int(ii, jj, kk);
        auto F = [&](int v) { return y + v * np; };
        auto val = [&](int v) { return F(v)[c]; };
        // ---- point values
        const double phi = val(PHI), trK = val(TRK), alpha = val(ALPHA), Aux = val(AUXA);
        double gt[3][3], At[3][3], Xt[3], beta[3], B[3];
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) {
            gt[i][j] = val(GT + sym(i, j));
            At[i][j] = val(AT + sym(i, j));
          }
        for (int i = 0; i < 3; ++i) { Xt[i] = val(XT + i); beta[i] = val(BETA + i); B[i] = val(BB + i); }
        // ---- centered first derivatives d[l] f
        double dphi[3], dtrK[3], dalpha[3], dgt[3][3][3], dbeta[3][3], dXt[3][3];
        // dgt[l][i][j] = d_l gt_ij ; dbeta[l][k] = d_l beta^k ; dXt[l][k] = d_l Xt^k
        for (int l = 0; l < 3; ++l) {
          dphi[l] = d1(F(PHI), c, st[l], h[l]);
          dtrK[l] = d1(F(TRK), c, st[l], h[l]);
          dalpha[l] = d1(F(ALPHA), c, st[l], h[l]);
          for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) dgt[l][i][j] = d1(F(GT + sym(i, j)), c, st[l], h[l]);
          for (int kx = 0; kx < 3; ++kx) {
            dbeta[l][kx] = d1(F(BETA + kx), c, st[l], h[l]);
            dXt[l][kx] = d1(F(XT + kx), c, st[l], h[l]);
          }
        }
        // ---- second derivatives dd[l][m] f (pure D2 on the diagonal, D1 x D1 mixed)
        auto dd = [&](int v, int l, int m) {
          if (l == m) return d2(F(v), c, st[l], h[l]);
          return d11(F(v), c, st[l], h[l], st[m], h[m]);
        };
        double ddphi[3][3], ddalpha[3][3], ddgt[3][3][3][3], ddbeta[3][3][3];
        for (int l = 0; l < 3; ++l)
          for (int m = 0; m < 3; ++m) {
            ddphi[l][m] = dd(PHI, l, m);
            ddalpha[l][m] = dd(ALPHA, l, m);
            for (int i = 0; i < 3; ++i)
              for (int j = 0; j < 3; ++j) ddgt[l][m][i][j] = dd(GT + sym(i, j), l, m);
            for (int kx = 0; kx < 3; ++kx) ddbeta[l][m][kx] = dd(BETA + kx, l, m);
          }
        // ---- advection Adv(f) = sum_k [max(beta^k,0) D+_k f + min(beta^k,0) D-_k f]
        auto adv = [&](int v) {
          double s = 0.0;
          for (int l = 0; l < 3; ++l) {
            const double bp = beta[l] > 0.0 ? beta[l] : 0.0;
            const double bm = beta[l] < 0.0 ? beta[l] : 0.0;
            s += bp * dplus(F(v), c, st[l], h[l]) + bm * dminus(F(v), c, st[l], h[l]);
          }
          return s;
        };
        // ---- inverse conformal metric: cofactor / det (det computed, App. A.2)
        const double det = gt[0][0] * (gt[1][1] * gt[2][2] - gt[1][2] * gt[2][1]) -
                           gt[0][1] * (gt[1][0] * gt[2][2] - gt[1][2] * gt[2][0]) +
                           gt[0][2] * (gt[1][0] * gt[2][1] - gt[1][1] * gt[2][0]);
        double gu[3][3];
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) {
            // cofactor C_ji, i.e. adjugate entry (i,j)
            const int r0 = (j + 1) % 3, r1 = (j + 2) % 3, c0 = (i + 1) % 3, c1 = (i + 2) % 3;
            gu[i][j] = (gt[r0][c0] * gt[r1][c1] - gt[r0][c1] * gt[r1][c0]) / det;
          }
        const double em4phi = std::exp(-4.0 * phi);
        // ---- Christoffels: Gl[i][j][k] = 1/2 (d_j gt_ik + d_k gt_ij - d_i gt_jk)
        double Gl[3][3][3], Gu[3][3][3], Xtn[3];
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j)
            for (int kx = 0; kx < 3; ++kx)
              Gl[i][j][kx] = 0.5 * (dgt[j][i][kx] + dgt[kx][i][j] - dgt[i][j][kx]);
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j)
            for (int kx = 0; kx < 3; ++kx) {
              double s = 0.0;
              for (int l = 0; l < 3; ++l) s += gu[i][l] * Gl[l][j][kx];
              Gu[i][j][kx] = s;
            }
        for (int i = 0; i < 3; ++i) {
          double s = 0.0;
          for (int j = 0; j < 3; ++j)
            for (int kx = 0; kx < 3; ++kx) s += gu[j][kx] * Gu[i][j][kx];
          Xtn[i] = s;
        }
        // ---- conformal Ricci R~_ij
        double Rt[3][3];
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) {
            double s = 0.0;
            for (int l = 0; l < 3; ++l)
              for (int m = 0; m < 3; ++m) s += gu[l][m] * ddgt[l][m][i][j];
            double r = -0.5 * s;
            for (int kx = 0; kx < 3; ++kx)
              r += 0.5 * (gt[kx][i] * dXt[j][kx] + gt[kx][j] * dXt[i][kx]);
            for (int kx = 0; kx < 3; ++kx) r += 0.5 * Xtn[kx] * (Gl[i][j][kx] + Gl[j][i][kx]);
            for (int l = 0; l < 3; ++l)
              for (int m = 0; m < 3; ++m)
                for (int kx = 0; kx < 3; ++kx)
                  r += gu[l][m] * (Gu[kx][l][i] * Gl[j][kx][m] + Gu[kx][l][j] * Gl[i][kx][m] +
                                   Gu[kx][i][m] * Gl[kx][l][j]);
            Rt[i][j] = r;
          }
        // ---- phi part of the Ricci tensor
        double DDphi[3][3];
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) {
            double s = ddphi[i][j];
            for (int kx = 0; kx < 3; ++kx) s -= Gu[kx][i][j] * dphi[kx];
            DDphi[i][j] = s;
          }
        double trDDphi = 0.0, dphi2 = 0.0;
        for (int l = 0; l < 3; ++l)
          for (int m = 0; m < 3; ++m) {
            trDDphi += gu[l][m] * DDphi[l][m];
            dphi2 += gu[l][m] * dphi[l] * dphi[m];
          }
        double R[3][3];
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) {
            const double Rphi = -2.0 * DDphi[i][j] - 2.0 * gt[i][j] * trDDphi +
                                4.0 * dphi[i] * dphi[j] - 4.0 * gt[i][j] * dphi2;
            R[i][j] = Rt[i][j] + Rphi;
          }
        // ---- physical Christoffel and D_i D_j alpha
        double DDalpha[3][3];
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) {
            double s = ddalpha[i][j];
            for (int kx = 0; kx < 3; ++kx) {
              double gphys = Gu[kx][i][j];
              double corr = (kx == i ? dphi[j] : 0.0) + (kx == j ? dphi[i] : 0.0);
              double t = 0.0;
              for (int l = 0; l < 3; ++l) t += gu[kx][l] * dphi[l];
              corr -= gt[i][j] * t;
              gphys += 2.0 * corr;
              s -= gphys * dalpha[kx];
            }
            DDalpha[i][j] = s;
          }
        double trDDalpha = 0.0;
        {
          double s1 = 0.0, s2 = 0.0, s3 = 0.0;
          for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) {
              s1 += gu[i][j] * ddalpha[i][j];
              s3 += gu[i][j] * dphi[i] * dalpha[j];
            }
          for (int kx = 0; kx < 3; ++kx) s2 += Xtn[kx] * dalpha[kx];
          trDDalpha = em4phi * (s1 - s2 + 2.0 * s3);
        }
        // ---- raised At
        double Atm[3][3], Atu[3][3];  // Atm[i][j] = At^i_j ; Atu = At^ij
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) {
            double s = 0.0;
            for (int kx = 0; kx < 3; ++kx) s += gu[i][kx] * At[kx][j];
            Atm[i][j] = s;
          }
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) {
            double s = 0.0;
            for (int kx = 0; kx < 3; ++kx)
              for (int l = 0; l < 3; ++l) s += gu[i][kx] * gu[j][l] * At[kx][l];
            Atu[i][j] = s;
          }
        double AA = 0.0;
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) AA += At[i][j] * Atu[i][j];
        double divbeta = 0.0;
        for (int kx = 0; kx < 3; ++kx) divbeta += dbeta[kx][kx];
        // ---- right-hand sides (App. A.3)
        double rhs[NBSSN];
        rhs[PHI] = -alpha * trK / 6.0 + divbeta / 6.0 + adv(PHI);
        for (int i = 0; i < 3; ++i)
          for (int j = i; j < 3; ++j) {
            double r = -2.0 * alpha * At[i][j];
            for (int kx = 0; kx < 3; ++kx) r += gt[i][kx] * dbeta[j][kx] + gt[j][kx] * dbeta[i][kx];
            r -= (2.0 / 3.0) * gt[i][j] * divbeta;
            rhs[GT + sym(i, j)] = r + adv(GT + sym(i, j));
          }
        const double rhs_trK = -trDDalpha + alpha * (AA + trK * trK / 3.0) + adv(TRK);
        rhs[TRK] = rhs_trK;
        double X[3][3], trX = 0.0;
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) X[i][j] = -DDalpha[i][j] + alpha * R[i][j];
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) trX += gu[i][j] * X[i][j];
        for (int i = 0; i < 3; ++i)
          for (int j = i; j < 3; ++j) {
            double AAm = 0.0;
            for (int kx = 0; kx < 3; ++kx) AAm += At[i][kx] * Atm[kx][j];
            double r = em4phi * (X[i][j] - trX * gt[i][j] / 3.0) + alpha * (trK * At[i][j] - 2.0 * AAm);
            for (int kx = 0; kx < 3; ++kx) r += At[i][kx] * dbeta[j][kx] + At[j][kx] * dbeta[i][kx];
            r -= (2.0 / 3.0) * At[i][j] * divbeta;
            rhs[AT + sym(i, j)] = r + adv(AT + sym(i, j));
          }
        double ddivbeta[3];  // d_j (d . beta) = sum_k d_j d_k beta^k
        for (int j = 0; j < 3; ++j) {
          double s = 0.0;
          for (int kx = 0; kx < 3; ++kx) s += ddbeta[j][kx][kx];
          ddivbeta[j] = s;
        }
        double rhs_Xt[3];
        for (int i = 0; i < 3; ++i) {
          double r = 0.0;
          for (int j = 0; j < 3; ++j)
            for (int kx = 0; kx < 3; ++kx) r += gu[j][kx] * ddbeta[j][kx][i];
          for (int j = 0; j < 3; ++j) r += gu[i][j] * ddivbeta[j] / 3.0;
          for (int j = 0; j < 3; ++j) r -= Xtn[j] * dbeta[j][i];
          r += (2.0 / 3.0) * Xtn[i] * divbeta;
          for (int j = 0; j < 3; ++j) r -= 2.0 * Atu[i][j] * dalpha[j];
          double s = 0.0;
          for (int j = 0; j < 3; ++j)
            for (int kx = 0; kx < 3; ++kx) s += Gu[i][j][kx] * Atu[j][kx];
          for (int j = 0; j < 3; ++j) s += 6.0 * Atu[i][j] * dphi[j];
          for (int j = 0; j < 3; ++j) s -= (2.0 / 3.0) * gu[i][j] * dtrK[j];
          r += 2.0 * alpha * s;
          rhs_Xt[i] = r + adv(XT + i);
          rhs[XT + i] = rhs_Xt[i];
        }
        // ---- gauge (App. A.3)
        rhs[ALPHA] = -P.F_alpha * std::pow(alpha, P.n_alpha) * (P.L * Aux + (1.0 - P.L) * trK) +
                     P.c_alpha_adv * adv(ALPHA);
        rhs[AUXA] = P.L * (rhs_trK - P.eta_alpha * Aux) + P.c_alpha_adv * adv(AUXA);
        for (int i = 0; i < 3; ++i) {
          rhs[BETA + i] = P.C_beta * std::pow(alpha, P.p_beta) *
                              (P.S_B * B[i] + (1.0 - P.S_B) * (Xt[i] - P.eta * beta[i])) +
                          P.c_beta_adv * adv(BETA + i);
          rhs[BB + i] = P.S_B * (rhs_Xt[i] - P.eta * B[i]) +
                        P.c_beta_adv * (adv(BB + i) - adv(XT + i));
        }
        for (int v = 0; v < NBSSN; ++v) kout[v * ni + o] = rhs[v];
      }
}

// ---------------------------------------------------------------- BSSN constraints
// Vacuum constraints of the BSSN variables (PAPER.md:472-473
// "constraint equations"), evaluated with the same 4th-order stencils:
//   H   = R + 2/3 K^2 - At_ij At^ij,   R = e^{-4 phi} gt^ij (R~_ij + R^phi_ij)   (App. A.2)
//   M^i = D~_j At^ij + 6 At^ij d_j phi - 2/3 gt^ij d_j K,
//         D~_j At^ij = d_j At^ij + Gt^i_jk At^jk + Gt^j_jk At^ik  (full conformal covariant
//         divergence: det gt is computed, not assumed 1 -- App. A.2; R16)
//   G^i = Xt^i - gt^jk Gt^i_jk
// out: 7 interior fields [H, M1, M2, M3, G1, G2, G3].
void bssn_constraints(const double* y, double* out, const Grid& G) {
  const int64_t np = G.npad(), ni = G.nint();
  const int64_t st[3] = {1, G.p[0], G.p[0] * G.p[1]};
  const double* h = G.h;
#pragma omp parallel for schedule(static)
  for (int64_t kk = 0; kk < G.n[2]; ++kk)
    for (int64_t jj = 0; jj < G.n[1]; ++jj)
      for (int64_t ii = 0; ii < G.n[0]; ++ii) {
        const int64_t c = G.at(ii, jj, kk), o = G.at_int(ii, jj, kk);
        auto F = [&](int v) { return y + v * np; };
        const double phi = F(PHI)[c], trK = F(TRK)[c];
        double gt[3][3], At[3][3], Xt[3];
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) { gt[i][j] = F(GT + sym(i, j))[c]; At[i][j] = F(AT + sym(i, j))[c]; }
        for (int i = 0; i < 3; ++i) Xt[i] = F(XT + i)[c];
        double dphi[3], dtrK[3], dgt[3][3][3], dAt[3][3][3], dXt[3][3];
        for (int l = 0; l < 3; ++l) {
          dphi[l] = d1(F(PHI), c, st[l], h[l]);
          dtrK[l] = d1(F(TRK), c, st[l], h[l]);
          for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) {
              dgt[l][i][j] = d1(F(GT + sym(i, j)), c, st[l], h[l]);
              dAt[l][i][j] = d1(F(AT + sym(i, j)), c, st[l], h[l]);
            }
          for (int kx = 0; kx < 3; ++kx) dXt[l][kx] = d1(F(XT + kx), c, st[l], h[l]);
        }
        auto dd = [&](int v, int l, int m) {
          if (l == m) return d2(F(v), c, st[l], h[l]);
          return d11(F(v), c, st[l], h[l], st[m], h[m]);
        };
        const double det = gt[0][0] * (gt[1][1] * gt[2][2] - gt[1][2] * gt[2][1]) -
                           gt[0][1] * (gt[1][0] * gt[2][2] - gt[1][2] * gt[2][0]) +
                           gt[0][2] * (gt[1][0] * gt[2][1] - gt[1][1] * gt[2][0]);
        double gu[3][3];
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) {
            const int r0 = (j + 1) % 3, r1 = (j + 2) % 3, c0 = (i + 1) % 3, c1 = (i + 2) % 3;
            gu[i][j] = (gt[r0][c0] * gt[r1][c1] - gt[r0][c1] * gt[r1][c0]) / det;
          }
        double Gl[3][3][3], Gu[3][3][3], Xtn[3];
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j)
            for (int kx = 0; kx < 3; ++kx)
              Gl[i][j][kx] = 0.5 * (dgt[j][i][kx] + dgt[kx][i][j] - dgt[i][j][kx]);
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j)
            for (int kx = 0; kx < 3; ++kx) {
              double s = 0.0;
              for (int l = 0; l < 3; ++l) s += gu[i][l] * Gl[l][j][kx];
              Gu[i][j][kx] = s;
            }
        for (int i = 0; i < 3; ++i) {
          double s = 0.0;
          for (int j = 0; j < 3; ++j)
            for (int kx = 0; kx < 3; ++kx) s += gu[j][kx] * Gu[i][j][kx];
          Xtn[i] = s;
        }
        // Ricci scalar: gt^ij (R~_ij + R^phi_ij), as in the RHS
        double Rsum = 0.0;
        double trDDphi = 0.0, dphi2 = 0.0, DDphi[3][3];
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) {
            double s = dd(PHI, i, j);
            for (int kx = 0; kx < 3; ++kx) s -= Gu[kx][i][j] * dphi[kx];
            DDphi[i][j] = s;
          }
        for (int l = 0; l < 3; ++l)
          for (int m = 0; m < 3; ++m) {
            trDDphi += gu[l][m] * DDphi[l][m];
            dphi2 += gu[l][m] * dphi[l] * dphi[m];
          }
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) {
            double s = 0.0;
            for (int l = 0; l < 3; ++l)
              for (int m = 0; m < 3; ++m) s += gu[l][m] * dd(GT + sym(i, j), l, m);
            double r = -0.5 * s;
            for (int kx = 0; kx < 3; ++kx)
              r += 0.5 * (gt[kx][i] * dXt[j][kx] + gt[kx][j] * dXt[i][kx]);
            for (int kx = 0; kx < 3; ++kx) r += 0.5 * Xtn[kx] * (Gl[i][j][kx] + Gl[j][i][kx]);
            for (int l = 0; l < 3; ++l)
              for (int m = 0; m < 3; ++m)
                for (int kx = 0; kx < 3; ++kx)
                  r += gu[l][m] * (Gu[kx][l][i] * Gl[j][kx][m] + Gu[kx][l][j] * Gl[i][kx][m] +
                                   Gu[kx][i][m] * Gl[kx][l][j]);
            const double Rphi = -2.0 * DDphi[i][j] - 2.0 * gt[i][j] * trDDphi + 4.0 * dphi[i] * dphi[j] -
                                4.0 * gt[i][j] * dphi2;
            Rsum += gu[i][j] * (r + Rphi);
          }
        const double Rscal = std::exp(-4.0 * phi) * Rsum;
        double Atu[3][3];
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) {
            double s = 0.0;
            for (int kx = 0; kx < 3; ++kx)
              for (int l = 0; l < 3; ++l) s += gu[i][kx] * gu[j][l] * At[kx][l];
            Atu[i][j] = s;
          }
        double AA = 0.0;
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) AA += At[i][j] * Atu[i][j];
        out[0 * ni + o] = Rscal + (2.0 / 3.0) * trK * trK - AA;
        // d_l gu^{ab} = -gu^{ai} gu^{bj} d_l gt_ij
        double dgu[3][3][3];
        for (int l = 0; l < 3; ++l)
          for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) {
              double s = 0.0;
              for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) s -= gu[a][i] * gu[b][j] * dgt[l][i][j];
              dgu[l][a][b] = s;
            }
        for (int i = 0; i < 3; ++i) {
          // d_j At^ij = d_j (gu^ik gu^jl At_kl)
          double div = 0.0;
          for (int j = 0; j < 3; ++j)
            for (int kx = 0; kx < 3; ++kx)
              for (int l = 0; l < 3; ++l)
                div += dgu[j][i][kx] * gu[j][l] * At[kx][l] + gu[i][kx] * dgu[j][j][l] * At[kx][l] +
                       gu[i][kx] * gu[j][l] * dAt[j][kx][l];
          double m = div;
          for (int j = 0; j < 3; ++j)
            for (int kx = 0; kx < 3; ++kx) m += Gu[i][j][kx] * Atu[j][kx];
          for (int j = 0; j < 3; ++j)
            for (int kx = 0; kx < 3; ++kx) m += Gu[j][j][kx] * Atu[i][kx];
          for (int j = 0; j < 3; ++j) m += 6.0 * Atu[i][j] * dphi[j] - (2.0 / 3.0) * gu[i][j] * dtrK[j];
          out[(1 + i) * ni + o] = m;
          out[(4 + i) * ni + o] = Xt[i] - Xtn[i];
        }
      }
}

int n_gf_of(int system) { return system == 1 ? 5 : (system == 2 ? 25 : -1); }

const double kDefaultBssnParams[10] = {2.0, 1.0, 1.0, 0.0, 1.0, 0.75, 0.0, 1.0, 1.0, 1.0};

void rhs_any(int system, const double* y, double* k, const Grid& G, const double* prm) {
  if (system == 1) wave_rhs(y, k, G);
  else bssn_rhs(y, k, G, prm ? prm : kDefaultBssnParams);
}

}  // namespace

extern "C" {

// All functions return 0 on success, nonzero on invalid arguments.

int chemora_oracle_n_gf(int system) { return n_gf_of(system); }

void chemora_oracle_default_bssn_params(double* out10) {
  for (int i = 0; i < 10; ++i) out10[i] = kDefaultBssnParams[i];
}

// Periodic ghost fill of n_gf padded arrays.
int chemora_oracle_fill_ghosts(double* f, int n_gf, const int64_t* ext, int g) {
  const double one[3] = {1, 1, 1};
  Grid G(ext, g, one);
  for (int a = 0; a < 3; ++a)
    if (ext[a] < 2 * g || g < 0) return 1;
  for (int v = 0; v < n_gf; ++v) fill_ghosts_one(f + v * G.npad(), G);
  return 0;
}

// k = F(y) at interior points, ghosts of y used as they are.  y: padded, k: interior.
// fd_order: accuracy order of the wave system's centered D1 (2, 4, 6, 8); BSSN: 4 only.
int chemora_oracle_rhs_order(int system, const double* y, double* k, const int64_t* ext, int g,
                             const double* spacing, const double* params, int fd_order) {
  if (n_gf_of(system) < 0) return 1;
  if (fd_order != 2 && fd_order != 4 && fd_order != 6 && fd_order != 8) return 3;
  if (system == 2 && fd_order != 4) return 3;
  if (g < (system == 1 ? fd_order / 2 : 3)) return 2;
  Grid G(ext, g, spacing);
  G.order = fd_order;
  rhs_any(system, y, k, G, params);
  return 0;
}

int chemora_oracle_rhs(int system, const double* y, double* k, const int64_t* ext, int g,
                       const double* spacing, const double* params) {
  return chemora_oracle_rhs_order(system, y, k, ext, g, spacing, params, 4);
}

// nsteps classical RK4 steps in place on the padded state y (textbook k1..k4 form).
// On return the ghosts of y are filled.
int chemora_oracle_rk4_order(int system, double* y, const int64_t* ext, int g, const double* spacing,
                             double dt, int nsteps, const double* params, int fd_order) {
  const int nf = n_gf_of(system);
  if (nf < 0) return 1;
  if (fd_order != 2 && fd_order != 4 && fd_order != 6 && fd_order != 8) return 3;
  if (system == 2 && fd_order != 4) return 3;
  if (g < (system == 1 ? fd_order / 2 : 3)) return 2;
  Grid G(ext, g, spacing);
  G.order = fd_order;
  const int64_t np = G.npad(), ni = G.nint();
  std::vector<double> Y(static_cast<size_t>(nf * np));
  std::vector<double> k1(nf * ni), k2(nf * ni), k3(nf * ni), k4(nf * ni);
  auto fill = [&](double* f) { for (int v = 0; v < nf; ++v) fill_ghosts_one(f + v * np, G); };
  // Y = y + a * k at interior points (ghosts filled afterwards)
  auto axpy = [&](double a, const std::vector<double>& kk) {
    for (int v = 0; v < nf; ++v)
#pragma omp parallel for schedule(static)
      for (int64_t z = 0; z < G.n[2]; ++z)
        for (int64_t j = 0; j < G.n[1]; ++j)
          for (int64_t i = 0; i < G.n[0]; ++i) {
            const int64_t c = v * np + G.at(i, j, z), o = v * ni + G.at_int(i, j, z);
            Y[c] = y[c] + a * kk[o];
          }
    fill(Y.data());
  };
  for (int step = 0; step < nsteps; ++step) {
    fill(y);
    rhs_any(system, y, k1.data(), G, params);
    axpy(dt / 2.0, k1);
    rhs_any(system, Y.data(), k2.data(), G, params);
    axpy(dt / 2.0, k2);
    rhs_any(system, Y.data(), k3.data(), G, params);
    axpy(dt, k3);
    rhs_any(system, Y.data(), k4.data(), G, params);
    for (int v = 0; v < nf; ++v)
#pragma omp parallel for schedule(static)
      for (int64_t z = 0; z < G.n[2]; ++z)
        for (int64_t j = 0; j < G.n[1]; ++j)
          for (int64_t i = 0; i < G.n[0]; ++i) {
            const int64_t c = v * np + G.at(i, j, z), o = v * ni + G.at_int(i, j, z);
            y[c] = y[c] + dt / 6.0 * (k1[o] + 2.0 * k2[o] + 2.0 * k3[o] + k4[o]);
          }
  }
  fill(y);
  return 0;
}

int chemora_oracle_rk4(int system, double* y, const int64_t* ext, int g, const double* spacing,
                       double dt, int nsteps, const double* params) {
  return chemora_oracle_rk4_order(system, y, ext, g, spacing, dt, nsteps, params, 4);
}

// Norms over the interior: out[3*v+0] = L2 = sqrt(h^3 sum f^2),
// out[3*v+1] = Linf = max |f|, out[3*v+2] = h^3 sum f; for the wave system
// out[3*n_gf] = E = h^3 sum 1/2 (rho^2 + v1^2 + v2^2 + v3^2).
// Summation order: serial within a z-plane, then planes in z order.
int chemora_oracle_norms(int system, const double* y, const int64_t* ext, int g,
                         const double* spacing, double* out) {
  const int nf = n_gf_of(system);
  if (nf < 0) return 1;
  Grid G(ext, g, spacing);
  const int64_t np = G.npad();
  const double vol = spacing[0] * spacing[1] * spacing[2];
  const int64_t nz = G.n[2];
  std::vector<double> s2(nf * nz), mx(nf * nz), s1(nf * nz), en(nz);
#pragma omp parallel for schedule(static)
  for (int64_t z = 0; z < nz; ++z) {
    for (int v = 0; v < nf; ++v) {
      double a = 0.0, m = 0.0, b = 0.0;
      for (int64_t j = 0; j < G.n[1]; ++j)
        for (int64_t i = 0; i < G.n[0]; ++i) {
          const double f = y[v * np + G.at(i, j, z)];
          a += f * f;
          b += f;
          m = std::max(m, std::fabs(f));
        }
      s2[v * nz + z] = a; mx[v * nz + z] = m; s1[v * nz + z] = b;
    }
    double e = 0.0;
    if (system == 1)
      for (int64_t j = 0; j < G.n[1]; ++j)
        for (int64_t i = 0; i < G.n[0]; ++i) {
          const int64_t c = G.at(i, j, z);
          const double r = y[np + c], a = y[2 * np + c], b = y[3 * np + c], d = y[4 * np + c];
          e += 0.5 * (r * r + a * a + b * b + d * d);
        }
    en[z] = e;
  }
  for (int v = 0; v < nf; ++v) {
    double a = 0.0, m = 0.0, b = 0.0;
    for (int64_t z = 0; z < nz; ++z) {
      a += s2[v * nz + z]; b += s1[v * nz + z]; m = std::max(m, mx[v * nz + z]);
    }
    out[3 * v + 0] = std::sqrt(vol * a);
    out[3 * v + 1] = m;
    out[3 * v + 2] = vol * b;
  }
  if (system == 1) {
    double e = 0.0;
    for (int64_t z = 0; z < nz; ++z) e += en[z];
    out[3 * nf] = vol * e;
  }
  return 0;
}

// BSSN constraint fields at interior points, ghosts of y used as they are.
// out: 7 interior arrays [H, M1, M2, M3, G1, G2, G3] (see bssn_constraints above).
int chemora_oracle_constraints(const double* y, const int64_t* ext, int g, const double* spacing,
                               double* out) {
  if (g < 3) return 2;
  Grid G(ext, g, spacing);
  bssn_constraints(y, out, G);
  return 0;
}

}  // extern "C"
