"""Exact vacuum solutions used to pin the BSSN oracle.

Pure-gauge Minkowski: flat spacetime in coordinates X^a = x^a + eps xi^a(t, x, y, z).  The
ADM data are obtained from g_{mu nu} = eta_{ab} dX^a/dx^mu dX^b/dx^nu with exact (sympy)
derivatives of xi, converted to BSSN variables with the standard definitions
(phi = ln det(gamma)/12, gt = det^-1/3 gamma, At = det^-1/3 (K_ij - gamma_ij K/3),
Xt^i = gt^jk Gt^i_jk), and the time derivatives of the BSSN variables are taken by a
5-point central difference in t.  Nothing here shares code with oracle/.
"""
from __future__ import annotations

import functools

import numpy as np
import sympy as sp

EPS = 0.1


@functools.lru_cache(maxsize=None)
def _xi_functions():
    t, x, y, z = sp.symbols("t x y z")
    X = (t, x, y, z)
    xi = [sp.Rational(1, 2) * sp.sin(x + 2 * y) * sp.cos(t),
          sp.sin(y - z + t) * sp.cos(x),
          sp.cos(z + x) * sp.sin(2 * t + y),
          sp.sin(x + y + z - t)]
    d1 = [[sp.lambdify(X, sp.diff(xi[a], X[m]), "numpy") for m in range(4)] for a in range(4)]
    d2 = [[[sp.lambdify(X, sp.diff(xi[a], X[m], X[n]), "numpy") for n in range(4)] for m in range(4)]
          for a in range(4)]
    return d1, d2


def _bcast(v, shape):
    return np.broadcast_to(np.asarray(v, dtype=float), shape)


def adm_data(t, x, y, z):
    """gamma_ij, d_k gamma_ij, d_t gamma_ij, beta_i (lower), d_k beta_i, g00 on arrays."""
    d1, d2 = _xi_functions()
    shape = np.broadcast(x, y, z).shape
    eta = np.diag([-1.0, 1.0, 1.0, 1.0])
    J = np.zeros((4, 4) + shape)      # J[a][mu] = dX^a/dx^mu
    dJ = np.zeros((4, 4, 4) + shape)  # dJ[k][a][mu] = d_k J[a][mu], k over (t,x,y,z)
    for a in range(4):
        for m in range(4):
            J[a, m] = (1.0 if a == m else 0.0) + EPS * _bcast(d1[a][m](t, x, y, z), shape)
            for k in range(4):
                dJ[k, a, m] = EPS * _bcast(d2[a][m][k](t, x, y, z), shape)
    g = np.einsum("ab,am...,bn...->mn...", eta, J, J)
    dg = np.einsum("ab,kam...,bn...->kmn...", eta, dJ, J) + np.einsum("ab,am...,kbn...->kmn...", eta, J, dJ)
    gam = g[1:, 1:]
    dgam = dg[1:, 1:, 1:]      # [k][i][j], spatial k
    dtgam = dg[0, 1:, 1:]
    beta_l = g[0, 1:]
    dbeta_l = dg[1:, 0, 1:]    # [k][i]
    return gam, dgam, dtgam, beta_l, dbeta_l, g[0, 0]


def _mat_last(a):
    """[3][3][...] -> [...][3][3]"""
    return np.moveaxis(np.moveaxis(a, 0, -1), 0, -1)


def _mat_first(a):
    return np.moveaxis(np.moveaxis(a, -1, 0), -1, 0)


def bssn_vars(t, x, y, z):
    """Dict of the 17 ADM-part BSSN variables plus alpha and beta^i at time t."""
    gam, dgam, dtgam, beta_l, dbeta_l, g00 = adm_data(t, x, y, z)
    G = _mat_last(gam)
    Gi = np.linalg.inv(G)
    gu = _mat_first(Gi)                          # gamma^ij
    det = np.linalg.det(G)
    beta_u = np.einsum("ij...,j...->i...", gu, beta_l)
    alpha = np.sqrt(np.einsum("i...,i...->...", beta_l, beta_u) - g00)
    # Christoffel Gamma^k_ij = 1/2 g^kl (d_i g_lj + d_j g_li - d_l g_ij)
    low = 0.5 * (np.einsum("ilj...->lij...", dgam) + np.einsum("jli...->lij...", dgam) - dgam)
    # low[l][i][j] = 1/2 (d_i g_lj + d_j g_li - d_l g_ij)
    Gam = np.einsum("kl...,lij...->kij...", gu, low)
    Dbeta = dbeta_l - np.einsum("kij...,k...->ij...", Gam, beta_l)   # D_i beta_j, [i][j]
    K = (-dtgam + Dbeta + np.einsum("ij...->ji...", Dbeta)) / (2 * alpha)
    trK = np.einsum("ij...,ij...->...", gu, K)
    w = det ** (-1.0 / 3.0)
    gt = w * gam
    At = w * (K - gam * trK / 3.0)
    # d_k gt_ij = w (d_k g_ij - g_ij d_k ln det / 3), d_k ln det = g^lm d_k g_lm
    dlndet = np.einsum("lm...,klm...->k...", gu, dgam)
    dgt = w * (dgam - gam[None] * dlndet[:, None, None] / 3.0)
    gtu = gu / w
    lowt = 0.5 * (np.einsum("ilj...->lij...", dgt) + np.einsum("jli...->lij...", dgt) - dgt)
    Gamt = np.einsum("kl...,lij...->kij...", gtu, lowt)
    Xt = np.einsum("ij...,kij...->k...", gtu, Gamt)
    out = {"phi": np.log(det) / 12.0, "trK": trK, "alpha": alpha}
    names = ["11", "12", "13", "22", "23", "33"]
    idx = [(0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2)]
    for nm, (i, j) in zip(names, idx):
        out["gt" + nm] = gt[i, j]
        out["At" + nm] = At[i, j]
    for i in range(3):
        out[f"Xt{i + 1}"] = Xt[i]
        out[f"beta{i + 1}"] = beta_u[i]
    return out


ADM_PART = ["phi", "gt11", "gt12", "gt13", "gt22", "gt23", "gt33", "trK", "At11", "At12", "At13",
            "At22", "At23", "At33", "Xt1", "Xt2", "Xt3"]


def bssn_time_derivative(t, x, y, z, delta=1e-3):
    """5-point central difference in t of the BSSN variables (error ~ delta^4)."""
    f = {s: bssn_vars(t + s * delta, x, y, z) for s in (-2, -1, 1, 2)}
    return {k: (f[-2][k] - 8 * f[-1][k] + 8 * f[1][k] - f[2][k]) / (12 * delta) for k in ADM_PART}
