"""Independent continuum evaluation of the BSSN right-hand side and constraints at a point
(test infrastructure for the oracle pins; shares nothing with oracle/ or the CUDA path).

The oracle's RHS of polynomial data of degree <= 4 (ghosts = the polynomial's values,
HOST_PADDED) equals the CONTINUUM right-hand side of SURVEY.md App. A at every interior
point up to rounding, because every stencil it applies (centered D1, D2, mixed D1 x D1,
lopsided upwind) is exact on such polynomials (pinned separately).  This
module computes that continuum value by a different route from the oracle's index-loop
transcription:

* every field is carried as a second-order jet (value, gradient, Hessian) obtained exactly
  from its polynomial, and all algebra is jet arithmetic (product / quotient / exp rules),
  so derivatives of composite quantities (inverse metrics, Christoffel symbols) are
  differentiated exactly instead of being assembled from App. A's expanded formulas;
* the curvature comes from first principles: the Ricci tensor of the PHYSICAL metric
  gamma_ij = e^{4 phi} gt_ij from its own Christoffel symbols,
      R_ij = d_k G^k_ij - d_j G^k_ik + G^k_kl G^l_ij - G^k_jl G^l_ik,
  plus the one place where the BSSN Ricci tensor deliberately differs from it -- the
  evolved Xt^k replaces gt^jk Gt^k_jk under the derivative (App. A.2, R8):
      R^BSSN_ij = R_ij[gamma] + 1/2 (gt_ki d_j D^k + gt_kj d_i D^k),   D^k = Xt^k - Xtn^k
  (the identity R~_ij[gt] = -1/2 gt^lm d_l d_m gt_ij + gt_k(i d_j) Xtn^k + ... holds for any
  metric, and the conformal split R = R~ + R^phi for any conformal factor);
* D_i D_j alpha from the physical Christoffel symbols; traces with the physical inverse
  metric; Lie derivatives of the tensor densities gt (weight -2/3) and At by the general
  formula L_b T_ij = b^k d_k T_ij + T_kj d_i b^k + T_ik d_j b^k;
* the Gamma-tilde equation, the constraints' divergence D~_j At^ij (with the full
  conformal Christoffel symbols, det gt not assumed 1) and the gauge equations are App. A.3
  as printed in SURVEY.md, written in tensor notation over these objects.

Only plain numpy; index conventions: t[i][j] full 3x3 (symmetric where the field is).
"""
from __future__ import annotations

import math

import numpy as np

NAN3 = np.full((3, 3), np.nan)


class Jet:
    """f(p + d) = v + g.d + 1/2 d.H.d + O(|d|^3).  A derivative of a jet is a first-order
    jet (H unknown = NaN), which is all the first-principles formulas need."""
    __slots__ = ("v", "g", "H")

    def __init__(self, v, g=None, H=None):
        self.v = float(v)
        self.g = np.zeros(3) if g is None else np.asarray(g, dtype=np.float64)
        self.H = np.zeros((3, 3)) if H is None else np.asarray(H, dtype=np.float64)

    @staticmethod
    def c(v):
        return Jet(v)

    def __add__(self, o):
        o = o if isinstance(o, Jet) else Jet(o)
        return Jet(self.v + o.v, self.g + o.g, self.H + o.H)
    __radd__ = __add__

    def __neg__(self):
        return Jet(-self.v, -self.g, -self.H)

    def __sub__(self, o):
        return self + (-(o if isinstance(o, Jet) else Jet(o)))

    def __rsub__(self, o):
        return Jet(o) - self

    def __mul__(self, o):
        if not isinstance(o, Jet):
            return Jet(self.v * o, self.g * o, self.H * o)
        return Jet(self.v * o.v, self.g * o.v + self.v * o.g,
                   self.H * o.v + self.v * o.H + np.outer(self.g, o.g) + np.outer(o.g, self.g))
    __rmul__ = __mul__

    def recip(self):
        v = 1.0 / self.v
        return Jet(v, -self.g * v * v, -self.H * v * v + 2.0 * np.outer(self.g, self.g) * v ** 3)

    def __truediv__(self, o):
        return self * (o.recip() if isinstance(o, Jet) else 1.0 / o)

    def d(self, i):
        """Partial derivative along axis i (a first-order jet)."""
        return Jet(self.g[i], self.H[i], NAN3)


def jexp(a: Jet) -> Jet:
    e = math.exp(a.v)
    return Jet(e, e * a.g, e * (a.H + np.outer(a.g, a.g)))


def jpow(a: Jet, p: float) -> Jet:
    v = a.v ** p
    return Jet(v, p * a.v ** (p - 1) * a.g,
               p * a.v ** (p - 1) * a.H + p * (p - 1) * a.v ** (p - 2) * np.outer(a.g, a.g))


def poly_jet(coeffs, p, scale=1.0, base=0.0) -> Jet:
    """Jet of base + scale * sum c_abc x^a y^b z^c at the point p (exact)."""
    x = p
    v, g, H = 0.0, np.zeros(3), np.zeros((3, 3))
    for (a, b, c), w in coeffs.items():
        e = (a, b, c)

        def mono(e2):
            if min(e2) < 0:
                return 0.0
            return x[0] ** e2[0] * x[1] ** e2[1] * x[2] ** e2[2]
        v += w * mono(e)
        for i in range(3):
            ei = list(e)
            ei[i] -= 1
            g[i] += w * e[i] * mono(ei)
            for j in range(3):
                eij = list(ei)
                eij[j] -= 1
                f = e[i] * (e[j] - (1 if i == j else 0))
                H[i, j] += w * f * mono(eij)
    return Jet(base + scale * v, scale * g, scale * H)


def inverse3(m):
    """Inverse of a symmetric 3x3 matrix of jets via the adjugate (jet arithmetic)."""
    cof = [[None] * 3 for _ in range(3)]
    for i in range(3):
        for j in range(3):
            r = [k for k in range(3) if k != i]
            c = [k for k in range(3) if k != j]
            minor = m[r[0]][c[0]] * m[r[1]][c[1]] - m[r[0]][c[1]] * m[r[1]][c[0]]
            cof[i][j] = minor if (i + j) % 2 == 0 else -minor
    det = m[0][0] * cof[0][0] + m[0][1] * cof[0][1] + m[0][2] * cof[0][2]
    idet = det.recip()
    return [[cof[j][i] * idet for j in range(3)] for i in range(3)], det


def christoffel(m, minv):
    """G[k][i][j] = 1/2 m^kl (d_i m_lj + d_j m_il - d_l m_ij)  (first-order jets)."""
    dm = [[[m[a][b].d(l) for b in range(3)] for a in range(3)] for l in range(3)]  # dm[l][a][b]
    G = [[[None] * 3 for _ in range(3)] for _ in range(3)]
    for k in range(3):
        for i in range(3):
            for j in range(3):
                s = Jet(0.0)
                for l in range(3):
                    s = s + minv[k][l] * (dm[i][l][j] + dm[j][i][l] - dm[l][i][j])
                G[k][i][j] = 0.5 * s
    return G


def ricci(G):
    """R_ij = d_k G^k_ij - d_j G^k_ik + G^k_kl G^l_ij - G^k_jl G^l_ik (values)."""
    R = np.zeros((3, 3))
    for i in range(3):
        for j in range(3):
            r = 0.0
            for k in range(3):
                r += G[k][i][j].g[k] - G[k][i][k].g[j]
                for l in range(3):
                    r += G[k][k][l].v * G[l][i][j].v - G[k][j][l].v * G[l][i][k].v
            R[i, j] = r
    return R


SYM = ((0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2))


def sym_full(vals):
    """6 packed (xx, xy, xz, yy, yz, zz) -> full 3x3 list."""
    t = [[None] * 3 for _ in range(3)]
    for s, (i, j) in enumerate(SYM):
        t[i][j] = vals[s]
        t[j][i] = vals[s]
    return t


def fields_at(polys, scales, bases, p):
    """Jets of the 25 App. A variables at point p (order phi, gt6, K, At6, Xt3, alpha, A,
    beta3, B3)."""
    return [poly_jet(polys[v], p, scales[v], bases[v]) for v in range(25)]


def bssn_rhs_and_constraints(J, prm):
    """Continuum App. A.3 right-hand sides (25) and the constraints [H, M1..3, G1..3] at a
    point, from the jets J of the 25 variables.  prm = (F_alpha, n_alpha, L, eta_alpha,
    c_alpha_adv, C_beta, p_beta, S_B, eta, c_beta_adv)."""
    Fa, na, Lg, eta_a, ca, Cb, pb, SB, eta, cb = prm
    phi = J[0]
    gt = sym_full(J[1:7])
    K = J[7]
    At = sym_full(J[8:14])
    Xt = J[14:17]
    alpha, Aux = J[17], J[18]
    beta, B = J[19:22], J[22:25]
    val = lambda t: np.array([[t[i][j].v for j in range(3)] for i in range(3)])

    # physical metric, its inverse and Christoffels; Ricci from first principles
    e4 = jexp(4.0 * phi)
    gam = [[e4 * gt[i][j] for j in range(3)] for i in range(3)]
    gaminv, _ = inverse3(gam)
    Gp = christoffel(gam, gaminv)
    Rphys = ricci(Gp)
    # conformal metric: inverse, Christoffels, contracted Xtn, D = Xt - Xtn
    gtinv, _ = inverse3(gt)
    Gc = christoffel(gt, gtinv)
    Xtn = []
    for k in range(3):
        s = Jet(0.0)
        for i in range(3):
            for j in range(3):
                s = s + gtinv[i][j] * Gc[k][i][j]
        Xtn.append(s)
    Dk = [Xt[k] - Xtn[k] for k in range(3)]      # first-order jets
    gtv, gtiv, Atv = val(gt), val(gtinv), val(At)
    R = Rphys.copy()
    for i in range(3):
        for j in range(3):
            for k in range(3):
                R[i, j] += 0.5 * (gtv[k, i] * Dk[k].g[j] + gtv[k, j] * Dk[k].g[i])
    # D_i D_j alpha with the physical Christoffels
    da = alpha.g
    DDa = alpha.H - np.einsum("kij,k->ij", np.array([[[Gp[k][i][j].v for j in range(3)] for i in range(3)]
                                                      for k in range(3)]), da)
    gaminv_v = val(gaminv)
    trDDa = np.sum(gaminv_v * DDa)
    # At with raised indices
    Au = gtiv @ Atv @ gtiv
    Am = gtiv @ Atv                                  # At^i_j
    AA = np.sum(Atv * Au)
    db = np.array([[beta[k].g[l] for k in range(3)] for l in range(3)])   # db[l][k] = d_l beta^k
    divb = np.trace(db)
    a, Kv = alpha.v, K.v
    adv = lambda f: sum(beta[k].v * f.g[k] for k in range(3))

    def lie(T):  # L_beta T_ij for a covariant 2-tensor (values)
        Tv = val(T)
        out = np.zeros((3, 3))
        for i in range(3):
            for j in range(3):
                out[i, j] = adv(T[i][j]) + sum(Tv[k, j] * db[i, k] + Tv[i, k] * db[j, k] for k in range(3))
        return out

    rhs = np.zeros(25)
    rhs[0] = -a * Kv / 6.0 + divb / 6.0 + adv(phi)
    dgt = -2.0 * a * Atv + lie(gt) - (2.0 / 3.0) * gtv * divb
    rhs_K = -trDDa + a * (AA + Kv * Kv / 3.0) + adv(K)
    X = -DDa + a * R
    trX = np.sum(gtiv * X)
    e4m = math.exp(-4.0 * phi.v)
    dAt = e4m * (X - gtv * trX / 3.0) + a * (Kv * Atv - 2.0 * Atv @ Am) + lie(At) - (2.0 / 3.0) * Atv * divb
    for s, (i, j) in enumerate(SYM):
        rhs[1 + s] = dgt[i, j]
        rhs[8 + s] = dAt[i, j]
    rhs[7] = rhs_K
    # Gamma-tilde equation (App. A.3)
    Gcv = np.array([[[Gc[k][i][j].v for j in range(3)] for i in range(3)] for k in range(3)])
    Xtnv = np.array([x.v for x in Xtn])
    ddb = np.array([[[beta[i].H[j, k] for k in range(3)] for j in range(3)] for i in range(3)])  # d_j d_k beta^i
    dphi, dK = phi.g, K.g
    ddivb = np.array([sum(ddb[k][j][k] for k in range(3)) for j in range(3)])
    rhs_Xt = np.zeros(3)
    for i in range(3):
        r = np.sum(gtiv * ddb[i]) + (gtiv[i] @ ddivb) / 3.0
        r += -sum(Xtnv[j] * db[j, i] for j in range(3)) + (2.0 / 3.0) * Xtnv[i] * divb
        r += -2.0 * sum(Au[i, j] * da[j] for j in range(3))
        r += 2.0 * a * (np.sum(Gcv[i] * Au) + 6.0 * Au[i] @ dphi - (2.0 / 3.0) * gtiv[i] @ dK)
        rhs_Xt[i] = r + adv(Xt[i])
        rhs[14 + i] = rhs_Xt[i]
    # gauge (App. A.3)
    rhs[17] = -Fa * a ** na * (Lg * Aux.v + (1.0 - Lg) * Kv) + ca * adv(alpha)
    rhs[18] = Lg * (rhs_K - eta_a * Aux.v) + ca * adv(Aux)
    for i in range(3):
        rhs[19 + i] = Cb * a ** pb * (SB * B[i].v + (1.0 - SB) * (Xt[i].v - eta * beta[i].v)) + cb * adv(beta[i])
        rhs[22 + i] = SB * (rhs_Xt[i] - eta * B[i].v) + cb * (adv(B[i]) - adv(Xt[i]))

    # constraints: H from the physical Ricci scalar, M^i = D~_j At^ij + ..., G^i = Xt^i - Xtn^i
    Rs = np.sum(gaminv_v * Rphys) + e4m * sum(Dk[k].g[k] for k in range(3))
    H = Rs + (2.0 / 3.0) * Kv * Kv - AA
    Auj = [[sum((gtinv[i][k] * gtinv[j][l]) * At[k][l] for k in range(3) for l in range(3))
            for j in range(3)] for i in range(3)]   # At^ij as jets
    M = np.zeros(3)
    for i in range(3):
        div = sum(Auj[i][j].g[j] for j in range(3))
        div += np.sum(Gcv[i] * Au)                                    # Gt^i_jk At^kj
        div += sum(Gcv[j, j, k] * Au[i, k] for j in range(3) for k in range(3))  # Gt^j_jk At^ik
        M[i] = div + 6.0 * Au[i] @ dphi - (2.0 / 3.0) * gtiv[i] @ dK
    G = np.array([Xt[i].v - Xtnv[i] for i in range(3)])
    return rhs, np.concatenate([[H], M, G])
