"""Energies of the Incremental Potential and the barrier-augmented Lagrangian terms.

TEST INFRASTRUCTURE (see oracle/__init__.py).

Inertia   E_I = sum_j m_j ||x_j - y_j||^2 / (2 h^2)           PAPER.md:143 (§3.1)
Elastic   Psi = sum_e V_e [mu/2 (tr F^T F - 3) - mu ln J + lam/2 (ln J)^2],  F = D_s D_m^{-1}
          (+inf if J <= 0)                                      SURVEY Q1 reading of "Neo-Hookean"
          ARAP tets (NEXT-4; DESIGN.md R-ARAP): Psi = mu ||F - R||_F^2, R the rotation of
          the polar decomposition F = R S, = mu (tr F^T F - 2 tr S + 3); tr S = sigma_1 + sigma_2 +
          sigma_3 is the largest root of s^4 - 2 I1 s^2 - 8 J s + I1^2 - 4 I2 = 0 (I1 = tr C, I2 = the
          second invariant of C = F^T F, J = det F), reached by Newton in AD arithmetic (+inf if J <= 0)
Barrier   b(d, dhat) = -(d - dhat)^2 ln(d / dhat) for 0 < d < dhat, else 0
                                                                PAPER.md:193-200 (eq:IPC-barrier)
Mollifier f(y) = -y^3/(3 eps^2) + y^2/eps (y < eps), y - eps/3 (y >= eps), eps = eps_v h
                                                                PAPER.md:339-340 (§4.1), SURVEY Q24
Derivatives of Psi come from oracle.ad (forward-mode second-order AD), never from closed forms.
"""
from __future__ import annotations

import numpy as np

from .ad import D2


# ---------------------------------------------------------------------------
# inertia
# ---------------------------------------------------------------------------
def inertia_energy(x, y, mass, h, free):
    dx = (x - y)[free]
    return float(np.sum(mass[free] * np.einsum("ij,ij->i", dx, dx)) / (2.0 * h * h))


def inertia_grad(x, y, mass, h, free):
    g = (mass[:, None] * (x - y)) / (h * h)
    g[~free] = 0.0
    return g


# ---------------------------------------------------------------------------
# Neo-Hookean
# ---------------------------------------------------------------------------
def _nh_psi_ad(xs, Dm_inv, vol, mu, lam):
    """xs: 12 D2 variables (node-major xyz); returns D2 of V * Psi."""
    p = [xs[3 * k:3 * k + 3] for k in range(4)]
    Ds = [[p[c + 1][r] - p[0][r] for c in range(3)] for r in range(3)]  # Ds[r][c]
    F = [[Ds[r][0] * Dm_inv[:, 0, c] + Ds[r][1] * Dm_inv[:, 1, c] + Ds[r][2] * Dm_inv[:, 2, c]
          for c in range(3)] for r in range(3)]
    J = (F[0][0] * (F[1][1] * F[2][2] - F[1][2] * F[2][1])
         - F[0][1] * (F[1][0] * F[2][2] - F[1][2] * F[2][0])
         + F[0][2] * (F[1][0] * F[2][1] - F[1][1] * F[2][0]))
    Ic = None
    for r in range(3):
        for c in range(3):
            t = F[r][c] * F[r][c]
            Ic = t if Ic is None else Ic + t
    lnJ = J.log()
    psi = (Ic - 3.0) * (mu / 2.0) - lnJ * mu + lnJ * lnJ * (lam / 2.0)
    return psi * vol


def _arap_psi_ad(xs, Dm_inv, vol, mu, newton=4):
    """xs: 12 D2 variables; returns D2 of V * mu ||F - R||^2 = V mu (I1 - 2 tr S + 3)."""
    p = [xs[3 * k:3 * k + 3] for k in range(4)]
    Ds = [[p[c + 1][r] - p[0][r] for c in range(3)] for r in range(3)]
    F = [[Ds[r][0] * Dm_inv[:, 0, c] + Ds[r][1] * Dm_inv[:, 1, c] + Ds[r][2] * Dm_inv[:, 2, c]
          for c in range(3)] for r in range(3)]
    J = (F[0][0] * (F[1][1] * F[2][2] - F[1][2] * F[2][1])
         - F[0][1] * (F[1][0] * F[2][2] - F[1][2] * F[2][0])
         + F[0][2] * (F[1][0] * F[2][1] - F[1][1] * F[2][0]))
    # C = F^T F, I1 = tr C, I2 = (I1^2 - tr C^2) / 2
    Cm = [[F[0][i] * F[0][j] + F[1][i] * F[1][j] + F[2][i] * F[2][j] for j in range(3)] for i in range(3)]
    I1 = Cm[0][0] + Cm[1][1] + Cm[2][2]
    trC2 = None
    for i in range(3):
        for j in range(3):
            t = Cm[i][j] * Cm[j][i]
            trC2 = t if trC2 is None else trC2 + t
    I2 = (I1 * I1 - trC2) * 0.5
    # tr S: start from the sum of singular values of the values, then Newton on the quartic in AD
    Fv = np.stack([np.stack([F[r][c].v for c in range(3)], -1) for r in range(3)], -2)
    s = J.const_like(np.linalg.svd(Fv, compute_uv=False).sum(axis=-1))
    for _ in range(newton):
        s2 = s * s
        f = s2 * s2 - I1 * s2 * 2.0 - J * s * 8.0 + I1 * I1 - I2 * 4.0
        fp = s2 * s * 4.0 - I1 * s * 4.0 - J * 8.0
        s = s - f / fp
    psi = (I1 - s * 2.0 + 3.0) * mu + J.log() * 0.0  # + 0 * ln J: nan (infeasible) when J <= 0
    return psi * vol


def nh_stencils(x, mesh, chunk=20000):
    """Per-tet AD value, gradient (T,12) and Hessian (T,12,12) of V_e Psi_e (no projection): Neo-Hookean,
    or ARAP for the tets mesh.arap marks.  Tets with J <= 0 give nan (the caller treats the energy as +inf)."""
    T = len(mesh.tets)
    val = np.empty(T)
    grad = np.empty((T, 12))
    hess = np.empty((T, 12, 12))
    arap = mesh.arap if mesh.arap is not None else np.zeros(T, bool)
    if len(arap) != T:
        raise ValueError("mesh.arap must have one entry per tet (subset it with the tets)")
    for model in (False, True):
        idx = np.nonzero(arap == model)[0]
        for s in range(0, len(idx), chunk):
            e = idx[s:s + chunk]
            xs = x[mesh.tets[e]].reshape(-1, 12)
            with np.errstate(invalid="ignore", divide="ignore"):
                if model:
                    r = _arap_psi_ad(D2.variables(xs), mesh.Dm_inv[e], mesh.vol[e], mesh.mu[e])
                else:
                    r = _nh_psi_ad(D2.variables(xs), mesh.Dm_inv[e], mesh.vol[e], mesh.mu[e], mesh.lam[e])
            val[e], grad[e], hess[e] = r.v, r.g, r.H
    return val, grad, hess


def nh_energy(x, mesh):
    """Plain (non-AD) evaluation of sum_e V_e Psi_e; +inf if any J <= 0."""
    t = mesh.tets
    Ds = np.stack([x[t[:, 1]] - x[t[:, 0]], x[t[:, 2]] - x[t[:, 0]], x[t[:, 3]] - x[t[:, 0]]], axis=2)
    F = Ds @ mesh.Dm_inv
    J = np.linalg.det(F)
    if np.any(J <= 0) or np.any(~np.isfinite(J)):
        return np.inf
    Ic = np.einsum("eij,eij->e", F, F)
    lnJ = np.log(J)
    psi = mesh.mu / 2 * (Ic - 3.0) - mesh.mu * lnJ + mesh.lam / 2 * lnJ ** 2
    if mesh.arap is not None and np.any(mesh.arap):
        a = mesh.arap
        trS = np.linalg.svd(F[a], compute_uv=False).sum(axis=-1)  # J > 0: tr S = sum of singular values
        psi[a] = mesh.mu[a] * (Ic[a] - 2.0 * trS + 3.0)
    return float(np.sum(mesh.vol * psi))


def nh_min_J(x, mesh):
    t = mesh.tets
    Ds = np.stack([x[t[:, 1]] - x[t[:, 0]], x[t[:, 2]] - x[t[:, 0]], x[t[:, 3]] - x[t[:, 0]]], axis=2)
    return float(np.min(np.linalg.det(Ds @ mesh.Dm_inv))) if len(t) else np.inf


# ---------------------------------------------------------------------------
# barrier
# ---------------------------------------------------------------------------
def barrier(d, dhat):
    """b(d, dhat) elementwise; d must be > 0 (the caller handles d <= 0 as infeasible)."""
    d = np.asarray(d, np.float64)
    dhat = np.broadcast_to(np.asarray(dhat, np.float64), d.shape)
    out = np.zeros_like(d)
    m = d < dhat
    out[m] = -((d[m] - dhat[m]) ** 2) * np.log(d[m] / dhat[m])
    return out


def barrier_ad(d: D2, dhat):
    """b(d, dhat) as a D2 (d a D2); zero where d >= dhat."""
    dhat = np.broadcast_to(np.asarray(dhat, np.float64), d.v.shape)
    m = d.v < dhat
    safe_v = np.where(m, d.v, dhat * 0.5)  # avoid log of garbage in the masked-out lanes
    ds = D2(safe_v, d.g, d.H)
    diff = ds - dhat
    b = -(diff * diff) * (ds * (1.0 / dhat)).log()
    zero = d.const_like(0.0)
    return b.select(m, zero)


# ---------------------------------------------------------------------------
# friction mollifier
# ---------------------------------------------------------------------------
def mollifier(y, eps):
    y = np.asarray(y, np.float64)
    return np.where(y < eps, -(y ** 3) / (3 * eps * eps) + y * y / eps, y - eps / 3.0)


def mollifier_of_sq_ad(q: D2, eps):
    """f(sqrt(q)) as a D2 of q = ||w||^2.  At q == 0 exactly the cubic term has zero value,
    gradient and Hessian, so f = q/eps there (exact, avoids 0*inf from sqrt)."""
    zero_mask = q.v <= 0.0
    qs = D2(np.where(zero_mask, 1.0, q.v), q.g, q.H)
    y = qs.sqrt()
    cubic = -(y * qs) * (1.0 / (3 * eps * eps)) + qs * (1.0 / eps)
    lin = y - eps / 3.0
    smooth = cubic.select(y.v < eps, lin)
    at0 = q * (1.0 / eps)
    return at0.select(zero_mask, smooth)
