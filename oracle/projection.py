"""PSD projection of stencil Hessians (§4.2.2).

TEST INFRASTRUCTURE (see oracle/__init__.py).

P(H) = V max(Lambda, 0) V^T on the full 3k x 3k DOF-space stencil Hessian ("projecting the local
Hessian to the closest symmetric positive semi-definite form", "eliminating negative
eigenvalues").  The per-stencil average clamped eigenvalue lambda_bar = tr P(H) / (3k) is the
stencil's contribution to Lambda (Q18).

``project_eigh`` uses LAPACK (numpy.linalg.eigh) as a library primitive; ``project_jacobi`` is a
plain cyclic Jacobi used only to cross-check it in the tests.
"""
from __future__ import annotations

import numpy as np


def project_eigh(H):
    """H: (B, n, n) symmetric -> (P(H) (B,n,n) exactly symmetric, clamped eigenvalues (B,n))."""
    H = 0.5 * (H + np.transpose(H, (0, 2, 1)))
    w, V = np.linalg.eigh(H)
    wc = np.maximum(w, 0.0)
    P = np.einsum("bij,bj,bkj->bik", V, wc, V)
    P = 0.5 * (P + np.transpose(P, (0, 2, 1)))
    return P, wc


def lambda_bar(P):
    """Average clamped eigenvalue per stencil = tr P(H) / n."""
    return np.trace(P, axis1=1, axis2=2) / P.shape[1]


def project_jacobi(H, tol=1e-15, max_sweeps=100):
    """Cyclic Jacobi eigen-decomposition of one symmetric matrix, then clamp (cross-check only)."""
    A = 0.5 * (np.array(H, dtype=np.float64) + np.array(H, dtype=np.float64).T)
    n = A.shape[0]
    V = np.eye(n)
    fro = np.linalg.norm(A)
    for _ in range(max_sweeps):
        off = np.sqrt(np.sum((A - np.diag(np.diag(A))) ** 2))
        if off <= tol * fro:
            break
        for p in range(n - 1):
            for q in range(p + 1, n):
                if A[p, q] == 0.0:
                    continue
                theta = (A[q, q] - A[p, p]) / (2.0 * A[p, q])
                t = np.sign(theta) / (abs(theta) + np.sqrt(theta * theta + 1.0)) if theta != 0 else 1.0
                c = 1.0 / np.sqrt(t * t + 1.0)
                s = t * c
                J = np.eye(n)
                J[p, p] = c
                J[q, q] = c
                J[p, q] = s
                J[q, p] = -s
                A = J.T @ A @ J
                V = V @ J
    w = np.diag(A)
    P = (V * np.maximum(w, 0.0)) @ V.T
    return 0.5 * (P + P.T), np.maximum(w, 0.0)
