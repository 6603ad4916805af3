"""Elementwise rules of the barrier-augmented Lagrangian loop (Alg. 1).

TEST INFRASTRUCTURE (see oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np

from .energy import barrier


def slack(mu, sigma, dhat, d):
    """s_i = max{-mu_i/sigma - dhat + d_i(x), 0}   (§3.2.2)."""
    return np.maximum(-np.asarray(mu) / sigma - dhat + np.asarray(d), 0.0)


def dual_update(mu, sigma, dhat, s, d):
    """mu_i <- mu_i + sigma b(d_i; dhat + s_i)   (Alg. 1 line 14; Q12 verbatim)."""
    return np.asarray(mu) + sigma * barrier(d, dhat + np.asarray(s))


def sigma_ls(gb, gE):
    """Least-squares sigma: -(gb . gE)/||gb||^2 (PAPER.md:285-289 with the squared norm, Q7).
    Returns None when gb = 0."""
    bb = float(np.dot(gb, gb))
    if bb == 0.0:
        return None
    return -float(np.dot(gb, gE)) / bb


def sigma_schedule(sigma, sigma0, dmin_new, dhat, cap=False, use_min=False):
    """sigma <- max(1.2 sigma, 100 sigma0) if min d(x^{l+1}) < 1e-2 dhat (Alg. 1 lines 15-16, Q8).
    cap=True: the NEXT-1 sigma-cap reading, an overall ceiling of 1e8 sigma0.
    use_min=True: min(1.2 sigma, 100 sigma0), capped growth (the SURVEY Q8 alternative)."""
    if dmin_new < 1e-2 * dhat:
        s = min(1.2 * sigma, 100.0 * sigma0) if use_min else max(1.2 * sigma, 100.0 * sigma0)
        return min(s, 1e8 * sigma0) if cap else s
    return sigma


def aprime_rule(dmin, dmin_prev, aprime_empty, dhat):
    """Alg. 1 lines 3-6: 'clear' if min d > 1e-2 dhat; 'rebuild' if min d decreased or A' empty;
    else 'keep'."""
    if dmin > 1e-2 * dhat:
        return "clear"
    if dmin < dmin_prev or aprime_empty:
        return "rebuild"
    return "keep"
