"""Narrow-phase continuous collision detection with conservative time of impact.

TEST INFRASTRUCTURE (see oracle/__init__.py).

Follows PAPER.md:464-482 (§5.3 "Narrow Phase") with the SURVEY readings Q31-Q34 and the
DESIGN.md reading R-CCD1:
 1. coplanarity cubic c(t) = det[x1(t)-x0(t), x2(t)-x0(t), x3(t)-x0(t)] for linear motion,
    on the inflated interval [-eps, 1+eps], eps = 1e-12.
 2. root finder (Yuksel-style Newton-bisection): split the interval at the
    real roots of c'(t); in the first monotone piece with a sign change run Newton with a
    bisection fallback until |dt| <= 1e-15 (<= 100 iterations); deflate
    (A=a, B=b+A t*, C=c+B t*; Q31 reading of the garbled P:466) and solve the quadratic in
    closed form; clamp roots to [0,1]; sort.
 3. activation: the first root (ascending) with d_TOC < eps + min(dhat, 1e-2 d_0), d_0 the pair's
    distance at t = 0 (PAPER.md:468 writes eps + dhat; DESIGN.md R-CCD2: with the full dhat margin a
    pair already within dhat that slides tangentially past a neighbouring primitive's plane is
    truncated to 0.9 t at every Newton iteration -- a Zeno stall observed on C1 step 3 -- while a
    genuine crossing has d_TOC = 0 up to root error either way).
 4. conservative TOI (fig:ccd_toi): reference frame t_ref = (t_prev + t)/2;
    R-CCD1: the root itself is the coplanar configuration whose signed distance is rounding
    noise, so the TOI is backtracked at least once: toi = 0.9 t, then while the signed distance
    at toi and at t_ref differ in sign (PT/EE-resolved pairs only; PP/PE lack a signed distance),
    toi <- 0.9 toi (<= 200 times, then 0); R-CCD3: if toi falls to or below the previous
    (non-contact) root t_prev, the sign can never match again, so toi = t_ref.
 5. identically-zero cubic: toi = 0.9 d(0) / (max_k |dx_k| of feature A + of feature B) (Q33).
Returns toi in [0,1] (1.0 = no collision on this step).
"""
from __future__ import annotations

import numpy as np

from .contact import PT, EE, resolve_features

EPS = 1e-12


def _cubic_coeffs(x0, dx):
    """x0, dx: (4,3) start positions and displacements; c(t) = det of edge matrix."""
    e0 = [x0[1] - x0[0], x0[2] - x0[0], x0[3] - x0[0]]
    f = [dx[1] - dx[0], dx[2] - dx[0], dx[3] - dx[0]]

    def det(a, b, c):
        return float(np.dot(a, np.cross(b, c)))

    # expand det(e1 + t f1, e2 + t f2, e3 + t f3) by multilinearity
    d = det(e0[0], e0[1], e0[2])
    c = det(f[0], e0[1], e0[2]) + det(e0[0], f[1], e0[2]) + det(e0[0], e0[1], f[2])
    b = det(f[0], f[1], e0[2]) + det(f[0], e0[1], f[2]) + det(e0[0], f[1], f[2])
    a = det(f[0], f[1], f[2])
    return a, b, c, d


def _poly(a, b, c, d, t):
    return ((a * t + b) * t + c) * t + d


def _quad_roots(A, B, C):
    if A == 0.0:
        if B == 0.0:
            return []
        return [-C / B]
    disc = B * B - 4.0 * A * C
    if disc < 0.0:
        return []
    sq = np.sqrt(disc)
    q = -0.5 * (B + (sq if B >= 0 else -sq))
    roots = [q / A]
    if q != 0.0:
        roots.append(C / q)
    return roots


def _newton_bisect(a, b, c, d, lo, hi):
    flo = _poly(a, b, c, d, lo)
    t = 0.5 * (lo + hi)
    for _ in range(100):
        ft = _poly(a, b, c, d, t)
        if ft == 0.0:
            return t
        if (ft < 0) == (flo < 0):
            lo, flo = t, ft
        else:
            hi = t
        dft = (3.0 * a * t + 2.0 * b) * t + c
        tn = t - ft / dft if dft != 0.0 else 0.5 * (lo + hi)
        if not (lo < tn < hi):
            tn = 0.5 * (lo + hi)
        if abs(tn - t) <= 1e-15:
            return tn
        t = tn
    return t


def cubic_roots(a, b, c, d, lo=-EPS, hi=1.0 + EPS):
    """Real roots of a t^3 + b t^2 + c t + d in [lo, hi], clamped to [0,1], ascending."""
    if a == 0.0:
        r = _quad_roots(b, c, d)
    else:
        crit = sorted(t for t in _quad_roots(3.0 * a, 2.0 * b, c) if lo < t < hi)
        knots = [lo] + crit + [hi]
        r = []
        for i in range(len(knots) - 1):
            l, h = knots[i], knots[i + 1]
            fl, fh = _poly(a, b, c, d, l), _poly(a, b, c, d, h)
            if fl == 0.0:
                r1 = l
            elif fh == 0.0:
                r1 = h
            elif (fl < 0) != (fh < 0):
                r1 = _newton_bisect(a, b, c, d, l, h)
            else:
                continue
            B = b + a * r1
            C = c + B * r1
            r = [r1] + _quad_roots(a, B, C)
            break
    out = sorted(min(max(t, 0.0), 1.0) for t in r if lo <= t <= hi)
    return out


def _signed_dist(ftype, P):
    if ftype == PT:
        p, a, b, c = P
        return float(np.dot(p - a, np.cross(b - a, c - a)))
    a0, a1, b0, b1 = P
    return float(np.dot(a0 - b0, np.cross(a1 - a0, b1 - b0)))


def pair_toi(ftype, x, dx, ids, dhat, d0frac=1e-2):
    """Conservative TOI of one PT or EE feature pair (role-ordered ids) moving by dx."""
    X0 = x[ids]
    DX = dx[ids]
    a, b, c, d = _cubic_coeffs(X0, DX)
    if a == 0.0 and b == 0.0 and c == 0.0 and d == 0.0:
        d0 = np.sqrt(resolve_features(x, ftype, ids[None])[0][0])
        na = 1 if ftype == PT else 2
        ma = max(np.linalg.norm(DX[k]) for k in range(na))
        mb = max(np.linalg.norm(DX[k]) for k in range(na, 4))
        if ma + mb == 0.0:
            return 1.0
        return min(1.0, 0.9 * d0 / (ma + mb))
    roots = cubic_roots(a, b, c, d)
    d0 = np.sqrt(resolve_features(x, ftype, ids[None])[0][0])
    thr = EPS + min(dhat, d0frac * d0)  # R-CCD2; d0frac = inf: P:468's literal eps + dhat
    t_prev = 0.0
    for t in roots:
        xt = x.copy()
        xt[ids] = X0 + t * DX
        D, sub, _ = resolve_features(xt, ftype, ids[None])
        if np.sqrt(D[0]) < thr:
            toi = 0.9 * t
            if sub[0] in (PT, EE):
                tref = 0.5 * (t_prev + t)
                sref = _signed_dist(ftype, X0 + tref * DX)
                n = 0
                while (_signed_dist(ftype, X0 + toi * DX) > 0) != (sref > 0):
                    toi *= 0.9
                    n += 1
                    if toi <= t_prev:  # DESIGN.md R-CCD3: crossed back over an earlier, non-contact root
                        toi = tref
                        break
                    if n >= 200:
                        toi = 0.0
                        break
            return toi
        t_prev = t
    return 1.0


def far_pairs(ftype, x, dx, pairs, dhat, d0frac=1e-2):
    """Broad-phase refinement (result-neutral; DESIGN.md R-CCD4): pairs for which pair_toi returns 1.
    The feature distance moves by at most ma + mb over the step (ma, mb = the largest displacement of
    a vertex of either primitive: every point of a primitive is a convex combination of its vertices),
    so if d(0) > ma + mb + 2 thr no root t in [0, 1] has d(t) < thr (2 thr + 1e-9 absorbs the rounding
    of the computed distances); if also 0.9 d(0) >= ma + mb the identically-zero-cubic branch returns
    min(1, 0.9 d(0) / (ma + mb)) = 1 as well."""
    D0 = np.sqrt(resolve_features(x, ftype, pairs)[0])
    na = 1 if ftype == PT else 2
    disp = np.linalg.norm(dx[pairs], axis=2)
    m = disp[:, :na].max(axis=1) + disp[:, na:].max(axis=1)
    thr = EPS + np.minimum(dhat, d0frac * D0)
    return (D0 > m + 2.0 * thr + 1e-9) & (0.9 * D0 >= m)


def step_toi(x, dx, pt, ee, dhat, d0frac=1e-2, prefilter=True):
    """alpha_CCD = min over candidate pairs of the conservative TOI (1.0 if none)."""
    tmin = 1.0
    for ftype, pairs in ((PT, pt), (EE, ee)):
        if prefilter and len(pairs):
            pairs = pairs[~far_pairs(ftype, x, dx, pairs, dhat, d0frac)]
        for ids in pairs:
            t = pair_toi(ftype, x, dx, ids, dhat, d0frac)
            if t < tmin:
                tmin = t
    return tmin
