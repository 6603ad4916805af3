"""Contact: primitive distances and their type resolution, constraint keys, broad phase,
contact potentials phi and friction stencils.

TEST INFRASTRUCTURE (see oracle/__init__.py).

Constraint model (PAPER.md:147-156 eq:problem, 193-211 eq:aug-lag):
 - feature pairs: every surface vertex p vs every surface triangle (p not in it), and every pair
   of surface edges sharing no node; pairs whose nodes are all fixed are skipped (Q29).
 - d = Euclidean distance between the two features (Q2), resolved to one of
   PP (point-point), PE (point-edge), PT (point-triangle interior), EE (edge-edge interior) (Q27):
     PT interior iff the projected barycentrics are all >= 0; else min over 3 point-segments.
     EE interior iff both closest-point parameters are in [0,1] and
       ||ea x eb||^2 > 1e-10 ||ea||^2 ||eb||^2 (DESIGN.md R-EE1); else min over 4 point-segments.
     point-segment: t = (p-a).(b-a)/|b-a|^2; t < 0 -> PP(p,a); t > 1 -> PP(p,b); else PE.
     Ties go to the higher-dimensional feature, then the lowest local index.
 - a constraint is identified by its key (type, canonical node ids); duplicates reached from
   several feature pairs count once (Q28).
 - stencil potential phi(d) = [i in A] sigma b(d; dhat) + [i in A'] (mu (dhat + s - d) + sigma b(d; dhat + s))
   (eq:aug-lag with R(x) of PAPER.md:210), projected once per stencil (Q22).
"""
from __future__ import annotations

import numpy as np

from .ad import D2
from .energy import barrier, barrier_ad

PP, PE, PT, EE = 0, 1, 2, 3
NNODES = {PP: 2, PE: 3, PT: 4, EE: 4}


# ---------------------------------------------------------------------------
# type resolution (plain numpy, vectorised over pairs)
# ---------------------------------------------------------------------------
def _dot(a, b):
    return np.einsum("ij,ij->i", a, b)


def _point_segment(p, a, b):
    """Returns (D squared distance, type, t clamp-param, which-end (0=a,1=b) for PP)."""
    e = b - a
    ee = _dot(e, e)
    t = _dot(p - a, e) / ee
    D_pe = _dot(np.cross(a - p, b - p), np.cross(a - p, b - p)) / ee
    D_a = _dot(p - a, p - a)
    D_b = _dot(p - b, p - b)
    typ = np.where((t >= 0) & (t <= 1), PE, PP)
    D = np.where(t < 0, D_a, np.where(t > 1, D_b, D_pe))
    end = np.where(t > 1, 1, 0)
    return D, typ, t, end


def _ps_locals(pl, al, bl, typ, end):
    """Local role-ordered node indices of a point-segment resolution (padded with -1)."""
    M = len(typ)
    loc = np.full((M, 4), -1, np.int64)
    loc[:, 0] = pl
    pe = typ == PE
    loc[pe, 1] = al
    loc[pe, 2] = bl
    pp = ~pe
    loc[pp, 1] = np.where(end[pp] == 1, bl, al)
    return loc


def _min_of_candidates(cands):
    """cands: list of (D, typ, loc) in increasing local-index order; pick min D, ties ->
    higher-dimensional type, then the earliest candidate."""
    Ds = np.stack([c[0] for c in cands], axis=1)
    ts = np.stack([c[1] for c in cands], axis=1)
    best = np.zeros(Ds.shape[0], np.int64)
    for j in range(1, Ds.shape[1]):
        cur_D = Ds[np.arange(len(best)), best]
        cur_t = ts[np.arange(len(best)), best]
        better = (Ds[:, j] < cur_D) | ((Ds[:, j] == cur_D) & (ts[:, j] > cur_t))
        best = np.where(better, j, best)
    r = np.arange(len(best))
    D = Ds[r, best]
    typ = ts[r, best]
    locs = np.stack([c[2] for c in cands], axis=1)
    loc = locs[r, best]
    return D, typ, loc


def resolve_pt(P, A, B, C):
    """Point-triangle feature pairs (role order p,a,b,c) -> (D, type, local role-ordered idx (M,4))."""
    M = len(P)
    e1, e2, w = B - A, C - A, P - A
    a11, a12, a22 = _dot(e1, e1), _dot(e1, e2), _dot(e2, e2)
    r1, r2 = _dot(e1, w), _dot(e2, w)
    det = a11 * a22 - a12 * a12
    u = (a22 * r1 - a12 * r2) / det
    v = (a11 * r2 - a12 * r1) / det
    inside = (u >= 0) & (v >= 0) & (u + v <= 1)
    n = np.cross(e1, e2)
    D_pt = _dot(w, n) ** 2 / _dot(n, n)
    cands = []
    for (al, bl, Aa, Bb) in [(1, 2, A, B), (2, 3, B, C), (3, 1, C, A)]:
        D, typ, _t, end = _point_segment(P, Aa, Bb)
        cands.append((D, typ, _ps_locals(0, al, bl, typ, end)))
    D_o, typ_o, loc_o = _min_of_candidates(cands)
    loc_pt = np.tile(np.array([0, 1, 2, 3]), (M, 1))
    D = np.where(inside, D_pt, D_o)
    typ = np.where(inside, PT, typ_o)
    loc = np.where(inside[:, None], loc_pt, loc_o)
    return D, typ, loc


def resolve_ee(A0, A1, B0, B1):
    """Edge-edge feature pairs (role order a0,a1,b0,b1) -> (D, type, local idx (M,4))."""
    M = len(A0)
    ea, eb, r = A1 - A0, B1 - B0, A0 - B0
    a, b, c = _dot(ea, ea), _dot(ea, eb), _dot(eb, eb)
    d, e = _dot(ea, r), _dot(eb, r)
    den = a * c - b * b
    with np.errstate(divide="ignore", invalid="ignore"):
        s = (b * e - c * d) / den
        t = (a * e - b * d) / den
    nondeg = den > 1e-10 * a * c  # R-EE1: sin^2 angle threshold above rounding noise
    inside = nondeg & (s >= 0) & (s <= 1) & (t >= 0) & (t <= 1)
    n = np.cross(ea, eb)
    with np.errstate(divide="ignore", invalid="ignore"):
        D_ee = _dot(r, n) ** 2 / _dot(n, n)
    cands = []
    for (pl, al, bl, Pp, Aa, Bb) in [(0, 2, 3, A0, B0, B1), (1, 2, 3, A1, B0, B1),
                                     (2, 0, 1, B0, A0, A1), (3, 0, 1, B1, A0, A1)]:
        D, typ, _t, end = _point_segment(Pp, Aa, Bb)
        cands.append((D, typ, _ps_locals(pl, al, bl, typ, end)))
    D_o, typ_o, loc_o = _min_of_candidates(cands)
    loc_ee = np.tile(np.array([0, 1, 2, 3]), (M, 1))
    D = np.where(inside, D_ee, D_o)
    typ = np.where(inside, EE, typ_o)
    loc = np.where(inside[:, None], loc_ee, loc_o)
    return D, typ, loc


def resolve_features(x, ftype, ids):
    """Resolve feature pairs of feature type ftype (PT pairs, EE pairs, or a key's own type)
    given role-ordered node ids (M,4) -> (D, sub-type, local idx into ids (M,4))."""
    M = len(ids)
    if M == 0:
        return np.zeros(0), np.zeros(0, np.int64), np.zeros((0, 4), np.int64)
    X = [x[np.maximum(ids[:, k], 0)] for k in range(4)]
    if ftype == PT:
        return resolve_pt(*X)
    if ftype == EE:
        return resolve_ee(*X)
    if ftype == PE:
        D, typ, _t, end = _point_segment(X[0], X[1], X[2])
        return D, typ, _ps_locals(0, 1, 2, typ, end)
    D = _dot(X[0] - X[1], X[0] - X[1])
    loc = np.full((M, 4), -1, np.int64)
    loc[:, 0], loc[:, 1] = 0, 1
    return D, np.full(M, PP, np.int64), loc


def canonical_keys(typ, gids):
    """(type, role-ordered global ids (M,4) padded -1) -> key rows (M,5) = [type, n0..n3]."""
    M = len(typ)
    k = np.full((M, 5), -1, np.int64)
    k[:, 0] = typ
    for i in range(M):
        t = typ[i]
        g = gids[i]
        if t == PP:
            a, b = sorted((g[0], g[1]))
            k[i, 1:3] = (a, b)
        elif t == PE:
            a, b = sorted((g[1], g[2]))
            k[i, 1:4] = (g[0], a, b)
        elif t == PT:
            k[i, 1] = g[0]
            k[i, 2:5] = sorted((g[1], g[2], g[3]))
        else:
            e1 = tuple(sorted((g[0], g[1])))
            e2 = tuple(sorted((g[2], g[3])))
            a, b = sorted((e1, e2))
            k[i, 1:5] = (*a, *b)
    return k


def key_feature_ids(keys):
    """Key rows -> (feature type, role-ordered ids (M,4)); canonical order is a valid role order."""
    return keys[:, 0], keys[:, 1:5]


# ---------------------------------------------------------------------------
# broad phase (result-neutral: any sound superset gives the same constraint set)
# ---------------------------------------------------------------------------
def _boxes(xa, xb, prims):
    lo = np.minimum(xa[prims].min(axis=1), xb[prims].min(axis=1))
    hi = np.maximum(xa[prims].max(axis=1), xb[prims].max(axis=1))
    return lo, hi


def _overlap_pairs(lo1, hi1, lo2, hi2, chunk=2048):
    out = []
    for s in range(0, len(lo1), chunk):
        l1, h1 = lo1[s:s + chunk, None, :], hi1[s:s + chunk, None, :]
        ov = np.all((l1 <= hi2[None]) & (lo2[None] <= h1), axis=2)
        i, j = np.nonzero(ov)
        out.append(np.stack([i + s, j], axis=1))
    return np.concatenate(out, axis=0) if out else np.zeros((0, 2), np.int64)


def candidates(mesh, xa, xb, inflate):
    """Feature pairs whose AABBs over the linear motion xa -> xb, each inflated by inflate/2
    per side, overlap.  Returns (pt (M,4) role order p,a,b,c ; ee (K,4) a0,a1,b0,b1)."""
    sv, tris, edges, fixed = mesh.surf_verts, mesh.tris, mesh.edges, mesh.fixed
    h = 0.5 * inflate
    vlo, vhi = _boxes(xa, xb, sv[:, None])
    tlo, thi = _boxes(xa, xb, tris)
    elo, ehi = _boxes(xa, xb, edges)
    ij = _overlap_pairs(vlo - h, vhi + h, tlo - h, thi + h)
    pt = np.concatenate([sv[ij[:, 0], None], tris[ij[:, 1]]], axis=1) if len(ij) else np.zeros((0, 4), np.int64)
    keep = (pt[:, 0] != pt[:, 1]) & (pt[:, 0] != pt[:, 2]) & (pt[:, 0] != pt[:, 3])
    keep &= ~np.all(fixed[pt], axis=1)
    pt = pt[keep]
    ij = _overlap_pairs(elo - h, ehi + h, elo - h, ehi + h)
    ij = ij[ij[:, 0] < ij[:, 1]]
    ee = np.concatenate([edges[ij[:, 0]], edges[ij[:, 1]]], axis=1) if len(ij) else np.zeros((0, 4), np.int64)
    keep = ((ee[:, 0] != ee[:, 2]) & (ee[:, 0] != ee[:, 3]) & (ee[:, 1] != ee[:, 2]) & (ee[:, 1] != ee[:, 3]))
    keep &= ~np.all(fixed[ee], axis=1)
    return pt.astype(np.int64), ee[keep].astype(np.int64)


def constraint_set(x, pt, ee, dhat):
    """Active constraints: the candidate feature pairs (vertex-triangle, edge-edge) whose feature
    distance is < dhat ("i-th primitive pair in the active primitive set").
    DESIGN.md R-DUP1: every feature pair is its own constraint with its own (continuous) feature
    distance; degenerate duplicates (two vertex-triangle pairs resolving to the same point-edge) are
    NOT merged, because merging makes the barrier sum jump when the vertex slides from the shared
    edge onto one triangle (SURVEY Q28 reading replaced).  Key = [PT|EE, role-ordered ids].
    Returns (keys (M,5) sorted lexicographically, d (M,))."""
    rows, ds = [], []
    for ftype, pairs in ((PT, pt), (EE, ee)):
        if len(pairs) == 0:
            continue
        D, _typ, _loc = resolve_features(x, ftype, pairs)
        m = D < dhat * dhat
        if not np.any(m):
            continue
        k = np.empty((int(m.sum()), 5), np.int64)
        k[:, 0] = ftype
        k[:, 1:] = pairs[m]
        rows.append(k)
        ds.append(np.sqrt(D[m]))
    if not rows:
        return np.zeros((0, 5), np.int64), np.zeros(0)
    keys = np.concatenate(rows)
    d = np.concatenate(ds)
    order = np.lexsort(keys.T[::-1])
    keys, d = keys[order], d[order]
    m = d < dhat
    return keys[m], d[m]


def activation_margin(x, pt, ee, dhat):
    """min over the candidate feature pairs of |d - dhat| / dhat: how close the d < dhat membership
    decision of the active set came to a tie (decision-trace tooling, SURVEY c.4)."""
    m = np.inf
    for ftype, pairs in ((PT, pt), (EE, ee)):
        if len(pairs):
            D, _t, _l = resolve_features(x, ftype, pairs)
            m = min(m, float(np.min(np.abs(np.sqrt(D) - dhat))) / dhat)
    return m


def key_distance(x, keys):
    """True feature distance d_i(x) of each key (re-resolving its sub-type at x)."""
    d = np.zeros(len(keys))
    for t in (PP, PE, PT, EE):
        m = keys[:, 0] == t
        if np.any(m):
            D, _, _ = resolve_features(x, t, keys[m, 1:5])
            d[m] = np.sqrt(D)
    return d


# ---------------------------------------------------------------------------
# squared distances as D2 (used only for derivatives)
# ---------------------------------------------------------------------------
def _sqdist_ad(sub, P):
    """P: role-ordered list of points, each a list of 3 D2; returns D2 of squared distance."""
    def dot(a, b):
        return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]

    def sub3(a, b):
        return [a[0] - b[0], a[1] - b[1], a[2] - b[2]]

    def cross(a, b):
        return [a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]]

    if sub == PP:
        r = sub3(P[0], P[1])
        return dot(r, r)
    if sub == PE:
        c = cross(sub3(P[1], P[0]), sub3(P[2], P[0]))
        e = sub3(P[2], P[1])
        return dot(c, c) / dot(e, e)
    if sub == PT:
        n = cross(sub3(P[2], P[1]), sub3(P[3], P[1]))
        w = dot(sub3(P[0], P[1]), n)
        return w * w / dot(n, n)
    n = cross(sub3(P[1], P[0]), sub3(P[3], P[2]))
    w = dot(sub3(P[0], P[2]), n)
    return w * w / dot(n, n)


def contact_stencils(x, keys, inA, inAp, mu, s, sigma, dhat):
    """Gradient and (unprojected) Hessian of phi_i(d_i(x)) for each key (Q22).  The stencil is the
    support of the resolved sub-type at x (its nodes in role order): d_i does not depend on the
    other nodes of the feature pair there (DESIGN.md R-DUP1).
    Returns list of (support node ids (k,), grad (3k,), hess (3k,3k), d, phi'(d)) in key order."""
    out = [None] * len(keys)
    kt, kid = keys[:, 0], keys[:, 1:5]
    for t in (PP, PE, PT, EE):
        sel = np.nonzero(kt == t)[0]
        if len(sel) == 0:
            continue
        _, sub, loc = resolve_features(x, t, kid[sel])
        # group by (sub-type, local pattern)
        pat = np.concatenate([sub[:, None], loc], axis=1)
        upat, inv = np.unique(pat, axis=0, return_inverse=True)
        for pi, pr in enumerate(upat):
            idx = sel[inv.ravel() == pi]
            st, lc = int(pr[0]), pr[1:]
            sup = lc[lc >= 0]
            k = len(sup)
            ids = kid[idx][:, sup]
            xs = x[ids].reshape(len(idx), 3 * k)
            V = D2.variables(xs)
            role = [V[3 * j:3 * j + 3] for j in range(k)]
            D = _sqdist_ad(st, role)
            d = D.sqrt()
            phi = _phi_ad(d, inA[idx], inAp[idx], mu[idx], s[idx], sigma, dhat)
            dphi = _dphi(d.v, inA[idx], inAp[idx], mu[idx], s[idx], sigma, dhat)
            for n_, i in enumerate(idx):
                out[i] = (ids[n_].copy(), phi.g[n_].copy(), phi.H[n_].copy(), d.v[n_], dphi[n_])
    return out


def _phi_ad(d, inA, inAp, mu, s, sigma, dhat):
    zero = d.const_like(0.0)
    phi = zero
    if np.any(inA):
        phi = phi + barrier_ad(d, dhat) * (sigma * inA.astype(np.float64))
    if np.any(inAp):
        w = inAp.astype(np.float64)
        al = (d * -1.0 + (dhat + s)) * mu + barrier_ad(d, dhat + s) * sigma
        phi = phi + al * w
    return phi


def _dphi(d, inA, inAp, mu, s, sigma, dhat):
    """phi'(d) by AD on the scalar d (used for the friction normal force, Q25)."""
    v = D2.variables(d[:, None])[0]
    return _phi_ad(v, inA, inAp, mu, s, sigma, dhat).g[:, 0]


def phi_energy(d, inA, inAp, mu, s, sigma, dhat):
    e = np.zeros_like(d)
    if np.any(inA):
        e += inA * sigma * barrier(d, dhat)
    if np.any(inAp):
        e += inAp * (mu * (dhat + s - d) + sigma * barrier(d, dhat + s))
    return e


# ---------------------------------------------------------------------------
# friction (§4.1)
# ---------------------------------------------------------------------------
def closest_point_weights(x, keys):
    """Signed closest-point weights Gamma (M,4) over each key's nodes and the unit normal n (M,3)
    at x (Q26): PT: +1 on p, -beta on the triangle; EE: (1-a, a) on edge A, -(1-b, b) on B;
    PE: +1 on p, -(1-t, t) on the edge; PP: +1, -1.  Computed on the resolved sub-type."""
    M = len(keys)
    G = np.zeros((M, 4))
    nrm = np.zeros((M, 3))
    for t in (PP, PE, PT, EE):
        sel = np.nonzero(keys[:, 0] == t)[0]
        if len(sel) == 0:
            continue
        ids = keys[sel, 1:5]
        _, sub, loc = resolve_features(x, t, ids)
        for n_, i in enumerate(sel):
            lc = loc[n_]
            pts = [x[ids[n_, j]] for j in lc if j >= 0]
            w = np.zeros(4)
            st = sub[n_]
            if st == PP:
                w[lc[0]], w[lc[1]] = 1.0, -1.0
            elif st == PE:
                p, a, b = pts
                tt = np.dot(p - a, b - a) / np.dot(b - a, b - a)
                w[lc[0]], w[lc[1]], w[lc[2]] = 1.0, -(1 - tt), -tt
            elif st == PT:
                p, a, b, c = pts
                e1, e2, ww = b - a, c - a, p - a
                a11, a12, a22 = e1 @ e1, e1 @ e2, e2 @ e2
                det = a11 * a22 - a12 * a12
                u = (a22 * (e1 @ ww) - a12 * (e2 @ ww)) / det
                v = (a11 * (e2 @ ww) - a12 * (e1 @ ww)) / det
                w[lc[0]], w[lc[1]], w[lc[2]], w[lc[3]] = 1.0, -(1 - u - v), -u, -v
            else:
                a0, a1, b0, b1 = pts
                ea, eb, r = a1 - a0, b1 - b0, a0 - b0
                A_, B_, C_ = ea @ ea, ea @ eb, eb @ eb
                D_, E_ = ea @ r, eb @ r
                den = A_ * C_ - B_ * B_
                s_ = (B_ * E_ - C_ * D_) / den
                t_ = (A_ * E_ - B_ * D_) / den
                w[lc[0]], w[lc[1]], w[lc[2]], w[lc[3]] = 1 - s_, s_, -(1 - t_), -t_
            kk = NNODES[t]
            diff = sum(w[j] * x[ids[n_, j]] for j in range(kk))
            G[i] = w
            nrm[i] = diff / np.linalg.norm(diff)
    return G, nrm


def friction_stencils(x, x_t, keys, Gam, nrm, lam, chi, eps_v, h):
    """Gradient and Hessian of D_j = chi lam_j f(||(I - n n^T) Gamma_j (x - x_t)||) per pair."""
    from .energy import mollifier_of_sq_ad
    eps = eps_v * h
    out = []
    for i in range(len(keys)):
        k = NNODES[int(keys[i, 0])]
        ids = keys[i, 1:1 + k]
        xs = x[ids].reshape(1, 3 * k)
        V = D2.variables(xs)
        n = nrm[i]
        u = [None, None, None]
        for c in range(3):
            acc = None
            for j in range(k):
                term = (V[3 * j + c] - x_t[ids[j], c]) * Gam[i, j]
                acc = term if acc is None else acc + term
            u[c] = acc
        un = u[0] * n[0] + u[1] * n[1] + u[2] * n[2]
        w = [u[c] - un * n[c] for c in range(3)]
        q = w[0] * w[0] + w[1] * w[1] + w[2] * w[2]
        Dj = mollifier_of_sq_ad(q, eps) * (chi * lam[i])
        out.append((ids.copy(), Dj.g[0].copy(), Dj.H[0].copy()))
    return out


def friction_energy(x, x_t, keys, Gam, nrm, lam, chi, eps_v, h):
    from .energy import mollifier
    if len(keys) == 0:
        return 0.0
    eps = eps_v * h
    tot = 0.0
    for i in range(len(keys)):
        k = NNODES[int(keys[i, 0])]
        ids = keys[i, 1:1 + k]
        u = np.sum(Gam[i, :k, None] * (x[ids] - x_t[ids]), axis=0)
        w = u - np.dot(u, nrm[i]) * nrm[i]
        tot += chi * lam[i] * float(mollifier(np.linalg.norm(w), eps))
    return tot
