"""Linear algebra of the inexact Newton step: SpMV, block-Jacobi PCG with the App. B policy,
and the stiffness-grouped block-Jacobi warm start.

TEST INFRASTRUCTURE (see oracle/__init__.py).

 - SpMV: y = (D + L + L^T + sum_i (C_i + C_i^T)) v, i.e. the plain product with the assembled
   symmetric matrix (§5.1).  Here: scipy CSR product (library primitive).
 - PCG: textbook preconditioned CG (Saad, Alg. 9.1) with M = blockdiag(D_j) (PAPER.md:384, 418
   "block diagonal ... also used for preconditioning").  Stop (App. B):
     ||r_k|| <= tol ||r^0||, r^0 := b (residual of the zero guess);
     stagnation (DESIGN.md R-PCG1, reading of "monitor the residual's decrease over the most recent
       100 PCG iterations.  If it stops decreasing"): the CG objective phi(x) = x'Ax/2 - b'x, which
       PCG decreases monotonically by alpha_k rho_k / 2 per iteration, decreased by no more than
       STALL_REL of its total decrease over the last W iterations.  (The residual norm itself
       oscillates by orders of magnitude on the stiff C4 systems, so a residual-minimum test stops
       CG before it ever improves on x0 -- measured, profiles/pcg_stagnation_r01.md.)
     iteration cap; NaN.
 - pcg_cg: the same block-Jacobi PCG in Chronopoulos-Gear form (one inner-product phase per
   iteration: (r,u) and (Au,u) together), the parity partner of the GPU's single-reduction PCG
   (SURVEY §8(c) c.1 step 7).  Equal to the textbook iterates in exact arithmetic (pinned in
   tests/test_oracle_solver.py); same stop rules.
 - warm start: for each stiffness group G an
   independent block-Jacobi PCG on A_GG (cross-group blocks skipped), zero initial guess,
   stop at ||r_G|| <= ws_tol ||b_G|| or ws_max iterations; the union is the initial guess x_0.
"""
from __future__ import annotations

import numpy as np

STOP_CONVERGED, STOP_STAGNATED, STOP_CAP, STOP_NAN = 0, 1, 2, 3
STALL_REL = 1e-10  # R-PCG1: "stops decreasing" = window decrease below 1e-10 of the total decrease


def block_inverse(Dblocks):
    return np.linalg.inv(Dblocks)


def apply_block(Dinv, r):
    N = Dinv.shape[0]
    return np.einsum("nij,nj->ni", Dinv, r.reshape(N, 3)).ravel()


def precond(M, r):
    """Apply the preconditioner: M is the block-Jacobi inverse (N,3,3) or, for the additive
    preconditioner of App. A, a callable r -> M^-1 r."""
    return M(r) if callable(M) else apply_block(M, r)


def additive_schwarz(A, Dinv, agg_nodes=9):
    """Two-level additive preconditioner of App. A ("comparison only, not
    adopted"): M^-1 = sum_b B_b^T (B_b A B_b^T)^-1 B_b over
      level 1: every node's 3x3 diagonal block (the block-Jacobi inverse Dinv), and
      level 2: aggregates of `agg_nodes` consecutive nodes [a0, a0 + agg_nodes) (the last one ragged),
               i.e. the 3 agg_nodes x 3 agg_nodes principal submatrices ("27x27" for 9 nodes),
    each inverse precomputed once per Newton step (the library inverse stands in for the
    paper's Gauss-Jordan elimination).  DESIGN.md R-AS1 states the reading.  Returns a callable."""
    N = A.shape[0] // 3
    A = A.tocsr()
    blocks = []
    for a0 in range(0, N, agg_nodes):
        a1 = min(a0 + agg_nodes, N)
        idx = np.arange(3 * a0, 3 * a1)
        blocks.append((3 * a0, 3 * a1, np.linalg.inv(A[idx][:, idx].toarray())))

    def apply(r):
        z = apply_block(Dinv, r)
        for i0, i1, Binv in blocks:
            z[i0:i1] += Binv @ r[i0:i1]
        return z

    apply.blocks = blocks
    return apply


def stop_threshold(st, tol):
    """||r_k|| threshold of the stop test: App. B's tol ||b|| (Q14), or one of App. B's alternatives
     when st.crit = (name, u kappa): (i) min(0.5, sqrt(||b||)) ||b|| (b = -grad E);
    (ii) u kappa ||x_k||; (iii) u kappa ||b||."""
    crit = getattr(st, "crit", None)
    if crit is None:
        return tol * st.bnorm
    name, ukappa = crit
    if name == "i":
        return min(0.5, np.sqrt(st.bnorm)) * st.bnorm
    if name == "ii":
        return ukappa * float(np.linalg.norm(st.x))
    return ukappa * st.bnorm


class PCGState:
    """Saved PCG state so App. B's 'return to PCG for an additional 100 iterations' can resume."""

    def __init__(self, x, r, z, p, rz, hist, bnorm):
        self.x, self.r, self.z, self.p, self.rz = x, r, z, p, rz
        self.hist = hist
        self.bnorm = bnorm
        self.k = len(hist) - 1
        self.stop = None
        self.dec = [0.0]  # cumulative decrease of the CG objective, dec[k] = phi_0 - phi_k


def pcg_start(A, b, x0, Dinv):
    r = b - A @ x0
    z = precond(Dinv, r)
    return PCGState(x0.copy(), r, z, z.copy(), float(r @ z), [float(np.linalg.norm(r))],
                    float(np.linalg.norm(b)))


def stalled(st, window, literal=False):
    """App. B stagnation at iteration st.k.  R-PCG1 (default): the CG objective decreased by
    no more than STALL_REL of its total decrease over the last `window` iterations.  literal (Q15, the
    residual reading): the best ||r_j|| of the last window is no better than the best before it."""
    k = st.k
    if window <= 0 or k < window:
        return False
    if literal:
        return min(st.hist[k - window + 1:k + 1]) >= min(st.hist[:k - window + 1])
    return (st.dec[k] - st.dec[k - window]) <= STALL_REL * st.dec[k]


def pcg_run(A, Dinv, st: PCGState, tol, window, max_iters, literal_stall=False):
    """Run PCG iterations on st until a stop condition or until st.k reaches max_iters."""
    while True:
        rn = st.hist[-1]
        if not np.isfinite(rn):
            st.stop = STOP_NAN
            return st
        if rn <= stop_threshold(st, tol):
            st.stop = STOP_CONVERGED
            return st
        k = st.k
        if stalled(st, window, literal_stall):
            st.stop = STOP_STAGNATED
            return st
        if k >= max_iters:
            st.stop = STOP_CAP
            return st
        q = A @ st.p
        pq = float(st.p @ q)
        alpha = st.rz / pq if pq != 0.0 else np.nan  # as the GPU: 0/0 -> NaN -> NaN stop next check
        st.dec.append(st.dec[-1] + 0.5 * alpha * st.rz)  # phi(x + a p) = phi(x) - a rho / 2
        st.x = st.x + alpha * st.p
        st.r = st.r - alpha * q
        st.z = precond(Dinv, st.r)
        rz_new = float(st.r @ st.z)
        beta = rz_new / st.rz if st.rz != 0.0 else 0.0  # r = 0 exactly: converged, next check stops
        st.rz = rz_new
        st.p = st.z + beta * st.p
        st.hist.append(float(np.linalg.norm(st.r)))
        st.k += 1


def stop_margin(st, tol):
    """How close the convergence test ||r_k|| <= tol ||b|| came to a tie at the last two iterates
    (relative): decision-trace tooling (SURVEY c.4); another PCG form may stop one iteration apart
    when this is at rounding level."""
    ref = tol * st.bnorm
    if ref <= 0.0:
        return np.inf
    return min(abs(h / ref - 1.0) for h in st.hist[-2:])


def pcg(A, b, x0, Dinv, tol=1e-4, window=100, max_iters=20000, literal_stall=False, crit=None):
    st = pcg_start(A, b, x0, Dinv)
    st.crit = crit
    return pcg_run(A, Dinv, st, tol, window, max_iters, literal_stall)


class CGState(PCGState):
    """Chronopoulos-Gear state (x, r, u, p, s, w and the scalars) for App. B resumes."""


def cg_start(A, b, x0, Dinv):
    """Chronopoulos-Gear PCG (Chronopoulos & Gear 1989, preconditioned form), M = blockdiag(D_j):
        r_0 = b - A x_0, u_0 = M^-1 r_0, w_0 = A u_0, gam_0 = (r_0,u_0), delta_0 = (w_0,u_0),
        alpha_0 = gam_0/delta_0, beta_0 = 0, p_-1 = s_-1 = 0;
        p_k = u_k + beta_k p_{k-1};  s_k = w_k + beta_k s_{k-1}   (s_k = A p_k)
        x_{k+1} = x_k + alpha_k p_k;  r_{k+1} = r_k - alpha_k s_k;  u_{k+1} = M^-1 r_{k+1};  w_{k+1} = A u_{k+1}
        gam_{k+1} = (r_{k+1},u_{k+1}); delta_{k+1} = (w_{k+1},u_{k+1});  beta_{k+1} = gam_{k+1}/gam_k
        alpha_{k+1} = gam_{k+1} / (delta_{k+1} - beta_{k+1} gam_{k+1} / alpha_k)."""
    x = x0.copy()
    r = b - A @ x
    u = precond(Dinv, r)
    st = CGState(x, r, u, np.zeros_like(b), float(r @ u), [float(np.linalg.norm(r))], float(np.linalg.norm(b)))
    st.u, st.w, st.s = u, A @ u, np.zeros_like(b)
    delta = float(st.w @ u)
    st.alpha = st.rz / delta if delta != 0.0 else 0.0
    st.beta = 0.0
    return st


def cg_run(A, Dinv, st, tol, window, max_iters, literal_stall=False):
    """Chronopoulos-Gear iterations on st until a stop condition or st.k reaches max_iters.  Stop
    rules and their order as pcg_run (App. B, Q14, R-PCG1), checked on ||r_k|| before step k."""
    while True:
        rn = st.hist[-1]
        k = st.k
        if not np.isfinite(rn):
            st.stop = STOP_NAN
            return st
        if rn <= stop_threshold(st, tol):
            st.stop = STOP_CONVERGED
            return st
        if stalled(st, window, literal_stall):
            st.stop = STOP_STAGNATED
            return st
        if k >= max_iters:
            st.stop = STOP_CAP
            return st
        st.p = st.u + st.beta * st.p
        st.s = st.w + st.beta * st.s
        st.x = st.x + st.alpha * st.p
        st.r = st.r - st.alpha * st.s
        st.u = precond(Dinv, st.r)
        st.w = A @ st.u
        gam_new = float(st.r @ st.u)
        delta = float(st.w @ st.u)
        st.dec.append(st.dec[-1] + 0.5 * st.alpha * st.rz)  # phi decrease of step k: alpha_k gam_k / 2
        beta = gam_new / st.rz if st.rz != 0.0 else 0.0
        den = delta - beta * gam_new / st.alpha if st.alpha != 0.0 else delta
        st.alpha = gam_new / den if den != 0.0 else 0.0  # r = 0 exactly: converged, next check stops
        st.beta = beta
        st.rz = gam_new
        st.hist.append(float(np.linalg.norm(st.r)))
        st.k += 1
        st.z = st.u


def pcg_cg(A, b, x0, Dinv, tol=1e-4, window=100, max_iters=20000, literal_stall=False, crit=None):
    st = cg_start(A, b, x0, Dinv)
    st.crit = crit
    return cg_run(A, Dinv, st, tol, window, max_iters, literal_stall)


def warm_start(A, b, groups, Dinv, fixed, tol=1e-2, max_iters=100):
    """Per-group independent block-Jacobi PCG on A_GG with zero guess (Q20).
    groups: (N,) int group id per node (ignored for fixed nodes).  Returns (x0, iters per group)."""
    N = len(groups)
    x0 = np.zeros(3 * N)
    iters = {}
    free = ~fixed
    for g in np.unique(groups[free]):
        nodes = np.nonzero(free & (groups == g))[0]
        dofs = (3 * nodes[:, None] + np.arange(3)[None]).ravel()
        Agg = A[dofs][:, dofs]
        bg = b[dofs]
        st = PCGState(np.zeros(len(dofs)), bg.copy(), None, None, 0.0, [float(np.linalg.norm(bg))],
                      float(np.linalg.norm(bg)))
        Dg = Dinv[nodes]
        st.z = apply_block(Dg, st.r)
        st.p = st.z.copy()
        st.rz = float(st.r @ st.z)
        it = 0
        while True:
            if st.hist[-1] <= tol * st.bnorm or it >= max_iters or not np.isfinite(st.hist[-1]):
                break
            q = Agg @ st.p
            alpha = st.rz / float(st.p @ q)
            st.x = st.x + alpha * st.p
            st.r = st.r - alpha * q
            st.z = apply_block(Dg, st.r)
            rz_new = float(st.r @ st.z)
            beta = rz_new / st.rz
            st.rz = rz_new
            st.p = st.z + beta * st.p
            st.hist.append(float(np.linalg.norm(st.r)))
            it += 1
        x0[dofs] = st.x
        iters[int(g)] = it
    return x0, iters
