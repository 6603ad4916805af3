"""The barrier-augmented Lagrangian time step (Alg. 1) with its inexact
Newton-PCG primal solve (§4) -- the oracle procedure of SURVEY.md §8(c) c.1.

TEST INFRASTRUCTURE (see oracle/__init__.py).

Per time step (backward Euler):  y = x_t + h v_t + h^2 G;  x^0 = x_t (Q5);
mu = {}, A' = {} (Alg. 1 data line); sigma^0 from the least-squares fit (Q7).
Per Newton iteration l (one inexact Newton iteration = one l, Q6):
  A = {d < dhat at x^l}; dmin; A' rules (Alg. 1 lines 3-6; Q9, Q10)
  friction anchors at x^l (Q25, Q26)
  e = grad L (line 7); assemble A, Lambda, groups; warm start; PCG (App. B) -> p
  line search: alpha_0 = min(1, alpha_CCD), halve on energy increase / budget (Q35-Q37),
    alpha < 1e-9 -> resume PCG +100 iterations (App. B, Q16)
  x^{l+1} = x^l + alpha p;  stop if ||e^l|| <= 1e-4 ||e^0|| (lines 9-11; Q13)
  s_i, mu_i on A' (lines 12-14; Q11, Q12);  sigma <- max(1.2 sigma, 100 sigma^0) if min d < 1e-2 dhat
  (lines 15-16; Q8)
v_{t+1} = (x_{t+1} - x_t)/h (eq:int:x).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import ccd as ccdm
from . import contact as cm
from . import linalg as la
from .assemble import floor_log10
from .auglag import aprime_rule, dual_update, sigma_ls, sigma_schedule, slack
from .energy import barrier, inertia_energy, inertia_grad, nh_energy, nh_stencils
from .mesh import precompute
from .projection import project_eigh

# R-LS1: energy comparisons tolerate 8 units of roundoff of the summed magnitudes
LS_ROUND = 8.0 * 2.0 ** -53

FLAG_NO_WARMSTART = 1
FLAG_NO_AUGLAG = 2
FLAG_SIGMA_CAP = 8  # NEXT-1: sigma ceiling 1e8 sigma0 (the GPU's BAL_SIGMA_CAP)
FLAG_SIGMA_MIN = 16  # min(1.2 sigma, 100 sigma0) reading of Alg. 1 line 16 (the GPU's BAL_SIGMA_MIN)
FLAG_FRICTION_NO_FREEZE = 32  # literal per-iteration anchors (disables R-FRIC1)
FLAG_CCD_LITERAL = 64  # literal P:468 CCD activation eps + dhat (disables R-CCD2; the GPU's BAL_CCD_LITERAL)
FLAG_PCG_LITERAL_STALL = 128  # literal residual stagnation test (Q15; disables R-PCG1; BAL_PCG_LITERAL_STALL)
FLAG_ADDITIVE_PRECOND = 512  # NEXT-1: global PCG with App. A's two-level additive preconditioner (R-AS1)
FLAG_PCG_CG = 1 << 20  # oracle only: global PCG in the Chronopoulos-Gear form (la.pcg_cg, pinned to the
# textbook iterates) -- the GPU's form, for decision-trace parity of PCG iteration counts (R-CG)
FLAG_PCG_CRIT_I = 1024  # NEXT-4: App. B criterion (i) (the GPU's BAL_PCG_CRIT_I)
FLAG_PCG_CRIT_II = 2048  # App. B criterion (ii) (BAL_PCG_CRIT_II)
FLAG_PCG_CRIT_III = 4096  # App. B criterion (iii) (BAL_PCG_CRIT_III)
AS_AGG_NODES = 9  # R-AS1: level-2 aggregates of 9 consecutive nodes (27x27 blocks)
FREEZE_WINDOW = 10  # R-FRIC1 window (the GPU's kFreezeWindow)


class NotConverged(RuntimeError):
    pass


class NonFinite(RuntimeError):
    """sigma^0 or ||e^l|| is not finite (the GPU's BAL_E_NAN)."""


def _coo_add(rows, cols, vals, ids, H):
    k = len(ids)
    dof = (3 * np.asarray(ids)[:, None] + np.arange(3)[None]).ravel()
    rows.append(np.repeat(dof, 3 * k))
    cols.append(np.tile(dof, 3 * k))
    vals.append(H.ravel())


def _pcg_window(pst, tol, drift=5e-2):
    """Trace only (DESIGN.md R-TRACE): the iterations k at which a PCG whose residual history
    differs from this one by a relative `drift` could have met ||r_k|| <= tol ||b||: from the first k
    with ||r_k|| <= (1 + drift) tol ||b|| to the first k with ||r_k|| <= (1 - drift) tol ||b|| (the stop
    iteration if none)."""
    h = np.asarray(pst.hist)
    thr = tol * pst.bnorm
    lo = np.nonzero(h <= (1.0 + drift) * thr)[0]
    hi = np.nonzero(h <= (1.0 - drift) * thr)[0]
    k = int(pst.k)
    return (int(lo[0]) if len(lo) else k, int(hi[0]) if len(hi) else k)


class Oracle:
    def __init__(self, scene, flags=0):
        self.scene = scene
        self.mesh = precompute(scene)
        p = scene["params"]
        self.p = p
        self.h = float(p["h"])
        self.g = np.asarray(p["gravity"], np.float64)
        self.dhat = float(p["dhat"])
        self.flags = flags
        self.free = ~self.mesh.fixed
        self.N = self.mesh.n

    # ------------------------------------------------------------------ energy
    def energy(self, x, st, pt, ee):
        """L(x) at fixed (y, sigma, A' with mu, s, friction anchors).  Returns (L, n_constraints, S)
        where S = sum of the magnitudes of all terms of L -- the scale of its FP64 evaluation error
        used by the line-search acceptance (DESIGN.md R-LS1)."""
        m = self.mesh
        if m.tets.size and nh_energy(x, m) == np.inf:
            return np.inf, 0, np.inf
        keys, d = cm.constraint_set(x, pt, ee, self.dhat)
        if len(d) and np.min(d) <= 0.0:
            return np.inf, len(d), np.inf
        dap = cm.key_distance(x, st["ap_keys"]) if len(st["ap_keys"]) else np.zeros(0)
        if len(dap) and np.min(dap) <= 0.0:
            return np.inf, len(d), np.inf
        ei = inertia_energy(x, st["y"], m.mass, self.h, self.free)
        ee_ = nh_energy(x, m)
        eb = float(np.sum(st["sigma"] * barrier(d, self.dhat)))
        L = ei + ee_ + eb
        S = abs(ei) + abs(ee_) + abs(eb)
        if len(dap):
            al = cm.phi_energy(dap, np.zeros(len(dap)), np.ones(len(dap)), st["ap_mu"], st["ap_s"], st["sigma"],
                               self.dhat)
            L += float(np.sum(al))
            S += float(np.sum(np.abs(al)))
        if st.get("fr_keys") is not None and len(st["fr_keys"]):
            ef = cm.friction_energy(x, st["x_t"], st["fr_keys"], st["fr_G"], st["fr_n"], st["fr_lam"],
                                    float(self.p["chi"]), float(self.p["eps_v"]), self.h)
            L += ef
            S += abs(ef)
        if not np.isfinite(L):
            return np.inf, len(d), np.inf
        return L, len(d), S

    # ---------------------------------------------------------------- stencils
    def contact_stencil_set(self, x, keys_A, st):
        """Merge A (resolved at x) and A' keys into one stencil list (Q22)."""
        ap = st["ap_keys"]
        allk = np.concatenate([keys_A, ap]) if len(ap) else keys_A
        if len(allk) == 0:
            return np.zeros((0, 5), np.int64), np.zeros(0), np.zeros(0), np.zeros(0), np.zeros(0)
        uk, inv = np.unique(allk, axis=0, return_inverse=True)
        inv = inv.ravel()
        inA = np.zeros(len(uk))
        inA[inv[:len(keys_A)]] = 1.0
        inAp = np.zeros(len(uk))
        mu = np.zeros(len(uk))
        s = np.zeros(len(uk))
        if len(ap):
            ia = inv[len(keys_A):]
            inAp[ia] = 1.0
            mu[ia] = st["ap_mu"]
            s[ia] = st["ap_s"]
        return uk, inA, inAp, mu, s

    def assemble(self, x, st, keys_A):
        """Returns dict with CSR A (fixed rows identity), gradient e, Dinv, e_j, groups, stencils."""
        m = self.mesh
        N, h = self.N, self.h
        rows, cols, vals = [], [], []
        grad = inertia_grad(x, st["y"], m.mass, h, np.ones(N, bool)).ravel()
        lam_diag = np.repeat(m.mass / (h * h), 3).reshape(N, 3).copy()
        # inertia
        dm = np.repeat(m.mass / (h * h), 3)
        rows.append(np.arange(3 * N))
        cols.append(np.arange(3 * N))
        vals.append(dm)
        out = {}
        # elastic (AD Hessian, projected on the full 12x12; Q21, Q23)
        if m.tets.size:
            _v, g, H = nh_stencils(x, m)
            P, wc = project_eigh(H)
            lb = wc.sum(axis=1) / 12.0
            for k in range(4):
                np.add.at(grad.reshape(N, 3), m.tets[:, k], g[:, 3 * k:3 * k + 3])
                np.add.at(lam_diag, m.tets[:, k], lb[:, None])
            dof = (3 * m.tets[:, :, None] + np.arange(3)[None, None]).reshape(-1, 12)
            rows.append(np.repeat(dof, 12, axis=1).ravel())
            cols.append(np.tile(dof, (1, 12)).ravel())
            vals.append(P.reshape(-1))
            out["elastic_P"] = P
            out["elastic_g"] = g
            out["elastic_lbar"] = lb
        # contact
        uk, inA, inAp, mu, s = self.contact_stencil_set(x, keys_A, st)
        cs = cm.contact_stencils(x, uk, inA, inAp, mu, s, st["sigma"], self.dhat) if len(uk) else []
        c_P, c_lb, c_ids, c_g = [], [], [], []
        for (ids, g, H, _d, _dp) in cs:
            P, wc = project_eigh(H[None])
            lb = wc.sum() / (3 * len(ids))  # Q18 over the stencil's support nodes (R-DUP1)
            grad.reshape(N, 3)[ids] += g.reshape(-1, 3)
            lam_diag[ids] += lb
            _coo_add(rows, cols, vals, ids, P[0])
            c_P.append(P[0])
            c_lb.append(lb)
            c_ids.append(ids)
            c_g.append(g)
        out["contact_keys"], out["contact_P"], out["contact_lbar"] = uk, c_P, c_lb
        out["contact_g"] = c_g
        out["contact_ids"] = c_ids
        out["contact_inA"], out["contact_inAp"] = inA, inAp
        # friction (PSD analytically; not projected, not in Lambda: Q17)
        if st.get("fr_keys") is not None and len(st["fr_keys"]):
            fs = cm.friction_stencils(x, st["x_t"], st["fr_keys"], st["fr_G"], st["fr_n"], st["fr_lam"],
                                      float(self.p["chi"]), float(self.p["eps_v"]), h)
            for (ids, g, H) in fs:
                grad.reshape(N, 3)[ids] += g.reshape(-1, 3)
                _coo_add(rows, cols, vals, ids, H)
            out["friction"] = fs
        A = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                          shape=(3 * N, 3 * N)).tocsr()
        A.sum_duplicates()
        fixed_dof = np.repeat(m.fixed, 3)
        if np.any(fixed_dof):
            keep = sp.diags((~fixed_dof).astype(np.float64))
            A = (keep @ A @ keep + sp.diags(fixed_dof.astype(np.float64))).tocsr()
            grad[fixed_dof] = 0.0
        A.eliminate_zeros()
        Dblk = np.zeros((N, 3, 3))
        for c1 in range(3):
            for c2 in range(3):
                Dblk[:, c1, c2] = np.asarray(A[3 * np.arange(N) + c1, 3 * np.arange(N) + c2]).ravel()
        e_j = lam_diag.sum(axis=1)
        groups = np.full(N, -999, np.int64)
        groups[self.free] = floor_log10(e_j[self.free])
        out.update(A=A, grad=grad, Dblk=Dblk, Dinv=np.linalg.inv(Dblk), e_j=e_j, groups=groups)
        return out

    # ------------------------------------------------------------- friction anchors
    def friction_anchors(self, x, st, keys_A):
        """lambda_j = -phi_j'(d_j) at x^l, Gamma, n (Q25, Q26); friction pairs = A at x^l."""
        if float(self.p["chi"]) <= 0.0 or len(keys_A) == 0:
            return None
        uk, inA, inAp, mu, s = self.contact_stencil_set(x, keys_A, st)
        sel = inA > 0
        keys = uk[sel]
        d = cm.key_distance(x, keys)
        dphi = cm._dphi(d, inA[sel], inAp[sel], mu[sel], s[sel], st["sigma"], self.dhat)
        G, n = cm.closest_point_weights(x, keys)
        return keys, G, n, -dphi

    # -------------------------------------------------------------------- sigma0
    def sigma0(self, x, st, keys):
        m = self.mesh
        N = self.N
        gE = inertia_grad(x, st["y"], m.mass, self.h, np.ones(N, bool)).ravel()
        if m.tets.size:
            _v, g, _H = nh_stencils(x, m)
            for k in range(4):
                np.add.at(gE.reshape(N, 3), m.tets[:, k], g[:, 3 * k:3 * k + 3])
        gb = np.zeros(3 * N)
        if len(keys):
            cs = cm.contact_stencils(x, keys, np.ones(len(keys)), np.zeros(len(keys)), np.zeros(len(keys)),
                                     np.zeros(len(keys)), 1.0, self.dhat)
            for (ids, g, _H, _d, _dp) in cs:
                gb.reshape(N, 3)[ids] += g.reshape(-1, 3)
        fd = np.repeat(m.fixed, 3)
        gE[fd] = 0.0
        gb[fd] = 0.0
        floor = float(np.mean(m.mass[self.free])) / (self.h * self.h)
        with np.errstate(over="ignore", invalid="ignore"):
            s_ls = sigma_ls(gb, gE)
        # a non-finite least-squares value (overflowing ||g_b||^2) falls back to the floor (Q7)
        return floor if (s_ls is None or not np.isfinite(s_ls)) else max(s_ls, floor)

    # ---------------------------------------------------------------------- step
    def step(self, x_t, v_t, trace=None):
        p = self.p
        m = self.mesh
        h, dhat = self.h, self.dhat
        x_t = np.asarray(x_t, np.float64).reshape(-1, 3)
        v_t = np.asarray(v_t, np.float64).reshape(-1, 3)
        y = x_t + h * v_t + h * h * self.g[None]
        y[m.fixed] = x_t[m.fixed]
        x = x_t.copy()
        st = dict(y=y, x_t=x_t, ap_keys=np.zeros((0, 5), np.int64), ap_mu=np.zeros(0), ap_s=np.zeros(0),
                  fr_keys=None)
        pt, ee = cm.candidates(m, x, x, dhat)
        keys, d = cm.constraint_set(x, pt, ee, dhat)
        if len(d) and d.min() <= 0:
            raise ValueError("infeasible input: surface distance <= 0")
        sig0 = self.sigma0(x, st, keys)
        if not (np.isfinite(sig0) and sig0 > 0.0):
            raise NonFinite("sigma0 is not a positive finite number")
        st["sigma"] = sig0
        dmin_prev = np.inf
        e0 = None
        dx_prev = None
        emin, frozen = [], False
        stats = dict(newton=0, pcg=0, ws=0, max_constraints=0)
        converged = False
        for l in range(int(p["max_newton"])):
            pt, ee = cm.candidates(m, x, x, dhat)
            keys, d = cm.constraint_set(x, pt, ee, dhat)
            dmin = float(d.min()) if len(d) else np.inf
            rebuilt = False
            rule = "keep" if self.flags & FLAG_NO_AUGLAG else aprime_rule(dmin, dmin_prev, len(st["ap_keys"]) == 0, dhat)
            if rule == "clear":
                st["ap_keys"], st["ap_mu"], st["ap_s"] = np.zeros((0, 5), np.int64), np.zeros(0), np.zeros(0)
            elif rule == "rebuild":
                newk = keys[d < 1e-2 * dhat]
                mu_new, s_new = np.zeros(len(newk)), np.zeros(len(newk))
                old = {tuple(k): (mu_, s_) for k, mu_, s_ in zip(st["ap_keys"], st["ap_mu"], st["ap_s"])}
                for i, k in enumerate(newk):
                    if tuple(k) in old:
                        mu_new[i], s_new[i] = old[tuple(k)]
                st["ap_keys"], st["ap_mu"], st["ap_s"] = newk, mu_new, s_new
                rebuilt = True
            dmin_prev = dmin
            if not frozen:  # friction anchors at x^l, unless frozen (R-FRIC1)
                fr = self.friction_anchors(x, st, keys)
                if fr is not None:
                    st["fr_keys"], st["fr_G"], st["fr_n"], st["fr_lam"] = fr
                else:
                    st["fr_keys"] = None
            asm = self.assemble(x, st, keys)
            e = asm["grad"]
            en = float(np.linalg.norm(e))
            if not np.isfinite(en):
                raise NonFinite("||e|| is not finite")
            if e0 is None:
                e0 = en
            # R-FRIC1: the per-iteration anchor update is a fixed-point iteration;
            # once the best ||e|| has not halved over FREEZE_WINDOW iterations the anchors are frozen for
            # the rest of the step (IPC's semi-implicit friction, convergent)
            emin.append(en if not emin else min(emin[-1], en))
            if (not frozen and not (self.flags & FLAG_FRICTION_NO_FREEZE) and float(p["chi"]) > 0.0
                    and l >= FREEZE_WINDOW and emin[l] > 0.5 * emin[l - FREEZE_WINDOW]):
                frozen = True
            if e0 == 0.0:
                converged = True
                break
            A, Dinv = asm["A"], asm["Dinv"]
            b = -e
            ws_it = {}
            if self.flags & FLAG_NO_WARMSTART:
                x0 = np.zeros_like(b)
            else:
                x0, ws_it = la.warm_start(A, b, asm["groups"], Dinv, m.fixed, float(p["ws_rel_tol"]),
                                          int(p["ws_max_iters"]))
                # DESIGN.md R-WS1: keep the warm start only if it is closer to the solution than 0 in
                # the A-norm, i.e. phi(x0) = x0'A x0 / 2 - b'x0 < phi(0) = 0
                if not (0.5 * float(x0 @ (A @ x0)) - float(b @ x0) < 0.0):
                    x0 = np.zeros_like(b)
            M = la.additive_schwarz(A, Dinv, AS_AGG_NODES) if self.flags & FLAG_ADDITIVE_PRECOND else Dinv
            solve = la.pcg_cg if self.flags & FLAG_PCG_CG else la.pcg
            crit = None
            if self.flags & (FLAG_PCG_CRIT_I | FLAG_PCG_CRIT_II | FLAG_PCG_CRIT_III):
                # App. B alternatives; kappa from the assembled eigenvalues (DESIGN.md R-KAPPA)
                ej = asm["e_j"][self.free]
                ukappa = np.finfo(np.float64).eps * float(ej.max() / ej.min())
                crit = ("i" if self.flags & FLAG_PCG_CRIT_I else "ii" if self.flags & FLAG_PCG_CRIT_II else "iii",
                        ukappa)
            pst = solve(A, b, x0, M, float(p["pcg_rel_tol"]), int(p["pcg_stall_window"]),
                        int(p["max_pcg"]), bool(self.flags & FLAG_PCG_LITERAL_STALL), crit=crit)
            resumes = 0
            while True:
                dirn = pst.x.copy()
                safeguard = False
                # Q38 descent safeguard; a NaN dot product (PCG stopped on NaN) also falls back
                if not (float(dirn @ e) < 0.0):
                    dirn = -la.apply_block(Dinv, e)
                    safeguard = True
                P = dirn.reshape(-1, 3)
                cpt, cee = cm.candidates(m, x, x + P, dhat)
                a_ccd = ccdm.step_toi(x, P, cpt, cee, dhat,
                                      np.inf if self.flags & FLAG_CCD_LITERAL else 1e-2)
                alpha = min(1.0, a_ccd)
                ccd_sens = 0.0
                if trace is not None and a_ccd < 1.0:
                    # conditioning of alpha_CCD (trace only, DESIGN.md R-TRACE): relative change of
                    # the TOI under a 1e-6 relative perturbation of the direction, the size by which
                    # two PCG implementations' directions differ; a near-double cubic root amplifies it
                    xi = np.random.default_rng(l).standard_normal(P.shape)
                    a_pert = ccdm.step_toi(x, P * (1.0 + 1e-6 * xi), cpt, cee, dhat,
                                           np.inf if self.flags & FLAG_CCD_LITERAL else 1e-2)
                    ccd_sens = abs(a_pert - a_ccd) / a_ccd
                L0, _n0, S0 = self.energy(x, st, cpt, cee)
                halvings = 0
                ls_margin = np.inf  # closest accept/reject decision to its threshold, relative to S
                while alpha >= float(p["alpha_min"]):
                    L1, n1, S1 = self.energy(x + alpha * P, st, cpt, cee)
                    if np.isfinite(L1):
                        ls_margin = min(ls_margin, abs(L1 - L0 - LS_ROUND * max(S0, S1)) / max(S0, S1))
                    # R-LS1: accept when L does not increase beyond its FP64 evaluation error; an
                    # infeasible trial (J <= 0, d <= 0, NaN) has L = +inf and is never accepted
                    if (n1 <= int(p["max_constraints"]) and np.isfinite(L1)
                            and L1 <= L0 + LS_ROUND * max(S0, S1)):
                        break
                    alpha *= 0.5
                    halvings += 1
                if alpha >= float(p["alpha_min"]):
                    break
                if resumes >= 50 or pst.k >= int(p["max_pcg"]):
                    raise NotConverged("line search failed after PCG resumes")
                resumes += 1
                pst.crit = None  # App. B resume: exactly pcg_resume_iters more iterations
                pst = (la.cg_run if self.flags & FLAG_PCG_CG else la.pcg_run)(A, M, pst, 0.0, 10 ** 9, min(pst.k + int(p["pcg_resume_iters"]),
                                                                  int(p["max_pcg"])))
            x_new = x + alpha * P
            if trace is not None:
                dx_prev_next = (alpha * P).ravel()
            stats["newton"] += 1
            stats["pcg"] += pst.k
            stats["ws"] += sum(ws_it.values()) if ws_it else 0
            stats["max_constraints"] = max(stats["max_constraints"], len(keys))
            if trace is not None:
                gvals, gcnt = np.unique(asm["groups"][self.free], return_counts=True)
                trace.append(dict(l=l, nA=len(keys), nAp=len(st["ap_keys"]), rebuilt=rebuilt, dmin=dmin,
                                  sigma=st["sigma"], groups=dict(zip(gvals.tolist(), gcnt.tolist())),
                                  ws_iters=ws_it, pcg_iters=pst.k, pcg_stop=pst.stop, alpha_ccd=a_ccd,
                                  alpha=alpha, halvings=halvings, resumes=resumes, safeguard=safeguard,
                                  rel_e=en / e0, e_sens=(1e-6 * float(np.linalg.norm(A @ dx_prev)) / e0
                                                         if dx_prev is not None else 0.0),
                                  nA_margin=cm.activation_margin(x, pt, ee, dhat),
                                  ls_margin=ls_margin, ccd_sens=ccd_sens,
                                  pcg_window=_pcg_window(pst, float(p["pcg_rel_tol"])),
                                  pcg_margin=la.stop_margin(pst, float(p["pcg_rel_tol"]))))
            if trace is not None:
                # trace only (DESIGN.md R-TRACE): ||e|| at the next iterate moves by ~||A dx|| when the
                # step moves by dx; two PCG forms' steps agree to ~1e-6 relative
                dx_prev = dx_prev_next
            if en <= float(p["newton_rel_tol"]) * e0:
                x = x_new
                converged = True
                break
            # AL updates on A' (lines 12-14)
            if len(st["ap_keys"]):
                dn = cm.key_distance(x_new, st["ap_keys"])
                s_new = slack(st["ap_mu"], st["sigma"], dhat, dn)
                st["ap_s"] = s_new
                st["ap_mu"] = dual_update(st["ap_mu"], st["sigma"], dhat, s_new, dn)
            # sigma schedule (lines 15-16)
            if not (self.flags & FLAG_NO_AUGLAG):
                _k2, d2 = cm.constraint_set(x_new, cpt, cee, dhat)
                st["sigma"] = sigma_schedule(st["sigma"], sig0, float(d2.min()) if len(d2) else np.inf, dhat,
                                             cap=bool(self.flags & FLAG_SIGMA_CAP),
                                             use_min=bool(self.flags & FLAG_SIGMA_MIN))
            x = x_new
        if not converged:
            raise NotConverged("Newton iteration cap reached")
        x[m.fixed] = x_t[m.fixed]
        v = (x - x_t) / h
        stats["sigma0"] = sig0
        return x, v, stats
