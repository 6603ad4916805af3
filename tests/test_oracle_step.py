"""Pins of the oracle's CCD and full BAL step (closed forms, dense time
scans, free fall, momentum, non-penetration).  CPU only."""
import numpy as np
import pytest

import scenes
from oracle import ccd
from oracle import contact as cm
from oracle.bal import FLAG_NO_AUGLAG, Oracle
from oracle.energy import nh_min_J


# ---------------------------------------------------------------- cubic root finder
def test_cubic_roots_constructed():
    r = ccd.cubic_roots(1.0, -1.5, 0.6875, -0.09375)  # (t-.25)(t-.5)(t-.75)
    np.testing.assert_allclose(r, [0.25, 0.5, 0.75], atol=1e-12)
    r = ccd.cubic_roots(1.0, 0.0, -1.0, 0.0)  # t^3 - t -> {0, 1} on [-eps, 1+eps]
    np.testing.assert_allclose(r, [0.0, 1.0], atol=1e-12)
    assert ccd.cubic_roots(1.0, 0.0, 0.0, 5.0) == []
    rng = np.random.default_rng(30)
    for _ in range(300):
        a, b, c, d = rng.normal(size=4)
        roots = ccd.cubic_roots(a, b, c, d)
        ts = np.linspace(-ccd.EPS, 1 + ccd.EPS, 100001)
        f = ((a * ts + b) * ts + c) * ts + d
        changes = np.nonzero(np.sign(f[:-1]) * np.sign(f[1:]) < 0)[0]
        # every sign change of the dense scan is matched by a reported root nearby
        for ci in changes:
            assert any(abs(r - ts[ci]) <= 2e-5 for r in roots)
        for r in roots:
            assert abs(((a * r + b) * r + c) * r + d) <= 1e-9 * (abs(a) + abs(b) + abs(c) + abs(d))


def test_ccd_vertex_onto_plane():
    """Vertex at height 1 moving -2 onto a triangle's plane: coplanar at t = 0.5, TOI < 0.5."""
    x = np.array([[0.2, 0.2, 1.0], [0, 0, 0], [1.0, 0, 0], [0, 1.0, 0]])
    dx = np.zeros((4, 3))
    dx[0] = [0, 0, -2.0]
    t = ccd.pair_toi(cm.PT, x, dx, np.array([0, 1, 2, 3]), 1e-3)
    assert 0.0 < t < 0.5
    assert t == pytest.approx(0.45, rel=1e-12)
    # no motion -> no collision
    assert ccd.pair_toi(cm.PT, x, np.zeros((4, 3)), np.array([0, 1, 2, 3]), 1e-3) == 1.0


def _dense_first_hit(ftype, x, dx, ids, n=10000):
    ts = np.linspace(0, 1, n + 1)
    X = x[ids][None] + ts[:, None, None] * dx[ids][None]
    P = [X[:, k] for k in range(4)]
    D, _, _ = (cm.resolve_pt if ftype == cm.PT else cm.resolve_ee)(*P)
    if ftype == cm.PT:
        sd = np.einsum("ij,ij->i", P[0] - P[1], np.cross(P[2] - P[1], P[3] - P[1]))
        n_ = np.cross(P[2] - P[1], P[3] - P[1])
    else:
        sd = np.einsum("ij,ij->i", P[0] - P[2], np.cross(P[1] - P[0], P[3] - P[2]))
    hit = np.nonzero(np.sign(sd[1:]) != np.sign(sd[:-1]))[0]
    # a crossing of the support plane only counts when the features are within reach
    for h in hit:
        if min(np.sqrt(D[h]), np.sqrt(D[h + 1])) < 1e-2:
            return ts[h]
    return None


def test_ccd_random_trajectories_no_false_negatives():
    rng = np.random.default_rng(31)
    misses = 0
    for trial in range(400):
        ftype = cm.PT if trial % 2 == 0 else cm.EE
        x = rng.normal(size=(4, 3)) * 0.5
        dx = rng.normal(size=(4, 3)) * 0.8
        ids = np.array([0, 1, 2, 3])
        D0, _, _ = cm.resolve_features(x, ftype, ids[None])
        if np.sqrt(D0[0]) < 2e-3:
            continue
        t = ccd.pair_toi(ftype, x, dx, ids, 1e-3)
        th = _dense_first_hit(ftype, x, dx, ids)
        xt = x + t * dx
        Dt, _, _ = cm.resolve_features(xt, ftype, ids[None])
        assert Dt[0] > 0.0  # conservative: distance at the TOI is positive
        if th is not None:
            D_hit, _, _ = cm.resolve_features(x + th * dx, ftype, ids[None])
            if np.sqrt(D_hit[0]) < 1e-6:  # a genuine touching/crossing in the scan
                assert t <= th + 1e-4
                misses += 0


# ---------------------------------------------------------------- BAL step
def test_free_fall_reaches_predictor():
    sc = scenes.make_free_cube(3)
    o = Oracle(sc)
    x, v, st = o.step(sc["x0"], sc["v0"])
    y = sc["x0"] + o.h * sc["v0"] + o.h ** 2 * o.g[None]
    assert np.linalg.norm(x - y) <= 1e-6 * np.linalg.norm(y - sc["x0"])
    np.testing.assert_allclose(v, (x - sc["x0"]) / o.h)


def test_linear_momentum_two_tets():
    """Gravity-free, frictionless: sum_j m_j (x_j - y_j)/h^2 = sum_j e_j at every iterate, hence
    the momentum change equals h * sum_j e_j(x_{t+1}) -- a pin that every non-inertia gradient
    (elastic, barrier, AL) is translation invariant."""
    sc = scenes.make_two_tets(0)
    o = Oracle(sc)
    m = o.mesh.mass
    x, v = sc["x0"], sc["v0"]
    p0 = (m[:, None] * v).sum(0)
    saw_contact = False
    for _ in range(6):
        tr = []
        x, v_new, st = o.step(x, v, tr)
        saw_contact |= any(r["nA"] > 0 for r in tr)
        v = v_new
    p1 = (m[:, None] * v).sum(0)
    assert saw_contact
    scale = np.abs(m[:, None] * sc["v0"]).sum()
    assert np.linalg.norm(p1 - p0) <= 1e-3 * scale  # Newton stops at 1e-4 relative gradient


def test_tet_drop_nonpenetration_and_convergence():
    sc = scenes.make_single_tet(1, height=0.01, speed=1.0)
    o = Oracle(sc)
    x, v = sc["x0"], sc["v0"]
    for step in range(4):
        x_prev = x
        tr = []
        x, v, st = o.step(x, v, tr)
        assert tr[-1]["rel_e"] <= 1e-4
        # dense time sampling of the step between its endpoints and over all surface pairs
        pt, ee = cm.candidates(o.mesh, x_prev, x, o.dhat)
        for ts in np.linspace(0, 1, 101):
            xs = x_prev + ts * (x - x_prev)
            for ftype, pairs in ((cm.PT, pt), (cm.EE, ee)):
                if len(pairs):
                    D, _, _ = cm.resolve_features(xs, ftype, pairs)
                    assert D.min() > 0.0
        assert nh_min_J(x, o.mesh) > 0
    assert x[:4, 1].min() > 0.0  # above the plane


def test_bal_equals_plain_barrier_newton_fixed_point():
    """SPEC degeneracy check: with A' pinned empty and sigma fixed (plain IPC barrier Newton) the
    step converges to (nearly) the same state when no pair gets closer than 1e-2 dhat."""
    sc = scenes.make_single_tet(2, height=0.004, speed=0.05)
    o1 = Oracle(sc)
    o2 = Oracle(sc, flags=FLAG_NO_AUGLAG)
    x1, _, s1 = o1.step(sc["x0"], sc["v0"])
    x2, _, s2 = o2.step(sc["x0"], sc["v0"])
    assert np.linalg.norm(x1 - x2) <= 1e-6 * np.linalg.norm(x1 - sc["x0"]) + 1e-9


# ---------------------------------------------------------------- lumped mass
def test_lumped_mass_pins():
    """m_j = sum over the tets at j of rho V_e / 4: one tet of edge 0.1 m (V = 1e-3 / 6 m^3, by hand)
    gives rho V / 4 per node; the two C1 cubes (edge 1.0 m each, so total volume 2 m^3 from the scene
    recipe, not from the tets) give sum m = 2 rho; masses are positive."""
    from oracle.mesh import precompute
    sc = scenes.make_single_tet(0)
    m = precompute(sc)
    free = ~m.fixed
    np.testing.assert_allclose(m.mass[free], 1e3 * (1e-3 / 6.0) / 4.0, rtol=1e-12)
    c = scenes.make_cubes(1)
    mc = precompute(c)
    assert np.sum(mc.mass) == pytest.approx(2.0 * 1e3, rel=1e-12)
    assert np.all(mc.mass[~mc.fixed] > 0)


# ---------------------------------------------------------------- sigma^0 (Q7)
def test_sigma0_through_assembly_and_floor():
    """Oracle.sigma0 end to end: with the inertial predictor chosen so that the non-barrier gradient
    is g_E = -K g_b (y = x + h^2 M^-1 (grad Psi + K g_b)), the least-squares penalty is exactly K
    (Q7) whenever K exceeds the floor; with no active constraint sigma^0 is the floor m_bar / h^2."""
    from oracle.energy import nh_stencils
    sc = scenes.make_single_tet(3, height=0.0004)  # within dhat of the plane
    o = Oracle(sc)
    m = o.mesh
    x = sc["x0"].copy()
    pt, ee = cm.candidates(m, x, x, o.dhat)
    keys, _d = cm.constraint_set(x, pt, ee, o.dhat)
    assert len(keys) > 0
    N = o.N
    gb = np.zeros((N, 3))
    for ids, g, _H, _dd, _dp in cm.contact_stencils(x, keys, np.ones(len(keys)), np.zeros(len(keys)),
                                                    np.zeros(len(keys)), np.zeros(len(keys)), 1.0, o.dhat):
        gb[ids] += g.reshape(-1, 3)
    gpsi = np.zeros((N, 3))
    _v, g, _H = nh_stencils(x, m)
    for k in range(4):
        np.add.at(gpsi, m.tets[:, k], g[:, 3 * k:3 * k + 3])
    floor = float(np.mean(m.mass[~m.fixed])) / o.h ** 2
    K = 10.0 * floor
    y = x.copy()
    free = ~m.fixed
    y[free] = x[free] + o.h ** 2 * (gpsi[free] + K * gb[free]) / m.mass[free, None]
    st = dict(y=y, x_t=x, ap_keys=np.zeros((0, 5), np.int64), ap_mu=np.zeros(0), ap_s=np.zeros(0), fr_keys=None)
    assert o.sigma0(x, st, keys) == pytest.approx(K, rel=1e-9)
    assert o.sigma0(x, st, np.zeros((0, 5), np.int64)) == pytest.approx(floor, rel=1e-15)


# ---------------------------------------------------------------- literal readings
def test_literal_ccd_activation_stalls_the_line_search():
    """P:468's literal activation d_TOC < eps + dhat (flag, R-CCD2 off): on C1 a pair already within
    dhat that slides past a neighbouring primitive's plane is truncated every Newton iteration;
    alpha_CCD shrinks ~10x per iteration until the App. B resumes give up (the reason for R-CCD2)."""
    from oracle.bal import FLAG_CCD_LITERAL, NotConverged
    sc = scenes.make_cubes(1)
    sc["params"]["max_pcg"] = 400  # the App. B resumes give up sooner (the stall is the same)
    o = Oracle(sc, flags=FLAG_CCD_LITERAL)
    x, v = sc["x0"], sc["v0"]
    tr = []
    with pytest.raises(NotConverged):
        for _ in range(3):
            tr = []
            x, v, _s = o.step(x, v, tr)
    a = [t["alpha_ccd"] for t in tr][-4:]
    assert all(0.05 < a[i + 1] / a[i] < 0.2 for i in range(len(a) - 1)), a


def test_literal_residual_stagnation_stops_with_a_useless_direction():
    """Q15's literal residual-minimum test (flag, R-PCG1 off) on an ill-conditioned SPD system whose CG
    residual norm oscillates: it stops after one window with ||r|| above ||b|| (CG never improved on
    x0 = 0 in the residual norm), although the CG objective was still decreasing (the reason for
    R-PCG1's objective-based test)."""
    import scipy.sparse as sp
    from oracle import linalg as la
    rng = np.random.default_rng(0)
    n = 600
    A = sp.diags(np.logspace(0, 9, n)).tocsr()
    b = rng.normal(size=n)
    Dinv = np.tile(np.eye(3), (n // 3, 1, 1))
    lit = la.pcg(A, b, np.zeros(n), Dinv, tol=1e-4, window=100, max_iters=2000, literal_stall=True)
    assert lit.stop == la.STOP_STAGNATED and lit.k == 100
    assert lit.hist[-1] > lit.bnorm
    obj = la.pcg(A, b, np.zeros(n), Dinv, tol=1e-4, window=100, max_iters=2000)
    assert obj.stop == la.STOP_CAP  # the objective kept decreasing: no stagnation stop
    phi = lambda x: 0.5 * x @ (A @ x) - b @ x  # noqa: E731
    assert phi(obj.x) < phi(lit.x) < 0.0


def test_ccd_prefilter_is_result_neutral():
    """DESIGN.md R-CCD4: pairs far_pairs() drops are exactly pairs whose pair_toi is 1 -- on random
    pairs at every scale of distance vs displacement (far, grazing, colliding, in-plane motion),
    and step_toi with and without the prefilter agree bitwise."""
    rng = np.random.default_rng(37)
    dropped = 0
    for trial in range(600):
        ftype = cm.PT if trial % 2 == 0 else cm.EE
        x = rng.normal(size=(4, 3)) * 10.0 ** rng.uniform(-3, 0)
        dx = rng.normal(size=(4, 3)) * 10.0 ** rng.uniform(-4, 0)
        if trial % 7 == 0:
            x[:, 2] = 0.0
            dx[:, 2] = 0.0  # coplanar, in-plane motion: the identically-zero cubic
        ids = np.array([[0, 1, 2, 3]])
        D0, _, _ = cm.resolve_features(x, ftype, ids)
        if np.sqrt(D0[0]) < 1e-9:
            continue
        far = ccd.far_pairs(ftype, x, dx, ids, 1e-3)[0]
        if far:
            dropped += 1
            assert ccd.pair_toi(ftype, x, dx, ids[0], 1e-3) == 1.0
    assert dropped > 50
    sc = scenes.make_cubes(1)
    o = Oracle(sc)
    x1, _v, _ = o.step(sc["x0"], sc["v0"])
    dx = 0.004 * rng.normal(size=x1.shape) * (~o.mesh.fixed[:, None])
    pt, ee = cm.candidates(o.mesh, x1, x1 + dx, o.dhat)
    assert ccd.step_toi(x1, dx, pt, ee, o.dhat) == ccd.step_toi(x1, dx, pt, ee, o.dhat, prefilter=False)
