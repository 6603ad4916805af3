"""Pins of the oracle's distances, constraint keys, contact potentials and AL rules
(brute force, closed forms, FD).  CPU only."""
import numpy as np
import pytest

from oracle import contact as cm
from oracle.auglag import aprime_rule, dual_update, sigma_ls, sigma_schedule, slack
from oracle.energy import barrier


def brute_pt(p, a, b, c, n=400):
    u, v = np.meshgrid(np.linspace(0, 1, n + 1), np.linspace(0, 1, n + 1), indexing="ij")
    m = u + v <= 1
    q = a[None] + u[m][:, None] * (b - a)[None] + v[m][:, None] * (c - a)[None]
    return np.min(np.sum((q - p) ** 2, axis=1))


def brute_ee(a0, a1, b0, b1, n=400):
    s, t = np.meshgrid(np.linspace(0, 1, n + 1), np.linspace(0, 1, n + 1), indexing="ij")
    pa = a0[None] + s.ravel()[:, None] * (a1 - a0)[None]
    pb = b0[None] + t.ravel()[:, None] * (b1 - b0)[None]
    return np.min(np.sum((pa - pb) ** 2, axis=1))


def test_pt_distance_vs_grid_search():
    rng = np.random.default_rng(10)
    for _ in range(60):
        P, A, B, C = rng.normal(size=(4, 3))
        D, typ, loc = cm.resolve_pt(P[None], A[None], B[None], C[None])
        Dg = brute_pt(P, A, B, C)
        diam = max(np.linalg.norm(B - A), np.linalg.norm(C - A), np.linalg.norm(C - B))
        assert D[0] <= Dg * (1 + 1e-12)
        assert np.sqrt(Dg) - np.sqrt(D[0]) <= 2.0 * diam / 400


def test_ee_distance_vs_grid_search():
    rng = np.random.default_rng(11)
    for _ in range(60):
        A0, A1, B0, B1 = rng.normal(size=(4, 3))
        D, typ, loc = cm.resolve_ee(A0[None], A1[None], B0[None], B1[None])
        Dg = brute_ee(A0, A1, B0, B1)
        L = max(np.linalg.norm(A1 - A0), np.linalg.norm(B1 - B0))
        assert D[0] <= Dg * (1 + 1e-12)
        assert np.sqrt(Dg) - np.sqrt(D[0]) <= 2.0 * L / 400


def test_axis_aligned_cases():
    a, b, c = np.array([0.0, 0, 0]), np.array([1.0, 0, 0]), np.array([0.0, 1, 0])
    # interior: PT, d = 1
    D, t, loc = cm.resolve_pt(np.array([[0.2, 0.2, 1.0]]), a[None], b[None], c[None])
    assert t[0] == cm.PT and D[0] == pytest.approx(1.0, rel=1e-15)
    # beyond edge ab: PE with the edge (local 1,2), d^2 = 0.5^2 + 2^2
    D, t, loc = cm.resolve_pt(np.array([[0.5, -0.5, 2.0]]), a[None], b[None], c[None])
    assert t[0] == cm.PE and list(loc[0, :3]) == [0, 1, 2] and D[0] == pytest.approx(4.25, rel=1e-14)
    # beyond vertex b: PP
    D, t, loc = cm.resolve_pt(np.array([[2.0, -1.0, 0.0]]), a[None], b[None], c[None])
    assert t[0] == cm.PP and list(loc[0, :2]) == [0, 2] and D[0] == pytest.approx(2.0, rel=1e-14)
    # parallel unit edges offset by (0,1,0): degenerate -> point-edge, d = 1
    D, t, loc = cm.resolve_ee(np.array([[0.0, 0, 0]]), np.array([[1.0, 0, 0]]),
                              np.array([[0.0, 1, 0]]), np.array([[1.0, 1, 0]]))
    assert D[0] == pytest.approx(1.0, rel=1e-14) and t[0] == cm.PE
    # crossing skew edges: EE interior, d = 2
    D, t, loc = cm.resolve_ee(np.array([[-1.0, 0, 0]]), np.array([[1.0, 0, 0]]),
                              np.array([[0.0, -1, 2]]), np.array([[0.0, 1, 2]]))
    assert t[0] == cm.EE and D[0] == pytest.approx(4.0, rel=1e-14)


def test_feature_pairs_are_constraints_and_barrier_is_continuous():
    """R-DUP1: each vertex-triangle / edge-edge pair is its own constraint with its own feature
    distance, so the barrier sum is continuous when a vertex slides across a shared edge (merging
    the two point-edge duplicates, makes it jump by ~b(d))."""
    dhat = 1e-3
    x = np.array([[0.0, 0, 0], [1.0, 0, 0], [0.5, 1.0, -1.0], [0.5, -1.0, -1.0], [0.5, 0.0001, 0.0005]])
    # roof: triangles (0,1,2) and (0,3,1) share the ridge edge (0,1); point 4 hovers over the ridge
    pt = np.array([[4, 0, 1, 2], [4, 0, 3, 1]])
    keys, d = cm.constraint_set(x, pt, np.zeros((0, 4), np.int64), dhat)
    assert len(keys) == 2 and set(keys[:, 0]) == {cm.PT}
    np.testing.assert_allclose(d, np.hypot(0.0001, 0.0005), rtol=1e-12)
    # slide the vertex across the ridge at constant height above the roof: the sum stays smooth
    ys = np.linspace(-4e-4, 4e-4, 801)
    tot = []
    for yy in ys:
        xx = x.copy()
        xx[4] = [0.5, yy, 0.0005 - abs(yy)]
        k, dd = cm.constraint_set(xx, pt, np.zeros((0, 4), np.int64), dhat)
        tot.append(np.sum(barrier(dd, dhat)))
    jumps = np.abs(np.diff(tot))
    assert jumps.max() <= 0.02 * max(tot)


def test_contact_stencil_derivatives_fd():
    rng = np.random.default_rng(12)
    dhat = 1e-3
    # a PT pair in the interior region, distance 0.3 dhat, plus AL terms
    a, b, c = np.array([0.0, 0, 0]), np.array([1.0, 0.1, 0]), np.array([0.2, 1.0, 0.05])
    n = np.cross(b - a, c - a)
    n /= np.linalg.norm(n)
    p = 0.3 * a + 0.3 * b + 0.4 * c + 0.3 * dhat * n
    x = np.stack([p, a, b, c])
    for (ftype, ids) in ((cm.PT, np.array([0, 1, 2, 3])),):
        keys, d = cm.constraint_set(x, ids[None], np.zeros((0, 4), np.int64), dhat)
        assert len(keys) == 1 and keys[0, 0] == cm.PT
        inA, inAp = np.ones(1), np.ones(1)
        mu, s, sigma = np.array([3.0]), np.array([1e-4]), 50.0
        (sid, g, H, dd, _dp), = cm.contact_stencils(x, keys, inA, inAp, mu, s, sigma, dhat)

        def energy(xx):
            return cm.phi_energy(cm.key_distance(xx, keys), inA, inAp, mu, s, sigma, dhat)[0]

        eps = 1e-9
        gfd = np.zeros(12)
        for i in range(12):
            dx = np.zeros(12)
            dx[i] = eps
            xp = x.copy()
            xm = x.copy()
            xp[sid] += dx.reshape(4, 3)
            xm[sid] -= dx.reshape(4, 3)
            gfd[i] = (energy(xp) - energy(xm)) / (2 * eps)
        assert np.linalg.norm(gfd - g) <= 1e-5 * np.linalg.norm(g)
        # Hessian: FD of the AD gradient
        Hfd = np.zeros((12, 12))
        for i in range(12):
            dx = np.zeros(12)
            dx[i] = 1e-10
            xp = x.copy()
            xm = x.copy()
            xp[sid] += dx.reshape(4, 3)
            xm[sid] -= dx.reshape(4, 3)
            gp = cm.contact_stencils(xp, keys, inA, inAp, mu, s, sigma, dhat)[0][1]
            gm = cm.contact_stencils(xm, keys, inA, inAp, mu, s, sigma, dhat)[0][1]
            Hfd[:, i] = (gp - gm) / 2e-10
        assert np.linalg.norm(Hfd - H) <= 1e-4 * np.linalg.norm(H)
        assert np.allclose(H, H.T, rtol=0, atol=1e-10 * np.abs(H).max())


def test_slack_closed_form_vs_grid():
    """Eq. P:181 is the argmin over s >= 0 of mu c + sigma/2 c^2, c = dhat + s - d (eq:problem-s)."""
    rng = np.random.default_rng(13)
    dhat = 1e-3
    sgrid = np.arange(0, 5e-3, 1e-6)
    for _ in range(100):
        mu = rng.uniform(0, 5)
        sigma = 10 ** rng.uniform(2, 5)
        d = rng.uniform(0, 4e-3)
        c = dhat + sgrid - d
        obj = mu * c + 0.5 * sigma * c * c
        s_grid = sgrid[np.argmin(obj)]
        assert abs(slack(mu, sigma, dhat, d) - s_grid) <= 1e-6
    assert slack(0.0, 1.0, dhat, dhat) == 0.0
    assert slack(0.0, 1.0, dhat, 2 * dhat) == pytest.approx(1e-3, rel=1e-12)


def test_dual_update_and_schedules():
    dhat = 1e-3
    assert dual_update(1.0, 10.0, dhat, 0.0, 5e-4) == pytest.approx(1.0 + 10.0 * barrier(np.array([5e-4]), dhat)[0])
    assert dual_update(1.0, 10.0, dhat, 0.0, 2e-3) == 1.0
    assert sigma_schedule(5.0, 1.0, 0.5e-5, dhat) == 100.0   # first trigger jumps to 100 sigma0
    assert sigma_schedule(200.0, 1.0, 0.5e-5, dhat) == 240.0  # then x1.2
    assert sigma_schedule(200.0, 1.0, 2e-5, dhat) == 200.0    # strict < 1e-2 dhat
    assert aprime_rule(2e-5, 1e-5, False, dhat) == "clear"
    assert aprime_rule(5e-6, 6e-6, False, dhat) == "rebuild"
    assert aprime_rule(5e-6, 4e-6, True, dhat) == "rebuild"
    assert aprime_rule(5e-6, 4e-6, False, dhat) == "keep"


def test_sigma_ls_pins():
    rng = np.random.default_rng(14)
    gE = rng.normal(size=30)
    assert sigma_ls(-gE, gE) == pytest.approx(1.0, rel=1e-15)
    gb = rng.normal(size=30)
    s1 = sigma_ls(gb, gE)
    assert sigma_ls(7.0 * gb, 7.0 * gE) == pytest.approx(s1, rel=1e-14)
    # least squares: minimises ||sigma gb + gE||^2
    ss = np.linspace(s1 - 1, s1 + 1, 2001)
    r = [np.sum((s * gb + gE) ** 2) for s in ss]
    assert abs(ss[int(np.argmin(r))] - s1) <= 1e-3
    assert sigma_ls(np.zeros(3), gE[:3]) is None


def test_friction_closest_point_weights():
    """Gamma applied to the stencil equals closest-point difference; n is unit (Q26)."""
    rng = np.random.default_rng(15)
    x = rng.normal(size=(8, 3))
    keys = np.array([[cm.PT, 0, 1, 2, 3], [cm.EE, 4, 5, 6, 7], [cm.PE, 0, 4, 5, -1], [cm.PP, 1, 6, -1, -1]])
    G, n = cm.closest_point_weights(x, keys)
    d = cm.key_distance(x, keys)
    for i, k in enumerate(keys):
        kk = cm.NNODES[int(k[0])]
        diff = sum(G[i, j] * x[k[1 + j]] for j in range(kk))
        assert np.linalg.norm(diff) == pytest.approx(d[i], rel=1e-10)
        assert np.linalg.norm(n[i]) == pytest.approx(1.0, rel=1e-14)
        assert abs(G[i, :kk].sum()) < 1e-12  # weights sum to zero (translation invariance)
