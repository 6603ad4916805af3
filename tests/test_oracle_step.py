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
