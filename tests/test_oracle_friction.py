"""Pins of the oracle's friction (§4.1; SPEC S:195-223, S:580,
S:587): finite differences of D against its AD stencils for every resolved sub-type, the force
closed form, lambda = -phi'(d) written out by hand, anchor invariances, and the incline physics
(closed-form creep velocity when sticking, closed-form acceleration when sliding).  CPU only."""
import numpy as np
import pytest

import scenes
from oracle import contact as cm
from oracle.bal import Oracle

CHI, EPS_V, H = 0.3, 1e-3, 1.0 / 30.0
EPS = EPS_V * H


def _config(rng, sub):
    """Positions (4,3) and a key whose resolved sub-type at x is `sub`."""
    if sub == cm.PT:   # point above the interior of a triangle
        tri = np.array([[0.0, 0, 0], [1.0, 0, 0], [0.0, 1.0, 0]]) + rng.normal(scale=0.05, size=(3, 3))
        p = np.array([0.25, 0.3, 0.0]) + np.array([0, 0, 0.3 + rng.uniform()])
        x = np.vstack([p, tri])
        key = [cm.PT, 0, 1, 2, 3]
    elif sub == cm.EE:  # two crossing edges
        a = np.array([[-1.0, 0, 0], [1.0, 0, 0]]) + rng.normal(scale=0.05, size=(2, 3))
        b = np.array([[0.0, -1.0, 0.4], [0.0, 1.0, 0.4]]) + rng.normal(scale=0.05, size=(2, 3))
        x = np.vstack([a, b])
        key = [cm.EE, 0, 1, 2, 3]
    elif sub == cm.PE:
        e = np.array([[-1.0, 0, 0], [1.0, 0, 0]]) + rng.normal(scale=0.05, size=(2, 3))
        p = np.array([0.1, 0.5, 0.2]) + rng.normal(scale=0.05, size=3)
        x = np.vstack([p, e, [[5.0, 5.0, 5.0]]])
        key = [cm.PE, 0, 1, 2, -1]
    else:
        x = np.vstack([rng.normal(size=3), rng.normal(size=3) + 2.0, [[5.0, 5, 5], [6.0, 6, 6]]])
        key = [cm.PP, 0, 1, -1, -1]
    keys = np.array([key], np.int64)
    _, s, _ = cm.resolve_features(x, int(key[0]), keys[:, 1:5])
    assert int(s[0]) == sub
    return x, keys


def _start_state(rng, x, keys, y_over_eps):
    """x_t such that the tangential displacement of the pair at x is y_over_eps * EPS."""
    G, n = cm.closest_point_weights(x, keys)
    t = np.cross(n[0], rng.normal(size=3))
    t /= np.linalg.norm(t)
    k = cm.NNODES[int(keys[0, 0])]
    ids = keys[0, 1:1 + k]
    # move only the first node back: Gamma[0] = +1 (or 1-a for EE) scales the relative motion
    x_t = x.copy()
    x_t[ids[0]] -= (y_over_eps * EPS / G[0, 0]) * t
    return x_t, G, n


@pytest.mark.parametrize("sub", [cm.PT, cm.EE, cm.PE, cm.PP])
def test_friction_stencil_fd_all_subtypes(sub):
    """AD gradient / Hessian of D_j (frozen anchors) against central differences of the separately
    coded energy, 20 random configurations per sub-type, both the sticking (y < eps) and sliding
    (y > eps) branches of f (SPEC S:580 acceptance 2: rel err < 1e-4)."""
    rng = np.random.default_rng(40 + sub)
    for trial in range(20):
        x, keys = _config(rng, sub)
        r = [0.3, 0.7, 1.5, 3.0][trial % 4]
        x_t, G, n = _start_state(rng, x, keys, r)
        # evaluate at a perturbed point (anchors stay those of x)
        xe = x + rng.normal(scale=0.02 * EPS, size=x.shape)
        lam = np.array([rng.uniform(0.5, 50.0)])
        (ids, g, Hs), = cm.friction_stencils(xe, x_t, keys, G, n, lam, CHI, EPS_V, H)
        k = len(ids)

        def energy(z):
            xx = xe.copy()
            xx[ids] = z.reshape(k, 3)
            return cm.friction_energy(xx, x_t, keys, G, n, lam, CHI, EPS_V, H)

        z0 = xe[ids].ravel()
        step = 1e-4 * EPS
        fd = np.array([(energy(z0 + step * e) - energy(z0 - step * e)) / (2 * step) for e in np.eye(3 * k)])
        assert np.linalg.norm(fd - g) <= 1e-4 * np.linalg.norm(g) + 1e-14
        def gfun(z):
            return cm.friction_stencils(_put(xe, ids, z), x_t, keys, G, n, lam, CHI, EPS_V, H)[0][1]

        fdH = np.array([(gfun(z0 + step * e) - gfun(z0 - step * e)) / (2 * step) for e in np.eye(3 * k)])
        assert np.linalg.norm(fdH - Hs) <= 1e-4 * np.linalg.norm(Hs)
        # symmetric, PSD (analytically, P:340 Q24 reading; projection is not applied to friction)
        assert np.allclose(Hs, Hs.T, rtol=0, atol=1e-12 * np.abs(Hs).max())
        assert np.linalg.eigvalsh(Hs).min() >= -1e-10 * np.abs(Hs).max()


def _put(x, ids, z):
    xx = x.copy()
    xx[ids] = z.reshape(len(ids), 3)
    return xx


def test_friction_force_closed_form():
    """Point over a triangle interior: grad_p D = chi lam f'(y) w_hat with w the tangential part of
    the relative displacement, f'(y) = 1 when sliding, 2y/eps - y^2/eps^2 when sticking; the triangle
    nodes carry -beta_k times it (action = reaction), no normal component (P_n)."""
    rng = np.random.default_rng(50)
    for y_over in (0.25, 0.6, 2.0, 7.0):
        x, keys = _config(rng, cm.PT)
        x_t, G, n = _start_state(rng, x, keys, y_over)
        lam = np.array([3.7])
        (ids, g, _H), = cm.friction_stencils(x, x_t, keys, G, n, lam, CHI, EPS_V, H)
        u = sum(G[0, j] * (x[ids[j]] - x_t[ids[j]]) for j in range(4))
        w = u - np.dot(u, n[0]) * n[0]
        y = np.linalg.norm(w)
        assert y == pytest.approx(y_over * EPS, rel=1e-9)
        fp = 1.0 if y >= EPS else 2 * y / EPS - y * y / EPS ** 2
        f_p = CHI * lam[0] * fp * w / y
        np.testing.assert_allclose(g[0:3], f_p, rtol=1e-10, atol=1e-14 * CHI * lam[0])
        for j in (1, 2, 3):
            np.testing.assert_allclose(g[3 * j:3 * j + 3], G[0, j] * f_p, rtol=1e-10, atol=1e-14 * CHI * lam[0])
        assert abs(np.dot(g[0:3], n[0])) <= 1e-12 * np.linalg.norm(g[0:3])


def _barrier_prime(d, dh):
    """d/dd of b(d, dh) = -(d - dh)^2 ln(d/dh) (eq:IPC-barrier), by hand."""
    return -2.0 * (d - dh) * np.log(d / dh) - (d - dh) ** 2 / d


def test_lambda_is_minus_phi_prime_by_hand():
    """lambda_j = -phi_j'(d_j) at x^l (Q25): for a pair in A only, sigma |b'(d; dhat)|; for a pair
    also in A' (multiplier mu, slack s), + mu - sigma b'(d; dhat + s) (eq:aug-lag)."""
    sc = scenes.make_incline(0, ratio=0.8, chi=CHI)
    o = Oracle(sc)
    x = sc["x0"].copy()
    pt, ee = cm.candidates(o.mesh, x, x, o.dhat)
    keys, d = cm.constraint_set(x, pt, ee, o.dhat)
    assert len(keys) == 3
    sigma, dh = 7.5, o.dhat
    st = dict(ap_keys=np.zeros((0, 5), np.int64), ap_mu=np.zeros(0), ap_s=np.zeros(0), sigma=sigma)
    fk, G, n, lam = o.friction_anchors(x, st, keys)
    np.testing.assert_array_equal(fk, keys)
    np.testing.assert_allclose(lam, -sigma * _barrier_prime(d, dh), rtol=1e-12)
    assert np.all(lam > 0)
    # the first pair also in A' with mu = 2.5, s = 1e-4
    st = dict(ap_keys=keys[:1].copy(), ap_mu=np.array([2.5]), ap_s=np.array([1e-4]), sigma=sigma)
    _fk, _G, _n, lam2 = o.friction_anchors(x, st, keys)
    hand = -sigma * _barrier_prime(d[0], dh) + 2.5 - sigma * _barrier_prime(d[0], dh + 1e-4)
    assert lam2[0] == pytest.approx(hand, rel=1e-12)
    np.testing.assert_allclose(lam2[1:], lam[1:], rtol=1e-15)
    # normals point from the triangle to the vertex, i.e. along the incline normal here
    # (d = 5e-4 m between points of magnitude ~0.3 m: n carries ~u |x| / d rounding)
    np.testing.assert_allclose(n, np.tile(sc["incline_normal"], (3, 1)), atol=1e-10)


def test_anchors_static_and_rigid_invariance():
    """Static configuration across two iterations -> identical anchors; a rigid translation
    of everything leaves Gamma, n and lambda unchanged (they depend on relative geometry only)."""
    sc = scenes.make_incline(3, ratio=0.8, chi=CHI)
    o = Oracle(sc)
    x = sc["x0"].copy()
    pt, ee = cm.candidates(o.mesh, x, x, o.dhat)
    keys, _d = cm.constraint_set(x, pt, ee, o.dhat)
    st = dict(ap_keys=np.zeros((0, 5), np.int64), ap_mu=np.zeros(0), ap_s=np.zeros(0), sigma=3.0)
    a1 = o.friction_anchors(x, st, keys)
    a2 = o.friction_anchors(x.copy(), st, keys)
    for u, v in zip(a1, a2):
        np.testing.assert_array_equal(u, v)
    a3 = o.friction_anchors(x + np.array([0.3, -0.2, 0.7]), st, keys)
    for u, v in zip(a1[1:], a3[1:]):
        np.testing.assert_allclose(u, v, rtol=1e-7, atol=1e-9)


def _run_incline(ratio, steps):
    sc = scenes.make_incline(0, ratio=ratio, chi=CHI)
    o = Oracle(sc)
    x, v = sc["x0"], sc["v0"]
    vd = []
    for _ in range(steps):
        tr = []
        x, v, _s = o.step(x, v, trace=tr)
        assert tr[-1]["rel_e"] <= 1e-4
        vd.append(float(v[:4].mean(0) @ sc["incline_down"]))
    return sc, np.array(vd)


def test_incline_sticks_with_closed_form_creep():
    """tan(theta) = 0.8 chi: quasi-static.  In the mollified stick branch the friction
    force chi lam f'(y) balances m g sin(theta) with lam = m g cos(theta), so f'(y) = tan(theta)/chi
    = r and the steady creep is y = eps (1 - sqrt(1 - r)) per step, i.e. v = eps_v (1 - sqrt(1 - r))
    -- below eps_v h drift per step, as S:587 requires."""
    _sc, vd = _run_incline(0.8, 8)
    v_star = EPS_V * (1.0 - np.sqrt(1.0 - 0.8))
    assert vd[-1] == pytest.approx(v_star, rel=2e-3)
    assert vd[-1] * H < EPS_V * H
    assert abs(vd[-1] - vd[-2]) <= 1e-3 * v_star


def test_incline_slides_with_closed_form_acceleration():
    """tan(theta) = 1.2 chi: slides persistently; in the sliding branch (f' = 1) the net force is
    m g (sin(theta) - chi cos(theta)), so backward Euler gains dv = g h (sin - chi cos) per step."""
    _sc, vd = _run_incline(1.2, 6)
    th = np.arctan(1.2 * CHI)
    dv = 9.81 * H * (np.sin(th) - CHI * np.cos(th))
    assert np.all(np.diff(vd) > 0)
    np.testing.assert_allclose(np.diff(vd)[2:], dv, rtol=2e-3)
