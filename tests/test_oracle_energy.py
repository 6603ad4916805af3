"""Pins of the oracle's energies against closed forms, textbook special cases, invariants and
finite differences.  CPU only."""
import numpy as np
import pytest

from oracle.ad import D2
from oracle.energy import (barrier, barrier_ad, inertia_energy, inertia_grad, mollifier,
                           mollifier_of_sq_ad, nh_energy, nh_stencils)
from oracle.mesh import precompute


def one_tet_scene(X, E=1e5, nu=0.4, rho=1e3):
    return dict(rest_x=X, tets=np.array([[0, 1, 2, 3]]), node_fixed=np.zeros(4, np.uint8),
                tet_material=np.zeros(1, np.int32), materials=np.array([[E, nu, rho]]),
                obstacle_tris=np.zeros((0, 3), np.int32))


def rand_tet(rng):
    while True:
        X = rng.normal(size=(4, 3))
        if np.linalg.det(np.stack([X[1] - X[0], X[2] - X[0], X[3] - X[0]], 1)) > 0.3:
            return X


# ---------------------------------------------------------------- inertia
def test_inertia_closed_form():
    x = np.array([[1.0, 0, 0]])
    y = np.zeros((1, 3))
    m = np.array([2.0])
    assert inertia_energy(x, y, m, 1.0, np.array([True])) == pytest.approx(1.0, rel=1e-15)
    g = inertia_grad(x, y, m, 0.5, np.array([True]))
    np.testing.assert_allclose(g, [[8.0, 0, 0]], rtol=1e-15)


# ---------------------------------------------------------------- Neo-Hookean (Q1)
def test_nh_rest_zero_energy_and_gradient():
    rng = np.random.default_rng(0)
    for _ in range(5):
        X = rand_tet(rng)
        m = precompute(one_tet_scene(X))
        v, g, _ = nh_stencils(X, m)
        assert abs(v[0]) < 1e-12 * m.mu[0] * m.vol[0]
        L = np.cbrt(m.vol[0])
        assert np.max(np.abs(g)) <= 1e-12 * m.mu[0] * m.vol[0] / L


def test_nh_rest_hessian_is_linear_elastic_stiffness():
    """Textbook special case: Bonet-Wood NH linearises to mu eps:eps + lam/2 tr(eps)^2, whose tet
    stiffness is K_ab = V[mu((g_a.g_b)I + g_b g_a^T) + lam g_a g_b^T], g_a = grad of shape fn a."""
    rng = np.random.default_rng(1)
    for _ in range(5):
        X = rand_tet(rng)
        m = precompute(one_tet_scene(X))
        _, _, H = nh_stencils(X, m)
        Dm_inv = m.Dm_inv[0]
        G = np.zeros((4, 3))
        G[1:] = Dm_inv  # rows of D_m^{-1} are grad N_1..N_3
        G[0] = -G[1:].sum(0)
        mu, lam, V = m.mu[0], m.lam[0], m.vol[0]
        K = np.zeros((12, 12))
        for a in range(4):
            for b in range(4):
                K[3 * a:3 * a + 3, 3 * b:3 * b + 3] = V * (mu * (G[a] @ G[b] * np.eye(3) + np.outer(G[b], G[a]))
                                                         + lam * np.outer(G[a], G[b]))
        assert np.linalg.norm(H[0] - K) <= 1e-12 * np.linalg.norm(K)


def test_nh_uniform_scaling_closed_form():
    rng = np.random.default_rng(2)
    X = rand_tet(rng)
    m = precompute(one_tet_scene(X))
    mu, lam, V = m.mu[0], m.lam[0], m.vol[0]
    for s in (0.7, 1.0, 1.3, 2.0):
        x = X[0] + s * (X - X[0])
        v, g, _ = nh_stencils(x, m)
        psi = 1.5 * mu * (s * s - 1) - 3 * mu * np.log(s) + 4.5 * lam * np.log(s) ** 2
        assert v[0] == pytest.approx(V * psi, rel=1e-13, abs=1e-13 * mu * V)
        # dE/ds = V tr(P), P = (mu(s - 1/s) + 3 lam ln s / s) I
        dEds = float(g[0] @ (X - X[0]).ravel())
        P = mu * (s - 1 / s) + 3 * lam * np.log(s) / s
        assert dEds == pytest.approx(V * 3 * P, rel=1e-12, abs=1e-12 * mu * V)
        assert nh_energy(x, m) == pytest.approx(v[0], rel=1e-13, abs=1e-13 * mu * V)


def test_nh_invariances_and_fd():
    rng = np.random.default_rng(3)
    X = rand_tet(rng)
    m = precompute(one_tet_scene(X, E=1e6))
    x = X + 0.15 * rng.normal(size=(4, 3))
    v, g, H = nh_stencils(x, m)
    # translation null space
    for c in range(3):
        t = np.zeros((4, 3))
        t[:, c] = 1.0
        assert np.linalg.norm(H[0] @ t.ravel()) <= 1e-12 * np.linalg.norm(H[0])
        assert abs(g[0] @ t.ravel()) <= 1e-12 * np.linalg.norm(g[0])
    # rotation invariance
    Q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
    if np.linalg.det(Q) < 0:
        Q[:, 0] *= -1
    assert nh_energy(x @ Q.T, m) == pytest.approx(v[0], rel=1e-12)
    # central finite differences: gradient of energy, Hessian from gradient
    eps = 1e-6
    gfd = np.zeros(12)
    Hfd = np.zeros((12, 12))
    for i in range(12):
        dx = np.zeros(12)
        dx[i] = eps
        xp, xm = x + dx.reshape(4, 3), x - dx.reshape(4, 3)
        gfd[i] = (nh_energy(xp, m) - nh_energy(xm, m)) / (2 * eps)
        Hfd[:, i] = (nh_stencils(xp, m)[1][0] - nh_stencils(xm, m)[1][0]) / (2 * eps)
    assert np.linalg.norm(gfd - g[0]) <= 1e-6 * np.linalg.norm(g[0])
    assert np.linalg.norm(Hfd - H[0]) <= 1e-4 * np.linalg.norm(H[0])


def test_nh_inverted_is_infinite():
    rng = np.random.default_rng(4)
    X = rand_tet(rng)
    m = precompute(one_tet_scene(X))
    x = X.copy()
    x[3] = x[0] - (X[3] - X[0])  # reflect the apex through node 0's face region
    x[3] = X[0] + (X[0] - X[3])
    assert nh_energy(x, m) == np.inf


# ---------------------------------------------------------------- barrier
def test_barrier_values():
    dhat = 1e-3
    assert barrier(np.array([5e-4]), dhat)[0] == pytest.approx(1.732868e-7, rel=1e-6)
    assert barrier(np.array([5e-4]), dhat)[0] == pytest.approx(-(5e-4) ** 2 * np.log(0.5), rel=1e-15)
    assert np.all(barrier(np.array([dhat, 1.5 * dhat, 10.0]), dhat) == 0.0)
    d = np.linspace(1e-6, dhat * (1 - 1e-9), 1000)
    b = barrier(d, dhat)
    assert np.all(b > 0) and np.all(np.diff(b) < 0)  # strictly decreasing on (0, dhat)


def _b_derivs_by_hand(d, dh):
    """Hand differentiation of -(d-dh)^2 ln(d/dh) -- an independent check of the AD."""
    b1 = -2 * (d - dh) * np.log(d / dh) - (d - dh) ** 2 / d
    b2 = -2 * np.log(d / dh) - 4 * (d - dh) / d + (d - dh) ** 2 / d ** 2
    return b1, b2


def test_barrier_derivatives():
    dhat = 1e-3
    d = np.array([0.1 * dhat, 0.3 * dhat, 0.77 * dhat, dhat * (1 - 1e-6)])
    v = D2.variables(d[:, None])[0]
    b = barrier_ad(v, dhat)
    b1, b2 = _b_derivs_by_hand(d, dhat)
    np.testing.assert_allclose(b.g[:, 0], b1, rtol=1e-12)
    np.testing.assert_allclose(b.H[:, 0, 0], b2, rtol=1e-12)
    # survey pins at d = 0.1 dhat
    assert b.g[0, 0] == pytest.approx(-12.24465 * dhat, rel=1e-5)
    assert b.H[0, 0, 0] == pytest.approx(121.605, rel=1e-5)
    assert np.all(b.g[:, 0] < 0) and np.all(b.H[:, 0, 0] > 0)
    # C2 clamp at dhat: value, first and second derivatives -> 0
    v2 = D2.variables(np.array([[dhat * (1 - 1e-9)], [dhat], [2 * dhat]]))[0]
    b2_ = barrier_ad(v2, dhat)
    assert np.all(np.abs(b2_.v) < 1e-20) and np.all(np.abs(b2_.g) < 1e-14) and np.all(np.abs(b2_.H) < 1e-7)


# ---------------------------------------------------------------- mollifier (Q24)
def test_mollifier():
    eps = 1e-3 / 30
    assert mollifier(np.array(eps), eps) == pytest.approx(2 * eps / 3, rel=1e-15)
    assert mollifier(np.array(0.0), eps) == 0.0
    # AD of f(sqrt(q)) along w = (y, 0, 0): f'(y) from both sides of eps equals 1 (C^1)
    for y in (eps * (1 - 1e-9), eps * (1 + 1e-9)):
        w = D2.variables(np.array([[y]]))[0]
        f = mollifier_of_sq_ad(w * w, eps)
        assert f.g[0, 0] == pytest.approx(1.0, rel=1e-6)
    # inside: f'(y) = -y^2/eps^2 + 2y/eps, f'' = -2y/eps^2 + 2/eps
    y = 0.4 * eps
    w = D2.variables(np.array([[y]]))[0]
    f = mollifier_of_sq_ad(w * w, eps)
    assert f.g[0, 0] == pytest.approx(-y * y / eps ** 2 + 2 * y / eps, rel=1e-12)
    assert f.H[0, 0, 0] == pytest.approx(-2 * y / eps ** 2 + 2 / eps, rel=1e-12)
    # at w = 0 exactly: f = |w|^2/eps, Hessian 2/eps I
    w3 = D2.variables(np.zeros((1, 3)))
    q = w3[0] * w3[0] + w3[1] * w3[1] + w3[2] * w3[2]
    f0 = mollifier_of_sq_ad(q, eps)
    np.testing.assert_allclose(f0.H[0], 2 / eps * np.eye(3), rtol=1e-15)


# ---------------------------------------------------------------- ARAP (NEXT-4, R-ARAP)
def arap_tet_scene(X, E=1e5, nu=0.4, rho=1e3):
    sc = one_tet_scene(X, E, nu, rho)
    sc["material_model"] = np.array([1])
    return sc


def test_arap_is_zero_on_rotations_and_matches_scaling_closed_form():
    """Psi = mu ||F - R||^2 vanishes with its gradient for EVERY rotation of the rest shape (not only
    at rest); F = sI gives V * 3 mu (s - 1)^2 and gradient V P Dm^-T with P = 2 mu (s - 1) I."""
    rng = np.random.default_rng(50)
    for _ in range(5):
        X = rand_tet(rng)
        m = precompute(arap_tet_scene(X))
        Q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
        Q *= np.sign(np.linalg.det(Q))
        x = X @ Q.T + rng.normal(size=3)
        v, g, _ = nh_stencils(x, m)
        L = np.cbrt(m.vol[0])
        assert abs(v[0]) < 1e-12 * m.mu[0] * m.vol[0] and np.max(np.abs(g)) <= 1e-12 * m.mu[0] * m.vol[0] / L
        s = 1.0 + rng.uniform(-0.3, 0.5)
        v, g, _ = nh_stencils(s * X, m)
        assert v[0] == pytest.approx(m.vol[0] * 3 * m.mu[0] * (s - 1) ** 2, rel=1e-12)
        Gd = m.vol[0] * 2 * m.mu[0] * (s - 1) * m.Dm_inv[0].T  # columns: nodes 1..3
        np.testing.assert_allclose(g[0, 3:].reshape(3, 3), Gd.T, rtol=1e-11, atol=1e-12 * np.abs(Gd).max())


def test_arap_rest_hessian_and_twist_eigenvalues():
    """Rest Hessian = the linear-elastic tet stiffness with lam = 0 (||F - R||^2 -> eps:eps); at
    F = diag(s1, s2, s3) (a tet with D_m = I) the F-space Hessian along the twist direction
    e_i e_j^T - e_j e_i^T is V 4 mu (1 - 2 / (s_i + s_j)) (analytic ARAP eigensystem), and along the
    scaling direction e_i e_i^T it is V 2 mu."""
    rng = np.random.default_rng(51)
    X = rand_tet(rng)
    m = precompute(arap_tet_scene(X))
    _, _, H = nh_stencils(X, m)
    G = np.zeros((4, 3))
    G[1:] = m.Dm_inv[0]
    G[0] = -G[1:].sum(0)
    K = np.zeros((12, 12))
    for a in range(4):
        for b in range(4):
            K[3 * a:3 * a + 3, 3 * b:3 * b + 3] = m.vol[0] * m.mu[0] * (G[a] @ G[b] * np.eye(3) + np.outer(G[b], G[a]))
    assert np.linalg.norm(H[0] - K) <= 1e-11 * np.linalg.norm(K)
    X1 = np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]])
    m1 = precompute(arap_tet_scene(X1))
    sig = np.array([0.7, 1.1, 1.6])
    x = X1 * sig[None, :]  # F = diag(sig)
    _, _, H = nh_stencils(x, m1)
    HF = H[0][3:, 3:]  # F_rc = x[c+1][r]: index 3 c + r after dropping node 0
    V, mu = m1.vol[0], m1.mu[0]
    for i in range(3):
        for j in range(i + 1, 3):
            T = np.zeros((3, 3))
            T[i, j], T[j, i] = 1.0, -1.0
            t = T.T.ravel()  # t[3 c + r] = T[r, c]
            assert t @ HF @ t == pytest.approx(V * 4 * mu * (1 - 2 / (sig[i] + sig[j])), rel=1e-10)
        t = np.zeros(9)
        t[3 * i + i] = 1.0
        assert t @ HF @ t == pytest.approx(V * 2 * mu, rel=1e-10)


def test_arap_fd_and_energy_consistency():
    """AD gradient / Hessian vs central differences of the plain energy (nh_energy with the SVD) at
    random deformations; J <= 0 is +inf like NH."""
    rng = np.random.default_rng(52)
    for _ in range(3):
        X = rand_tet(rng)
        m = precompute(arap_tet_scene(X))
        x = X + 0.15 * rng.normal(size=X.shape)
        v, g, H = nh_stencils(x, m)
        assert v[0] == pytest.approx(nh_energy(x, m), rel=1e-12)
        h = 1e-6
        gfd = np.zeros(12)
        for k in range(12):
            xp, xm = x.copy().ravel(), x.copy().ravel()
            xp[k] += h
            xm[k] -= h
            gfd[k] = (nh_energy(xp.reshape(4, 3), m) - nh_energy(xm.reshape(4, 3), m)) / (2 * h)
        assert np.linalg.norm(gfd - g[0]) <= 1e-6 * np.linalg.norm(g[0])
        Hfd = np.zeros((12, 12))
        for k in range(12):
            xp, xm = x.copy().ravel(), x.copy().ravel()
            xp[k] += h
            xm[k] -= h
            Hfd[:, k] = (nh_stencils(xp.reshape(4, 3), m)[1][0] - nh_stencils(xm.reshape(4, 3), m)[1][0]) / (2 * h)
        assert np.linalg.norm(Hfd - H[0]) <= 1e-6 * np.linalg.norm(H[0])
    xi = X.copy()
    xi[[1, 2]] = xi[[2, 1]]
    assert nh_energy(xi, m) == np.inf
