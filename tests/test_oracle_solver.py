"""Pins of the oracle's projection, assembly, stiffness groups, SpMV, PCG and warm start
(SURVEY.md §8(c) c.3).  CPU only."""
import numpy as np
import pytest

import scenes
from oracle import linalg as la
from oracle.assemble import BlockSystem, floor_log10, stiffness_groups
from oracle.bal import Oracle
from oracle.projection import lambda_bar, project_eigh, project_jacobi


# ---------------------------------------------------------------- projection (Q21)
def test_projection_properties():
    rng = np.random.default_rng(20)
    for n in (6, 9, 12):
        A = rng.normal(size=(n, n))
        H = A + A.T
        P, wc = project_eigh(H[None])
        P = P[0]
        assert np.array_equal(P, P.T)
        assert np.linalg.eigvalsh(P).min() >= -1e-14 * np.linalg.norm(H)
        P2, _ = project_eigh(P[None])  # idempotent
        assert np.linalg.norm(P2[0] - P) <= 1e-13 * np.linalg.norm(H)
        Pj, _ = project_jacobi(H)       # unique nearest PSD matrix: any correct eigensolver agrees
        assert np.linalg.norm(Pj - P) <= 1e-13 * np.linalg.norm(H)
        # Frobenius-nearest: no random PSD matrix is closer
        for _ in range(20):
            B = rng.normal(size=(n, n))
            Q = P + 1e-3 * (B @ B.T)
            assert np.linalg.norm(H - Q) >= np.linalg.norm(H - P)
        assert lambda_bar(P[None])[0] == pytest.approx(np.mean(wc[0]), rel=1e-12)
        # PSD input unchanged
        S = A @ A.T
        Ps, _ = project_eigh(S[None])
        assert np.linalg.norm(Ps[0] - S) <= 1e-13 * np.linalg.norm(S)


# ---------------------------------------------------------------- groups (Q17-Q19)
def test_floor_log10_exact_decades():
    e = np.array([1.0, 9.999999999999999, 10.0, 1e4, 30003.0, 1e-3, 0.00099999999, 1e12 * (1 - 1e-16)])
    assert list(floor_log10(e)) == [0, 0, 1, 4, 4, -3, -4, 11]


def test_stiffness_group_examples():
    # one stencil over nodes 0-3 with lambda_bar = 1e4, m/h^2 = 1 -> e = 3(1e4 + 1) = 30003 -> group 4
    mass = np.ones(8)
    e, g = stiffness_groups(mass, 1.0, [np.array([0, 1, 2, 3])], [1e4], np.zeros(8, bool))
    assert e[0] == pytest.approx(30003.0) and g[0] == 4
    # two disjoint stencils 1e4 and 1e6 -> groups {4, 6}
    e, g = stiffness_groups(mass, 1.0, [np.array([0, 1, 2, 3]), np.array([4, 5, 6, 7])], [1e4, 1e6],
                            np.zeros(8, bool))
    assert set(g[:4]) == {4} and set(g[4:]) == {6}


# ---------------------------------------------------------------- assembly vs dense brute force
def _dense_brute(o, x, asm):
    """Sum_i S_i^T P(H_i) S_i + M/h^2 with explicit dense selection matrices (N small)."""
    m = o.mesh
    N = o.N
    A = np.diag(np.repeat(m.mass / o.h ** 2, 3))
    for e, tet in enumerate(m.tets):
        S = np.zeros((12, 3 * N))
        for a, n in enumerate(tet):
            S[3 * a:3 * a + 3, 3 * n:3 * n + 3] = np.eye(3)
        A += S.T @ asm["elastic_P"][e] @ S
    for ids, P in zip(asm["contact_ids"], asm["contact_P"]):
        S = np.zeros((3 * len(ids), 3 * N))
        for a, n in enumerate(ids):
            S[3 * a:3 * a + 3, 3 * n:3 * n + 3] = np.eye(3)
        A += S.T @ P @ S
    fd = np.repeat(m.fixed, 3)
    A[fd, :] = 0
    A[:, fd] = 0
    A[fd, fd] = 1.0
    return A


def test_assembly_matches_dense_and_is_spd():
    sc = scenes.make_single_tet(0, height=0.0004)  # within dhat of the plane: contact stencils too
    o = Oracle(sc)
    x = sc["x0"] + 1e-4 * np.random.default_rng(21).normal(size=sc["x0"].shape) * (~o.mesh.fixed[:, None])
    from oracle import contact as cm
    pt, ee = cm.candidates(o.mesh, x, x, o.dhat)
    keys, d = cm.constraint_set(x, pt, ee, o.dhat)
    assert len(keys) > 0
    st = dict(y=x.copy(), x_t=x.copy(), sigma=1e3, ap_keys=np.zeros((0, 5), np.int64), ap_mu=np.zeros(0),
              ap_s=np.zeros(0), fr_keys=None)
    asm = o.assemble(x, st, keys)
    A = asm["A"].toarray()
    Ad = _dense_brute(o, x, asm)
    assert np.linalg.norm(A - Ad) <= 1e-13 * np.linalg.norm(Ad)
    assert np.allclose(A, A.T, rtol=0, atol=1e-12 * np.abs(A).max())
    assert np.linalg.eigvalsh(A).min() > 0


def test_elastic_rows_annihilate_translations(cubes):
    o = Oracle(cubes)
    rng = np.random.default_rng(22)
    x = cubes["x0"] + 0.01 * rng.normal(size=cubes["x0"].shape) * (~o.mesh.fixed[:, None])
    from oracle.energy import nh_stencils
    from oracle.projection import project_eigh as pe
    _v, _g, H = nh_stencils(x, o.mesh)
    P, _ = pe(H)
    for c in range(3):
        t = np.zeros(12)
        t[c::3] = 1.0
        assert np.max(np.linalg.norm(P @ t, axis=1)) <= 1e-10 * np.max(np.linalg.norm(P, axis=(1, 2)))


# ---------------------------------------------------------------- SpMV / PCG / warm start
def _rand_spd_blocks(rng, N, density=0.3, cond_scale=1.0):
    bs = BlockSystem(N)
    for i in range(N):
        for j in range(i):
            if rng.uniform() < density:
                B = rng.normal(size=(3, 3)) * 0.3
                bs.add(i, j, B)
                bs.add(j, i, B.T)
    A = bs.to_dense()
    lam = np.linalg.eigvalsh(A).min()
    for i in range(N):
        bs.add(i, i, (abs(lam) + 1.0) * np.eye(3) * cond_scale ** rng.uniform(0, 1))
    return bs


def test_spmv_is_dense_product_and_symmetric():
    rng = np.random.default_rng(23)
    bs = _rand_spd_blocks(rng, 30)
    A = bs.to_csr()
    Ad = bs.to_dense()
    v, w = rng.normal(size=90), rng.normal(size=90)
    np.testing.assert_allclose(A @ v, Ad @ v, rtol=1e-13, atol=1e-13 * np.abs(Ad).max())
    assert float(v @ (A @ w)) == pytest.approx(float(w @ (A @ v)), rel=1e-12)


def test_pcg_special_cases_and_dense_solve():
    rng = np.random.default_rng(24)
    import scipy.sparse as sp
    # identity -> 1 iteration
    N = 10
    Dinv = np.tile(np.eye(3), (N, 1, 1))
    b = rng.normal(size=3 * N)
    st = la.pcg(sp.identity(3 * N, format="csr"), b, np.zeros(3 * N), Dinv, tol=1e-12)
    assert st.k == 1 and np.allclose(st.x, b)
    # diagonal with 3 distinct eigenvalues, identity preconditioner -> <= 3 iterations
    dg = np.repeat([1.0, 2.0, 3.0], N)
    A = sp.diags(dg).tocsr()
    st = la.pcg(A, b, np.zeros(3 * N), Dinv, tol=1e-12)
    assert st.k <= 3 and np.allclose(st.x, b / dg, rtol=1e-10)
    # random SPD vs dense solve
    bs = _rand_spd_blocks(rng, 25, cond_scale=1e3)
    A = bs.to_csr()
    Dinv = np.linalg.inv(bs.diag_blocks())
    b = rng.normal(size=75)
    st = la.pcg(A, b, np.zeros(75), Dinv, tol=1e-13, window=10 ** 9)
    xd = np.linalg.solve(bs.to_dense(), b)
    assert np.linalg.norm(st.x - xd) <= 1e-9 * np.linalg.norm(xd)
    # App. B stagnation: a stalled residual history stops the solve
    s2 = la.PCGState(np.zeros(3), np.ones(3), np.ones(3), np.ones(3), 1.0, [1.0] * 101, 1.0)
    s2.dec = [1.0] * 101  # CG objective did not decrease over the last 100 iterations (R-PCG1)
    la.pcg_run(sp.identity(3, format="csr"), np.tile(np.eye(3), (1, 1, 1)), s2, 1e-4, 100, 10 ** 6)
    assert s2.stop == la.STOP_STAGNATED


def test_pcg_chronopoulos_gear_special_cases_and_textbook_iterates():
    """pcg_cg (the GPU's single-reduction form) against closed forms and the textbook recurrences:
    identity -> 1 iteration; 3 distinct eigenvalues -> <= 3 iterations; dense solve; and for k <= 20
    the same iterates as Saad Alg. 9.1 (the two are equal in exact arithmetic)."""
    rng = np.random.default_rng(26)
    import scipy.sparse as sp
    N = 10
    Dinv = np.tile(np.eye(3), (N, 1, 1))
    b = rng.normal(size=3 * N)
    st = la.pcg_cg(sp.identity(3 * N, format="csr"), b, np.zeros(3 * N), Dinv, tol=1e-12)
    assert st.k == 1 and np.allclose(st.x, b)
    dg = np.repeat([1.0, 2.0, 3.0], N)
    st = la.pcg_cg(sp.diags(dg).tocsr(), b, np.zeros(3 * N), Dinv, tol=1e-12)
    assert st.k <= 3 and np.allclose(st.x, b / dg, rtol=1e-10)
    bs = _rand_spd_blocks(rng, 25, cond_scale=1e3)
    A = bs.to_csr()
    Dinv = np.linalg.inv(bs.diag_blocks())
    b = rng.normal(size=75)
    xd = np.linalg.solve(bs.to_dense(), b)
    st = la.pcg_cg(A, b, np.zeros(75), Dinv, tol=1e-13, window=10 ** 9)
    assert np.linalg.norm(st.x - xd) <= 1e-9 * np.linalg.norm(xd)
    x0 = rng.normal(size=75)
    for k in (1, 2, 5, 10, 20):
        a = la.pcg_cg(A, b, x0, Dinv, tol=0.0, window=10 ** 9, max_iters=k)
        t = la.pcg(A, b, x0, Dinv, tol=0.0, window=10 ** 9, max_iters=k)
        assert a.k == t.k == k
        assert np.linalg.norm(a.x - t.x) <= 1e-10 * np.linalg.norm(t.x)
        assert np.max(np.abs(np.subtract(a.hist, t.hist))) <= 1e-10 * t.hist[0]
        assert np.max(np.abs(np.subtract(a.dec, t.dec))) <= 1e-10 * t.dec[-1]


def test_warm_start_exact_on_decoupled_groups():
    rng = np.random.default_rng(25)
    b1 = _rand_spd_blocks(rng, 8)
    b2 = _rand_spd_blocks(rng, 6)
    bs = BlockSystem(14)
    for (i, j), B in b1.blocks.items():
        bs.add(i, j, B)
    for (i, j), B in b2.blocks.items():
        bs.add(i + 8, j + 8, 1e4 * B)
    A = bs.to_csr()
    Dinv = np.linalg.inv(bs.diag_blocks())
    groups = np.array([2] * 8 + [6] * 6)
    b = rng.normal(size=42)
    x0, it = la.warm_start(A, b, groups, Dinv, np.zeros(14, bool), tol=1e-14, max_iters=1000)
    xd = np.linalg.solve(bs.to_dense(), b)
    assert np.linalg.norm(x0 - xd) <= 1e-11 * np.linalg.norm(xd)
    st = la.pcg(A, b, x0, Dinv, tol=1e-10)
    assert st.k <= 1
    x0z, _ = la.warm_start(A, np.zeros(42), groups, Dinv, np.zeros(14, bool))
    assert np.all(x0z == 0)


def test_additive_schwarz_is_the_printed_sum_and_its_special_cases():
    """App. A two-level additive preconditioner, DESIGN.md R-AS1.
    (1) apply(r) equals the printed M^-1 = sum_i B_i^T (B_i A B_i^T)^-1 B_i with explicit 0/1
        block-mapping matrices B_i (3x3 node blocks + 9-node aggregates, a ragged last one);
    (2) A with no coupling between nodes: the aggregate inverses are blockdiag(D_j^-1), so
        M^-1 = 2 A^-1 and PCG from 0 lands on A^-1 b after ONE iteration (alpha = 1/2);
    (3) symmetric positive definite on a C1 system; (4) Chronopoulos-Gear == textbook iterates with it."""
    import scipy.sparse as sp
    rng = np.random.default_rng(31)
    bs = _rand_spd_blocks(rng, 22, cond_scale=1e2)  # 22 nodes: aggregates 9, 9, 4
    A = bs.to_csr()
    Dinv = np.linalg.inv(bs.diag_blocks())
    M = la.additive_schwarz(A, Dinv, 9)
    n = A.shape[0]
    Ad = A.toarray()
    Mi = np.zeros((n, n))
    sets = [[j] for j in range(22)] + [list(range(0, 9)), list(range(9, 18)), list(range(18, 22))]
    for nodes in sets:
        B = np.zeros((3 * len(nodes), n))
        for a, j in enumerate(nodes):
            B[3 * a:3 * a + 3, 3 * j:3 * j + 3] = np.eye(3)
        Mi += B.T @ np.linalg.inv(B @ Ad @ B.T) @ B
    for _ in range(3):
        r = rng.normal(size=n)
        assert np.linalg.norm(M(r) - Mi @ r) <= 1e-12 * np.linalg.norm(Mi @ r)
    # (2) decoupled nodes
    blocks = np.stack([np.eye(3) * (1.0 + j) + 0.1 * np.ones((3, 3)) for j in range(12)])
    Ab = sp.block_diag(list(blocks)).tocsr()
    Db = np.linalg.inv(blocks)
    b = rng.normal(size=36)
    st = la.pcg(Ab, b, np.zeros(36), la.additive_schwarz(Ab, Db, 9), tol=1e-13, window=10 ** 9)
    assert st.k == 1
    assert np.linalg.norm(st.x - np.linalg.solve(Ab.toarray(), b)) <= 1e-13 * np.linalg.norm(st.x)
    # (3) SPD on a C1 system (436 nodes: 48 aggregates of 9 + one of 4)
    sc = scenes.make_cubes(1)
    o = Oracle(sc)
    x = sc["x0"]
    st0 = dict(y=x.copy(), x_t=x.copy(), sigma=1.0, ap_keys=np.zeros((0, 5), np.int64), ap_mu=np.zeros(0),
               ap_s=np.zeros(0), fr_keys=None)
    asm = o.assemble(x, st0, np.zeros((0, 5), np.int64))
    Mc = la.additive_schwarz(asm["A"], asm["Dinv"], 9)
    Md = np.stack([Mc(e) for e in np.eye(asm["A"].shape[0])[:120]], axis=1)  # first 40 nodes' columns
    assert np.allclose(Md[:120], Md[:120].T, rtol=0, atol=1e-12 * np.abs(Md).max())
    assert np.linalg.eigvalsh(0.5 * (Md[:120] + Md[:120].T)).min() > 0
    # (4) both PCG forms with the additive preconditioner
    b = rng.normal(size=n)
    for k in (1, 5, 20):
        a = la.pcg_cg(A, b, np.zeros(n), M, tol=0.0, window=10 ** 9, max_iters=k)
        t = la.pcg(A, b, np.zeros(n), M, tol=0.0, window=10 ** 9, max_iters=k)
        assert np.linalg.norm(a.x - t.x) <= 1e-10 * np.linalg.norm(t.x)


def test_app_b_alternative_criteria_stop_where_defined():
    """NEXT-4, App. B criteria (i) ||r|| <= min(0.5, sqrt||b||) ||b||, (ii) ||r_k|| <=
    u kappa ||x_k||, (iii) ||r_k|| <= u kappa ||b|| in both PCG forms: each stops at the FIRST
    iteration whose residual meets its threshold (checked from outside: the run capped one iteration
    earlier does not meet it), and (iii) with u kappa = tol is the default relative-residual test."""
    rng = np.random.default_rng(41)
    bs = _rand_spd_blocks(rng, 30, cond_scale=1e4)
    A = bs.to_csr()
    Dinv = np.linalg.inv(bs.diag_blocks())
    n = A.shape[0]
    for scale in (1e-3, 1e2):  # sqrt||b|| below and above 0.5 for criterion (i)
        b = scale * rng.normal(size=n)
        bn = np.linalg.norm(b)
        for solve in (la.pcg, la.pcg_cg):
            for crit, thr in ((("i", 0.0), lambda st: min(0.5, np.sqrt(bn)) * bn),
                              (("ii", 1e-9), lambda st: 1e-9 * np.linalg.norm(st.x)),
                              (("iii", 1e-7), lambda st: 1e-7 * bn)):
                st = solve(A, b, np.zeros(n), Dinv, tol=1e-4, window=10 ** 9, crit=crit)
                assert st.stop == la.STOP_CONVERGED
                assert st.hist[-1] <= thr(st)
                if st.k > 0:
                    prev = solve(A, b, np.zeros(n), Dinv, tol=1e-4, window=10 ** 9, max_iters=st.k - 1, crit=crit)
                    assert prev.stop == la.STOP_CAP and prev.hist[-1] > thr(prev)
        a = la.pcg(A, b, np.zeros(n), Dinv, tol=1e-4, window=10 ** 9, crit=("iii", 1e-4))
        d = la.pcg(A, b, np.zeros(n), Dinv, tol=1e-4, window=10 ** 9)
        assert a.k == d.k and np.array_equal(a.x, d.x)
