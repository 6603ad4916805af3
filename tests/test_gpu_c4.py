"""GPU parity at BASELINE.json's full size (configs[3], the C4 puffer-net scene, ~1.75M tets) in the
launch configuration bench.py times: sampled outputs the oracle computes one by one (elastic
stencils of sampled tets, assembled rows of sampled nodes), the SpMV against the CSR product of the
assembled blocks over every row, and fixed-iteration PCG against the oracle's textbook PCG on the
same (GPU-assembled) system.  SURVEY §8(c) c.4; tolerances as north_star states."""
import numpy as np
import pytest

import scenes
from tests.gpu_helpers import bsr_to_csr, dinv_full, lower_blocks_to_full

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2407_00046_b200 as bal  # noqa: E402
from oracle import linalg as la  # noqa: E402
from oracle.energy import nh_stencils  # noqa: E402
from oracle.mesh import precompute  # noqa: E402
from oracle.projection import lambda_bar, project_eigh  # noqa: E402

DEV = torch.device("cuda:0")


def _t(a):
    return torch.as_tensor(np.ascontiguousarray(a, np.float64).ravel(), device=DEV)


def _np(t):
    return t.detach().cpu().numpy()


@pytest.fixture(scope="module")
def c4():
    sc = scenes.make_puffer_net(seed=4)
    m = precompute(sc)
    rng = np.random.default_rng(44)
    # a deformed, generic configuration: small random displacement of every free node
    x = sc["x0"] + 2e-4 * rng.normal(size=sc["x0"].shape) * (1 - sc["node_fixed"][:, None])
    p = sc["params"]
    y = x + p["h"] * sc["v0"] + p["h"] ** 2 * np.array(p["gravity"])[None]
    ctx = bal.bal_init(sc)
    out = bal.bal_assemble(ctx, _t(x), y=y)
    A = bsr_to_csr(_np(out["static_row_ptr"]), _np(out["static_col"]), _np(out["static_val"]), len(x))
    return sc, m, x, y, ctx, out, A


def _sub_mesh(m, sel):
    return type(m)(**{**m.__dict__, "tets": m.tets[sel], "Dm_inv": m.Dm_inv[sel], "vol": m.vol[sel],
                      "mu": m.mu[sel], "lam": m.lam[sel], "arap": m.arap[sel]})


def test_c4_sampled_elastic_stencils(c4):
    sc, m, x, y, ctx, out, A = c4
    rng = np.random.default_rng(1)
    sel = np.sort(rng.choice(len(m.tets), size=3000, replace=False))
    _v, _g, H = nh_stencils(x, _sub_mesh(m, sel))
    P, _ = project_eigh(H)
    lb = lambda_bar(P)
    Pg = _np(out["elastic_blocks"]).reshape(-1, 90)[sel]
    err = max(np.linalg.norm(lower_blocks_to_full(Pg[i], 4) - P[i]) / max(np.linalg.norm(P[i]), 1e-300)
              for i in range(len(sel)))
    assert err <= 1e-12, err
    np.testing.assert_allclose(_np(out["elastic_lbar"])[sel], lb, rtol=1e-12, atol=0)


def test_c4_sampled_assembled_rows(c4):
    """Rows of sampled free nodes: M/h^2 + sum over incident tets of S^T P(H) S, summed densely."""
    sc, m, x, y, ctx, out, A = c4
    rng = np.random.default_rng(2)
    N = len(x)
    free = np.flatnonzero(sc["node_fixed"] == 0)
    nodes = rng.choice(free, size=150, replace=False)
    p = sc["params"]
    flat = m.tets.ravel()
    order = np.argsort(flat, kind="stable")
    starts = np.searchsorted(flat[order], np.arange(N + 1))
    for i in nodes:
        tsel = np.unique(order[starts[i]:starts[i + 1]] // 4)
        _v, _g, H = nh_stencils(x, _sub_mesh(m, tsel))
        P, _ = project_eigh(H)
        row = np.zeros((3, 3 * N))
        row[:, 3 * i:3 * i + 3] += np.eye(3) * m.mass[i] / p["h"] ** 2
        for t, e in enumerate(tsel):
            a = int(np.flatnonzero(m.tets[e] == i)[0])
            for b in range(4):
                j = m.tets[e, b]
                if sc["node_fixed"][j]:
                    continue  # fixed DOFs: identity rows/columns (App. C, Q23)
                row[:, 3 * j:3 * j + 3] += P[t][3 * a:3 * a + 3, 3 * b:3 * b + 3]
        g = A[3 * i:3 * i + 3].toarray()
        scale = np.abs(row).sum()
        assert np.abs(g - row).sum() <= 1e-12 * scale, i


def test_c4_spmv_every_row(c4):
    sc, m, x, y, ctx, out, A = c4
    rng = np.random.default_rng(3)
    v = rng.normal(size=A.shape[0])
    yg = torch.empty(A.shape[0], dtype=torch.float64, device=DEV)
    bal.bal_spmv(ctx, _t(v), yg)
    yo = A @ v
    bound = abs(A) @ np.abs(v)
    assert np.all(np.abs(_np(yg) - yo) <= 1e-12 * bound + 1e-300)
    # bitwise deterministic run to run
    y2 = torch.empty_like(yg)
    bal.bal_spmv(ctx, _t(v), y2)
    assert torch.equal(yg, y2)


def test_c4_pcg_fixed_iterations(c4):
    """k block-Jacobi PCG iterations (no stopping) from x0 = 0 on the assembled C4 system: the GPU's
    single-reduction (Chronopoulos-Gear) PCG against the oracle's pcg_cg (1e-10) and the textbook
    recurrences (1e-8)."""
    sc, m, x, y, ctx, out, A = c4
    b = -_np(out["grad"])
    Dinv = dinv_full(_np(out["diag_inv"]))
    xg = torch.empty(A.shape[0], dtype=torch.float64, device=DEV)
    k = 50
    s = bal.bal_pcg(ctx, _t(b), _t(np.zeros_like(b)), xg, warm_start=0, rel_tol=0.0, stall_window=0, max_iters=k)
    st = la.pcg_cg(A, b, np.zeros_like(b), Dinv, tol=0.0, window=10 ** 9, max_iters=k)
    assert s["iters"] == k == st.k
    assert np.linalg.norm(_np(xg) - st.x) <= 1e-10 * np.linalg.norm(st.x)
    tb = la.pcg(A, b, np.zeros_like(b), Dinv, tol=0.0, window=10 ** 9, max_iters=k)
    assert np.linalg.norm(_np(xg) - tb.x) <= 1e-8 * np.linalg.norm(tb.x)


def test_c4_pcg_to_app_b_stop(c4):
    """A full solve on the C4 system under the App. B policy (Q14, R-PCG1): the GPU stops
    converged with ||b - A x|| <= 1e-4 ||b|| recomputed on the CPU from the returned x, or stagnated
    with the CG objective phi(x) = x'Ax/2 - b'x below phi(0) = 0 (a descent direction)."""
    sc, m, x, y, ctx, out, A = c4
    b = -_np(out["grad"])
    xg = torch.empty(A.shape[0], dtype=torch.float64, device=DEV)
    s = bal.bal_pcg(ctx, _t(b), _t(np.zeros_like(b)), xg, warm_start=0)
    xs = _np(xg)
    r = b - A @ xs
    assert s["stop_reason"] in (0, 1), s
    if s["stop_reason"] == 0:
        assert np.linalg.norm(r) <= 1.0001e-4 * np.linalg.norm(b)
    assert 0.5 * xs @ (A @ xs) - b @ xs < 0.0
    assert abs(np.linalg.norm(r) / np.linalg.norm(b) - s["rel_residual"]) <= 1e-6 * max(s["rel_residual"], 1e-4)


@pytest.fixture(scope="module")
def c4_contact():
    """C4 with one free ring translated (as a rigid body) until its closest feature pair to a
    neighbouring ring is 0.4 mm apart: a few hundred ring-ring constraints below dhat, found by the
    oracle's brute-force broad phase on the surface primitives of a 12 cm box around them."""
    import types

    import scipy.sparse as sp
    from scipy.sparse.csgraph import connected_components

    from oracle import contact as cm
    sc = scenes.make_puffer_net(seed=4)
    m = precompute(sc)
    N = len(sc["x0"])
    x = sc["x0"].copy()
    e = m.tets[:, [0, 1, 1, 2, 2, 3]].reshape(-1, 2)
    _nc, lab = connected_components(sp.coo_matrix((np.ones(len(e)), (e[:, 0], e[:, 1])), shape=(N, N)),
                                    directed=False)
    net = np.zeros(N, bool)
    net[np.unique(m.tets[sc["tet_material"] == 1])] = True
    free_net = np.flatnonzero(net & ~m.fixed)
    c = x[free_net[len(free_net) // 2]]
    inside = np.all(np.abs(x - c) < 0.06, axis=1)
    sub = types.SimpleNamespace(surf_verts=m.surf_verts[inside[m.surf_verts]], tris=m.tris[inside[m.tris].all(1)],
                                edges=m.edges[inside[m.edges].all(1)], fixed=m.fixed)
    dhat = sc["params"]["dhat"]
    pt, ee = cm.candidates(sub, x, x, 8e-3)
    keys8, d8 = cm.constraint_set(x, pt, ee, 8e-3)
    k = keys8[np.argmin(d8)][None]
    body = lab == lab[k[0, 1]]
    for _ in range(3):  # Newton on the rigid translation of `body` along grad d
        d0 = cm.key_distance(x, k)[0]
        g = np.zeros(3)
        for a in range(3):
            x3 = x.copy()
            x3[body, a] += 1e-6
            g[a] = (cm.key_distance(x3, k)[0] - d0) / 1e-6
        x[body] -= (d0 - 4e-4) * g / (g @ g)
    keys, d = cm.constraint_set(x, pt, ee, dhat)
    assert len(keys) > 50 and d.min() > 3e-4
    return sc, m, x, keys, d


def test_c4_contact_stencils_and_spmv_with_contacts(c4_contact):
    from oracle import contact as cm
    sc, m, x, keys, d = c4_contact
    dhat = sc["params"]["dhat"]
    sigma = 2.3e4
    ctx = bal.bal_init(sc)
    out = bal.bal_assemble(ctx, _t(x), active_keys=keys, sigma=sigma)
    n = len(keys)
    cs = cm.contact_stencils(x, keys, np.ones(n), np.zeros(n), np.zeros(n), np.zeros(n), sigma, dhat)
    nodes = _np(out["contact_stencil_nodes"]).reshape(-1, 4)
    blocks = _np(out["contact_blocks"]).reshape(-1, 90)
    assert len(nodes) == n
    worst = 0.0
    for i, (ids, _g, H, dd, _dp) in enumerate(cs):
        k = len(ids)
        assert list(nodes[i, :k]) == list(ids) and np.all(nodes[i, k:] == -1)
        P, _ = project_eigh(H[None])
        Hg = lower_blocks_to_full(blocks[i], k)
        tol = 1e-12 + 4e-15 * np.abs(x).max() / dd  # DESIGN.md contact parity tolerance
        worst = max(worst, np.linalg.norm(Hg - P[0]) / max(np.linalg.norm(P[0]), 1e-300) / tol)
    assert worst <= 1.0, worst
    # SpMV over the full system (static + contact BSR) in the bench's launch configuration
    N = len(x)
    A = bsr_to_csr(_np(out["static_row_ptr"]), _np(out["static_col"]), _np(out["static_val"]), N)
    assert out["contact_col"].numel() > 0
    A = A + bsr_to_csr(_np(out["contact_row_ptr"]), _np(out["contact_col"]), _np(out["contact_val"]), N)
    v = np.random.default_rng(5).normal(size=3 * N)
    yg = torch.empty(3 * N, dtype=torch.float64, device=DEV)
    bal.bal_spmv(ctx, _t(v), yg)
    assert np.all(np.abs(_np(yg) - A @ v) <= 1e-12 * (abs(A) @ np.abs(v)) + 1e-300)


# --------------------------------------------------------------------------- contact-rich C4 start
@pytest.fixture(scope="module")
def c4_settled():
    """The bench workload: C4's contact-rich start (scenes.make_puffer_net(settled=True)), after one
    inexact-Newton iteration of its first frame (the library's own constraint set, ~2.5e5 pairs)."""
    sc = scenes.make_puffer_net(seed=4, settled=True)
    ctx = bal.bal_init(sc)
    x = torch.as_tensor(sc["x0"].ravel(), device=DEV)
    v = torch.as_tensor(sc["v0"].ravel(), device=DEV)
    bal.bal_frame_begin(ctx, x, v)
    bal.bal_frame_iterate(ctx, 1)
    out = bal.bal_get_system(ctx)
    return sc, ctx, out


def test_c4_settled_spmv_every_row_with_paper_scale_contacts(c4_settled):
    """SpMV over every row of the static + contact system at paper-scale contact load (228K
    avg / 292K max constraints) in the bench's launch configuration: element-wise 1e-12 of |A||v|
    against the CSR product of the assembled blocks, bitwise repeatable."""
    sc, ctx, out = c4_settled
    assert bal.bal_get_trace(ctx, max_records=8)[-1]["nA"] > 2e5
    N = len(sc["x0"])
    A = bsr_to_csr(_np(out["static_row_ptr"]), _np(out["static_col"]), _np(out["static_val"]), N)
    assert out["contact_col"].numel() > 5e5
    A = A + bsr_to_csr(_np(out["contact_row_ptr"]), _np(out["contact_col"]), _np(out["contact_val"]), N)
    v = np.random.default_rng(6).normal(size=3 * N)
    yg = torch.empty(3 * N, dtype=torch.float64, device=DEV)
    bal.bal_spmv(ctx, _t(v), yg)
    assert np.all(np.abs(_np(yg) - A @ v) <= 1e-12 * (abs(A) @ np.abs(v)) + 1e-300)
    y2 = torch.empty_like(yg)
    bal.bal_spmv(ctx, _t(v), y2)
    assert torch.equal(yg, y2)


def test_c4_settled_pcg_iterates(c4_settled):
    """20 single-reduction PCG iterations on the contact-rich system vs the oracle's pcg_cg (1e-10)."""
    sc, ctx, out = c4_settled
    N = len(sc["x0"])
    A = bsr_to_csr(_np(out["static_row_ptr"]), _np(out["static_col"]), _np(out["static_val"]), N)
    A = A + bsr_to_csr(_np(out["contact_row_ptr"]), _np(out["contact_col"]), _np(out["contact_val"]), N)
    b = -_np(out["grad"])
    Dinv = dinv_full(_np(out["diag_inv"]))
    xg = torch.empty(3 * N, dtype=torch.float64, device=DEV)
    s = bal.bal_pcg(ctx, _t(b), _t(np.zeros_like(b)), xg, warm_start=0, rel_tol=0.0, stall_window=0, max_iters=20)
    st = la.pcg_cg(A, b, np.zeros_like(b), Dinv, tol=0.0, window=10 ** 9, max_iters=20)
    assert s["iters"] == 20 == st.k
    assert np.linalg.norm(_np(xg) - st.x) <= 1e-10 * np.linalg.norm(st.x)


def test_c4_settled_fp32_matrix_spmv():
    """BAL_FP32_MATRIX on the bench workload: static blocks streamed in FP32, contact blocks FP64: the
    product over every row equals the CSR product of (FP32-rounded static + FP64 contact) blocks."""
    sc = scenes.make_puffer_net(seed=4, settled=True)
    ctx = bal.bal_init(sc, flags=bal.BAL_FP32_MATRIX)
    x = torch.as_tensor(sc["x0"].ravel(), device=DEV)
    v0 = torch.as_tensor(sc["v0"].ravel(), device=DEV)
    bal.bal_frame_begin(ctx, x, v0)
    bal.bal_frame_iterate(ctx, 1)
    out = bal.bal_get_system(ctx)
    N = len(sc["x0"])
    As = bsr_to_csr(_np(out["static_row_ptr"]), _np(out["static_col"]), _np(out["static_val"]), N)
    As.data = As.data.astype(np.float32).astype(np.float64)
    A = As + bsr_to_csr(_np(out["contact_row_ptr"]), _np(out["contact_col"]), _np(out["contact_val"]), N)
    v = np.random.default_rng(7).normal(size=3 * N)
    yg = torch.empty(3 * N, dtype=torch.float64, device=DEV)
    bal.bal_spmv(ctx, _t(v), yg)
    assert np.all(np.abs(_np(yg) - A @ v) <= 1e-12 * (abs(A) @ np.abs(v)) + 1e-300)
