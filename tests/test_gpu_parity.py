"""GPU parity: the CUDA path through the C ABI vs the CPU oracle on identical seeded inputs
(SURVEY.md §8(c) c.4).  Requires a B200 and the built libbal.so."""
import numpy as np
import pytest

import scenes
from tests.gpu_helpers import (assembly_bounds, bsr_to_csr, check_assembly_bounds, csr_to_bsr, dinv_full,
                               lower_blocks_to_full, oracle_state)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2407_00046_b200 as bal  # noqa: E402  (fails loudly if libbal.so is missing)
from oracle import contact as cm  # noqa: E402
from oracle import linalg as la  # noqa: E402
from oracle.bal import Oracle  # noqa: E402

DEV = torch.device("cuda:0")


def _t(a):
    return torch.as_tensor(np.ascontiguousarray(a, np.float64).ravel(), device=DEV)


def _np(t):
    return t.detach().cpu().numpy()


@pytest.fixture(scope="module")
def cubes_state():
    """C1 after one oracle step: contact-rich, deformed, generic."""
    sc = scenes.make_cubes(1)
    o = Oracle(sc)
    x1, v1, _ = o.step(sc["x0"], sc["v0"])
    return sc, o, x1, v1


# --------------------------------------------------------------------------- elastic (a3, a6)
def test_elastic_stencils_and_static_assembly_parity():
    sc = scenes.perturbed(scenes.make_cubes(1), seed=5, scale=0.02)
    o = Oracle(sc)
    ctx = bal.bal_init(sc)
    x = sc["x0"]
    rng = np.random.default_rng(6)
    y = x + 0.01 * rng.normal(size=x.shape)
    out = bal.bal_assemble(ctx, _t(x), y=y)
    st = oracle_state(o, x, y=y)
    asm = o.assemble(x, st, np.zeros((0, 5), np.int64))
    # per-stencil projected Hessians (lower blocks) and lambda_bar
    Pg = _np(out["elastic_blocks"]).reshape(-1, 90)
    worst = 0.0
    for e in range(len(sc["tets"])):
        Hg = lower_blocks_to_full(Pg[e], 4)
        Ho = asm["elastic_P"][e]
        err = np.linalg.norm(Hg - Ho) / max(np.linalg.norm(Ho), 1e-300)
        worst = max(worst, err)
    assert worst <= 1e-12, worst
    np.testing.assert_allclose(_np(out["elastic_lbar"]), asm["elastic_lbar"], rtol=1e-12, atol=0)
    # assembled system (static part only: no contacts), gradient, Lambda, groups, D^{-1}
    N = o.N
    Ag = bsr_to_csr(_np(out["static_row_ptr"]), _np(out["static_col"]), _np(out["static_val"]), N)
    Ao = asm["A"]
    D = (Ag - Ao).tocsr()
    absA = abs(Ao)
    rowscale = np.asarray(absA.sum(axis=1)).ravel() + 1e-300
    assert np.max(np.abs(D).sum(axis=1).A.ravel() / rowscale) <= 1e-12
    ge = _np(out["grad"])
    assert np.linalg.norm(ge - asm["grad"]) <= 1e-12 * np.linalg.norm(asm["grad"])
    np.testing.assert_allclose(_np(out["e_node"])[o.free], asm["e_j"][o.free], rtol=1e-13)
    assert np.array_equal(_np(out["group"])[o.free], asm["groups"][o.free])
    Dinv = dinv_full(_np(out["diag_inv"]))
    rel = np.linalg.norm(Dinv - asm["Dinv"], axis=(1, 2)) / np.linalg.norm(asm["Dinv"], axis=(1, 2))
    assert rel.max() <= 1e-12


# --------------------------------------------------------------------------- contact (a4, a6)
def test_contact_stencils_and_full_assembly_parity(cubes_state):
    sc, o, x1, v1 = cubes_state
    x = x1
    dhat = o.dhat
    pt, ee = cm.candidates(o.mesh, x, x, dhat)
    keys, d = cm.constraint_set(x, pt, ee, dhat)
    assert len(keys) > 10
    # an A' with the closest few pairs and nonzero multipliers / slacks exercises the AL terms
    rng = np.random.default_rng(7)
    ap = keys[np.argsort(d)[:5]]
    ap_mu = rng.uniform(0.5, 2.0, len(ap))
    ap_s = rng.uniform(0.0, 2e-4, len(ap))
    sigma = 3.7e5
    y = sc["x0"] + o.h * sc["v0"] + o.h ** 2 * o.g[None]
    st = oracle_state(o, x, y=y, sigma=sigma, ap_keys=ap, ap_mu=ap_mu, ap_s=ap_s)
    asm = o.assemble(x, st, keys)
    ctx = bal.bal_init(sc)
    out = bal.bal_assemble(ctx, _t(x), active_keys=keys, aprime_keys=ap, aprime_mu=ap_mu, aprime_s=ap_s,
                           sigma=sigma, y=y)
    # per-stencil: both sides order the stencils by feature-pair key; nodes are the resolved support
    nodes = _np(out["contact_stencil_nodes"]).reshape(-1, 4)
    blocks = _np(out["contact_blocks"]).reshape(-1, 90)
    lbg = _np(out["contact_lbar"])
    cg = _np(out["contact_grad"]).reshape(-1, 12)
    assert len(nodes) == len(asm["contact_keys"]) and out["n_friction_stencils"] == 0
    worst = 0.0
    tols = []
    for i, (k, ids, P, g, lb) in enumerate(zip(asm["contact_keys"], asm["contact_ids"], asm["contact_P"],
                                               asm["contact_g"], asm["contact_lbar"])):
        n = len(ids)
        assert list(nodes[i, :n]) == list(ids) and np.all(nodes[i, n:] == -1)
        Hg = lower_blocks_to_full(blocks[i], n)
        # FP64 distance cancellation: d carries ~u*|x| absolute error, so the stencil Hessian is
        # only determined to ~C*u*|x|/d relative (C = 18)
        dd = cm.key_distance(x, k[None])[0]
        tol = 1e-12 + 4e-15 * np.abs(x).max() / dd
        tols.append(tol)
        err = np.linalg.norm(Hg - P) / max(np.linalg.norm(P), 1e-300)
        gerr = np.linalg.norm(cg[i, :3 * n] - g) / max(np.linalg.norm(g), 1e-300)
        worst = max(worst, err / tol, gerr / tol)
        assert lbg[i] == pytest.approx(lb, rel=tol, abs=1e-300)
    assert worst <= 1.0, worst
    N = o.N
    Ag = bsr_to_csr(_np(out["static_row_ptr"]), _np(out["static_col"]), _np(out["static_val"]), N)
    if out["contact_col"].numel():
        Ag = Ag + bsr_to_csr(_np(out["contact_row_ptr"]), _np(out["contact_col"]), _np(out["contact_val"]), N)
    # per slot: |dA_ab| <= sum over the stencils writing (a, b) of tol_i ||P_i|| (c.4), and per node
    # for the gradient -- in place of a row-relative 1e-9
    B, gb = assembly_bounds(o, x, y, asm, contact_tol=tols)
    rs, rg = check_assembly_bounds(Ag, asm["A"], _np(out["grad"]), asm["grad"], B, gb, N, o.mesh.fixed)
    assert rs <= 1.0 and rg <= 1.0, (rs, rg)
    assert np.array_equal(_np(out["group"])[o.free], asm["groups"][o.free])


# --------------------------------------------------------------------------- SpMV (a7)
def test_spmv_parity_on_oracle_system(cubes_state):
    sc, o, x1, _ = cubes_state
    pt, ee = cm.candidates(o.mesh, x1, x1, o.dhat)
    keys, d = cm.constraint_set(x1, pt, ee, o.dhat)
    asm = o.assemble(x1, oracle_state(o, x1, sigma=4e5), keys)
    A = asm["A"]
    ctx = bal.bal_init(sc)
    rp, col, val = csr_to_bsr(A, o.N)
    bal.bal_load_bsr(ctx, rp, col, val)
    rng = np.random.default_rng(8)
    for _ in range(3):
        v = rng.normal(size=3 * o.N)
        yg = torch.empty(3 * o.N, dtype=torch.float64, device=DEV)
        bal.bal_spmv(ctx, _t(v), yg)
        yo = A @ v
        bound = abs(A) @ np.abs(v)
        assert np.all(np.abs(_np(yg) - yo) <= 1e-12 * bound + 1e-300)


def test_spmv_on_gpu_assembled_system(cubes_state):
    """y = A v on the library's own static+contact BSR equals the CSR product of its views."""
    sc, o, x1, _ = cubes_state
    pt, ee = cm.candidates(o.mesh, x1, x1, o.dhat)
    keys, d = cm.constraint_set(x1, pt, ee, o.dhat)
    ctx = bal.bal_init(sc)
    out = bal.bal_assemble(ctx, _t(x1), active_keys=keys, sigma=4e5)
    N = o.N
    A = bsr_to_csr(_np(out["static_row_ptr"]), _np(out["static_col"]), _np(out["static_val"]), N)
    if out["contact_col"].numel():
        A = A + bsr_to_csr(_np(out["contact_row_ptr"]), _np(out["contact_col"]), _np(out["contact_val"]), N)
    v = np.random.default_rng(9).normal(size=3 * N)
    yg = torch.empty(3 * N, dtype=torch.float64, device=DEV)
    bal.bal_spmv(ctx, _t(v), yg)
    assert np.all(np.abs(_np(yg) - A @ v) <= 1e-12 * (abs(A) @ np.abs(v)) + 1e-300)


@pytest.mark.parametrize("budget", [24, 96, 333])
def test_spmv_tile_budgets_on_oracle_system(cubes_state, budget, monkeypatch):
    """The tile-symmetric SpMV (k_spmv_ts) for several tile sizes (more tiles = more cross-tile
    partials, single-row tiles at 24): element-wise parity with the oracle's product and bitwise
    equality of repeated products."""
    monkeypatch.setenv("BAL_TS_BUDGET", str(budget))
    sc, o, x1, _ = cubes_state
    pt, ee = cm.candidates(o.mesh, x1, x1, o.dhat)
    keys, d = cm.constraint_set(x1, pt, ee, o.dhat)
    A = o.assemble(x1, oracle_state(o, x1, sigma=4e5), keys)["A"]
    ctx = bal.bal_init(sc)
    bal.bal_load_bsr(ctx, *csr_to_bsr(A, o.N))
    v = np.random.default_rng(10 + budget).normal(size=3 * o.N)
    yg = torch.empty(3 * o.N, dtype=torch.float64, device=DEV)
    bal.bal_spmv(ctx, _t(v), yg)
    assert np.all(np.abs(_np(yg) - A @ v) <= 1e-12 * (abs(A) @ np.abs(v)) + 1e-300)
    y2 = torch.empty_like(yg)
    bal.bal_spmv(ctx, _t(v), y2)
    assert torch.equal(yg, y2)


# --------------------------------------------------------------------------- PCG (a8, a9)
def _loaded_system(cubes_state):
    sc, o, x1, _ = cubes_state
    pt, ee = cm.candidates(o.mesh, x1, x1, o.dhat)
    keys, d = cm.constraint_set(x1, pt, ee, o.dhat)
    asm = o.assemble(x1, oracle_state(o, x1, sigma=4e5), keys)
    ctx = bal.bal_init(sc)
    rp, col, val = csr_to_bsr(asm["A"], o.N)
    bal.bal_load_bsr(ctx, rp, col, val, group=np.where(asm["groups"] < -900, 0, asm["groups"]))
    return sc, o, asm, ctx


def test_pcg_fixed_iterates_and_converged_parity(cubes_state):
    sc, o, asm, ctx = _loaded_system(cubes_state)
    A, Dinv = asm["A"], asm["Dinv"]
    b = -asm["grad"]
    N = o.N
    xg = torch.empty(3 * N, dtype=torch.float64, device=DEV)
    # (i) same system, x0 = 0, exactly k iterations (tolerance and stagnation disabled)
    for k in (1, 5, 20):
        s = bal.bal_pcg(ctx, _t(b), _t(np.zeros(3 * N)), xg, warm_start=0, rel_tol=0.0, stall_window=0,
                        max_iters=k)
        st = la.pcg_cg(A, b, np.zeros(3 * N), Dinv, tol=0.0, window=10 ** 9, max_iters=k)
        assert s["iters"] == k == st.k
        assert np.linalg.norm(_np(xg) - st.x) <= 1e-10 * np.linalg.norm(st.x)
        tb = la.pcg(A, b, np.zeros(3 * N), Dinv, tol=0.0, window=10 ** 9, max_iters=k)
        assert np.linalg.norm(_np(xg) - tb.x) <= 1e-8 * np.linalg.norm(tb.x)
        hg = bal.bal_pcg_history(ctx, k + 1)
        assert np.max(np.abs(hg - np.asarray(st.hist))) <= 1e-10 * st.hist[0]
    # (ii) converged to 1e-12: vs oracle and vs a direct solve
    s = bal.bal_pcg(ctx, _t(b), None, xg, warm_start=0, rel_tol=1e-12, stall_window=0, max_iters=20000)
    xd = np.linalg.solve(A.toarray(), b)
    assert s["stop_reason"] == 0
    assert np.linalg.norm(_np(xg) - xd) <= 1e-8 * np.linalg.norm(xd)
    # (iii) App. B default policy: same iteration count and stop reason as the oracle
    s = bal.bal_pcg(ctx, _t(b), None, xg, warm_start=0)
    st = la.pcg_cg(A, b, np.zeros(3 * N), Dinv, tol=1e-4, window=100, max_iters=20000)
    assert s["stop_reason"] == st.stop
    assert abs(s["iters"] - st.k) <= 1
    r = b - A @ _np(xg)
    assert np.linalg.norm(r) <= 1.0001e-4 * np.linalg.norm(b)


def test_warm_start_parity(cubes_state):
    sc, o, asm, ctx = _loaded_system(cubes_state)
    A, Dinv = asm["A"], asm["Dinv"]
    b = -asm["grad"]
    N = o.N
    xg = torch.empty(3 * N, dtype=torch.float64, device=DEV)
    s = bal.bal_pcg(ctx, _t(b), None, xg, warm_start=1, max_iters=0)
    x0, its = la.warm_start(A, b, asm["groups"], Dinv, o.mesh.fixed, 1e-2, 100)
    assert s["ws_iters_max"] == max(its.values())
    phi0 = 0.5 * x0 @ (A @ x0) - b @ x0
    assert phi0 < 0.0  # R-WS1 keeps it (phi(x0) < phi(0))
    assert np.linalg.norm(_np(xg) - x0) <= 1e-10 * np.linalg.norm(x0)
    # and the full warm-started solve reaches the App. B tolerance
    s = bal.bal_pcg(ctx, _t(b), None, xg, warm_start=1)
    r = b - A @ _np(xg)
    assert np.linalg.norm(r) <= 1.0001e-4 * np.linalg.norm(b)


def test_bad_mesh_and_args_fail_loudly():
    sc = scenes.make_single_tet(0)
    bad = dict(sc)
    t = sc["tets"].copy()
    t[0, [2, 3]] = t[0, [3, 2]]  # inverted
    bad["tets"] = t
    with pytest.raises(bal.BalError) as ei:
        bal.bal_init(bad)
    assert ei.value.status == -2


# --------------------------------------------------------------------------- friction (a5)
def test_friction_stencils_and_assembly_parity(cubes_state):
    sc, o, x1, v1 = cubes_state
    sc = dict(sc)
    sc["params"] = dict(sc["params"], chi=0.5)
    o = Oracle(sc)
    x = x1
    pt, ee = cm.candidates(o.mesh, x, x, o.dhat)
    keys, d = cm.constraint_set(x, pt, ee, o.dhat)
    sigma = 3.7e5
    y = sc["x0"] + o.h * sc["v0"] + o.h ** 2 * o.g[None]
    x_t = x - 0.004 * np.random.default_rng(3).normal(size=x.shape) * (~o.mesh.fixed[:, None])
    st = oracle_state(o, x, y=y, sigma=sigma)
    st["x_t"] = x_t
    fk, G, n, lam = o.friction_anchors(x, st, keys)
    st["fr_keys"], st["fr_G"], st["fr_n"], st["fr_lam"] = fk, G, n, lam
    asm = o.assemble(x, st, keys)
    ctx = bal.bal_init(sc)
    out = bal.bal_assemble(ctx, _t(x), active_keys=keys, sigma=sigma, y=y, x_t=x_t,
                           friction=dict(keys=fk, gamma=G, n=n, lam=lam))
    N = o.N
    # per-stencil friction (K3): D_j's gradient and (unprojected, PSD) Hessian over its nodes.  w =
    # P_n Gamma (x - x_t) carries ~u|x| absolute error and H depends on w through f'(y)/y, f''(y) and
    # w/|w| with y = |w| floored by the mollifier width eps (f is polynomial below eps, Q24), so a
    # stencil is determined to ~u|x| / max(y, eps) relative
    nf = out["n_friction_stencils"]
    assert nf == len(fk) > 10
    nc = len(asm["contact_keys"])
    blocks = _np(out["contact_blocks"]).reshape(-1, 90)[nc:]
    cg = _np(out["contact_grad"]).reshape(-1, 12)[nc:]
    nodes = _np(out["contact_stencil_nodes"]).reshape(-1, 4)[nc:]
    eps = float(o.p["eps_v"]) * o.h
    ftol, worst = [], 0.0
    for j, (ids, g, H) in enumerate(asm["friction"]):
        kk = len(ids)
        assert list(nodes[j, :kk]) == list(ids)
        w = np.sum(G[j, :kk, None] * (x[ids] - x_t[ids]), axis=0)
        w = w - np.dot(w, n[j]) * n[j]
        tol = 1e-12 + 4e-15 * np.abs(x).max() / max(np.linalg.norm(w), eps)
        ftol.append(tol)
        e_h = np.linalg.norm(lower_blocks_to_full(blocks[j], kk) - H) / max(np.linalg.norm(H), 1e-300)
        e_g = np.linalg.norm(cg[j, :3 * kk] - g) / max(np.linalg.norm(g), 1e-300)
        worst = max(worst, e_h / tol, e_g / tol)
    assert worst <= 1.0, worst
    ctol = [1e-12 + 4e-15 * np.abs(x).max() / cm.key_distance(x, k[None])[0] for k in asm["contact_keys"]]
    Ag = bsr_to_csr(_np(out["static_row_ptr"]), _np(out["static_col"]), _np(out["static_val"]), N)
    Ag = Ag + bsr_to_csr(_np(out["contact_row_ptr"]), _np(out["contact_col"]), _np(out["contact_val"]), N)
    B, gb = assembly_bounds(o, x, y, asm, contact_tol=ctol, friction=asm["friction"], friction_tol=ftol)
    rs, rg = check_assembly_bounds(Ag, asm["A"], _np(out["grad"]), asm["grad"], B, gb, N, o.mesh.fixed)
    assert rs <= 1.0 and rg <= 1.0, (rs, rg)


# --------------------------------------------------------------------------- NEXT-3 FP32 storage
def test_fp32_matrix_spmv_and_pcg_parity(cubes_state):
    """BAL_FP32_MATRIX ("single-precision version"): the global PCG's SpMV streams the stored
    blocks rounded to FP32, arithmetic stays FP64.  The product equals the oracle's product with the
    entrywise FP32-rounded matrix (1e-12 of |A32||v|; bitwise repeatable) and 20 PCG iterates match
    the oracle's pcg_cg on that matrix with the FP64 block-Jacobi preconditioner (1e-10)."""
    sc, o, x1, _ = cubes_state
    pt, ee = cm.candidates(o.mesh, x1, x1, o.dhat)
    keys, d = cm.constraint_set(x1, pt, ee, o.dhat)
    asm = o.assemble(x1, oracle_state(o, x1, sigma=4e5), keys)
    A, Dinv = asm["A"], asm["Dinv"]
    A32 = A.copy()
    A32.data = A32.data.astype(np.float32).astype(np.float64)
    assert np.abs(A32 - A).max() > 0  # the rounding is visible
    ctx = bal.bal_init(sc, flags=bal.BAL_FP32_MATRIX)
    bal.bal_load_bsr(ctx, *csr_to_bsr(A, o.N))
    v = np.random.default_rng(11).normal(size=3 * o.N)
    yg = torch.empty(3 * o.N, dtype=torch.float64, device=DEV)
    bal.bal_spmv(ctx, _t(v), yg)
    assert np.all(np.abs(_np(yg) - A32 @ v) <= 1e-12 * (abs(A32) @ np.abs(v)) + 1e-300)
    y2 = torch.empty_like(yg)
    bal.bal_spmv(ctx, _t(v), y2)
    assert torch.equal(yg, y2)
    b = -asm["grad"]
    xg = torch.empty(3 * o.N, dtype=torch.float64, device=DEV)
    s = bal.bal_pcg(ctx, _t(b), _t(np.zeros(3 * o.N)), xg, warm_start=0, rel_tol=0.0, stall_window=0, max_iters=20)
    st = la.pcg_cg(A32, b, np.zeros(3 * o.N), Dinv, tol=0.0, window=10 ** 9, max_iters=20)
    assert s["iters"] == 20 == st.k
    assert np.linalg.norm(_np(xg) - st.x) <= 1e-10 * np.linalg.norm(st.x)
