"""GPU parity on BASELINE.json configs[1] (C2, armadillo-like, ~95K tets, friction chi = 0.9) and
configs[2] (C3, stiff high-speed impact, ~317K tets, E = 1 GPa slab): the assembled system on
sampled outputs the oracle computes one by one (elastic stencils, assembled rows), the SpMV over
every row, fixed PCG iterations against the oracle's textbook PCG, and -- after GPU Newton
iterations of the first frame through the C ABI -- the invariants the method guarantees
(no inverted tet, no interpenetration, CCD-bounded progress)."""
import types

import numpy as np
import pytest

import scenes
from tests.gpu_helpers import bsr_to_csr, dinv_full, lower_blocks_to_full

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2407_00046_b200 as bal  # noqa: E402
from oracle import contact as cm  # noqa: E402
from oracle import linalg as la  # noqa: E402
from oracle.energy import nh_min_J, nh_stencils  # noqa: E402
from oracle.mesh import precompute  # noqa: E402
from oracle.projection import lambda_bar, project_eigh  # noqa: E402

DEV = torch.device("cuda:0")
SCENES = {"c2": scenes.make_armadillo_like, "c3": scenes.make_impact}


def _t(a):
    return torch.as_tensor(np.ascontiguousarray(a, np.float64).ravel(), device=DEV)


def _np(t):
    return t.detach().cpu().numpy()


def _sub_mesh(m, sel):
    return type(m)(**{**m.__dict__, "tets": m.tets[sel], "Dm_inv": m.Dm_inv[sel], "vol": m.vol[sel],
                      "mu": m.mu[sel], "lam": m.lam[sel], "arap": m.arap[sel]})


@pytest.fixture(scope="module", params=["c2", "c3"])
def assembled(request):
    sc = SCENES[request.param]()
    m = precompute(sc)
    rng = np.random.default_rng(12)
    x = sc["x0"] + 1e-4 * rng.normal(size=sc["x0"].shape) * (1 - sc["node_fixed"][:, None])
    p = sc["params"]
    y = x + p["h"] * sc["v0"] + p["h"] ** 2 * np.array(p["gravity"])[None]
    ctx = bal.bal_init(sc)
    out = bal.bal_assemble(ctx, _t(x), y=y)
    A = bsr_to_csr(_np(out["static_row_ptr"]), _np(out["static_col"]), _np(out["static_val"]), len(x))
    return request.param, sc, m, x, ctx, out, A


def test_sampled_stencils_and_rows(assembled):
    name, sc, m, x, ctx, out, A = assembled
    rng = np.random.default_rng(1)
    sel = np.sort(rng.choice(len(m.tets), size=2000, replace=False))
    _v, _g, H = nh_stencils(x, _sub_mesh(m, sel))
    P, _ = project_eigh(H)
    Pg = _np(out["elastic_blocks"]).reshape(-1, 90)[sel]
    err = max(np.linalg.norm(lower_blocks_to_full(Pg[i], 4) - P[i]) / max(np.linalg.norm(P[i]), 1e-300)
              for i in range(len(sel)))
    assert err <= 1e-12, (name, err)
    np.testing.assert_allclose(_np(out["elastic_lbar"])[sel], lambda_bar(P), rtol=1e-12, atol=0)
    N = len(x)
    flat = m.tets.ravel()
    order = np.argsort(flat, kind="stable")
    starts = np.searchsorted(flat[order], np.arange(N + 1))
    free = np.flatnonzero(sc["node_fixed"] == 0)
    h = sc["params"]["h"]
    for i in rng.choice(free, size=100, replace=False):
        tsel = np.unique(order[starts[i]:starts[i + 1]] // 4)
        _v, _g, H = nh_stencils(x, _sub_mesh(m, tsel))
        Pi, _ = project_eigh(H)
        row = np.zeros((3, 3 * N))
        row[:, 3 * i:3 * i + 3] += np.eye(3) * m.mass[i] / h ** 2
        for t, e in enumerate(tsel):
            a = int(np.flatnonzero(m.tets[e] == i)[0])
            for b in range(4):
                j = m.tets[e, b]
                if not sc["node_fixed"][j]:
                    row[:, 3 * j:3 * j + 3] += Pi[t][3 * a:3 * a + 3, 3 * b:3 * b + 3]
        assert np.abs(A[3 * i:3 * i + 3].toarray() - row).sum() <= 1e-12 * np.abs(row).sum(), (name, i)


def test_spmv_every_row_and_pcg_iterations(assembled):
    name, sc, m, x, ctx, out, A = assembled
    v = np.random.default_rng(3).normal(size=A.shape[0])
    yg = torch.empty(A.shape[0], dtype=torch.float64, device=DEV)
    bal.bal_spmv(ctx, _t(v), yg)
    assert np.all(np.abs(_np(yg) - A @ v) <= 1e-12 * (abs(A) @ np.abs(v)) + 1e-300), name
    b = -_np(out["grad"])
    Dinv = dinv_full(_np(out["diag_inv"]))
    xg = torch.empty(A.shape[0], dtype=torch.float64, device=DEV)
    s = bal.bal_pcg(ctx, _t(b), _t(np.zeros_like(b)), xg, warm_start=0, rel_tol=0.0, stall_window=0, max_iters=10)
    st = la.pcg_cg(A, b, np.zeros_like(b), Dinv, tol=0.0, window=10 ** 9, max_iters=10)
    assert s["iters"] == 10 == st.k
    assert np.linalg.norm(_np(xg) - st.x) <= 1e-10 * np.linalg.norm(st.x), name


def _min_distance_near(m, x, box_lo, box_hi, inflate):
    """Smallest feature-pair distance among surface primitives inside a box (oracle brute force)."""
    inside = np.all((x >= box_lo) & (x <= box_hi), axis=1)
    sub = types.SimpleNamespace(surf_verts=m.surf_verts[inside[m.surf_verts]], tris=m.tris[inside[m.tris].all(1)],
                                edges=m.edges[inside[m.edges].all(1)], fixed=m.fixed)
    pt, ee = cm.candidates(sub, x, x, inflate)
    keys, d = cm.constraint_set(x, pt, ee, inflate)
    return (d.min() if len(d) else np.inf), len(keys)


@pytest.mark.parametrize("name,newton", [("c2", 12), ("c3", 8)])
def test_first_frame_newton_iterations_keep_invariants(name, newton):
    """Newton iterations of frame 0 on the GPU (bal_frame_* slices): the accepted iterate keeps every
    tet un-inverted (J > 0) and every surface pair apart (d > 0: the CCD line search),
    and it moved (the step is not stalled)."""
    sc = SCENES[name]()
    m = precompute(sc)
    ctx = bal.bal_init(sc)
    x0 = _t(sc["x0"])
    v0 = _t(sc["v0"])
    xn, vn = torch.empty_like(x0), torch.empty_like(v0)
    bal.bal_frame_begin(ctx, x0, v0)
    bal.bal_frame_iterate(ctx, newton)
    st = bal.bal_frame_finish(ctx, xn, vn, allow_unconverged=True)
    x = _np(xn).reshape(-1, 3)
    assert st["newton_iters"] >= 1
    assert nh_min_J(x, m) > 0.0
    assert np.linalg.norm(x - sc["x0"]) > 0.0
    if name == "c2":  # the creature against the static plane y = 0
        assert x[~m.fixed, 1].min() > 0.0
        assert st["max_constraints"] > 0
    else:  # sphere against the slab: brute-force distances around the sphere
        sphere = np.zeros(len(x), bool)
        sphere[np.unique(m.tets[np.asarray(sc["tet_material"]) == 0])] = True
        lo, hi = x[sphere].min(0) - 0.03, x[sphere].max(0) + 0.03
        dmin, _n = _min_distance_near(m, x, lo, hi, 0.02)
        assert dmin > 0.0
