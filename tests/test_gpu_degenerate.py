"""Degenerate-contact robustness suite (§6.1 "Erleben tests"):
constructed exact ties -- a vertex over a triangle's interior, over an edge, over a vertex, exactly
parallel edges, an edge crossing an edge's interior, face on face -- where the feature-pair
sub-type resolution (PT -> PE / PP, EE -> PE / PP) has several correct answers.

What is unique is compared exactly: the active set A = {feature pairs with d < dhat} (its keys are
feature pairs, R-DUP1, so they do not depend on the resolution) bitwise, each pair's distance to
FP64 rounding, every stencil's gradient (first order, the same for every feature at a tie) and the
assembled gradient.  What may differ at a tie is checked for validity: where the two sides resolved
a pair to different supports, the GPU's choice must be a minimiser (its feature distance equals the
oracle's minimum); where they agree, the projected stencil Hessian must match too.  Then one time
step of each scene, GPU vs oracle positions.  Requires a B200."""
import numpy as np
import pytest

import scenes
from tests.gpu_helpers import lower_blocks_to_full, oracle_state

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2407_00046_b200 as bal  # noqa: E402
from oracle import contact as cm  # noqa: E402
from oracle.bal import Oracle  # noqa: E402

DEV = torch.device("cuda:0")
G = 5e-4  # gap = dhat / 2

# tet A: bottom face (a0, a1, a3) in the plane y = 0, body above it
A = np.array([[0.0, 0.0, 0.0], [0.1, 0.0, 0.0], [0.0, 0.1, 0.0], [0.0, 0.0, 0.1]])


def _apex_up(p):
    """Tet B with its apex p at the top and its base 8 cm below."""
    p = np.asarray(p, np.float64)
    return np.array([p, p + (-0.04, -0.08, -0.03), p + (0.05, -0.08, -0.02), p + (0.0, -0.08, 0.05)])


CASES = {
    "vertex_over_face_interior": _apex_up((0.03, -G, 0.03)),
    "vertex_over_edge": _apex_up((0.05, -G, 0.0)),
    "vertex_over_vertex": _apex_up((0.0, -G, 0.0)),
    "parallel_edges": np.array([[0.02, -G, 0.0], [0.08, -G, 0.0], [0.05, -0.08, 0.04], [0.05, -0.08, -0.04]]),
    "edge_crossing_edge": np.array([[0.05, -G, -0.03], [0.05, -G, 0.03], [0.02, -0.08, 0.0], [0.08, -0.08, 0.0]]),
    "face_on_face": np.array([[0.01, -G, 0.01], [0.06, -G, 0.01], [0.01, -G, 0.06], [0.02, -0.08, 0.02]]),
}


def scene(name, speed=0.3):
    sb = scenes.SceneBuilder()
    sb.add_body(A, scenes._orient(A, np.array([[0, 1, 2, 3]])), 0)
    B = CASES[name]
    sb.add_body(B, scenes._orient(B, np.array([[0, 1, 2, 3]])), 0, v0=(0.0, speed, 0.0))
    return sb.build([(1e5, 0.4, 1e3)], "degenerate-" + name, gravity=(0.0, 0.0, 0.0))


def _t(a):
    return torch.as_tensor(np.ascontiguousarray(a, np.float64).ravel(), device=DEV)


@pytest.mark.parametrize("name", list(CASES))
def test_degenerate_active_set_and_stencils(name):
    sc = scene(name)
    o = Oracle(sc)
    x = sc["x0"]
    dhat = o.dhat
    pt, ee = cm.candidates(o.mesh, x, x, dhat)
    keys_o, d_o = cm.constraint_set(x, pt, ee, dhat)
    assert len(keys_o) >= 1
    ctx = bal.bal_init(sc)
    keys_g, d_g = bal.bal_detect(ctx, _t(x))
    # the active set is unique: bitwise equal keys (no pair sits within rounding of d = dhat here)
    assert cm.activation_margin(x, pt, ee, dhat) > 1e-9
    assert np.array_equal(keys_g.astype(np.int64), keys_o), (keys_g, keys_o)
    tol_d = 4e-15 * np.abs(x).max() + 1e-13 * d_o
    assert np.all(np.abs(d_g - d_o) <= tol_d), np.abs(d_g - d_o) / tol_d

    sigma = 2.5e5
    st = oracle_state(o, x, sigma=sigma)
    asm = o.assemble(x, st, keys_o)
    out = bal.bal_assemble(ctx, _t(x), active_keys=keys_o, sigma=sigma)
    nodes = out["contact_stencil_nodes"].cpu().numpy().reshape(-1, 4)
    blocks = out["contact_blocks"].cpu().numpy().reshape(-1, 90)
    cg = out["contact_grad"].cpu().numpy().reshape(-1, 12)
    assert len(nodes) == len(asm["contact_keys"])
    same = 0
    for i, (k, ids, P, g) in enumerate(zip(asm["contact_keys"], asm["contact_ids"], asm["contact_P"],
                                           asm["contact_g"])):
        d = cm.key_distance(x, k[None])[0]
        tol = 1e-12 + 4e-15 * np.abs(x).max() / d
        gi = nodes[i][nodes[i] >= 0]
        # the gradient lives on the union of both supports: compare node by node
        gg, go = {}, {}
        for a, n in enumerate(gi):
            gg[int(n)] = gg.get(int(n), 0) + cg[i, 3 * a:3 * a + 3]
        for a, n in enumerate(ids):
            go[int(n)] = go.get(int(n), 0) + g[3 * a:3 * a + 3]
        gnorm = np.linalg.norm(g)
        for n in set(gg) | set(go):
            diff = np.asarray(gg.get(n, 0.0)) - np.asarray(go.get(n, 0.0))
            assert np.linalg.norm(diff) <= tol * gnorm, (name, i, n, diff)
        if list(gi) == list(ids):
            same += 1
            Hg = lower_blocks_to_full(blocks[i], len(ids))
            assert np.linalg.norm(Hg - P) <= tol * np.linalg.norm(P), (name, i)
        else:
            # a tie: the GPU's support must itself be a minimiser of the pair's distance
            sub = {2: cm.PP, 3: cm.PE, 4: cm.PT if k[0] == cm.PT else cm.EE}[len(gi)]
            kk = np.full((1, 5), -1, np.int64)
            kk[0, 0] = sub
            kk[0, 1:1 + len(gi)] = gi
            assert abs(cm.key_distance(x, kk)[0] - d) <= 4e-15 * np.abs(x).max() + 1e-13 * d, (name, i, gi, ids)
    ge = out["grad"].cpu().numpy()
    assert np.linalg.norm(ge - asm["grad"]) <= 1e-10 * np.linalg.norm(asm["grad"])
    assert same >= 1


@pytest.mark.parametrize("name", list(CASES))
def test_degenerate_step_parity(name):
    """One time step into the tie (B approaches A at 0.3 m/s, 1 cm per step against a 0.5 mm gap):
    GPU and oracle positions agree to 1e-5 of the displacement (DESIGN.md R-TRACE: the GPU's
    Chronopoulos-Gear and the oracle's textbook PCG directions agree to ~1e-6 per Newton iteration;
    a step takes 6-9 of them here)."""
    sc = scene(name)
    o = Oracle(sc)
    x1, _v1, _ = o.step(sc["x0"], sc["v0"])
    ctx = bal.bal_init(sc)
    xt = _t(sc["x0"])
    xn = torch.empty_like(xt)
    bal.bal_step(ctx, xt, _t(sc["v0"]), xn, torch.empty_like(xt))
    xg = xn.cpu().numpy().reshape(-1, 3)
    assert np.linalg.norm(xg - x1) <= 1e-5 * np.linalg.norm(x1 - sc["x0"])
    # intersection-free: every feature-pair distance stays positive
    pt, ee = cm.candidates(o.mesh, xg, xg, o.dhat)
    _k, d = cm.constraint_set(xg, pt, ee, o.dhat)
    assert np.all(d > 0)


def test_detect_rejects_a_short_output_buffer():
    """bal_detect (include/bal.h): |A| > max_n is BAL_E_INVALID_ARG, and *n_out still reports |A|."""
    sc = scene("vertex_over_vertex")
    ctx = bal.bal_init(sc)
    keys, _d = bal.bal_detect(ctx, _t(sc["x0"]))
    assert len(keys) > 1
    with pytest.raises(bal.BalError) as ei:
        bal.bal_detect(ctx, _t(sc["x0"]), max_n=1)
    assert ei.value.status == -1
