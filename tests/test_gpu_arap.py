"""NEXT-4: ARAP material and its coupling with Neo-Hookean (DESIGN.md R-ARAP) on the
GPU against the oracle's AD (sum of singular values through its quartic), through the C ABI.
Requires a B200."""
import numpy as np
import pytest

import scenes
from tests.gpu_helpers import bsr_to_csr, lower_blocks_to_full, oracle_state

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2407_00046_b200 as bal  # noqa: E402
from oracle.bal import Oracle  # noqa: E402

DEV = torch.device("cuda:0")


def _t(a):
    return torch.as_tensor(np.ascontiguousarray(a, np.float64).ravel(), device=DEV)


def test_arap_and_nh_stencils_and_assembly():
    """Every tet's projected 12x12 Hessian (ARAP bottom cube with compressed tets whose twist modes
    are negative and get clamped, NH top cube) and lambda_bar within 1e-12 of the oracle; assembled
    static system and gradient within 1e-12 relative."""
    sc = scenes.perturbed(scenes.make_nh_arap_cubes(1), seed=7, scale=0.03)
    o = Oracle(sc)
    assert o.mesh.arap.sum() == len(sc["tets"]) // 2
    x = sc["x0"]
    y = x + 0.01 * np.random.default_rng(8).normal(size=x.shape)
    ctx = bal.bal_init(sc)
    out = bal.bal_assemble(ctx, _t(x), y=y)
    asm = o.assemble(x, oracle_state(o, x, y=y), np.zeros((0, 5), np.int64))
    Pg = out["elastic_blocks"].cpu().numpy().reshape(-1, 90)
    worst = np.zeros(2)
    for e in range(len(sc["tets"])):
        Hg = lower_blocks_to_full(Pg[e], 4)
        Ho = asm["elastic_P"][e]
        err = np.linalg.norm(Hg - Ho) / max(np.linalg.norm(Ho), 1e-300)
        k = int(o.mesh.arap[e])
        worst[k] = max(worst[k], err)
    assert worst.max() <= 1e-12, worst
    np.testing.assert_allclose(out["elastic_lbar"].cpu().numpy(), asm["elastic_lbar"], rtol=1e-12, atol=0)
    # the ARAP cube really has indefinite (clamped) stencils
    from oracle.energy import nh_stencils
    _v, _g, H = nh_stencils(x, o.mesh)
    assert min(np.linalg.eigvalsh(H[e]).min() for e in np.nonzero(o.mesh.arap)[0]) < 0
    N = o.N
    Ag = bsr_to_csr(out["static_row_ptr"].cpu().numpy(), out["static_col"].cpu().numpy(),
                    out["static_val"].cpu().numpy(), N)
    assert abs(Ag - asm["A"]).max() <= 1e-12 * abs(asm["A"]).max()
    ge = out["grad"].cpu().numpy()
    assert np.linalg.norm(ge - asm["grad"]) <= 1e-12 * np.linalg.norm(asm["grad"])


def test_nh_arap_coupling_step_parity():
    """Two time steps of the NH-on-ARAP cubes falling onto the plane: GPU positions equal the oracle's
    to 1e-6 relative (the line search evaluates the ARAP energy in both)."""
    sc = scenes.make_nh_arap_cubes(1)
    o = Oracle(sc)
    ctx = bal.bal_init(sc)
    x, v = sc["x0"], sc["v0"]
    xt, vt = _t(x), _t(v)
    for _ in range(2):
        x, v, _st = o.step(x, v)
        xn, vn = torch.empty_like(xt), torch.empty_like(vt)
        bal.bal_step(ctx, xt, vt, xn, vn)
        xt, vt = xn, vn
        assert np.linalg.norm(xt.cpu().numpy().reshape(-1, 3) - x) <= 1e-6 * np.linalg.norm(x)
