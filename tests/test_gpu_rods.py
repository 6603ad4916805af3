"""NEXT-2: twisting rods (Table 1) with scripted Dirichlet ends.  A small
bundle (4 rods of 2 x 2 x 6 voxels, 1.5 mm apart) twisted at the paper's 5/12 rev/s: GPU and oracle
take the same steps from the same scripted end positions (positions to 1e-6 relative), every step
intersection-free.  Requires a B200."""
import numpy as np
import pytest

import scenes

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2407_00046_b200 as bal  # noqa: E402
from oracle import contact as cm  # noqa: E402
from oracle.bal import Oracle  # noqa: E402

DEV = torch.device("cuda:0")


def test_small_twisting_rods_parity():
    sc = scenes.make_twisting_rods(n=2, length=6, voxel=0.01, gap=0.0015)
    o = Oracle(sc)
    ctx = bal.bal_init(sc)
    h = sc["params"]["h"]
    fixed = sc["node_fixed"].astype(bool)
    xo, vo = sc["x0"].copy(), np.zeros_like(sc["x0"])
    vprev = vo
    for k in range(4):
        tgt = scenes.twist_targets(sc, (k + 1) * h)
        xo = xo.copy()
        xo[fixed] = tgt[fixed]
        xin = xo.copy()
        xo, vo, _st = o.step(xin, vprev)
        # the GPU takes the same step from the same input state (the oracle's x_t, v_t)
        xt = torch.as_tensor(xin.ravel(), device=DEV)
        vin = torch.as_tensor(np.ascontiguousarray(vprev).ravel(), device=DEV) if k else torch.zeros_like(xt)
        xn, vn = torch.empty_like(xt), torch.empty_like(xt)
        bal.bal_step(ctx, xt, vin, xn, vn)
        xg = xn.cpu().numpy().reshape(-1, 3)
        assert np.allclose(xg[fixed], tgt[fixed], rtol=0, atol=1e-15)
        assert np.linalg.norm(xg - xo) <= 1e-6 * np.linalg.norm(xo - xin), k
        pt, ee = cm.candidates(o.mesh, xg, xg, o.dhat)
        _k, d = cm.constraint_set(xg, pt, ee, o.dhat)
        assert np.all(d > 0)
        vprev = vo
