"""NEXT-4: App. B's alternative PCG termination criteria (BAL_PCG_CRIT_I / II / III,
DESIGN.md R-KAPPA) on the GPU against the oracle's pcg_cg with the same criterion, through the C ABI.
Requires a B200."""
import numpy as np
import pytest

import scenes
from tests.gpu_helpers import oracle_state

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2407_00046_b200 as bal  # noqa: E402
from oracle import contact as cm  # noqa: E402
from oracle import linalg as la  # noqa: E402
from oracle.bal import FLAG_PCG_CRIT_I, FLAG_PCG_CRIT_II, FLAG_PCG_CRIT_III, Oracle  # noqa: E402

DEV = torch.device("cuda:0")
CRITS = [("i", bal.BAL_PCG_CRIT_I, FLAG_PCG_CRIT_I), ("ii", bal.BAL_PCG_CRIT_II, FLAG_PCG_CRIT_II),
         ("iii", bal.BAL_PCG_CRIT_III, FLAG_PCG_CRIT_III)]


def _t(a):
    return torch.as_tensor(np.ascontiguousarray(a, np.float64).ravel(), device=DEV)


@pytest.fixture(scope="module")
def state():
    sc = scenes.make_cubes(1)
    o = Oracle(sc)
    x1, _v1, _ = o.step(sc["x0"], sc["v0"])
    pt, ee = cm.candidates(o.mesh, x1, x1, o.dhat)
    keys, _d = cm.constraint_set(x1, pt, ee, o.dhat)
    y = sc["x0"] + o.h * sc["v0"] + o.h ** 2 * o.g[None]
    asm = o.assemble(x1, oracle_state(o, x1, y=y, sigma=4e5), keys)
    return sc, o, x1, y, keys, asm


@pytest.mark.parametrize("name,gflag,oflag", CRITS)
def test_criterion_stop_matches_the_oracle(state, name, gflag, oflag):
    """The GPU assembles the system itself (kappa from its own e_j), solves -grad with the
    criterion; the oracle runs pcg_cg with the same criterion on its assembly: same stop reason,
    iteration counts within max(1, 2 %) (rounding of the same recurrences), and the GPU's final
    residual meets the criterion's threshold on the oracle's matrix."""
    sc, o, x1, y, keys, asm = state
    ctx = bal.bal_init(sc, flags=gflag)
    out = bal.bal_assemble(ctx, _t(x1), active_keys=keys, sigma=4e5, y=y)
    b = -out["grad"].cpu().numpy()
    xg = torch.empty_like(out["grad"])
    s = bal.bal_pcg(ctx, _t(b), None, xg, warm_start=0)
    ej = asm["e_j"][o.free]
    ukappa = np.finfo(np.float64).eps * float(ej.max() / ej.min())
    st = la.pcg_cg(asm["A"], -asm["grad"], np.zeros(3 * o.N), asm["Dinv"], tol=1e-4, window=100,
                   max_iters=20000, crit=(name, ukappa))
    assert s["stop_reason"] == st.stop
    assert abs(s["iters"] - st.k) <= max(1, 0.02 * st.k), (s["iters"], st.k)
    x = xg.cpu().numpy()
    if name == "i":
        # (i) stops early (a loose threshold): the true residual meets it too
        rn = np.linalg.norm(b - asm["A"] @ x)
        assert rn <= 1.01 * min(0.5, np.sqrt(np.linalg.norm(b))) * np.linalg.norm(b)
        assert np.linalg.norm(x - st.x) <= 1e-8 * np.linalg.norm(st.x)
    else:
        # (ii) / (iii): u kappa thresholds lie below the attainable accuracy of the true residual
        # (~u |A| |x|); only the recursive residual meets them (on both sides), and both solutions
        # have converged to rounding: compare them
        assert np.linalg.norm(x - st.x) <= 1e-6 * np.linalg.norm(st.x)


@pytest.mark.parametrize("name,gflag,oflag", CRITS)
def test_criterion_step_parity(name, gflag, oflag):
    """One C1 time step with the criterion in every Newton iteration: GPU positions equal the
    oracle's to 1e-6 relative."""
    sc = scenes.make_cubes(1)
    o = Oracle(sc, flags=oflag)
    x1, _v1, _ = o.step(sc["x0"], sc["v0"])
    ctx = bal.bal_init(sc, flags=gflag)
    xt = _t(sc["x0"])
    xn = torch.empty_like(xt)
    bal.bal_step(ctx, xt, _t(sc["v0"]), xn, torch.empty_like(xt))
    xg = xn.cpu().numpy().reshape(-1, 3)
    assert np.linalg.norm(xg - x1) <= 1e-6 * np.linalg.norm(x1)
