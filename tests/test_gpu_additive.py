"""NEXT-1: the two-level additive preconditioner of App. A (DESIGN.md R-AS1) on the
GPU (BAL_ADDITIVE_PRECOND) against the oracle's la.additive_schwarz, through the C ABI.
Requires a B200."""
import numpy as np
import pytest

import scenes
from tests.gpu_helpers import csr_to_bsr, oracle_state

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2407_00046_b200 as bal  # noqa: E402
from oracle import contact as cm  # noqa: E402
from oracle import linalg as la  # noqa: E402
from oracle.bal import FLAG_ADDITIVE_PRECOND, Oracle  # noqa: E402

DEV = torch.device("cuda:0")
U = np.finfo(np.float64).eps / 2


def _t(a):
    return torch.as_tensor(np.ascontiguousarray(a, np.float64).ravel(), device=DEV)


@pytest.fixture(scope="module")
def system():
    """C1 after one oracle step (contact-rich), assembled by the oracle, loaded into an AS context."""
    sc = scenes.make_cubes(1)
    o = Oracle(sc)
    x1, _v1, _ = o.step(sc["x0"], sc["v0"])
    pt, ee = cm.candidates(o.mesh, x1, x1, o.dhat)
    keys, _d = cm.constraint_set(x1, pt, ee, o.dhat)
    asm = o.assemble(x1, oracle_state(o, x1, sigma=4e5), keys)
    ctx = bal.bal_init(sc, flags=bal.BAL_ADDITIVE_PRECOND)
    rp, col, val = csr_to_bsr(asm["A"], o.N)
    bal.bal_load_bsr(ctx, rp, col, val, group=np.where(asm["groups"] < -900, 0, asm["groups"]))
    return sc, o, asm, ctx


def test_additive_pcg_iterates_match_the_oracle(system):
    """Fixed k PCG iterations from 0 with M^-1 = D^-1 + sum_agg B^T A_agg^-1 B: the GPU's Gauss-Jordan
    inverses (no pivoting, SPD) vs the oracle's library inverses differ by ~n kappa_agg u per
    aggregate, so the iterates agree to that level (the tolerance is derived from the measured
    largest aggregate condition number), and the converged solve equals a direct solve."""
    sc, o, asm, ctx = system
    A, Dinv = asm["A"], asm["Dinv"]
    M = la.additive_schwarz(A, Dinv, 9)
    kappa = max(np.linalg.cond(B) for (_i0, _i1, B) in M.blocks)
    tol = 1e-10 + 27 * 27 * kappa * U
    b = -asm["grad"]
    N = o.N
    xg = torch.empty(3 * N, dtype=torch.float64, device=DEV)
    for k in (1, 5, 20):
        s = bal.bal_pcg(ctx, _t(b), _t(np.zeros(3 * N)), xg, warm_start=0, rel_tol=0.0, stall_window=0,
                        max_iters=k)
        st = la.pcg_cg(A, b, np.zeros(3 * N), M, tol=0.0, window=10 ** 9, max_iters=k)
        assert s["iters"] == k == st.k
        err = np.linalg.norm(xg.cpu().numpy() - st.x) / np.linalg.norm(st.x)
        assert err <= tol, (k, err, tol)
        hg = bal.bal_pcg_history(ctx, k + 1)
        assert np.max(np.abs(hg - np.asarray(st.hist))) <= tol * st.hist[0]
    s = bal.bal_pcg(ctx, _t(b), None, xg, warm_start=0, rel_tol=1e-12, stall_window=0, max_iters=20000)
    xd = np.linalg.solve(A.toarray(), b)
    assert s["stop_reason"] == 0
    assert np.linalg.norm(xg.cpu().numpy() - xd) <= 1e-8 * np.linalg.norm(xd)
    # the preconditioner is stronger than block-Jacobi alone on this system (fewer iterations)
    s_bj = la.pcg_cg(A, b, np.zeros(3 * N), Dinv, tol=1e-8, window=10 ** 9)
    s_as = la.pcg_cg(A, b, np.zeros(3 * N), M, tol=1e-8, window=10 ** 9)
    assert s_as.k < s_bj.k


def test_additive_step_parity():
    """Two C1 time steps with the additive preconditioner in the global PCG (no warm start, the
    paper's "AP alone" comparison): GPU positions equal the oracle's (1e-6 relative)."""
    sc = scenes.make_cubes(1)
    flags_g = bal.BAL_ADDITIVE_PRECOND | bal.BAL_NO_WARMSTART
    o = Oracle(sc, flags=FLAG_ADDITIVE_PRECOND | 1)
    ctx = bal.bal_init(sc, flags=flags_g)
    x, v = sc["x0"], sc["v0"]
    xt, vt = _t(x), _t(v)
    for _ in range(2):
        x, v, _st = o.step(x, v)
        xn, vn = torch.empty_like(xt), torch.empty_like(vt)
        bal.bal_step(ctx, xt, vt, xn, vn)
        xt, vt = xn, vn
        xg = xt.cpu().numpy().reshape(-1, 3)
        assert np.linalg.norm(xg - x) <= 1e-6 * np.linalg.norm(x)
