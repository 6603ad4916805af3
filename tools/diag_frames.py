"""Diagnostic: run a few frames of a scene through bal_frame_* with a Newton cap (BAL_VERBOSE=1|2
prints the per-iteration trace / line-search energy deltas).

    python tools/diag_frames.py c2 --chi 0.9 --frames 2 --max-newton 60 [--vx 0.5] [--flags 8]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_00046_b200 as bal  # noqa: E402
import scenes  # noqa: E402


def arg(name, default, cast=float):
    return cast(sys.argv[sys.argv.index(name) + 1]) if name in sys.argv else default


def main():
    name = sys.argv[1]
    make = {"c1": lambda: scenes.make_cubes(1), "c2": lambda: scenes.make_armadillo_like(2),
            "c3": lambda: scenes.make_impact(3), "c4": lambda: scenes.make_puffer_net(4),
            "tet": lambda: scenes.make_single_tet(0, vt=1.0, speed=1.0)}[name]
    sc = make()
    sc["params"] = dict(sc["params"])
    if "--chi" in sys.argv:
        sc["params"]["chi"] = arg("--chi", 0.0)
    sc["params"]["max_newton"] = arg("--max-newton", 200, int)
    vx = arg("--vx", 0.0)
    v0 = sc["v0"].copy()
    v0[sc["node_fixed"] == 0, 0] += vx
    dev = torch.device("cuda:0")
    ctx = bal.bal_init(sc, flags=arg("--flags", 0, int))
    x = torch.as_tensor(sc["x0"].ravel(), device=dev)
    v = torch.as_tensor(v0.ravel(), device=dev)
    for f in range(arg("--frames", 1, int)):
        xn, vn = torch.empty_like(x), torch.empty_like(v)
        print(f"=== frame {f}", flush=True)
        try:
            bal.bal_frame_begin(ctx, x, v)
            bal.bal_frame_iterate(ctx, sc["params"]["max_newton"])
        except bal.BalError as e:
            print("ERROR", e, flush=True)
        s = bal.bal_frame_finish(ctx, xn, vn, allow_unconverged=True)
        print({k: s[k] for k in ("newton_iters", "pcg_iters", "converged", "sigma0", "sigma_final", "last_rel_grad",
                                 "ms_total", "max_constraints")}, flush=True)
        x, v = xn, vn


if __name__ == "__main__":
    main()
